#!/bin/bash
# compute-sanitizer memcheck + racecheck of the current build (bulk prefetch, factor-pair G, folded loop test)
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out; mkdir -p $O/san; : > $O/status.txt
CS=/usr/local/cuda/bin/compute-sanitizer
SAN_CASES=2:0,3:1,7:0,8:1,13:0,15:1 timeout 1700 $CS --tool memcheck --print-limit 10 python scripts/sanitize.py > $O/san/memcheck.log 2>&1; echo "memcheck rc=$?" >> $O/status.txt
SAN_CASES=2:0,7:0,8:1,15:0 HB_FUSED_UPDATE=0 timeout 1500 $CS --tool racecheck --print-limit 10 python scripts/sanitize.py > $O/san/racecheck.log 2>&1; echo "racecheck rc=$?" >> $O/status.txt
