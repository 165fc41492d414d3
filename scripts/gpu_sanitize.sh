#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out; mkdir -p $O; : > $O/status.txt
CS=/usr/local/cuda/bin/compute-sanitizer
SAN_CASES=2:0,4:1,8:1 HB_FUSED_UPDATE=0 timeout 1500 $CS --tool synccheck --print-limit 10 python scripts/sanitize.py > $O/san_sync_nocoop.log 2>&1; echo "synccheck partial no-coop rc=$?" >> $O/status.txt
SAN_CASES=2:0,4:1,8:1 timeout 1500 $CS --tool synccheck --print-limit 10 python scripts/sanitize.py > $O/san_sync_coop.log 2>&1; echo "synccheck partial coop rc=$?" >> $O/status.txt
SAN_CASES=1:0,3:1,7:0,15:0 HB_FUSED_UPDATE=0 timeout 1500 $CS --tool racecheck --print-limit 10 python scripts/sanitize.py > $O/san_race_w32.log 2>&1; echo "racecheck w32 rc=$?" >> $O/status.txt
SAN_CASES=2:0,4:1,8:1,12:0 HB_FUSED_UPDATE=0 timeout 1500 $CS --tool racecheck --print-limit 10 python scripts/sanitize.py > $O/san_race_partial.log 2>&1; echo "racecheck partial rc=$?" >> $O/status.txt
