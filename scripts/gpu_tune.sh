#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out; mkdir -p $O; : > $O/status.txt
HB_TUNE=1 timeout 3000 python scripts/opbench.py --tune 0,7,8 --reps 20 > $O/tune2.jsonl 2> $O/tune.err; echo "tune rc=$?" >> $O/status.txt
