#!/bin/bash
# N = 7 prefetch / shape variants at the C2 box (latency-bound size) and at C3
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out; mkdir -p $O; : > $O/status.txt
HB_TUNE=1 HB_TUNE_N=7 timeout 900 python scripts/opbench.py --tune 0,13,7,8,9,11,1,6 --degrees 7 --tune-box 16,16,16 --reps 50 > $O/tune_c2c.jsonl 2>> $O/tune.err; echo "tune c2 rc=$?" >> $O/status.txt
python -c "import __graft_entry__ as g; g.build()"
