#!/bin/bash
# N=7 launch-shape variants at the C2 box (latency-bound regime) vs C3
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out; mkdir -p $O
export HB_TUNE=1 HB_TUNE_N=7
timeout 1200 python scripts/opbench.py --tune 0,1,2,3,4,5,6,7,8 --degrees 7 --tune-box 16,16,16 --reps 50 > $O/tune_c2.jsonl 2> $O/tune_c2.err
echo "rc=$?"
timeout 600 python scripts/opbench.py --tune 0,3,5 --degrees 7 --reps 20 >> $O/tune_c2.jsonl 2>> $O/tune_c2.err
# restore the plain build for anything that follows
unset HB_TUNE HB_TUNE_N
python -c "import __graft_entry__ as g; g.build()"
