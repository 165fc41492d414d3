#!/bin/bash
# register-cap variants per degree with the current prefetch / layout choices (one tuning build per N)
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out; mkdir -p $O; : > $O/status.txt; : > $O/tune3.jsonl
for n in ${TUNE_DEGREES:-9 10 11 12 13 14 15}; do
  HB_TUNE=1 HB_TUNE_N=$n timeout 900 python scripts/opbench.py --tune ${TUNE_VARIANTS:-0,4,5,6} --degrees $n --reps 20 >> $O/tune3.jsonl 2>> $O/tune.err; echo "tune N=$n rc=$?" >> $O/status.txt
done
python -c "import __graft_entry__ as g; g.build()"
