#!/bin/bash
# N = 2 element-per-thread kernel (parity, EPB A/B vs the line kernel) and N = 7 register caps at C2
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out; mkdir -p $O; : > $O/status.txt
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "apply or cg_parity or C3 or jacobi or random_geometry or loopback" > $O/pytest_n2.log 2>&1; echo "pytest rc=$?" >> $O/status.txt
HB_N2_EPB=64 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "apply_all and 2" > $O/pytest_n2_64.log 2>&1; echo "pytest64 rc=$?" >> $O/status.txt
: > $O/n2.jsonl
for v in lines 32 64; do
  if [ $v = lines ]; then HB_N2_LINES=1 timeout 300 python scripts/opbench.py --N 2 --box 184,184,184 --reps 20 >> $O/n2.jsonl 2>> $O/opbench.err
  else HB_N2_EPB=$v timeout 300 python scripts/opbench.py --N 2 --box 184,184,184 --reps 20 >> $O/n2.jsonl 2>> $O/opbench.err; fi
  echo "n2 $v rc=$?" >> $O/status.txt
done
HB_TUNE=1 HB_TUNE_N=7 timeout 900 python scripts/opbench.py --tune 0,9,10,11 --degrees 7 --tune-box 16,16,16 --reps 50 > $O/tune_c2b.jsonl 2>> $O/tune.err; echo "tune c2 rc=$?" >> $O/status.txt
HB_TUNE=1 HB_TUNE_N=7 timeout 900 python scripts/opbench.py --tune 0,9,10,11 --degrees 7 --reps 20 >> $O/tune_c2b.jsonl 2>> $O/tune.err; echo "tune c3 rc=$?" >> $O/status.txt
python -c "import __graft_entry__ as g; g.build()"
