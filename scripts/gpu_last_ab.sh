#!/bin/bash
# N = 2 at 80 registers (tune variant 11) vs default; N = 13 alternative shared-memory padding
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out; mkdir -p $O; : > $O/status.txt; : > $O/last_ab.jsonl
for r in 1 2 3; do
  timeout 600 python scripts/opbench.py --N 13 --box 28,28,28 --reps 20 >> $O/last_ab.jsonl 2>> $O/ab.err
done
python -c "from paper_2202_12477_b200 import build as b; b.build(force=True, extra=['-DHB_N13_PAD_ALT'])" >> $O/status.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "apply_all and 13" > $O/pytest_pad.log 2>&1; echo "pytest rc=$?" >> $O/status.txt
for r in 1 2 3; do
  echo '{"pad_alt": 1}' >> $O/last_ab.jsonl
  timeout 600 python scripts/opbench.py --N 13 --box 28,28,28 --reps 20 >> $O/last_ab.jsonl 2>> $O/ab.err
done
for r in 1 2 3; do
  HB_TUNE=1 HB_TUNE_N=2 timeout 900 python scripts/opbench.py --tune 0,11 --degrees 2 --reps 20 >> $O/last_ab.jsonl 2>> $O/ab.err
done
python -c "import __graft_entry__ as g; g.build()"
