#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out; mkdir -p $O; : > $O/status.txt; : > $O/opbench_variants.jsonl
for v in 0 1 2 3 4; do
  HB_AX_VARIANT=$v timeout 300 python scripts/opbench.py --N 7 --box 52,52,52 >> $O/opbench_variants.jsonl 2>> $O/opbench.err
  HB_AX_VARIANT=$v timeout 300 python scripts/opbench.py --N 7 --box 16,16,16 >> $O/opbench_variants.jsonl 2>> $O/opbench.err
done
echo "variants done" >> $O/status.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ax_lines -s 5 -c 1 -o $O/prof_lines_c3 -f \
   python scripts/opbench.py --N 7 --box 52,52,52 --reps 3 > $O/ncu_full3.log 2>&1; echo "ncu-full3 rc=$?" >> $O/status.txt
timeout 900 python -m pytest tests -m gpu -q -x -rf > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/status.txt
timeout 900 python scripts/opbench.py --sweep > $O/opbench_sweep.jsonl 2>> $O/opbench.err; echo "sweep rc=$?" >> $O/status.txt
