#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out; mkdir -p $O; : > $O/status.txt; : > $O/opbench_bign.jsonl
for v in 0 1 2 3 4; do
  HB_AX_VN=15 HB_AX_VARIANT=$v timeout 300 python scripts/opbench.py --N 15 --box 24,24,24 >> $O/opbench_bign.jsonl 2>> $O/opbench.err
done
for v in 0 1 2; do
  HB_AX_VARIANT=$v timeout 300 python scripts/opbench.py --N 7 --box 52,52,52 >> $O/opbench_bign.jsonl 2>> $O/opbench.err
  HB_AX_VARIANT=$v timeout 300 python scripts/opbench.py --N 7 --box 16,16,16 >> $O/opbench_bign.jsonl 2>> $O/opbench.err
done
echo "var done" >> $O/status.txt
timeout 900 python scripts/opbench.py --sweep > $O/opbench_sweep.jsonl 2>> $O/opbench.err; echo "sweep rc=$?" >> $O/status.txt
