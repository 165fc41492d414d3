#!/bin/bash
# Kernel iteration batch: parity tests, variant timings, C3 sweep, bench.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out; mkdir -p $O; : > $O/status.txt
timeout 900 python -m pytest tests -m gpu -q -x -rf > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/status.txt
for v in 0 1 2 3 4 5 6; do
  HB_AX_VARIANT=$v timeout 300 python scripts/opbench.py --N 7 --box 52,52,52 >> $O/opbench_variants.jsonl 2>> $O/opbench.err
  HB_AX_VARIANT=$v timeout 300 python scripts/opbench.py --N 7 --box 16,16,16 >> $O/opbench_variants.jsonl 2>> $O/opbench.err
done
echo "variants done" >> $O/status.txt
timeout 900 python scripts/opbench.py --sweep > $O/opbench_sweep.jsonl 2>> $O/opbench.err; echo "sweep rc=$?" >> $O/status.txt
timeout 900 python bench.py --steps 5 --warmup 3 > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/status.txt
