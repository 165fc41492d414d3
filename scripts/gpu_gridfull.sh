#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out; mkdir -p $O; : > $O/status.txt; : > $O/gridfull.jsonl
HB_AX_GRID_FULL=1 timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "C2 or cg_parity" > $O/pytest_gf.log 2>&1; echo "pytest rc=$?" >> $O/status.txt
for r in 1 2; do for g in 0 1; do
  echo "{\"grid_full\": $g}" >> $O/gridfull.jsonl
  HB_AX_GRID_FULL=$g timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline >> $O/gridfull.jsonl 2>> $O/bench.err
done; done
echo done >> $O/status.txt
