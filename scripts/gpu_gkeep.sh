#!/bin/bash
# share of G kept L2-resident across CG iterations (evict_last policy) at C2 / C3
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out; mkdir -p $O; : > $O/status.txt; : > $O/gkeep.jsonl
HB_G_KEEP_MB=40 timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "C2 or cg_parity or apply_all" > $O/pytest_gkeep.log 2>&1; echo "pytest rc=$?" >> $O/status.txt
for mb in 0 20 40 60 80 100; do
  echo "{\"g_keep_mb\": $mb}" >> $O/gkeep.jsonl
  HB_G_KEEP_MB=$mb timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline >> $O/gkeep.jsonl 2>> $O/bench.err
done
for mb in 0 60; do
  echo "{\"g_keep_mb\": $mb, \"box\": \"52\"}" >> $O/gkeep.jsonl
  HB_G_KEEP_MB=$mb timeout 600 python bench.py --box 52,52,52 --steps 3 --warmup 3 --no-cpu-baseline >> $O/gkeep.jsonl 2>> $O/bench.err
done
echo "done" >> $O/status.txt
