#!/bin/bash
# vector update prefetching the next operator's first wave (HB_UPD_PF=1) vs off
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out; mkdir -p $O; : > $O/status.txt; : > $O/updpf.jsonl
HB_UPD_PF=1 timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "C2 or cg_parity or jacobi or tolerance" > $O/pytest_updpf.log 2>&1; echo "pytest rc=$?" >> $O/status.txt
for r in 1 2; do for g in 0 1; do
  echo "{\"upd_pf\": $g}" >> $O/updpf.jsonl
  HB_UPD_PF=$g timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline >> $O/updpf.jsonl 2>> $O/bench.err
done; done
for g in 0 1; do
  echo "{\"upd_pf\": $g, \"box\": \"24 N=7\"}" >> $O/updpf.jsonl
  HB_UPD_PF=$g timeout 600 python bench.py --box 24,24,24 --steps 5 --warmup 3 --no-cpu-baseline >> $O/updpf.jsonl 2>> $O/bench.err
done
echo done >> $O/status.txt
