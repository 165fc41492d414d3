#!/bin/bash
# G device layout A/B: six factor planes per k-slab (default build) vs interleaved pairs (-DHB_G_PAIRS)
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out; mkdir -p $O; : > $O/status.txt
SW="timeout 900 python scripts/opbench.py --sweep --reps 20 --degrees 1,2,3,4,5,6,7,8,9,10,11,12,13,14,15"
$SW > $O/gp_base.jsonl 2>> $O/opbench.err; echo "base rc=$?" >> $O/status.txt
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $O/gp_bench_base.json 2>> $O/bench.err
python -c "from paper_2202_12477_b200 import build as b; b.build(force=True, extra=['-DHB_G_PAIRS'])" >> $O/status.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x > $O/pytest_gp.log 2>&1; echo "pytest pairs rc=$?" >> $O/status.txt
$SW > $O/gp_pairs.jsonl 2>> $O/opbench.err; echo "pairs rc=$?" >> $O/status.txt
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $O/gp_bench_pairs.json 2>> $O/bench.err
