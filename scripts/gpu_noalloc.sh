#!/bin/bash
# G loads: ld.global.cs (default) vs ld.global.nc.L1::no_allocate (-DHB_G_NOALLOC)
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out; mkdir -p $O; : > $O/status.txt
SW="timeout 900 python scripts/opbench.py --sweep --reps 20"
$SW > $O/na_base.jsonl 2>> $O/opbench.err; echo "base rc=$?" >> $O/status.txt
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > $O/na_bench_base.json 2>> $O/bench.err
python -c "from paper_2202_12477_b200 import build as b; b.build(force=True, extra=['-DHB_G_NOALLOC'])" >> $O/status.txt 2>&1
$SW > $O/na_noalloc.jsonl 2>> $O/opbench.err; echo "noalloc rc=$?" >> $O/status.txt
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > $O/na_bench_noalloc.json 2>> $O/bench.err
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "apply_all" > $O/pytest_na.log 2>&1; echo "pytest rc=$?" >> $O/status.txt
python -c "import __graft_entry__ as g; g.build()"
