#!/bin/bash
# Operator A/B in a tuning build (HB_TUNE): opbench --tune over tune variants (op.cu tune_variant).
#   AB_C3="31,30" AB_C3_DEG="2,...,15" AB_C2="31,30" bash scripts/gpu_ab.sh
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out; mkdir -p $O; : > $O/status.txt
export HB_TUNE=1
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,clocks.mem,power.limit --format=csv > $O/nvsmi.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo "build rc=$?" >> $O/status.txt
if [ -n "$AB_TESTS" ]; then
  timeout 1500 python -m pytest tests/test_gpu_parity.py -q -x -rf -k "$AB_TESTS" > $O/ab_tests.log 2>&1; echo "tests rc=$?" >> $O/status.txt
fi
if [ -n "$AB_C2" ]; then
  for rep in 1 2; do
    timeout 600 python scripts/opbench.py --tune $AB_C2 --degrees 7 --tune-box 16,16,16 >> $O/ab_c2.jsonl 2>> $O/ab.err
  done; echo "ab c2 rc=$?" >> $O/status.txt
fi
if [ -n "$AB_C3" ]; then
  timeout 2400 python scripts/opbench.py --tune $AB_C3 --degrees ${AB_C3_DEG:-2,3,4,5,6,7,8,9,10,11,12,13,14,15} > $O/ab_c3.jsonl 2>> $O/ab.err; echo "ab c3 rc=$?" >> $O/status.txt
fi
if [ -n "$BENCH_VARIANTS" ]; then  # in-situ CG timing per variant (N=7 plain kernel), C2 and C3 N=7
  for v in $BENCH_VARIANTS; do
    HB_AX_VARIANT=$v HB_AX_VN=${BENCH_N:-7} timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-c3 | sed "s/^{/{\"variant\": \"$v\", /" >> $O/bench_variants.jsonl 2>> $O/ab.err
    HB_AX_VARIANT=$v HB_AX_VN=${BENCH_N:-7} timeout 600 python bench.py --box 52,52,52 --steps 3 --warmup 3 --no-cpu-baseline --no-c3 | sed "s/^{/{\"variant\": \"$v\", /" >> $O/bench_variants.jsonl 2>> $O/ab.err
  done; echo "bench variants done" >> $O/status.txt
fi
