#!/bin/bash
# Product build: GPU tests + smoke; tuning build: racecheck without the cooperative update and
# in-situ CG timing of the round-1 vs round-2 large-N operator configurations.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out; mkdir -p $O
STAGES="tests smoke" bash scripts/gpu_run.sh
cp $O/status.txt $O/status_product.txt
export HB_TUNE=1
python -c "import __graft_entry__ as g; g.build()" > $O/build_tune.log 2>&1; echo "tune build rc=$?" >> $O/status_product.txt
HB_FUSED_UPDATE=0 SAN_CASES="2:0,3:1,7:0,8:1,11:1,13:0,15:0" SAN_MULTIWAVE="1,2,7,11,12,13,15" timeout 2400 \
  compute-sanitizer --tool racecheck --print-limit 20 python scripts/sanitize.py > $O/san_racecheck.log 2>&1
echo "racecheck rc=$?" >> $O/status_product.txt
: > $O/bench_variants.jsonl
for nv in "11:0" "11:74" "12:0" "12:75" "13:0" "13:65"; do
  n=${nv%%:*}; v=${nv##*:}
  b=$(python -c "print({11:'33,33,33',12:'31,31,31',13:'28,28,28'}[$n])")
  HB_AX_VARIANT=$v HB_AX_VN=$n timeout 600 python bench.py --N $n --box $b --steps 3 --warmup 3 --no-cpu-baseline --no-c3 \
    | sed "s/^{/{\"variant\": \"$v\", /" >> $O/bench_variants.jsonl 2>> $O/bench_variants.err
done
echo "bench variants done" >> $O/status_product.txt
