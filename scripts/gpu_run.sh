#!/bin/bash
# One gpurun batch.  STAGES (env) picks from: tests smoke bench var sweep ncu ncuvec
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out
mkdir -p $O; : > $O/status.txt
nvidia-smi -L > $O/nvsmi.txt 2>&1
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,clocks.mem,power.limit --format=csv >> $O/nvsmi.txt 2>&1
STAGES=${STAGES:-"tests smoke bench ncu"}
VARIANTS=${VARIANTS:-"0 1 2 3 4"}
for s in $STAGES; do
  case $s in
    tests) timeout 1200 python -m pytest tests -m gpu -q -rf > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/status.txt ;;
    smoke) timeout 300 python __graft_entry__.py smoke > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/status.txt ;;
    bench) timeout 900 python bench.py --steps 10 --warmup 3 > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/status.txt
           timeout 900 python bench.py --box 52,52,52 --steps 3 --warmup 3 --no-cpu-baseline > $O/bench_c3n7.json 2>> $O/bench.err; echo "bench c3 rc=$?" >> $O/status.txt
           timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_ref.json 2>> $O/bench.err; echo "bench ref rc=$?" >> $O/status.txt
           HB_PDL=0 timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_nopdl.json 2>> $O/bench.err; echo "bench nopdl rc=$?" >> $O/status.txt ;;
    var) : > $O/opbench_variants.jsonl
         for v in $VARIANTS; do
           HB_AX_VARIANT=$v timeout 300 python scripts/opbench.py --N 7 --box 52,52,52 >> $O/opbench_variants.jsonl 2>> $O/opbench.err
           HB_AX_VARIANT=$v timeout 300 python scripts/opbench.py --N 7 --box 16,16,16 >> $O/opbench_variants.jsonl 2>> $O/opbench.err
         done; echo "var done" >> $O/status.txt ;;
    sweep) timeout 900 python scripts/opbench.py --sweep > $O/opbench_sweep.jsonl 2>> $O/opbench.err; echo "sweep rc=$?" >> $O/status.txt ;;
    ncu) timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $O/launches.csv \
           python bench.py --steps 1 --warmup 1 --iters 20 --no-cpu-baseline --no-profile > $O/ncu_launch.log 2>&1; echo "ncu-list rc=$?" >> $O/status.txt
         timeout 1200 ncu --set full --clock-control none --import-source on -k regex:ax_lines -s 5 -c 1 -o $O/prof_ax_c2 -f \
           python bench.py --steps 1 --warmup 1 --iters 5 --no-cpu-baseline --no-profile > $O/ncu_full.log 2>&1; echo "ncu-full rc=$?" >> $O/status.txt
         timeout 1200 ncu --set full --clock-control none --import-source on -k regex:ax_lines -s 5 -c 1 -o $O/prof_ax_c3 -f \
           python scripts/opbench.py --N 7 --box 52,52,52 --reps 3 > $O/ncu_full3.log 2>&1; echo "ncu-full3 rc=$?" >> $O/status.txt ;;
    ncuvec) timeout 1200 ncu --set full --clock-control none -k regex:cg_update -s 10 -c 1 -o $O/prof_vec_c2 -f \
           python bench.py --steps 1 --warmup 1 --iters 5 --no-cpu-baseline --no-profile > $O/ncu_vec.log 2>&1; echo "ncu-vec rc=$?" >> $O/status.txt
            timeout 1200 ncu --set full --clock-control none -k regex:cg_update -s 10 -c 1 -o $O/prof_vec_c3 -f \
           python bench.py --box 52,52,52 --steps 1 --warmup 1 --iters 5 --no-cpu-baseline --no-profile > $O/ncu_vec3.log 2>&1; echo "ncu-vec3 rc=$?" >> $O/status.txt ;;
    calib) timeout 300 python scripts/calib.py > $O/calib.json 2>> $O/calib.err; echo "calib rc=$?" >> $O/status.txt ;;
  esac
done
