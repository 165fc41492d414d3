#!/bin/bash
# One gpurun batch.  STAGES (env) picks from:
#   tests smoke bench ref ncu ncuvec ncun sweep cgsweep san race ipc2 big calib
# Every stage writes under gpurun_out/ and appends "<stage> rc=<code>" to gpurun_out/status.txt.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out
mkdir -p $O; : > $O/status.txt
nvidia-smi -L > $O/nvsmi.txt 2>&1
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,clocks.mem,power.limit --format=csv >> $O/nvsmi.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo "build rc=$?" >> $O/status.txt
STAGES=${STAGES:-"tests smoke bench ncu"}
NCU_BOX=${NCU_BOX:-16,16,16}
for s in $STAGES; do
  case $s in
    tests) timeout 1800 python -m pytest tests -m gpu -q -rf ${PYTEST_K:+-k "$PYTEST_K"} > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/status.txt ;;
    smoke) timeout 300 python __graft_entry__.py smoke > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/status.txt ;;
    bench) timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/status.txt
           timeout 900 python bench.py --box 52,52,52 --steps 3 --warmup 3 --no-cpu-baseline --no-c3 > $O/bench_c3n7.json 2>> $O/bench.err; echo "bench c3 rc=$?" >> $O/status.txt ;;
    ref) timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_ref.json 2> $O/bench_ref.err; echo "ref rc=$?" >> $O/status.txt ;;
    ncu) timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches.csv \
           python bench.py --steps 1 --warmup 1 --iters 20 --no-cpu-baseline --no-profile --no-c3 > $O/ncu_launch.log 2>&1; echo "ncu-list rc=$?" >> $O/status.txt
         timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -c 400 --csv --log-file $O/launches_warm.csv \
           python bench.py --steps 1 --warmup 1 --iters 20 --no-cpu-baseline --no-profile --no-c3 > $O/ncu_launch_warm.log 2>&1; echo "ncu-list-warm rc=$?" >> $O/status.txt
         timeout 1200 ncu --set full --clock-control none --import-source on -k regex:ax_ -s 5 -c 1 -o $O/prof_ax_c2 -f \
           python bench.py --steps 1 --warmup 1 --iters 5 --no-cpu-baseline --no-profile --no-c3 > $O/ncu_full.log 2>&1; echo "ncu-full rc=$?" >> $O/status.txt
         timeout 1200 ncu --set full --clock-control none --import-source on -k regex:ax_ -s 5 -c 1 -o $O/prof_ax_c3 -f \
           python scripts/opbench.py --N 7 --box 52,52,52 --reps 3 > $O/ncu_full3.log 2>&1; echo "ncu-full3 rc=$?" >> $O/status.txt ;;
    ncuvec) timeout 1200 ncu --set full --clock-control none -k regex:cg_update -s 10 -c 1 -o $O/prof_vec_c2 -f \
           python bench.py --steps 1 --warmup 1 --iters 5 --no-cpu-baseline --no-profile --no-c3 > $O/ncu_vec.log 2>&1; echo "ncu-vec rc=$?" >> $O/status.txt ;;
    sweep) timeout 1500 python scripts/opbench.py --sweep > $O/opbench_sweep.jsonl 2>> $O/opbench.err; echo "sweep rc=$?" >> $O/status.txt ;;
    cgsweep) : > $O/cg_sweep.jsonl
         for n in 1 2 3 4 5 6 7 8 9 10 11 12 13 14 15; do
           b=$(python -c "print({1:'120,100,91',2:'184,184,184',3:'122,122,122',4:'92,92,92',5:'73,73,73',6:'61,61,61',7:'52,52,52',8:'46,46,46',9:'41,41,41',10:'37,37,37',11:'33,33,33',12:'31,31,31',13:'28,28,28',14:'26,26,26',15:'24,24,24'}[$n])")
           timeout 600 python bench.py --N $n --box $b --steps 3 --warmup 3 --no-cpu-baseline --no-c3 >> $O/cg_sweep.jsonl 2>> $O/cgsweep.err
         done; echo "cgsweep done" >> $O/status.txt ;;
    san) for tool in memcheck racecheck; do
           SAN_CASES=${SAN_CASES:-"2:0,3:1,7:0,8:1,11:1,13:0,15:0"} SAN_MULTIWAVE=${SAN_MULTIWAVE:-"1,2,7,11,12,13,15"} timeout 1800 \
             compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize.py > $O/san_$tool.log 2>&1
           echo "san $tool rc=$?" >> $O/status.txt
         done ;;
    calib) timeout 300 python scripts/calib.py > $O/calib.json 2>> $O/calib.err; echo "calib rc=$?" >> $O/status.txt ;;
    ncun) mkdir -p $O/ncu_n  # per-degree operator captures at the C3 boxes, digested on the box (reports are large)
         for n in ${NCU_DEGREES:-2 4 15}; do
           b=$(python -c "print({1:'120,100,91',2:'184,184,184',3:'122,122,122',4:'92,92,92',5:'73,73,73',6:'61,61,61',7:'52,52,52',8:'46,46,46',9:'41,41,41',10:'37,37,37',11:'33,33,33',12:'31,31,31',13:'28,28,28',14:'26,26,26',15:'24,24,24'}[$n])")
           timeout 900 ncu --set full --clock-control none --import-source on -k regex:ax_ -s 5 -c 1 -o /tmp/prof_ax_n$n -f \
             python scripts/opbench.py --N $n --box $b --reps 3 > $O/ncu_n/ncu_n$n.log 2>&1; echo "ncu n$n rc=$?" >> $O/status.txt
           python scripts/ncu_digest.py $O/ncu_n /tmp/prof_ax_n$n.ncu-rep >> $O/status.txt 2>&1
           ncu -i /tmp/prof_ax_n$n.ncu-rep --page raw --csv > $O/ncu_n/raw_n$n.csv 2>/dev/null
         done ;;
    race) # racecheck in a tuning build without the cooperative update (the tool does not run it)
         HB_TUNE=1 python -c "import __graft_entry__ as g; g.build()" > $O/build_tune.log 2>&1
         HB_TUNE=1 HB_FUSED_UPDATE=0 SAN_CASES=${SAN_CASES:-"2:0,3:1,7:0,8:1,11:1,13:0,15:0"} SAN_MULTIWAVE=${SAN_MULTIWAVE:-"1,2,7,11,12,13,15"} \
           timeout 2400 compute-sanitizer --tool racecheck --print-limit 20 python scripts/sanitize.py > $O/san_racecheck.log 2>&1
         echo "racecheck rc=$?" >> $O/status.txt
         python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 ;;
    ipc2) timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 \
           bench.py --gpus 2 --transport ipc --box 8,8,8 --steps 2 --warmup 3 > $O/bench_ipc2.json 2>> $O/bench.err; echo "ipc2 rc=$?" >> $O/status.txt ;;
    big) timeout 900 python bench.py --box 66,66,66 --steps 3 --warmup 3 --no-cpu-baseline --no-c3 > $O/bench_c4_p1.json 2>> $O/bench.err; echo "c4 rc=$?" >> $O/status.txt
         timeout 900 python bench.py --N 15 --box 50,50,48 --steps 2 --warmup 3 --no-cpu-baseline --no-c3 > $O/bench_c5_p1.json 2>> $O/bench.err; echo "c5 rc=$?" >> $O/status.txt ;;
  esac
done
