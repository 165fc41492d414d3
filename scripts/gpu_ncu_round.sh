#!/bin/bash
# ncu evidence for the bench: launch list of the C2 bench command, --set full captures of the
# operator (C2, C3 N=7) and the fused vector update (C2, C3), summarised on the box (reports
# are too large to copy back): TAG=<round tag>
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out; mkdir -p $O; : > $O/status.txt
TAG=${TAG:-r1b_end}
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $O/launches.csv \
  python bench.py --steps 1 --warmup 1 --iters 20 --no-cpu-baseline --no-profile > $O/ncu_launch.log 2>&1; echo "ncu-list rc=$?" >> $O/status.txt
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:ax_lines -s 5 -c 1 -o $O/prof_ax_c2 -f \
  python bench.py --steps 1 --warmup 1 --iters 5 --no-cpu-baseline --no-profile > $O/ncu_full.log 2>&1; echo "ncu-full c2 rc=$?" >> $O/status.txt
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:ax_lines -s 5 -c 1 -o $O/prof_ax_c3 -f \
  python scripts/opbench.py --N 7 --box 52,52,52 --reps 3 > $O/ncu_full3.log 2>&1; echo "ncu-full c3 rc=$?" >> $O/status.txt
timeout 1200 ncu --set full --clock-control none -k regex:cg_update -s 10 -c 1 -o $O/prof_vec_c2 -f \
  python bench.py --steps 1 --warmup 1 --iters 5 --no-cpu-baseline --no-profile > $O/ncu_vec.log 2>&1; echo "ncu-vec c2 rc=$?" >> $O/status.txt
timeout 1200 ncu --set full --clock-control none -k regex:cg_update -s 10 -c 1 -o $O/prof_vec_c3 -f \
  python bench.py --box 52,52,52 --steps 1 --warmup 1 --iters 5 --no-cpu-baseline --no-profile > $O/ncu_vec3.log 2>&1; echo "ncu-vec c3 rc=$?" >> $O/status.txt
python scripts/ncu_summary.py $TAG $O/prof_ax_c2.ncu-rep:N7_16x16x16 $O/prof_ax_c3.ncu-rep:N7_52x52x52 \
  $O/prof_vec_c2.ncu-rep:vec_N7_16x16x16 $O/prof_vec_c3.ncu-rep:vec_N7_52x52x52 --launches $O/launches.csv > $O/summary.log 2>&1
echo "summary rc=$?" >> $O/status.txt
python scripts/ncu_digest.py $O/digest $O/prof_ax_c2.ncu-rep $O/prof_ax_c3.ncu-rep
mkdir -p $O/profiles_out; cp profiles/ncu_$TAG.md profiles/ncu_op_summary.json $O/profiles_out/
rm -f $O/*.ncu-rep
