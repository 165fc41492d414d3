#!/bin/bash
# BASELINE configs C4 / C5 at P = 1 (one GPU per gpurun call) + C1 smoke-size bench.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out; mkdir -p $O; [ "$1" = --append ] || : > $O/status.txt
free -g > $O/host_mem.txt; nproc >> $O/host_mem.txt
timeout 900 python bench.py --box 66,66,66 --N 7 --steps 3 --warmup 3 --no-cpu-baseline > $O/bench_c4_p1.json 2> $O/bench_cfg.err; echo "c4 rc=$?" >> $O/status.txt
timeout 1500 python bench.py --box 50,50,48 --N 15 --steps 2 --warmup 3 --no-cpu-baseline > $O/bench_c5_p1.json 2>> $O/bench_cfg.err; echo "c5 rc=$?" >> $O/status.txt
timeout 600 python bench.py --box 2,2,2 --N 3 --iters 50 --steps 10 --warmup 3 > $O/bench_c1.json 2>> $O/bench_cfg.err; echo "c1 rc=$?" >> $O/status.txt
