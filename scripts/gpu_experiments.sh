#!/bin/bash
# Experiments beyond the headline: assembled vs scattered storage (the paper's P:142-147
# argument), the deterministic assembly variant, and Jacobi PCG, on C2 / C3 N=7 / C3 N=15.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out; mkdir -p $O; : > $O/status.txt; : > $O/experiments.jsonl
run() { timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline "$@" >> $O/experiments.jsonl 2>> $O/exp.err; echo "$* rc=$?" >> $O/status.txt; }
for cfg in "--box 16,16,16 --N 7" "--box 52,52,52 --N 7" "--box 24,24,24 --N 15"; do
  run $cfg
  run $cfg --storage scattered
  run $cfg --variant 1
done
