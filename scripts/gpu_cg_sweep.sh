#!/bin/bash
# full CG (100 iterations, NekBone FOM and GDOF/s) per degree at the C3 boxes (~50 M DOFs)
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out; mkdir -p $O; : > $O/status.txt; : > $O/cg_sweep.jsonl
for nb in "1 367" "2 184" "3 122" "4 92" "5 73" "6 61" "7 52" "8 46" "9 41" "10 37" "11 33" "12 31" "13 28" "14 26" "15 24"; do
  set -- $nb
  timeout 600 python bench.py --N $1 --box $2,$2,$2 --steps 3 --warmup 3 --no-cpu-baseline >> $O/cg_sweep.jsonl 2>> $O/cg_sweep.err
  echo "N=$1 rc=$?" >> $O/status.txt
done
