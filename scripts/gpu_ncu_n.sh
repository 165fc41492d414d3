#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out; mkdir -p $O; : > $O/status.txt
for cfg in "15 24" "12 31" "2 184"; do
  set -- $cfg
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:ax_lines -s 5 -c 1 -o $O/prof_ax_n$1 -f \
     python scripts/opbench.py --N $1 --box $2,$2,$2 --reps 3 > $O/ncu_n$1.log 2>&1; echo "ncu N=$1 rc=$?" >> $O/status.txt
done
