#!/bin/bash
# ncu --set full captures of the operator at chosen degrees (C3 boxes): NCU_CFGS="N box ..."
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out; mkdir -p $O; : > $O/status.txt
CFGS=${NCU_CFGS:-"15 24 12 31 2 184"}
set -- $CFGS
while [ $# -ge 2 ]; do
  n=$1; b=$2; shift 2
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:ax_ -s 5 -c 1 -o $O/prof_ax_n$n -f \
     python scripts/opbench.py --N $n --box $b,$b,$b --reps 3 > $O/ncu_n$n.log 2>&1; echo "ncu N=$n rc=$?" >> $O/status.txt
done
python scripts/ncu_digest.py $O/digest $O/prof_ax_n*.ncu-rep
[ -n "$KEEP_REPS" ] || rm -f $O/prof_ax_n*.ncu-rep
