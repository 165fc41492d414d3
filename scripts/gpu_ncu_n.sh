#!/bin/bash
# ncu --set full of the operator at the C3 box of each degree in NCU_DEGREES (product build);
# digested on the box (reports exceed gpurun's copy-back limit): text digest + raw CSV per degree.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out; mkdir -p $O/ncu_n
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
for n in ${NCU_DEGREES:-2 4 15}; do
  b=$(python -c "print({1:'120,100,91',2:'184,184,184',3:'122,122,122',4:'92,92,92',5:'73,73,73',6:'61,61,61',7:'52,52,52',8:'46,46,46',9:'41,41,41',10:'37,37,37',11:'33,33,33',12:'31,31,31',13:'28,28,28',14:'26,26,26',15:'24,24,24'}[$n])")
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:ax_ -s 5 -c 1 -o /tmp/prof_ax_n$n -f \
    python scripts/opbench.py --N $n --box $b --reps 3 > $O/ncu_n/ncu_n$n.log 2>&1
  echo "ncu n$n rc=$?" >> $O/status.txt
  python scripts/ncu_digest.py $O/ncu_n /tmp/prof_ax_n$n.ncu-rep >> $O/status.txt 2>&1
  ncu -i /tmp/prof_ax_n$n.ncu-rep --page raw --csv > $O/ncu_n/raw_n$n.csv 2>/dev/null
done
