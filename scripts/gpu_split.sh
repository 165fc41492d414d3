#!/bin/bash
# dot_rows with two FMA chains per output from CNT >= HB_DOT_SPLIT_MIN: none (99) / default (6) / all (2)
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out; mkdir -p $O; : > $O/status.txt
SW="timeout 900 python scripts/opbench.py --sweep --reps 20 --degrees 3,5,7,8,9,10,11,12,13,14,15"
for v in 99 6 4 2; do
  python -c "from paper_2202_12477_b200 import build as b; b.build(force=True, extra=['-DHB_DOT_SPLIT_MIN=$v'])" >> $O/status.txt 2>&1
  $SW > $O/split_$v.jsonl 2>> $O/opbench.err; echo "split $v rc=$?" >> $O/status.txt
done
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "apply_all or apply_modes" > $O/pytest_split.log 2>&1; echo "pytest(2) rc=$?" >> $O/status.txt
python -c "import __graft_entry__ as g; g.build()"
