#!/bin/bash
# A/B of the operator kernel: this tree vs the worktree in _ab_old, same box, interleaved.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=$PWD/gpurun_out; mkdir -p $O; : > $O/status.txt; : > $O/ab.jsonl
for rep in 1 2; do
  for tree in . _ab_old _ab_b; do
    (cd $tree && timeout 600 python scripts/opbench.py --N 7 --box 52,52,52 --reps 30 2>>$O/ab.err | sed "s/^{/{\"tree\": \"$tree\", /" >> $O/ab.jsonl)
    (cd $tree && timeout 600 python scripts/opbench.py --N 15 --box 24,24,24 --reps 30 2>>$O/ab.err | sed "s/^{/{\"tree\": \"$tree\", /" >> $O/ab.jsonl)
    (cd $tree && timeout 600 python scripts/opbench.py --N 7 --box 16,16,16 --reps 30 2>>$O/ab.err | sed "s/^{/{\"tree\": \"$tree\", /" >> $O/ab.jsonl)
  done
done
echo done >> $O/status.txt
