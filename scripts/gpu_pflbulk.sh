#!/bin/bash
# per-line vs one bulk L2 prefetch of each element's G (rebuild with -DHB_PFL_BULK on the box)
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out; mkdir -p $O; : > $O/status.txt
SW="timeout 900 python scripts/opbench.py --sweep --reps 20 --degrees 6,7,8,9,10,11,12,13,14,15"
$SW > $O/pf_base.jsonl 2>> $O/opbench.err; echo "base rc=$?" >> $O/status.txt
python -c "from paper_2202_12477_b200 import build as b; b.build(force=True, extra=['-DHB_PFL_BULK'])" >> $O/status.txt 2>&1
$SW > $O/pf_bulk.jsonl 2>> $O/opbench.err; echo "bulk rc=$?" >> $O/status.txt
HB_AX_PIPE_PFN=1 HB_AX_PIPE=6,7,8,9,10,11,12,13,14,15 $SW > $O/pf_bulk_pipe_pfn.jsonl 2>> $O/opbench.err; echo "bulk pipe pfn rc=$?" >> $O/status.txt
