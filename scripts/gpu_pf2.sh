#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out; mkdir -p $O; : > $O/status.txt
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x > $O/pytest_pf2.log 2>&1; echo "pytest rc=$?" >> $O/status.txt
SW="timeout 900 python scripts/opbench.py --sweep --reps 20 --degrees"
$SW 1,2,3,4,5,6,7,8,9,10,11,12,13,14,15 > $O/pf2_sweep.jsonl 2>> $O/opbench.err; echo "sweep rc=$?" >> $O/status.txt
HB_AX_PFN=1 $SW 8,11,12,13,14,15 > $O/pf2_pfn.jsonl 2>> $O/opbench.err; echo "pfn rc=$?" >> $O/status.txt
