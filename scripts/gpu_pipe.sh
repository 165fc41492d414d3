#!/bin/bash
# PIPE (asynchronous gather) operator: parity under HB_AX_PIPE=all, then C3 sweeps A/B
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out; mkdir -p $O; : > $O/status.txt
HB_AX_PIPE=all timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "apply or cg_parity or C3 or random_geometry" > $O/pytest_pipe.log 2>&1; echo "pytest pipe rc=$?" >> $O/status.txt
D=${PIPE_DEGREES:-"2,3,4,5,6,7,8,9,10,11,12,13,14,15"}
timeout 900 python scripts/opbench.py --sweep --reps 20 --degrees $D > $O/sweep_base.jsonl 2>> $O/opbench.err; echo "base rc=$?" >> $O/status.txt
HB_AX_PIPE=all timeout 900 python scripts/opbench.py --sweep --reps 20 --degrees $D > $O/sweep_pipe.jsonl 2>> $O/opbench.err; echo "pipe rc=$?" >> $O/status.txt
HB_AX_PIPE=all HB_AX_PIPE_PFN=1 timeout 900 python scripts/opbench.py --sweep --reps 20 --degrees $D > $O/sweep_pipe_pfn.jsonl 2>> $O/opbench.err; echo "pipe pfn rc=$?" >> $O/status.txt
