#!/bin/bash
# Operator variant A/B at the C3 boxes: streaming contractions (N >= 8), async gather, G via bulk copy (N <= 5)
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out; mkdir -p $O; : > $O/status.txt
SW="timeout 900 python scripts/opbench.py --sweep --reps 20 --degrees"
HB_AX_GSM=2,3,4,5 HB_AX_STREAM=8,9,10,11,13,14,15 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "apply_all or apply_modes or single or C3" > $O/pytest_var.log 2>&1; echo "pytest rc=$?" >> $O/status.txt
$SW 2,3,4,5,8,9,10,11,12,13,14,15 > $O/v_base.jsonl 2>> $O/opbench.err; echo "base rc=$?" >> $O/status.txt
HB_AX_GSM=2,3,4,5 $SW 2,3,4,5 > $O/v_gsm.jsonl 2>> $O/opbench.err; echo "gsm rc=$?" >> $O/status.txt
HB_AX_STREAM=8,9,10,11,12,13,14,15 $SW 8,9,10,11,13,14,15 > $O/v_str.jsonl 2>> $O/opbench.err; echo "str rc=$?" >> $O/status.txt
HB_AX_STREAM=8,9,10,11,12,13,14,15 HB_AX_STREAM_MINB=1 $SW 8,9,10,11,12,13,14,15 > $O/v_str1.jsonl 2>> $O/opbench.err; echo "str1 rc=$?" >> $O/status.txt
HB_AX_STREAM=8,9,10,11,12,13,14,15 HB_AX_PIPE=8,9,10,11,12,13,14,15 $SW 8,9,10,11,12,13,14,15 > $O/v_strp.jsonl 2>> $O/opbench.err; echo "strp rc=$?" >> $O/status.txt
HB_AX_STREAM=8,9,10,11,12,13,14,15 HB_AX_PIPE=8,9,10,11,12,13,14,15 HB_AX_STREAM_MINB=1 $SW 8,9,10,11,12,13,14,15 > $O/v_strp1.jsonl 2>> $O/opbench.err; echo "strp1 rc=$?" >> $O/status.txt
