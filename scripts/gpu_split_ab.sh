#!/bin/bash
# Split-line kernel A/B (tuning build): parity of the split kernels, then line vs split operator timings.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out; mkdir -p $O; : > $O/status.txt
export HB_TUNE=1
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,clocks.mem,power.limit --format=csv > $O/nvsmi.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo "build rc=$?" >> $O/status.txt
HB_SPLIT=1 timeout 1500 python -m pytest tests/test_gpu_parity.py -q -x -rf -k "apply or cg_parity or C2 or C3 or jacobi or energy" > $O/split_tests.log 2>&1; echo "split tests rc=$?" >> $O/status.txt
timeout 600 python scripts/opbench.py --tune 0,20 --degrees 7 --tune-box 16,16,16 > $O/ab_c2.jsonl 2>> $O/ab.err; echo "ab c2 rc=$?" >> $O/status.txt
timeout 1800 python scripts/opbench.py --tune 0,20 --degrees ${DEGREES:-2,3,4,5,6,7,8,9,10,11,12,13,14,15} > $O/ab_c3.jsonl 2>> $O/ab.err; echo "ab c3 rc=$?" >> $O/status.txt
timeout 900 python scripts/opbench.py --tune 21,22,23,24,25 --degrees 7 --tune-box 16,16,16 > $O/regs_c2.jsonl 2>> $O/ab.err; echo "regs c2 rc=$?" >> $O/status.txt
