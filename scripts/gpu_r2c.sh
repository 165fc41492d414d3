#!/bin/bash
# Product build: ncu launch lists (cold and warm cache) and captures; tuning build: racecheck of
# the sanitizer workload without the cooperative update (racecheck does not run it).
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out; mkdir -p $O
STAGES="ncu ncuvec" bash scripts/gpu_run.sh
cp $O/status.txt $O/status_product.txt
export HB_TUNE=1
python -c "import __graft_entry__ as g; g.build()" > $O/build_tune.log 2>&1; echo "tune build rc=$?" >> $O/status_product.txt
HB_FUSED_UPDATE=0 SAN_CASES="2:0,3:1,7:0,8:1,11:1,13:0,15:0" SAN_MULTIWAVE="1,2,7,11,12,13,15" timeout 2400 \
  compute-sanitizer --tool racecheck --print-limit 20 python scripts/sanitize.py > $O/san_racecheck.log 2>&1
echo "racecheck rc=$?" >> $O/status_product.txt
