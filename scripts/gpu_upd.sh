#!/bin/bash
# cg_update_fused<U, MINB> A/B at C2 and C3 N=7 (bench, NekBone GFLOP/s + phase times)
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out; mkdir -p $O; : > $O/upd.jsonl
for box in 16,16,16 52,52,52; do
  for cfg in ${UPD_CFGS:-"0 2" "1 2" "0 2" "1 2" "2 1"}; do
    set -- $cfg
    HB_UPD_U=$1 HB_UPD_MINB=$2 timeout 600 python bench.py --no-cpu-baseline --steps 10 --warmup 3 --box $box 2>>$O/upd.err \
      | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'U':$1,'MINB':$2,'box':'$box','value':d['value'],'ph':d['phase_ms_per_iter']}))" >> $O/upd.jsonl
  done
done
cat $O/upd.jsonl
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "cg or jacobi" 2>&1 | tail -2
