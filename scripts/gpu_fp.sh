#!/bin/bash
# fused-p variant: parity + A/B against the default at C2 and C3 N=7 (and N=15 C5-size)
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "fused_p or cg_parity" > $O/fp_tests.log 2>&1; echo "tests rc=$?"; tail -3 $O/fp_tests.log
: > $O/fp_ab.jsonl
for args in "" "--box 52,52,52" "--N 15 --box 24,24,24"; do
  for v in 0 2 0 2; do
    timeout 600 python bench.py --no-cpu-baseline --steps 10 --warmup 3 --variant $v $args 2>>$O/fp_ab.err | tail -1 >> $O/fp_ab.jsonl
  done
done
python - <<'PY'
import json
for l in open("gpurun_out/fp_ab.jsonl"):
    try: d=json.loads(l)
    except Exception: print(l[:200]); continue
    print(d["config"]["box"], d["config"]["N"], d["config"]["assembly_variant"], d["value"], d["ms_per_step"], d["phase_ms_per_iter"], d["roofline"]["frac"])
PY
