#!/bin/bash
# C2 bench (tuning build) under a list of environment settings, REPS repeats each, interleaved.
#   ENV_LIST="HB_UPD_U=1;HB_UPD_U=2 HB_UPD_MINB=1" REPS=2 bash scripts/gpu_env_ab.sh
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out; mkdir -p $O
export HB_TUNE=1
python -c "import __graft_entry__ as g; g.build()" > $O/build_tune.log 2>&1; echo "tune build rc=$?" > $O/status.txt
: > $O/env_ab.jsonl
IFS=';' read -ra ENVS <<< "$ENV_LIST"
for rep in $(seq 1 ${REPS:-2}); do
  for e in "${ENVS[@]}"; do
    env $e timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-c3 ${BENCH_ARGS} \
      | sed "s/^{/{\"env\": \"$e\", /" >> $O/env_ab.jsonl 2>> $O/env_ab.err
  done
done
echo "env ab done" >> $O/status.txt
