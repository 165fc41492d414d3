#!/bin/bash
# In-situ (inside the CG) A/B in a tuning build (HB_TUNE: op.cu tune_variant, tune_env knobs):
#   BENCH_NV="7:30 7:31 ..." [REPS=1]   bench.py per (N, operator variant) at the C3 box of N
#   C2_VARIANTS="0 9" [C2_REPS=2]        C2 bench per N=7 operator variant
#   C2_ENV_AB="HB_X=1"                   C2 bench with and without an environment knob
#   ENV_LIST="HB_UPD_U=1;HB_UPD_U=2 HB_UPD_MINB=1" [REPS=2]   C2 bench per environment setting
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out; mkdir -p $O
export HB_TUNE=1
python -c "import __graft_entry__ as g; g.build()" > $O/build_tune.log 2>&1; echo "tune build rc=$?" > $O/status.txt
: > $O/insitu.jsonl
for rep in $(seq 1 ${REPS:-1}); do
for nv in ${BENCH_NV:-}; do
  n=${nv%%:*}; v=${nv##*:}
  b=$(python -c "print({1:'120,100,91',2:'184,184,184',3:'122,122,122',4:'92,92,92',5:'73,73,73',6:'61,61,61',7:'52,52,52',8:'46,46,46',9:'41,41,41',10:'37,37,37',11:'33,33,33',12:'31,31,31',13:'28,28,28',14:'26,26,26',15:'24,24,24'}[$n])")
  HB_AX_VARIANT=$v HB_AX_VN=$n timeout 600 python bench.py --N $n --box $b --steps 3 --warmup 3 --no-cpu-baseline --no-c3 \
    | sed "s/^{/{\"variant\": \"$v\", /" >> $O/insitu.jsonl 2>> $O/insitu.err
done
done
echo "insitu done" >> $O/status.txt
if [ -n "$C2_ENV_AB" ]; then  # C2 default bench with and without an env knob (tuning build)
  : > $O/c2_env.jsonl
  for rep in 1 2 3; do
    timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-c3 | sed 's/^{/{"knob": "off", /' >> $O/c2_env.jsonl 2>> $O/insitu.err
    env $C2_ENV_AB timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-c3 | sed 's/^{/{"knob": "on", /' >> $O/c2_env.jsonl 2>> $O/insitu.err
  done
  echo "c2 env done" >> $O/status.txt
fi
if [ -n "$C2_VARIANTS" ]; then  # C2 default bench per N=7 tune variant, interleaved repeats
  : > $O/c2_variants.jsonl
  for rep in $(seq 1 ${C2_REPS:-2}); do
    for v in $C2_VARIANTS; do
      HB_AX_VARIANT=$v HB_AX_VN=7 timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-c3 | sed "s/^{/{\"variant\": \"$v\", /" >> $O/c2_variants.jsonl 2>> $O/insitu.err
    done
  done
  echo "c2 variants done" >> $O/status.txt
fi
if [ -n "$ENV_LIST" ]; then
  : > $O/env_ab.jsonl
  IFS=';' read -ra ENVS <<< "$ENV_LIST"
  for rep in $(seq 1 ${REPS:-2}); do
    for e in "${ENVS[@]}"; do
      env $e timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-c3 \
        | sed "s/^{/{\"env\": \"$e\", /" >> $O/env_ab.jsonl 2>> $O/insitu.err
    done
  done
  echo "env ab done" >> $O/status.txt
fi
