#!/bin/bash
# Operator variants of one degree each from prebuilt tuning libraries (lib/t<N>/, built with
# HB_LIBDIR=.../lib/t<N> HB_TUNE=1 HB_TUNE_N=<N>): each is swapped in as lib/libhipbone_b200.so,
# its variants checked for parity (multi-wave apply, C3 sampled, CG) and timed inside the CG at
# the C3 box of N.  TUNE_NV="15:0,80,81 13:0,89" ; plain library restored at the end.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out; mkdir -p $O; L=paper_2202_12477_b200/lib
export HB_PREBUILT=1 HB_TUNE=1
cp $L/libhipbone_b200.so /tmp/plain.so
: > $O/tune_insitu.jsonl
for nv in ${TUNE_NV}; do
  n=${nv%%:*}; vs=${nv##*:}
  if [ "${n:0:1}" = "p" ]; then n=${n:1}; cp /tmp/plain.so $L/libhipbone_b200.so; tag=plain  # "p<N>": the plain library
  else cp $L/t$n/libhipbone_b200.so $L/libhipbone_b200.so; tag=t$n; fi
  b=${BOX:-}; [ -n "$b" ] || b=$(python -c "print({1:'120,100,91',2:'184,184,184',3:'122,122,122',4:'92,92,92',5:'73,73,73',6:'61,61,61',7:'52,52,52',8:'46,46,46',9:'41,41,41',10:'37,37,37',11:'33,33,33',12:'31,31,31',13:'28,28,28',14:'26,26,26',15:'24,24,24'}[$n])")
  for v in ${vs//,/ }; do
    if { [ "$v" != "0" ] || [ "$tag" != "plain" ]; } && [ -z "$NO_PARITY" ]; then
      HB_AX_VARIANT=$v HB_AX_VN=$n timeout 600 python -m pytest -q -x \
        "tests/test_gpu_parity.py::test_apply_multiwave_random_geometry[$n]" \
        "tests/test_gpu_parity.py::test_full_size_C3_sampled_and_properties[box$((n-1))-$n]" \
        $(python -m pytest tests/test_gpu_parity.py --collect-only -q 2>/dev/null | grep "random_geometry_both_mass_modes\[$n-0\]") \
        ${PAR_EXTRA} > $O/tune_par_${tag}_${n}_$v.log 2>&1
      echo "parity $tag n$n v$v rc=$?" >> $O/status.txt
    fi
    for rep in $(seq 1 ${REPS:-1}); do
      HB_AX_VARIANT=$v HB_AX_VN=$n timeout 600 python bench.py --N $n --box $b --steps ${STEPS:-3} --warmup 3 --no-cpu-baseline --no-c3 \
        | sed "s/^{/{\"lib\": \"$tag\", \"variant\": \"$v\", /" >> $O/tune_insitu.jsonl 2>> $O/tune.err
    done
  done
done
cp /tmp/plain.so $L/libhipbone_b200.so
echo "tune done" >> $O/status.txt
