#!/bin/bash
# A/B of compile-time variants (scripts/build_variant.py) against the in-tree library:
#   gpurun -- 'VARIANTS="su1 foo" WL="c2k8 c2" bash scripts/abv.sh'
# Each workload is timed default, variants, default again (gpurun_out/abv.txt); then
# the evaluator parity tests run against each variant (gpurun_out/pytest_abv_<v>.log).
mkdir -p gpurun_out; rm -f gpurun_out/abv.txt
for w in ${WL:-c2k8 c2}; do
  for v in default $VARIANTS default; do
    if [ "$v" = default ]; then unset MOIRAI_B200_LIB; else export MOIRAI_B200_LIB=build/variants/$v/libmoirai_b200.so; fi
    echo "[$w] $v" >> gpurun_out/abv.txt
    timeout 300 python scripts/prof_eval.py --workload $w --rows 1048576 --iters 3 >> gpurun_out/abv.txt 2>&1
  done
done
if [ -z "$AB_NO_TESTS" ]; then
  for v in $VARIANTS; do
    MOIRAI_B200_LIB=build/variants/$v/libmoirai_b200.so timeout 1500 python -m pytest tests/test_gpu_parity.py \
      tests/test_gpu_scale.py -x -q -k "eval or workload or local or scale or trace" > gpurun_out/pytest_abv_$v.log 2>&1
    echo "rc=$?" >> gpurun_out/pytest_abv_$v.log
  done
fi
