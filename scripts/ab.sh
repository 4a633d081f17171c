#!/bin/bash
# A/B timing of evaluator variants (scripts/prof_eval.py flags) on the named workloads,
# then the evaluator parity tests.  AB_FLAGS: ';'-separated flag sets, each timed
# after the default configuration, e.g.
#   gpurun -- 'WL="c2 c2k8" AB_FLAGS="--no-tail;--no-tail --no-evict-first" bash scripts/ab.sh'
mkdir -p gpurun_out; rm -f gpurun_out/ab.txt
IFS=';' read -ra VARIANTS <<< "${AB_FLAGS:---round1}"
for w in ${WL:-c2 c2k8 c1 c4}; do
  for f in "" "${VARIANTS[@]}"; do
    echo "[$w] flags: ${f:-default}" >> gpurun_out/ab.txt
    timeout 300 python scripts/prof_eval.py --workload $w --rows 1048576 --iters 3 $f >> gpurun_out/ab.txt 2>&1
  done
done
if [ -z "$AB_NO_TESTS" ]; then
  timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py -x -q -k "eval or workload or local or scale or trace" > gpurun_out/pytest_ab.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_ab.log
fi
