#!/bin/bash
# A/B timing of the thread-per-placement evaluator against the round-1 one
# (scripts/prof_eval.py --round1) on the named workloads, then the evaluator parity tests.
#   gpurun -- 'WL="c2 c2k8" bash scripts/ab.sh'
mkdir -p gpurun_out; rm -f gpurun_out/ab.txt
for w in ${WL:-c2 c2k8 c1 c4}; do
  for f in "" ${AB_FLAGS:-"--round1"}; do timeout 300 python scripts/prof_eval.py --workload $w --rows 1048576 --iters 3 $f >> gpurun_out/ab.txt 2>&1; done
done
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py -x -q -k "eval or workload or local or scale or trace" > gpurun_out/pytest_ab.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_ab.log
