#!/bin/bash
# A/B of the off-chip group kernel on the C5 sweep points (scripts/prof_eval.py), each
# point also with C5_AB (a prof_eval flag, e.g. --no-rhead) when set, + its parity tests.
mkdir -p gpurun_out; rm -f gpurun_out/c5ab.txt
for spec in "c5:1000:4 65536" "c5:2000:4 32768" "c5:5000:8 16384" "c5:10000:8 16384" "c5:20000:8 9472" "c3 1048576"; do
  set -- $spec
  for f in "" ${C5_AB:+"$C5_AB"}; do
    timeout 900 python scripts/prof_eval.py --workload $1 --rows $2 --iters 2 $f >> gpurun_out/c5ab.txt 2>&1
  done
done
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py -x -q -k "eval or workload or local or scale or trace" > gpurun_out/pytest_c5ab.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_c5ab.log
