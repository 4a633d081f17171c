#!/bin/bash
mkdir -p gpurun_out; rm -f gpurun_out/exp.txt
for args in "--rows 1048576" "--rows 1048576 --rcap 4" "--rows 1048576 --rcap 3"; do
  timeout 300 python scripts/prof_eval.py --workload c2 --iters 3 $args >> gpurun_out/exp.txt 2>&1
done
