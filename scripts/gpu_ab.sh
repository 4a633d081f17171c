#!/bin/bash
mkdir -p gpurun_out; rm -f gpurun_out/ab.txt
for w in c1 c2; do
  timeout 300 python scripts/prof_eval.py --workload $w --rows 1048576 --iters 3 >> gpurun_out/ab.txt 2>&1
done
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
