#!/bin/bash
mkdir -p gpurun_out
for w in c2 c4 c3 c1; do
  timeout 300 python scripts/prof_eval.py --workload $w --rows 262144 --iters 3 >> gpurun_out/tpp.txt 2>&1
  timeout 300 python scripts/prof_eval.py --workload $w --rows 262144 --iters 3 --no-tpp >> gpurun_out/tpp.txt 2>&1
done
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
