#!/bin/bash
mkdir -p gpurun_out; rm -f gpurun_out/pred.txt
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
for w in c1 c2 c2k8 c3 c4; do timeout 300 python scripts/prof_eval.py --workload $w --rows 1048576 --iters 3 >> gpurun_out/pred.txt 2>&1; done
for spec in "c5:1000:4 65536" "c5:5000:8 16384" "c5:10000:8 16384" "c5:20000:8 4096"; do set -- $spec; timeout 400 python scripts/prof_eval.py --workload $1 --rows $2 --iters 3 >> gpurun_out/pred.txt 2>&1; done
