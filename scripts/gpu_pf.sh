#!/bin/bash
mkdir -p gpurun_out; rm -f gpurun_out/pf.txt
for spec in "c3 1048576" "c5:1000:4 65536" "c5:2000:4 32768" "c5:5000:8 16384" "c5:10000:8 16384" "c5:20000:8 9472"; do set -- $spec; timeout 400 python scripts/prof_eval.py --workload $1 --rows $2 --iters 3 >> gpurun_out/pf.txt 2>&1; done
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/pytest_pf.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_pf.log
