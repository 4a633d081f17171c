#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/pytest_parity.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_parity.log
timeout 600 python bench.py --steps 5 --no-cpu > gpurun_out/bench_quick.json 2> gpurun_out/bench_quick.err
