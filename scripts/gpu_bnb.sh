#!/bin/bash
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_bnb.py -x -q > gpurun_out/pytest_bnb.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_bnb.log
timeout 900 python scripts/bench_bnb.py --oracle --accept8 > gpurun_out/bench_bnb.jsonl 2> gpurun_out/bench_bnb.err
