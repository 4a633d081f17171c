#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "gcof or fuse or smoke or coarsen or cycle or golden or aux" > gpurun_out/pytest_gcof.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gcof.log
timeout 600 python scripts/time_coarsen_native.py > gpurun_out/coarsen_native.txt 2>&1
timeout 900 python scripts/bench_gcof.py > gpurun_out/gcof.txt 2>&1
