#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "gcof or fuse or smoke or coarsen or cycle" > gpurun_out/pytest_gcof.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gcof.log
timeout 900 python scripts/bench_gcof.py 20000 50000 100000 > gpurun_out/gcof.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/gcof_launches.csv python scripts/gcof_kernels.py 100000 > gpurun_out/gcof_ncu.log 2>&1
