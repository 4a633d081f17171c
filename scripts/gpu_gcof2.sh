#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "gcof or fuse or smoke or coarsen" > gpurun_out/pytest_gcof.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gcof.log
timeout 900 python scripts/bench_gcof.py > gpurun_out/gcof.txt 2>&1
timeout 600 python scripts/prof_gcof_host.py > gpurun_out/gcof_prof.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_dfs -c 1 -o gpurun_out/dfs_full -f python scripts/gcof_kernels.py 100000 > gpurun_out/ncu_dfs.log 2>&1
