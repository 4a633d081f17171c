#!/bin/bash
bash scripts/gpu_c5c.sh
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_dfs -c 1 -o gpurun_out/dfs_full -f python scripts/gcof_kernels.py 100000 > gpurun_out/ncu_dfs.log 2>&1
