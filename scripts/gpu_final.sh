#!/bin/bash
bash scripts/gpu_round.sh
bash scripts/gpu_sweep.sh
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/gcof_launches.csv python scripts/gcof_kernels.py 100000 > gpurun_out/gcof_ncu.log 2>&1
