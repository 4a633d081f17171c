#!/bin/bash
mkdir -p gpurun_out
for w in c2 c3; do timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/gcof_launches_$w.csv python scripts/gcof_kernels.py $w > gpurun_out/gcof_ncu_$w.log 2>&1; done
