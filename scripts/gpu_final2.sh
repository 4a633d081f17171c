#!/bin/bash
mkdir -p gpurun_out
bash scripts/gpu_round.sh
bash scripts/gpu_sweep.sh
timeout 1500 compute-sanitizer --tool memcheck --print-limit 20 python scripts/sanitize.py > gpurun_out/sanitize_memcheck.log 2>&1; echo "rc=$?" >> gpurun_out/sanitize_memcheck.log
timeout 1500 compute-sanitizer --tool racecheck --print-limit 20 python scripts/sanitize.py > gpurun_out/sanitize_racecheck.log 2>&1; echo "rc=$?" >> gpurun_out/sanitize_racecheck.log
timeout 900 compute-sanitizer --tool synccheck --print-limit 20 python scripts/sanitize.py > gpurun_out/sanitize_synccheck.log 2>&1; echo "rc=$?" >> gpurun_out/sanitize_synccheck.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/gcof_launches.csv python scripts/gcof_kernels.py 100000 > gpurun_out/gcof_ncu.log 2>&1
