#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "gcof or fuse or smoke or coarsen or cycle" > gpurun_out/pytest_gcof.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gcof.log
timeout 900 python scripts/bench_gcof.py > gpurun_out/gcof.txt 2>&1
bash scripts/gpu_gcof_small.sh
timeout 1500 compute-sanitizer --tool racecheck --print-limit 20 python scripts/sanitize.py > gpurun_out/sanitize_racecheck.log 2>&1; echo "rc=$?" >> gpurun_out/sanitize_racecheck.log
