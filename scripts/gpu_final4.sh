#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "gcof or fuse or coarsen or cycle" > gpurun_out/pytest_gcof.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gcof.log
timeout 1500 compute-sanitizer --tool racecheck --print-limit 20 python scripts/sanitize.py > gpurun_out/sanitize_racecheck.log 2>&1; echo "rc=$?" >> gpurun_out/sanitize_racecheck.log
timeout 1500 compute-sanitizer --tool memcheck --print-limit 20 python scripts/sanitize.py > gpurun_out/sanitize_memcheck.log 2>&1; echo "rc=$?" >> gpurun_out/sanitize_memcheck.log
timeout 600 python scripts/time_coarsen_native.py 100000 > gpurun_out/cn100k.txt 2>&1
