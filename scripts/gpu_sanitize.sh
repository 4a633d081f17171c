#!/bin/bash
mkdir -p gpurun_out
timeout 300 python scripts/sanitize.py > gpurun_out/sanitize_plain.log 2>&1; echo "rc=$?" >> gpurun_out/sanitize_plain.log
timeout 1500 compute-sanitizer --tool memcheck --print-limit 20 python scripts/sanitize.py > gpurun_out/sanitize_memcheck.log 2>&1; echo "rc=$?" >> gpurun_out/sanitize_memcheck.log
timeout 1500 compute-sanitizer --tool racecheck --print-limit 20 python scripts/sanitize.py > gpurun_out/sanitize_racecheck.log 2>&1; echo "rc=$?" >> gpurun_out/sanitize_racecheck.log
timeout 900 compute-sanitizer --tool synccheck --print-limit 20 python scripts/sanitize.py > gpurun_out/sanitize_synccheck.log 2>&1; echo "rc=$?" >> gpurun_out/sanitize_synccheck.log
