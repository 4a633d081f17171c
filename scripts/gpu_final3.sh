#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 1500 compute-sanitizer --tool memcheck --print-limit 20 python scripts/sanitize.py > gpurun_out/sanitize_memcheck.log 2>&1; echo "rc=$?" >> gpurun_out/sanitize_memcheck.log
timeout 1500 compute-sanitizer --tool racecheck --print-limit 20 python scripts/sanitize.py > gpurun_out/sanitize_racecheck.log 2>&1; echo "rc=$?" >> gpurun_out/sanitize_racecheck.log
timeout 1500 compute-sanitizer --tool synccheck --print-limit 20 python scripts/sanitize.py > gpurun_out/sanitize_synccheck.log 2>&1; echo "rc=$?" >> gpurun_out/sanitize_synccheck.log
