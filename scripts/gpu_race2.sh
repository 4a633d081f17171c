#!/bin/bash
mkdir -p gpurun_out
timeout 1500 compute-sanitizer --tool racecheck --print-limit 20 python scripts/sanitize.py > gpurun_out/sanitize_racecheck.log 2>&1; echo "rc=$?" >> gpurun_out/sanitize_racecheck.log
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
rm -f gpurun_out/race_perf.txt
for spec in "c3 1048576" "c5:1000:4 65536" "c5:5000:8 16384"; do set -- $spec; timeout 300 python scripts/prof_eval.py --workload $1 --rows $2 --iters 3 >> gpurun_out/race_perf.txt 2>&1; done
timeout 900 python scripts/bench_gcof.py 100000 > gpurun_out/gcof_race.txt 2>&1
