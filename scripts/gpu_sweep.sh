#!/bin/bash
# Throughput of the default launch shape on every SURVEY §8(d) configuration, plus GCOF timings.
mkdir -p gpurun_out; rm -f gpurun_out/sweep.txt gpurun_out/gcof.txt
for w in c1 c2 c2k8 c3 c4 c4pcie; do
  timeout 300 python scripts/prof_eval.py --workload $w --rows 1048576 --iters 3 >> gpurun_out/sweep.txt 2>&1
done
for spec in "c5:1000:2 65536" "c5:1000:4 65536" "c5:1000:8 65536" "c5:2000:4 32768" "c5:5000:8 16384" "c5:10000:8 16384" "c5:20000:8 4096" "c5:50000:8 2048" "c5:100000:8 1024"; do
  set -- $spec
  timeout 900 python scripts/prof_eval.py --workload $1 --rows $2 --iters 2 >> gpurun_out/sweep.txt 2>&1
done
timeout 900 python scripts/bench_gcof.py > gpurun_out/gcof.txt 2>&1
