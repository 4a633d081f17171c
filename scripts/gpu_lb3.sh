#!/bin/bash
mkdir -p gpurun_out; rm -f gpurun_out/lb3.txt
for spec in "c3 1048576" "c5:1000:4 65536" "c5:2000:4 32768" "c5:5000:8 16384" "c5:10000:8 16384"; do set -- $spec; timeout 400 python scripts/prof_eval.py --workload $1 --rows $2 --iters 3 --ctas-per-sm 3 >> gpurun_out/lb3.txt 2>&1; done
