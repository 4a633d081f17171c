#!/bin/bash
mkdir -p gpurun_out; rm -f gpurun_out/c5big.txt
for spec in "c5:20000:8 9472" "c5:50000:8 4736" "c5:100000:8 4736"; do set -- $spec; timeout 900 python scripts/prof_eval.py --workload $1 --rows $2 --iters 2 >> gpurun_out/c5big.txt 2>&1; done
