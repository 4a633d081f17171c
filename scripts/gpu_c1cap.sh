#!/bin/bash
mkdir -p gpurun_out; rm -f gpurun_out/c1cap.txt
for c in 0 8 10 12 14 16; do timeout 300 python scripts/prof_eval.py --workload c1 --rows 1048576 --iters 3 --rcap $c >> gpurun_out/c1cap.txt 2>&1; done
for c in 0 3; do timeout 300 python scripts/prof_eval.py --workload c2 --rows 1048576 --iters 3 --rcap $c >> gpurun_out/c1cap.txt 2>&1; done
