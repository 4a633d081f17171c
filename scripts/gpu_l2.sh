#!/bin/bash
mkdir -p gpurun_out; rm -f gpurun_out/l2.txt
for mb in 0 32 64 96 128; do
  for w in c2 c1; do echo "MB=$mb" >> gpurun_out/l2.txt; MP_L2_PERSIST_MB=$mb timeout 300 python scripts/prof_eval.py --workload $w --rows 1048576 --iters 3 >> gpurun_out/l2.txt 2>&1; done
done
