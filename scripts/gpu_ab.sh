#!/bin/bash
mkdir -p gpurun_out; rm -f gpurun_out/ab.txt
for w in c2 c4; do
  timeout 300 python scripts/prof_eval.py --workload $w --rows 1048576 --iters 3 >> gpurun_out/ab.txt 2>&1
  MOIRAI_B200_LIB=$PWD/paper_2312_04025_b200/libmoirai_b200_su2.so timeout 300 python scripts/prof_eval.py --workload $w --rows 1048576 --iters 3 >> gpurun_out/ab.txt 2>&1
done
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "eval or workload or local" > gpurun_out/pytest_quick.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_quick.log
