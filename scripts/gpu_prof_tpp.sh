#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/pytest_parity.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_parity.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:mp_tpp -s 1 -c 1 -o gpurun_out/tpp_c2 -f python scripts/prof_eval.py --workload c2 --rows 262144 --iters 1 > gpurun_out/ncu_tpp.log 2>&1
