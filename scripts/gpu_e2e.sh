#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "large_graph or device_pointer or edge_case or workload" > gpurun_out/pytest_e2e.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_e2e.log
timeout 600 python bench.py --steps 10 --no-cpu > gpurun_out/bench_e2e.json 2> gpurun_out/bench_e2e.err
