#!/bin/bash
# quick perf + parity check: prof_eval on the given workloads, then the eval parity tests
mkdir -p gpurun_out; rm -f gpurun_out/quick.txt
for w in ${WL:-c2 c4}; do timeout 300 python scripts/prof_eval.py --workload $w --rows 1048576 --iters 3 $PE_ARGS >> gpurun_out/quick.txt 2>&1; done
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "eval or workload or local" > gpurun_out/pytest_quick.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_quick.log
