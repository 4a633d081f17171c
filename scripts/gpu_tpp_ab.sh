#!/bin/bash
# TPP kernels: parity suite + default-shape throughput on C1-C4 + shared-memory conflict counters
mkdir -p gpurun_out; rm -f gpurun_out/tpp_ab.txt
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_tpp_ab.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_tpp_ab.log
for w in c1 c2 c2k8 c4; do
  timeout 300 python scripts/prof_eval.py --workload $w --rows 1048576 --iters 3 >> gpurun_out/tpp_ab.txt 2>&1
done
timeout 300 python scripts/prof_eval.py --workload c2 --rows 1048576 --iters 3 --tpp-reg >> gpurun_out/tpp_ab.txt 2>&1
timeout 600 ncu --clock-control none -k regex:mp_tpps -s 1 -c 1 --metrics l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed,gpu__time_duration.sum python scripts/prof_eval.py --workload c2 --rows 1048576 --iters 1 > gpurun_out/ncu_tpp_ab.log 2>&1
