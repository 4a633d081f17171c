#!/bin/bash
# One parameterised GPU runner (run under gpurun from the repo root):
#   gpurun --timeout 1800 -- 'bash scripts/gpu.sh tests bench ncu'
# Tasks (any order, each bounded by its own timeout, logs under gpurun_out/):
#   tests       pytest -m gpu (whole suite)        smoke      __graft_entry__.smoke()
#   bench       bench.py (default workload)        benchref   bench.py --impl reference
#   launches    ncu launch list of a short bench   ncu        ncu --set full of the headline kernel
#   sweep       scripts/prof_eval.py on C1-C5      gcof       GCOF timings (scripts/bench_gcof.py)
#   sanitize    compute-sanitizer memcheck/racecheck/synccheck over scripts/sanitize.py
#   bnb         branch-and-bound tests + bench     peaks      on-chip bandwidth microbenchmarks
# Environment: WL (bench/ncu workload, default c2k8), PYTEST_K (pytest -k filter),
# BENCH_ARGS (extra bench.py args), TAG (suffix of the output names).
mkdir -p gpurun_out
WL=${WL:-c2k8}
TAG=${TAG:-}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks_event_reasons.active --format=csv > gpurun_out/gpu$TAG.txt 2>&1
for task in "$@"; do
  echo "=== $task $(date +%T)" >> gpurun_out/tasks$TAG.log
  case $task in
    tests)
      if [ -n "$PYTEST_K" ]; then K=(-k "$PYTEST_K"); else K=(); fi
      timeout 2400 python -m pytest tests -m gpu -x -q "${K[@]}" > gpurun_out/pytest_gpu$TAG.log 2>&1
      echo "rc=$?" >> gpurun_out/pytest_gpu$TAG.log ;;
    smoke)
      timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke$TAG.log 2>&1
      echo "rc=$?" >> gpurun_out/smoke$TAG.log ;;
    bench)
      timeout 900 python bench.py --workload $WL $BENCH_ARGS > gpurun_out/bench_$WL$TAG.json 2> gpurun_out/bench_$WL$TAG.err ;;
    benchref)
      timeout 900 python bench.py --impl reference --workload $WL > gpurun_out/benchref_$WL$TAG.json 2> gpurun_out/benchref_$WL$TAG.err ;;
    launches)
      timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
        --log-file gpurun_out/launches_$WL$TAG.csv python bench.py --workload $WL --steps 2 --warmup 3 --no-cpu \
        --no-local-search > gpurun_out/launches_$WL$TAG.log 2>&1 ;;
    ncu)
      timeout 1200 ncu --set full --clock-control none --import-source on -k regex:${NCU_KERNEL:-mp_tpps_kernel} -s 3 -c 1 \
        -o gpurun_out/ncu_$WL$TAG -f python bench.py --workload $WL --steps 1 --warmup 3 --no-cpu --no-local-search \
        > gpurun_out/ncu_$WL$TAG.log 2>&1 ;;
    sweep)
      rm -f gpurun_out/sweep$TAG.txt
      for w in c1 c2 c2k8 c3 c4 c4pcie; do
        timeout 300 python scripts/prof_eval.py --workload $w --rows 1048576 --iters 3 >> gpurun_out/sweep$TAG.txt 2>&1
      done
      for spec in "c5:1000:2 65536" "c5:1000:4 65536" "c5:1000:8 65536" "c5:2000:4 32768" "c5:5000:8 16384" \
                  "c5:10000:8 16384" "c5:20000:8 9472" "c5:50000:8 4736" "c5:100000:8 4736"; do
        set -- $spec
        timeout 900 python scripts/prof_eval.py --workload $1 --rows $2 --iters 2 >> gpurun_out/sweep$TAG.txt 2>&1
      done ;;
    gcof)
      timeout 900 python scripts/bench_gcof.py > gpurun_out/gcof$TAG.txt 2>&1 ;;
    sanitize)
      for tool in memcheck racecheck synccheck; do
        timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize.py \
          > gpurun_out/sanitize_$tool$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/sanitize_$tool$TAG.log
      done ;;
    bnb)
      timeout 900 python -m pytest tests/test_gpu_bnb.py -x -q > gpurun_out/pytest_bnb$TAG.log 2>&1
      timeout 900 python scripts/bench_bnb.py --oracle --accept8 > gpurun_out/bench_bnb$TAG.jsonl 2> gpurun_out/bench_bnb$TAG.err ;;
    *)
      echo "unknown task $task" >> gpurun_out/tasks$TAG.log ;;
  esac
done
echo "=== done $(date +%T)" >> gpurun_out/tasks$TAG.log
