#!/bin/bash
# One GPU call: parity tests, bench, ncu launch list, ncu full capture of the top kernel.
# Usage (from the repo root, under gpurun): bash scripts/gpu_check.sh <tag> [config]
TAG=${1:-r01}; CFG=${2:-2}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > gpurun_out/gpu_$TAG.txt
lscpu | grep -E "Model name|^CPU\(s\)" >> gpurun_out/gpu_$TAG.txt
if [ -z "$SKIP_TESTS" ]; then
  timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gpu_tests_$TAG.log 2>&1
  echo "tests exit=$?"; tail -3 gpurun_out/gpu_tests_$TAG.log
fi
timeout 600 python bench.py --config $CFG --steps 20 --warmup 5 > gpurun_out/bench_${TAG}_c$CFG.json 2> gpurun_out/bench_${TAG}_c$CFG.err
echo "bench exit=$?"; cat gpurun_out/bench_${TAG}_c$CFG.json; tail -3 gpurun_out/bench_${TAG}_c$CFG.err
if [ -n "$NCU" ]; then
  timeout 600 python bench.py --config $CFG --steps 2 --warmup 3 --no-cpu-baseline --settle-s 0 > gpurun_out/plain_$TAG.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}_c$CFG.csv \
     python bench.py --config $CFG --steps 2 --warmup 3 --no-cpu-baseline --settle-s 0 > gpurun_out/ncu_list_$TAG.log 2>&1
  echo "ncu list exit=$?"
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:af_rows_kernel -s 2 -c 1 \
     -o gpurun_out/prof_${TAG}_c$CFG python bench.py --config $CFG --steps 2 --warmup 3 --no-cpu-baseline --settle-s 0 > gpurun_out/ncu_full_$TAG.log 2>&1
  echo "ncu full exit=$?"
fi
