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
  python scripts/ncu_summary.py gpurun_out/prof_${TAG}_c$CFG.ncu-rep gpurun_out/sum_${TAG}_c$CFG.txt > /dev/null 2>&1
  python scripts/ncu_mix.py gpurun_out/prof_${TAG}_c$CFG.ncu-rep > gpurun_out/mix_${TAG}_c$CFG.txt 2>&1
  ncu -i gpurun_out/prof_${TAG}_c$CFG.ncu-rep --page source --csv --print-source cuda > gpurun_out/src_${TAG}_c$CFG.csv 2>/dev/null
  SZ=$(stat -c %s gpurun_out/prof_${TAG}_c$CFG.ncu-rep 2>/dev/null || echo 0)
  if [ "$SZ" -gt 25000000 ]; then rm -f gpurun_out/prof_${TAG}_c$CFG.ncu-rep; fi
fi
