#!/bin/bash
# Usage (under gpurun): bash scripts/gpu_prof.sh <tag> <config> [kernel-regex] [skip]
TAG=$1; CFG=$2; KRE=${3:-af_rows_kernel}; SKIP=${4:-2}
mkdir -p gpurun_out
timeout 600 python bench.py --config $CFG --steps 2 --warmup 3 --no-cpu-baseline --settle-s 0 > gpurun_out/plain_${TAG}.log 2>&1
echo "plain exit=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:$KRE -s $SKIP -c 1 \
  -o gpurun_out/prof_${TAG} python bench.py --config $CFG --steps 2 --warmup 3 --no-cpu-baseline --settle-s 0 > gpurun_out/ncu_${TAG}.log 2>&1
echo "ncu exit=$?"
