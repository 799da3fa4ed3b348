#!/bin/bash
# Usage (under gpurun): [EXTRA="--mode forward"] bash scripts/gpu_prof.sh <tag> <config> [kernel-regex] [skip]
# Runs the bench command once plain (must exit 0), then one ncu --set full capture of the kernel.
TAG=$1; CFG=$2; KRE=${3:-af_rows_kernel}; SKIP=${4:-2}
mkdir -p gpurun_out
timeout 600 python bench.py --config $CFG $EXTRA --steps 5 --warmup 3 --no-cpu-baseline --settle-s 0.5 > gpurun_out/plain_${TAG}.json 2> gpurun_out/plain_${TAG}.err
echo "plain $TAG exit=$?"; cat gpurun_out/plain_${TAG}.json | python -c "import json,sys; d=json.load(sys.stdin); print(d['ms_per_step'], d['roofline']['frac'], d['roofline']['kernel_ms'])" 2>/dev/null
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:$KRE -s $SKIP -c 1 \
  -o gpurun_out/prof_${TAG} python bench.py --config $CFG $EXTRA --steps 1 --warmup 3 --no-cpu-baseline --settle-s 0 > gpurun_out/ncu_${TAG}.log 2>&1
echo "ncu $TAG exit=$?"
# summarise on the box (reports of the big kernels exceed gpurun's 64 MiB return limit)
python scripts/ncu_summary.py gpurun_out/prof_${TAG}.ncu-rep gpurun_out/sum_${TAG}.txt > /dev/null 2>&1
python scripts/ncu_mix.py gpurun_out/prof_${TAG}.ncu-rep > gpurun_out/mix_${TAG}.txt 2>&1
SZ=$(stat -c %s gpurun_out/prof_${TAG}.ncu-rep 2>/dev/null || echo 0)
if [ "$SZ" -gt 25000000 ]; then rm -f gpurun_out/prof_${TAG}.ncu-rep; fi
