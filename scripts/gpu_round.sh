#!/bin/bash
# Under gpurun: GPU tests (new files first), then the default bench line and the per-config lines.
# Usage: TAG=r02a bash scripts/gpu_round.sh
TAG=${TAG:-r02}
mkdir -p gpurun_out
FILES="${FILES:-tests/test_gpu_softpsl_parity.py tests/test_gpu_c3_pins.py}" NOSUITE=${NOSUITE:-} bash scripts/gpu_tests.sh
timeout 900 python bench.py > gpurun_out/bench_${TAG}_default.json 2> gpurun_out/bench_${TAG}_default.err
echo "default rc=$?" >> gpurun_out/bench_${TAG}_default.err
bash scripts/bench_all.sh ${TAG} ${CFGS:-2 3 4} > gpurun_out/bench_${TAG}_summary.txt 2>&1
timeout 600 python bench.py --config 3 --mode forward --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_${TAG}_c3fwd.json 2>> gpurun_out/bench_${TAG}_summary.txt
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_${TAG}_ref.json 2>> gpurun_out/bench_${TAG}_summary.txt
