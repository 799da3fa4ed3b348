#!/bin/bash
# GPU test run under gpurun: new parity files first (with achieved-error log), then the suite.
mkdir -p gpurun_out
export GRAF_PARITY_LOG=gpurun_out/parity_errors.jsonl
rm -f $GRAF_PARITY_LOG
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
timeout ${T1:-1200} python -m pytest ${FILES:-tests/test_gpu_softpsl_parity.py tests/test_gpu_c3_pins.py} -q -s -m gpu -p no:cacheprovider --timeout=600 > gpurun_out/pytest_new.log 2>&1
echo "new tests exit $?" >> gpurun_out/pytest_new.log
if [ -z "$NOSUITE" ]; then
timeout ${T2:-1800} python -m pytest tests -q -m gpu -x -p no:cacheprovider --timeout=600 > gpurun_out/pytest_all.log 2>&1
echo "suite exit $?" >> gpurun_out/pytest_all.log
fi
