#!/bin/bash
# Local: build (must succeed), CPU tests, then one GPU iteration.  Usage: bash scripts/iter.sh <tag> [configs]
set -o pipefail
TAG=$1; shift
python -c "from paper_2506_22935_b200 import _build; _build.build()" || { echo BUILD_FAILED; exit 1; }
timeout 600 python -m pytest tests -x -q -m "not gpu" 2>&1 | tail -1
/usr/local/graft/bin/gpurun --timeout 1500 -- "bash scripts/gpu_iter.sh $TAG $*" > /tmp/gpu_$TAG.log 2>&1
tail -9 /tmp/gpu_$TAG.log
