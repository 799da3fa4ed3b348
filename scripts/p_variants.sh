#!/bin/bash
# Forced-P variant libraries (scripts/tune.py build <cfg> "<tag>:GRAF_FORCE_P=..") against the
# launch model on the config's batch blocks B, B/2, B/4, B/8.  Usage (under gpurun):
#   bash scripts/p_variants.sh <cfg> [forward]
C=$1; MODE=$2
mkdir -p gpurun_out
OUT=gpurun_out/p_variants_c$C$MODE.txt; : > $OUT
for L in "" paper_2506_22935_b200/variants/libgraf_c${C}_*.so; do
  if [ -n "$L" ]; then export GRAF_LIB_PATH=$PWD/$L; else unset GRAF_LIB_PATH; fi
  [ "$MODE" = forward ] && export GRAF_TUNE_MODE=forward
  timeout 300 python scripts/batch_shard_times.py $C 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read()); lib=d.pop('lib')
for c,v in d.items(): print(lib, c, ' '.join(f\"B={x['B_per_rank']}:{x['ms']:.4f}\" for x in v.values()))" | tee -a $OUT
done
