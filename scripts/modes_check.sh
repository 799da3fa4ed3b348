#!/bin/bash
# Under gpurun: every kernel path once (all_paths.py) and every bench mode once (short runs).
mkdir -p gpurun_out
timeout 600 python scripts/all_paths.py > gpurun_out/all_paths.log 2>&1; echo "all_paths rc=$?" >> gpurun_out/all_paths.log
for m in "--mode lpi" "--mode mlw" "--config 2 --mode match" "--config 2 --mode cross" "--config 2 --periodic" "--config 3 --mode match" "--config 1"; do
  tag=$(echo $m | tr -d ' -')
  timeout 600 python bench.py $m --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/mode_${tag}.json 2> gpurun_out/mode_${tag}.err
  echo "$m rc=$? $(head -c 300 gpurun_out/mode_${tag}.json)" >> gpurun_out/modes_summary.txt
done
