#!/bin/bash
# ncu A/B of a variant library (vlib/libgraf_f2.so, built with scripts/ab_lib.sh conventions) against
# the in-tree one on c5/c4/c2; run under gpurun.  Development tool.
mkdir -p gpurun_out
for c in 5 4 2; do
 for L in "" vlib/libgraf_f2.so; do
  tag=$([ -z "$L" ] && echo base || echo f2)
  if [ -n "$L" ]; then export GRAF_LIB_PATH=$L; else unset GRAF_LIB_PATH; fi
  sk=2; [ $c = 4 ] && sk=3
  timeout 900 ncu --section InstructionStats --section WarpStateStats --section SpeedOfLight --section ComputeWorkloadAnalysis --section LaunchStats --section Occupancy \
    --clock-control none -k regex:af_rows_kernel -s $sk -c 1 -o gpurun_out/ab_${tag}_c$c python bench.py --config $c --steps 1 --warmup 3 --no-cpu-baseline --settle-s 0 > gpurun_out/abncu_${tag}_c$c.log 2>&1
  echo "$tag c$c exit=$?"
 done
done
