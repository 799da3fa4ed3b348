#!/bin/bash
# Under gpurun: ncu --set full captures of c4's two passes (af_rows_kernel<8192, K_FWD> with the band
# cache write, af_rows_kernel<8192, K_PASS2> reading it), summaries + per-phase stall split.
TAG=${TAG:-c4}
mkdir -p gpurun_out
for K in 0 2; do
  timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k "regex:af_rows_kernel<\\(int\\)8192, \\(int\\)$K," -s 2 -c 1 -o gpurun_out/prof_${TAG}_k$K \
    python bench.py --config 4 --steps 1 --warmup 3 --no-cpu-baseline --settle-s 0 > gpurun_out/ncu_${TAG}_k$K.log 2>&1
  echo "ncu k$K exit=$?"
  python scripts/ncu_summary.py gpurun_out/prof_${TAG}_k$K.ncu-rep gpurun_out/sum_${TAG}_k$K.txt > /dev/null 2>&1
  ncu -i gpurun_out/prof_${TAG}_k$K.ncu-rep --page source --csv --print-source sass > gpurun_out/sass_${TAG}_k$K.csv 2>/dev/null
  python scripts/ncu_phases.py gpurun_out/sass_${TAG}_k$K.csv > gpurun_out/phases_${TAG}_k$K.txt 2>&1
  rm -f gpurun_out/sass_${TAG}_k$K.csv
done
