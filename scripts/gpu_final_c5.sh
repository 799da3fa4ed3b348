#!/bin/bash
# Under gpurun: the default (c5) bench line, its ncu launch list, and one --set full capture of
# the single-pass kernel af_rows_kernel<16384, 2, 0, 0> (the 3rd such launch = step 2's main pass;
# each step also runs two guarded fallback launches whose CTAs exit at once).
TAG=${TAG:-r02g}
mkdir -p gpurun_out
if [ -z "$ONLY_NCU" ]; then
timeout 900 python bench.py > gpurun_out/bench_${TAG}_default.json 2> gpurun_out/bench_${TAG}_default.err
echo "bench exit=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --settle-s 0 > gpurun_out/ncu_launches_${TAG}.log 2>&1
echo "launch list exit=$?"
fi
timeout 1500 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k "regex:af_rows_kernel<\\(int\\)16384, \\(int\\)2," -s 2 -c 1 -o gpurun_out/prof_${TAG}_c5 \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline --settle-s 0 > gpurun_out/ncu_${TAG}_c5.log 2>&1
echo "ncu exit=$?"
python scripts/ncu_summary.py gpurun_out/prof_${TAG}_c5.ncu-rep gpurun_out/sum_${TAG}_c5.txt > /dev/null 2>&1
python scripts/ncu_mix.py gpurun_out/prof_${TAG}_c5.ncu-rep > gpurun_out/mix_${TAG}_c5.txt 2>&1
ncu -i gpurun_out/prof_${TAG}_c5.ncu-rep --page source --csv --print-source sass > gpurun_out/sass_${TAG}_c5.csv 2>/dev/null
python scripts/ncu_phases.py gpurun_out/sass_${TAG}_c5.csv > gpurun_out/phases_${TAG}_c5.txt 2>&1
rm -f gpurun_out/sass_${TAG}_c5.csv
SZ=$(stat -c %s gpurun_out/prof_${TAG}_c5.ncu-rep 2>/dev/null || echo 0)
if [ -z "$KEEP_REP" ] && [ "$SZ" -gt 25000000 ]; then rm -f gpurun_out/prof_${TAG}_c5.ncu-rep; fi
