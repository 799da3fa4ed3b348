#!/bin/bash
# A/B of a variant library against the in-tree one: parity subset, then bench lines.
# Usage (under gpurun): bash scripts/ab_lib.sh <variant.so> [tests]
V=$1; T=${2:-1}
mkdir -p gpurun_out
if [ "$T" = 1 ]; then
  GRAF_LIB_PATH=$V timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_periodic.py \
     tests/test_gpu_cross.py tests/test_gpu_match.py tests/test_gpu_section7.py -x -q -p no:cacheprovider > gpurun_out/ab_tests.log 2>&1
  echo "variant tests exit=$?"; tail -2 gpurun_out/ab_tests.log
fi
run() {  # lib tag args...
  local L=$1; shift; local tag=$1; shift
  if [ -n "$L" ]; then export GRAF_LIB_PATH=$L; else unset GRAF_LIB_PATH; fi
  timeout 600 python bench.py "$@" --no-cpu-baseline > gpurun_out/ab_$tag.json 2> gpurun_out/ab_$tag.err
  python -c "import json; d=json.load(open('gpurun_out/ab_$tag.json')); r=d['roofline']; print('$tag', round(d['ms_per_step'],4), r['bound'], round(r['frac'],3), 'e2e', round(d['e2e']['value'],1))"
}
for cfg in "2 --steps 20 --warmup 5" "3 --mode forward --steps 10 --warmup 3" "3 --steps 5 --warmup 3" "4 --steps 10 --warmup 3" "5 --steps 3 --warmup 3"; do
  set -- $cfg; c=$1; shift
  m=$(echo "$cfg" | grep -q forward && echo fwd || echo "")
  run "" base_c$c$m --config $c "$@"
  run "$V" var_c$c$m --config $c "$@"
done
