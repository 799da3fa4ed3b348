#!/bin/bash
# Usage (under gpurun): bash scripts/bench_all.sh <tag> [configs...]
TAG=$1; shift; CFGS=${@:-1 2 3 4 5}
mkdir -p gpurun_out
for c in $CFGS; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_${TAG}_c$c.json 2> gpurun_out/bench_${TAG}_c$c.err
  rc=$?
  python - "$c" "$rc" "gpurun_out/bench_${TAG}_c$c.json" <<'PY'
import json, sys
c, rc, f = sys.argv[1:]
try:
    d = json.load(open(f)); r = d["roofline"]
    print(f"c{c} ms/step={d['ms_per_step']:.4f} surf/s={d['value']:.4g} {r['bound']} frac={r['frac']:.3f} kern_ms={r['kernel_ms']:.4f} e2e={d['e2e']['value']:.4g} clk={d['clocks'].get('sm_mhz')}")
except Exception as e:
    print(f"c{c} rc={rc} failed: {e}")
PY
done
