#!/bin/bash
# One development iteration on the GPU box: parity tests, then every bench line.
# Usage (under gpurun): [SKIP_TESTS=1] bash scripts/gpu_iter.sh <tag> [configs...]
TAG=$1; shift; CFGS=${@:-2 3 4 5}
mkdir -p gpurun_out
if [ -z "$SKIP_TESTS" ]; then
  timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/tests_$TAG.log 2>&1
  echo "tests exit=$?"; tail -3 gpurun_out/tests_$TAG.log
fi
bash scripts/bench_all.sh $TAG $CFGS
timeout 600 python bench.py --config 3 --mode forward --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_${TAG}_c3fwd.json 2> gpurun_out/bench_${TAG}_c3fwd.err
python -c "import json; d=json.load(open('gpurun_out/bench_${TAG}_c3fwd.json')); r=d['roofline']; print('c3fwd', d['ms_per_step'], r['bound'], r['frac'])"
timeout 600 python bench.py --config 2 --periodic --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_${TAG}_c2per.json 2> gpurun_out/bench_${TAG}_c2per.err
python -c "import json; d=json.load(open('gpurun_out/bench_${TAG}_c2per.json')); r=d['roofline']; print('c2per', d['ms_per_step'], r['bound'], r['frac'])"
timeout 600 python bench.py --mode lpi --steps 10 --warmup 3 > gpurun_out/bench_${TAG}_lpi.json 2> gpurun_out/bench_${TAG}_lpi.err
python -c "import json; d=json.load(open('gpurun_out/bench_${TAG}_lpi.json')); print('lpi it/s', d['value'], 'full2000 ms', d['config']['full_2000_iterations_ms'], 'loss', d['config']['final_loss_median'])"
timeout 600 python bench.py --config 2 --mode match --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_${TAG}_c2match.json 2> gpurun_out/bench_${TAG}_c2match.err
timeout 900 python bench.py --config 3 --mode match --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_${TAG}_c3match.json 2> gpurun_out/bench_${TAG}_c3match.err
python -c "
import json
for c in ('c2match','c3match'):
    d=json.load(open('gpurun_out/bench_${TAG}_'+c+'.json')); r=d['roofline']; print(c, d['ms_per_step'], r['bound'], r['frac'])"
timeout 600 python bench.py --config 2 --mode cross --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_${TAG}_c2cross.json 2> gpurun_out/bench_${TAG}_c2cross.err
python -c "import json; d=json.load(open('gpurun_out/bench_${TAG}_c2cross.json')); r=d['roofline']; print('c2cross', d['ms_per_step'], r['bound'], r['frac'])"
timeout 300 python bench.py --mode mlw --steps 20 --warmup 3 > gpurun_out/bench_${TAG}_mlw.json 2> gpurun_out/bench_${TAG}_mlw.err
python -c "import json; d=json.load(open('gpurun_out/bench_${TAG}_mlw.json')); print('mlw', d['ms_per_step'], d['value'])"
