#!/bin/bash
# CTAs-per-waveform sweep (GRAF_FORCE_P) for c2, c4, c5; run under gpurun
for P in 0 1 3 4 5 8; do echo "P=$P $(GRAF_FORCE_P=$P python scripts/c2_rows.py 64 256 2>/dev/null | head -1)"; done
for P in 0 6 8 12 16 18; do GRAF_FORCE_P=$P python bench.py --config 4 --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c4 P=$P', d['ms_per_step'])"; done
for P in 0 19 74; do GRAF_FORCE_P=$P python bench.py --config 5 --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c5 P=$P', d['ms_per_step'])"; done
