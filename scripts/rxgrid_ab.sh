#!/bin/bash
# C5 launch-phase A/B of the receiver-grid cell size (NRT_RX_GRID_V, metres; default 0.5)
for r in 1 2; do for v in 0.5 0.35 0.75 1.0; do
NRT_RX_GRID_V=$v timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "
import json,statistics,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); ph=d['phase_ms_build_launch_refine']
print('v=$v', 'step', round(d['ms_per_step'],1), 'launch median', round(statistics.median(p[1] for p in ph),1), 'trace', round(d['breakdown_ms']['trace'],1), 'coarse', d['coarse_paths'], d['bounces_per_step'])"
done; done
