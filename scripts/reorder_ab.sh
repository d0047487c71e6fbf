#!/bin/bash
# C5 A/B of the per-bounce live-list reorder (NRT_REORDER: unset = automatic, 0 = never, 1 = always)
for r in 1 2; do for m in auto 0 1; do
  if [ $m = auto ]; then unset NRT_REORDER; else export NRT_REORDER=$m; fi
  timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "
import json,statistics,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); ph=d['phase_ms_build_launch_refine']
print('reorder=$m', 'step', round(d['ms_per_step'],1), 'launch median', round(statistics.median(p[1] for p in ph),1), 'trace', round(d['breakdown_ms']['trace'],1), d['coarse_paths'])"
done; done
