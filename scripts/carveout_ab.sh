#!/bin/bash
# k_refine_w L1/shared-memory carveout A/B on C5 (NRT_REFINE_CARVEOUT = shared-memory share, %)
for r in 1 2; do for cv in none 0 40 60 80 100; do
  if [ $cv = none ]; then unset NRT_REFINE_CARVEOUT; else export NRT_REFINE_CARVEOUT=$cv; fi
  timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline 2> /tmp/cv.err | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('cv=$cv', round(d['ms_per_step'],1), {k:round(v,1) for k,v in d['breakdown_ms'].items()})"
  grep -m1 "k_refine_w smem" /tmp/cv.err
done; done
