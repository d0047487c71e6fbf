#!/bin/bash
# C5 launch-phase A/B (scene build + coarse launch, median over steps) of the default library and
# each variant (build.py -DNAME=VALUE variants/x.so), three times
for r in 1 2 3; do for lib in paper_2403_06648_b200/libnrt.so variants/*.so; do
NRT_LIB=$PWD/$lib timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "
import json,statistics,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); ph=d['phase_ms_build_launch_refine']
print('$lib', 'step', round(d['ms_per_step'],1), 'launch median', round(statistics.median(p[1] for p in ph),1), 'trace', round(d['breakdown_ms']['trace'],1))"
done; done
