#!/bin/bash
# C5 (RR, 10M surfels, 879 RX) voxel sweep at 1e7 rays, no refinement
for v in 0.0625 0.04 0.03125 0.025 0.02; do
  NRT_PROF_NO_REFINE=1 python scripts/prof_step.py C5 2 $v 1e7 | python -c "
import json,sys; d=json.load(sys.stdin); r=d[-1]; c=d[0]
print({'v':$v,'ms_trace':round(r['ms_trace'],2),'launch_ms':round(r['launch_ms'],2),'build':round(r['build_ms'],1),'tests/b':round(c['surfel_tests']/c['bounces'],1),'cells/b':round(c['cells_visited']/c['bounces'],1),'bounces':r['bounces']})"
done
