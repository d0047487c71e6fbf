#!/bin/bash
# time one C2 launch at several voxel sizes (results are voxel-invariant; speed is not)
for v in 0.0625 0.05 0.04 0.03125 0.025; do
  echo "voxel $v"
  python scripts/prof_step.py C2 2 $v | python -c "
import json,sys; d=json.load(sys.stdin); r=d[-1]; c=d[0]
print({'v':$v,'ms_trace':round(r['ms_trace'],2),'ms_fans':round(r['ms_fans'],2),'launch_ms':round(r['launch_ms'],2),'build_ms':round(r['build_ms'],2),'tests/b':round(c['surfel_tests']/c['bounces'],1),'cells/b':round(c['cells_visited']/c['bounces'],1),'nonempty/b':round(c['cells_nonempty']/c['bounces'],2),'refs':r['scene']['n_refs']})"
done
