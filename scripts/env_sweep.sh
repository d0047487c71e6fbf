#!/bin/bash
# time the launch of config $1 (n_rays $2 optional) under each env assignment in $ENVS (space-separated)
cfg=${1:-C2}; nr=${2:-}
for e in $ENVS; do
  env $e NRT_PROF_NO_REFINE=1 python scripts/prof_step.py $cfg 3 0 $nr 2>/dev/null | python -c "
import json,sys; d=json.load(sys.stdin); r=d[-1]
print({'cfg':'$cfg','env':'$e','ms_trace':round(r['ms_trace'],2),'ms_fans':round(r['ms_fans'],2),'launch_ms':round(r['launch_ms'],2),'n':r['n']})"
done
