#!/bin/bash
# time the launch of config $1 (optional n_rays $2) with each library variant (NRT_LIB)
cfg=${1:-C2}; nr=${2:-}
for lib in paper_2403_06648_b200/libnrt.so variants/*.so; do
  NRT_PROF_NO_REFINE=1 NRT_LIB=$PWD/$lib python scripts/prof_step.py $cfg 3 0 $nr 2>/dev/null | python -c "
import json,sys; d=json.load(sys.stdin); r=d[-1]
print({'cfg':'$cfg','lib':'$lib','ms_trace':round(r['ms_trace'],2),'ms_fans':round(r['ms_fans'],2),'launch_ms':round(r['launch_ms'],2)})"
done
