#!/bin/bash
# time one C2 launch with each library variant (NRT_LIB)
for lib in paper_2403_06648_b200/libnrt.so variants/*.so; do
  NRT_LIB=$PWD/$lib python scripts/prof_step.py C2 3 2>/dev/null | python -c "
import json,sys; d=json.load(sys.stdin); r=d[-1]; f=d[-2]
print({'lib':'$lib','ms_trace':round(r['ms_trace'],2),'ms_fans':round(r['ms_fans'],2),'launch_ms':round(r['launch_ms'],2),'refine':round(f['ms_refine_kernel'],2)})"
done
