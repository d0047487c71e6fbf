#!/bin/bash
for b in 0 512 2048 8192 32768; do
  NRT_SORT_BAND=$b python scripts/prof_step.py C2 3 | python -c "
import json,sys; d=json.load(sys.stdin); r=d[-1]
print({'band':$b,'ms_trace':round(r['ms_trace'],2),'ms_fans':round(r['ms_fans'],2),'launch_ms':round(r['launch_ms'],2)})"
done
