#!/bin/bash
# C5 receiver-capture strategies at 1e7 rays (no refinement)
for cfg in "NRT_RX_GRID_MIN=1000000" "NRT_RX_GRID_V=0.25" "NRT_RX_GRID_V=0.5" "NRT_RX_GRID_V=1.0"; do
  env $cfg NRT_PROF_NO_REFINE=1 python scripts/prof_step.py C5 2 0 1e7 | python -c "
import json,sys; d=json.load(sys.stdin); r=d[-1]
print({'cfg':'$cfg','ms_trace':round(r['ms_trace'],2),'launch_ms':round(r['launch_ms'],2)})"
done
