#!/bin/bash
# DRAM bytes per k_trace launch (all launches of a 2-rep C2 prof_step) and one full ncu capture
# of k_refine (the longest kernel of the step).  Outputs in gpurun_out/.
TAG=${1:-tr}
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct \
    --clock-control none -k regex:k_trace --csv --log-file gpurun_out/$TAG.trace_dram.csv \
    python scripts/prof_step.py C2 2 0.03125 > gpurun_out/$TAG.trace_dram.log 2>&1
echo "dram rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_refine \
    --launch-skip 1 --launch-count 1 -o gpurun_out/$TAG.k_refine -f \
    python scripts/prof_step.py C2 2 0.03125 > gpurun_out/$TAG.refine_full.log 2>&1
echo "refine full rc=$?"
