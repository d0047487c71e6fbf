#!/bin/bash
# ncu launch list of one C2 step (2 reps; the second is steady state) + summary
python scripts/prof_step.py C2 2 0.03125 > gpurun_out/ll_plain.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python scripts/prof_step.py C2 2 0.03125 > /dev/null 2>&1
echo rc=$?
