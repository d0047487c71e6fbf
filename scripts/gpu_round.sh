#!/bin/bash
# One gpurun call: GPU tests, bench (no profiler), ncu launch list of one C2 step, and one
# `ncu --set full` capture of the dominant kernel (k_trace).  Outputs land in gpurun_out/.
# Usage: scripts/gpu_round.sh [tag]   (each stage only after the previous exited 0)
TAG=${1:-r01}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/$TAG.smi.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/$TAG.pytest.log 2>&1
echo "pytest rc=$?" | tee -a gpurun_out/$TAG.status
timeout 900 python bench.py > gpurun_out/$TAG.bench.json 2> gpurun_out/$TAG.bench.err
echo "bench rc=$?" | tee -a gpurun_out/$TAG.status
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/$TAG.launches.csv \
    python scripts/prof_step.py C2 2 0.03125 > gpurun_out/$TAG.prof_step.log 2>&1
echo "launches rc=$?" | tee -a gpurun_out/$TAG.status
# one full capture of the primary k_trace launch of the second rep (steady state)
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_trace \
    --launch-skip 8 --launch-count 1 -o gpurun_out/$TAG.k_trace -f \
    python scripts/prof_step.py C2 2 0.03125 > gpurun_out/$TAG.ncu_full.log 2>&1
echo "ncu full rc=$?" | tee -a gpurun_out/$TAG.status
