#!/bin/bash
# quick GPU check: refine parity tests, refine timing diagnostics, C2 bench line (no CPU leg)
TAG=${1:-q}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/$TAG.pytest.log 2>&1
echo "pytest rc=$?" | tee -a gpurun_out/$TAG.status
NRT_REFINE_TIMING=1 timeout 300 python scripts/prof_step.py C2 2 0.03125 > gpurun_out/$TAG.refine_timing.json 2> gpurun_out/$TAG.refine_timing.err
echo "refine timing rc=$?" | tee -a gpurun_out/$TAG.status
timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/$TAG.bench.json 2> gpurun_out/$TAG.bench.err
echo "bench rc=$?" | tee -a gpurun_out/$TAG.status
