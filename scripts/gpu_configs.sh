#!/bin/bash
# Refinement timing diagnostics on C2 + bench lines for the other BASELINE configs (C1, C3-C5).
TAG=${1:-cfg}
mkdir -p gpurun_out
NRT_REFINE_TIMING=1 timeout 300 python scripts/prof_step.py C2 2 0.03125 > gpurun_out/$TAG.refine_timing.json 2> gpurun_out/$TAG.refine_timing.err
echo "refine timing rc=$?" | tee -a gpurun_out/$TAG.status
for c in C1 C3 C4 C5; do
  timeout 900 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/$TAG.bench_$c.json 2> gpurun_out/$TAG.bench_$c.err
  echo "bench $c rc=$?" | tee -a gpurun_out/$TAG.status
done
