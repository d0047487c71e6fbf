#!/bin/bash
# One gpurun call producing the round's evidence under gpurun_out/ (copy to profiles/ after):
# GPU tests, the default bench line (C5), the C2 secondary line, the launch list of one C5 step
# (per-kernel device time + DRAM bytes), and a sanitizer pass on small cases.
TAG=${1:-r02}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/$TAG.smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -s -p no:warnings > gpurun_out/$TAG.pytest.log 2>&1
echo "pytest rc=$?" | tee -a gpurun_out/$TAG.status
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/$TAG.bench_C5.json 2> gpurun_out/$TAG.bench_C5.err
echo "bench C5 rc=$?" | tee -a gpurun_out/$TAG.status
timeout 900 python bench.py --config C2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/$TAG.bench_C2.json 2> gpurun_out/$TAG.bench_C2.err
echo "bench C2 rc=$?" | tee -a gpurun_out/$TAG.status
