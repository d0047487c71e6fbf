#!/bin/bash
# One gpurun call producing the round's evidence under gpurun_out/ (copy to profiles/ after):
# GPU tests, the default bench line (C5), the C2 secondary line, the NEXT-1 SDF lines (C4, C2)
# and the NEXT-1 path-quality comparison.
TAG=${1:-r02}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/$TAG.smi.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q -s -p no:warnings > gpurun_out/$TAG.pytest.log 2>&1
echo "pytest rc=$?" | tee -a gpurun_out/$TAG.status
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/$TAG.bench_C5.json 2> gpurun_out/$TAG.bench_C5.err
echo "bench C5 rc=$?" | tee -a gpurun_out/$TAG.status
timeout 900 python bench.py --config C2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/$TAG.bench_C2.json 2> gpurun_out/$TAG.bench_C2.err
echo "bench C2 rc=$?" | tee -a gpurun_out/$TAG.status
timeout 900 python bench.py --config C4 --intersect sdf --steps 5 --warmup 3 > gpurun_out/$TAG.bench_C4_sdf.json 2> gpurun_out/$TAG.bench_C4_sdf.err
echo "bench C4 sdf rc=$?" | tee -a gpurun_out/$TAG.status
timeout 900 python bench.py --config C2 --intersect sdf --steps 10 --warmup 3 > gpurun_out/$TAG.bench_C2_sdf.json 2> gpurun_out/$TAG.bench_C2_sdf.err
echo "bench C2 sdf rc=$?" | tee -a gpurun_out/$TAG.status
PYTHONPATH=. timeout 900 python scripts/sdf_quality.py > gpurun_out/$TAG.sdf_quality.jsonl 2> gpurun_out/$TAG.sdf_quality.err
echo "sdf quality rc=$?" | tee -a gpurun_out/$TAG.status
