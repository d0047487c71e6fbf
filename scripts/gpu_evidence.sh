#!/bin/bash
# One gpurun call producing the round's evidence under gpurun_out/ (copy to profiles/ after):
# smoke(), GPU tests, the default bench line (C5), the C2 secondary line, the NEXT-1 SDF lines
# (C4, C2), NEXT-2 cone tracing (C2), NEXT-1 + NEXT-4 (C2) and the NEXT-1 path-quality study.
TAG=${1:-r02}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/$TAG.smi.txt 2>&1
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/$TAG.smoke.log 2>&1
echo "smoke rc=$?" | tee -a gpurun_out/$TAG.status
timeout 3000 python -m pytest tests -m gpu -q -s -p no:warnings > gpurun_out/$TAG.pytest.log 2>&1
echo "pytest rc=$?" | tee -a gpurun_out/$TAG.status
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/$TAG.bench_C5.json 2> gpurun_out/$TAG.bench_C5.err
echo "bench C5 rc=$?" | tee -a gpurun_out/$TAG.status
timeout 900 python bench.py --config C2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/$TAG.bench_C2.json 2> gpurun_out/$TAG.bench_C2.err
echo "bench C2 rc=$?" | tee -a gpurun_out/$TAG.status
timeout 900 python bench.py --config C4 --intersect sdf --steps 5 --warmup 3 > gpurun_out/$TAG.bench_C4_sdf.json 2> gpurun_out/$TAG.bench_C4_sdf.err
echo "bench C4 sdf rc=$?" | tee -a gpurun_out/$TAG.status
timeout 900 python bench.py --config C2 --intersect sdf --steps 10 --warmup 3 > gpurun_out/$TAG.bench_C2_sdf.json 2> gpurun_out/$TAG.bench_C2_sdf.err
echo "bench C2 sdf rc=$?" | tee -a gpurun_out/$TAG.status
timeout 900 python bench.py --config C2 --tracer env --steps 5 --warmup 3 > gpurun_out/$TAG.bench_C2_env.json 2> gpurun_out/$TAG.bench_C2_env.err
echo "bench C2 env rc=$?" | tee -a gpurun_out/$TAG.status
timeout 900 python bench.py --config C2 --intersect sdf --refine gd --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/$TAG.bench_C2_sdf_gd.json 2> gpurun_out/$TAG.bench_C2_sdf_gd.err
echo "bench C2 sdf gd rc=$?" | tee -a gpurun_out/$TAG.status
# launch lists (per-kernel time + DRAM bytes) of one C5 step and of the NEXT kernels
timeout 1800 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/$TAG.launches_C5.csv python scripts/prof_step.py C5 2 > /dev/null 2>&1
echo "launch list C5 rc=$?" | tee -a gpurun_out/$TAG.status
PYTHONPATH=. timeout 1800 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv -k regex:"k_trace_sdf|k_env_tx|k_env_prop|k_refine_gd" --log-file gpurun_out/$TAG.launches_next.csv python scripts/prof_next.py > /dev/null 2>&1
echo "launch list next rc=$?" | tee -a gpurun_out/$TAG.status
