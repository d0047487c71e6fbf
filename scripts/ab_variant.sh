# A/B of libnrt.so against variants/$1.so: C2 and C5 (1e7 rays) launch timings (no refine)
for l in paper_2403_06648_b200/libnrt.so variants/$1.so; do
  n=$(basename $l .so)
  NRT_LIB=$PWD/$l NRT_PROF_NO_REFINE=1 timeout 300 python scripts/prof_step.py C2 4 > gpurun_out/ab_c2_$n.json 2>/dev/null
  NRT_LIB=$PWD/$l NRT_PROF_NO_REFINE=1 timeout 300 python scripts/prof_step.py C5 3 0 1e7 > gpurun_out/ab_c5_$n.json 2>/dev/null
done
