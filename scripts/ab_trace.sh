# launch timings (no refine) for libnrt.so and the given variants: C2 (4 reps), C5 (1e7 rays), C3
for l in paper_2403_06648_b200/libnrt.so "$@"; do
  n=$(basename $l .so)
  NRT_LIB=$PWD/$l NRT_PROF_NO_REFINE=1 timeout 300 python scripts/prof_step.py C2 4 > gpurun_out/abt_c2_$n.json 2>/dev/null
  NRT_LIB=$PWD/$l NRT_PROF_NO_REFINE=1 timeout 300 python scripts/prof_step.py C5 3 0 1e7 > gpurun_out/abt_c5_$n.json 2>/dev/null
  NRT_LIB=$PWD/$l NRT_PROF_NO_REFINE=1 timeout 300 python scripts/prof_step.py C3 2 > gpurun_out/abt_c3_$n.json 2>/dev/null
done
