# refine timings for libnrt.so and variants: C2 probe + C4 (one rep, refine kernel ms)
for l in paper_2403_06648_b200/libnrt.so "$@"; do
  n=$(basename $l .so)
  NRT_LIB=$PWD/$l timeout 300 python scripts/refine_probe.py > gpurun_out/abr_c2_$n.json 2>/dev/null
  NRT_LIB=$PWD/$l timeout 600 python scripts/prof_step.py C4 1 > gpurun_out/abr_c4_$n.json 2>/dev/null
done
