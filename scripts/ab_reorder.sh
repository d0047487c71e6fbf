# A/B of the per-bounce coherence reorder: C2 and C5 (1e7 rays) launch timings
for v in 0 1; do
  if [ $v = 0 ]; then export NRT_NO_REORDER=1; else unset NRT_NO_REORDER; fi
  NRT_PROF_NO_REFINE=1 timeout 300 python scripts/prof_step.py C2 3 > gpurun_out/ab_c2_$v.json 2>/dev/null
  NRT_PROF_NO_REFINE=1 timeout 300 python scripts/prof_step.py C5 2 0 1e7 > gpurun_out/ab_c5_$v.json 2>/dev/null
done
