#!/bin/bash
# C5 step / trace / refine ms of the default library and each variant (build.py -DNAME=VALUE variants/x.so), twice
for r in 1 2; do for lib in paper_2403_06648_b200/libnrt.so variants/*.so; do
NRT_LIB=$PWD/$lib timeout 300 python bench.py --steps 3 --warmup 3 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$lib', round(d['ms_per_step'],1), {k:round(v,1) for k,v in d['breakdown_ms'].items()})"
done; done
