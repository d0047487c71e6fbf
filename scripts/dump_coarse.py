"""Save the C2 coarse path set (GPU launch) to gpurun_out/ for offline analysis with the oracle."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import nrt_gen as G  # noqa: E402
import paper_2403_06648_b200 as N  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
case = G.case(cfg)
p = N.launch_case(N.build_case_scene(case), case)
np.save(os.path.join(ROOT, "gpurun_out", f"{cfg}_coarse.npy"), p.export())
print(cfg, p.count())
