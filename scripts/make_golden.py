"""Whole-configuration coarse sets of the CPU oracle (tier-1 grid, oracle/grid.c — pinned to the
brute-force definition by tests/test_oracle_grid_pins.py) -> tests/golden/fullsize_sets.json.

For every configuration it stores what the GPU parity test compares: the number of records, the
raw-record count, the ray-bounce count, the event count and the SHA-256 of the deduped record
bytes (184-byte records in R17 key order).  This script calls only oracle/ and nrt_gen (no
CUDA path).  Usage: python scripts/make_golden.py [C2 C3 C4 C5 C2s0 C2s5 C2s20 ...]
"""
import hashlib
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import nrt_gen as G  # noqa: E402
from oracle import oracle as O  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden", "fullsize_sets.json")
# the oracle's own grid cell (m): independent of the GPU's voxel (DESIGN.md §3 lists those)
ORACLE_VOXEL = {"SR": 0.05, "RR": 0.03}


def case_of(name):
    if name.startswith("C2s") and name[3:].isdigit():  # full C2 at another noise level (mm)
        return G.case("C2", sigma=int(name[3:]) / 1000.0), "SR"
    c = G.case(name)
    return c, "RR" if name in ("C4", "C5") else "SR"


def main():
    names = sys.argv[1:] or ["C2", "C3", "C4", "C5"]
    procs = os.cpu_count() or 1
    db = json.load(open(OUT)) if os.path.exists(OUT) else {}
    for name in names:
        case, kind = case_of(name)
        t0 = time.time()
        recs, n_raw, nb, ev = O.launch_phased(case, procs=procs, return_events=True,
                                              grid_voxel=ORACLE_VOXEL[kind])
        dt = time.time() - t0
        db[name] = {"records": int(len(recs)), "n_raw": int(n_raw), "bounces": int(nb),
                    "events": int(len(ev)),
                    "sha256": hashlib.sha256(recs.tobytes()).hexdigest(),
                    "events_sha256": hashlib.sha256(ev.tobytes()).hexdigest(),
                    "n_rays": int(case.n_rays), "n_surfels": int(case.scene.n),
                    "oracle": f"tier-1 grid {ORACLE_VOXEL[kind]} m, {procs} processes, {dt:.0f} s"}
        print(name, db[name], flush=True)
        json.dump(db, open(OUT, "w"), indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
