"""Builds libnrt.so (the CUDA C-ABI library) in-tree for sm_100a with nvcc.

Every csrc/*.cu compiles to its own object (in parallel), then one link.  All files are
compiled without FMA contraction (R3: the coarse path and the post-processing decisions are
bit-exact against the oracle) except refine.cu, whose results are compared with a tolerance
(1e-5 m / 1e-12 s) and whose FP64 dependency chains are shorter with fused multiply-adds.
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libnrt.so")
SOURCES = ["api.cu", "scene.cu", "launch.cu", "dedupe.cu", "refine.cu", "post.cu"]
COMMON = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-prec-div=true", "-prec-sqrt=true", "-ftz=false",
    "-Xcompiler", "-fPIC,-ffp-contract=off,-fno-fast-math",
    "-Xptxas", "-v",
]
FMAD = {"refine.cu": "-fmad=true"}  # default -fmad=false (R3: no FMA contraction on the parity path)
if os.environ.get("NRT_REFINE_FMAD") == "0":  # A/B switch
    FMAD = {}
NVCC_FLAGS = COMMON + ["-fmad=false", "--shared"]  # (kept for reference: the single-command form)


def build(force: bool = False, verbose: bool = False, defines=(), out: str | None = None) -> str:
    """Compile every .cu of csrc/ into one shared library (out, default libnrt.so).
    `defines` (e.g. ["NRT_TRACE_MINB=8"]) are tuning variants for experiments."""
    lib = out or LIB
    srcs = [os.path.join(CSRC, s) for s in SOURCES]
    deps = srcs + [os.path.join(CSRC, "internal.cuh"), os.path.join(CSRC, "refine.cu"), os.path.join(ROOT, "include", "nrt.h"),
                   os.path.abspath(__file__)]
    if not force and os.path.exists(lib):
        mt = os.path.getmtime(lib)
        if all(os.path.getmtime(s) <= mt for s in deps):
            return lib
    nvcc = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
    tag = "" if out is None else os.path.basename(lib) + "."
    objdir = os.path.join(HERE, "build", tag or "default")
    os.makedirs(objdir, exist_ok=True)
    procs, logs = [], []
    for s in SOURCES:
        obj = os.path.join(objdir, s + ".o")
        cmd = [nvcc, *COMMON, FMAD.get(s, "-fmad=false"), *[f"-D{d}" for d in defines],
               "-I", os.path.join(ROOT, "include"), "-c", os.path.join(CSRC, s), "-o", obj]
        procs.append((s, obj, cmd, subprocess.Popen(cmd, stdout=subprocess.PIPE,
                                                    stderr=subprocess.PIPE, text=True)))
    ok = True
    for s, obj, cmd, p in procs:
        o, e = p.communicate()
        logs.append(" ".join(cmd) + "\n" + o + e)
        if p.returncode != 0:
            ok = False
            sys.stderr.write(e[-8000:])
    link = [nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "--shared", "-o", lib + ".tmp",
            *[obj for _, obj, _, _ in procs]]
    if ok:
        r = subprocess.run(link, capture_output=True, text=True)
        logs.append(" ".join(link) + "\n" + r.stdout + r.stderr)
        ok = r.returncode == 0
        if not ok:
            sys.stderr.write(r.stderr[-8000:])
    log = os.path.join(HERE, "build.log" if out is None else os.path.basename(lib) + ".log")
    with open(log, "w") as f:
        f.write("\n".join(logs))
    if not ok:
        raise RuntimeError(f"nvcc failed (see {log})")
    if verbose:
        sys.stderr.write("\n".join(logs))
    os.replace(lib + ".tmp", lib)
    return lib


if __name__ == "__main__":
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    defs = [a[2:] for a in args if a.startswith("-D")]
    outs = [a for a in args if a.endswith(".so")]
    build(force="--force" in sys.argv, verbose="--verbose" in sys.argv, defines=defs,
          out=os.path.abspath(outs[0]) if outs else None)
