"""Builds libnrt.so (the CUDA C-ABI library) in-tree for sm_100a with nvcc."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libnrt.so")
SOURCES = ["api.cu", "scene.cu", "launch.cu", "dedupe.cu", "refine.cu", "post.cu"]
NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-fmad=false",            # R3: no FMA contraction anywhere on the parity path
    "-prec-div=true", "-prec-sqrt=true", "-ftz=false",
    "-Xcompiler", "-fPIC,-ffp-contract=off,-fno-fast-math",
    "-Xptxas", "-v",
    "--shared",
]


def build(force: bool = False, verbose: bool = False, defines=(), out: str | None = None) -> str:
    """Compile every .cu of csrc/ into one shared library (out, default libnrt.so).
    `defines` (e.g. ["NRT_TRACE_MINB=8"]) are tuning variants for experiments."""
    lib = out or LIB
    srcs = [os.path.join(CSRC, s) for s in SOURCES]
    deps = srcs + [os.path.join(CSRC, "internal.cuh"), os.path.join(ROOT, "include", "nrt.h")]
    if not force and os.path.exists(lib):
        mt = os.path.getmtime(lib)
        if all(os.path.getmtime(s) <= mt for s in deps):
            return lib
    nvcc = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
    cmd = [nvcc, *NVCC_FLAGS, *[f"-D{d}" for d in defines], "-I", os.path.join(ROOT, "include"),
           "-o", lib + ".tmp", *srcs]
    r = subprocess.run(cmd, capture_output=True, text=True)
    log = os.path.join(HERE, "build.log" if out is None else os.path.basename(lib) + ".log")
    with open(log, "w") as f:
        f.write(" ".join(cmd) + "\n" + r.stdout + r.stderr)
    if r.returncode != 0:
        sys.stderr.write(r.stderr[-8000:])
        raise RuntimeError(f"nvcc failed (see {log})")
    if verbose:
        sys.stderr.write(r.stderr)
    os.replace(lib + ".tmp", lib)
    return lib


if __name__ == "__main__":
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    defs = [a[2:] for a in args if a.startswith("-D")]
    outs = [a for a in args if a.endswith(".so")]
    build(force="--force" in sys.argv, verbose="--verbose" in sys.argv, defines=defs,
          out=os.path.abspath(outs[0]) if outs else None)
