"""Build libgna_b200.so in-tree with nvcc for sm_100a (no JIT cache, no torch extension)."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
SOURCES = ["api.cu", "attn_sm100.cu", "permute.cu", "sim.cpp"]
HEADERS = ["geom.cuh", "ptx.cuh", "kernels.h", "attn_common.cuh", os.path.join("..", "..", "include", "gna.h")]
OUT = os.path.join(HERE, "libgna_b200.so")
NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
              "-Xcompiler", "-fPIC", "-shared", "--expt-relaxed-constexpr"]


def _stale() -> bool:
    if not os.path.exists(OUT):
        return True
    t = os.path.getmtime(OUT)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS] + [__file__]
    return any(os.path.getmtime(d) > t for d in deps)


TRACE_OUT = os.path.join(HERE, "libgna_b200_trace.so")


def build(force: bool = False, verbose: bool = False, trace: bool = False) -> str:
    out = TRACE_OUT if trace else OUT
    if not force and not trace and not _stale():
        return OUT
    nvcc = os.environ.get("NVCC", "nvcc")
    tmp = out + f".tmp{os.getpid()}"
    cmd = [nvcc, *NVCC_FLAGS, *(["-DGNA_TRACE"] if trace else []), "-o", tmp,
           *[os.path.join(CSRC, s) for s in SOURCES]]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.check_call(cmd)
    os.replace(tmp, out)
    return out


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True, trace="--trace" in sys.argv))
