"""Build libchfilter.so in-tree with nvcc for sm_100a.

    python -m paper_2303_10581_b200.build

Device code: -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo
-fmad=false (no FMA contraction anywhere; the predicate also uses explicit
__d*_rn intrinsics).  Host code: -ffp-contract=off (the host octagon
builder and the exact hull must round exactly like the device).
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libchfilter.so")
SOURCES = ["chfilter.cu", "comm.cu", "hull_gpu.cu", "hull.cpp"]
DEPS = SOURCES + ["octagon.cuh", "exact.cuh", "internal.h"]

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVFLAGS = ["-O3", "-lineinfo", "-std=c++17", "-fmad=false", "--expt-relaxed-constexpr",
           "-Xcompiler", "-fPIC,-ffp-contract=off,-O2", "-Xptxas", "-v"]


def nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if c and os.path.exists(c):
            return c
    raise RuntimeError("nvcc not found")


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, d) for d in DEPS] + [os.path.join(ROOT, "include", "chfilter.h")]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return LIB
    tmp = LIB + ".tmp%d" % os.getpid()
    extra = os.environ.get("CH_NVCC_EXTRA", "").split()  # developer experiments only
    cmd = [nvcc(), *ARCH, *NVFLAGS, *extra, "-shared", "-o", tmp,
           *[os.path.join(CSRC, s) for s in SOURCES], "-cudart", "static"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc failed")
    if verbose:
        sys.stderr.write(r.stderr)
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
