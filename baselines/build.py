"""Build baselines/libchcub.so (the CUB Variant #4 baseline)."""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, ROOT)
from paper_2303_10581_b200 import build as pb  # noqa: E402

LIB = os.path.join(HERE, "libchcub.so")


def build(force=False):
    src = os.path.join(HERE, "cub_variant.cu")
    if not force and os.path.exists(LIB) and os.path.getmtime(LIB) > os.path.getmtime(src):
        return LIB
    pb.build()
    cmd = [pb.nvcc(), *pb.ARCH, "-O3", "-std=c++17", "-Xcompiler", "-fPIC", "-shared", "-o", LIB, src,
           "-L" + os.path.dirname(pb.LIB), "-lchfilter", "-Xlinker", "-rpath,$ORIGIN/../paper_2303_10581_b200",
           "-cudart", "static"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode:
        sys.stderr.write(r.stderr)
        raise RuntimeError("nvcc failed")
    return LIB


if __name__ == "__main__":
    print(build(force=True))
