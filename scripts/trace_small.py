#!/usr/bin/env python
"""Phase clocks of K5 / K6 (needs a build with CH_NVCC_EXTRA=-DCH_TRACE):
python scripts/trace_small.py [lib]"""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2303_10581_b200 as chf  # noqa: E402
from paper_2303_10581_b200 import _lib  # noqa: E402
import synth  # noqa: E402

lib = _lib.load()
tr = (ctypes.c_longlong * 32)()
for dist in ("normal", "circle"):
    for n in (1000, 4000, 10000, 30000):
        xy = synth.points(dist, n, seed=0, device="cuda")
        ws = chf.Workspace(n)
        out = torch.empty(n, dtype=torch.int64, device="cuda")
        cnt = torch.empty(1, dtype=torch.int64, device="cuda")
        rows = []
        for it in range(20):
            chf.filter_async(xy, ws, out, cnt)
            torch.cuda.synchronize()
            lib.ch_debug_trace(tr, 32)
            rows.append(list(tr))
        r = rows[-1]
        b = 0 if n <= 4096 else 10
        last = 8 if b == 0 else 20
        ks = [k for k in range(b, last + 1) if k != 15]  # (K6 has no phase 15 since the octagon push went)
        ph = [r[k] - r[b] for k in ks]
        bo = [r[k] - r[14 if b else 3] for k in (21, 22, 23, 24)]
        print(f"{dist:7s} {n:6d} " + " ".join(f"{v:6d}" for v in ph) + "  | octagon " + " ".join(f"{v:6d}" for v in bo))
