#!/usr/bin/env python
"""Run the small-n one-launch step (K5 / K6) a few times, for ncu:
python scripts/k6_prof.py DIST N [iters]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2303_10581_b200 as chf  # noqa: E402
import synth  # noqa: E402

dist, n = sys.argv[1], int(float(sys.argv[2]))
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 5
xy = synth.points(dist, n, seed=0, device="cuda")
ws = chf.Workspace(n)
out = torch.empty(n, dtype=torch.int64, device="cuda")
cnt = torch.empty(1, dtype=torch.int64, device="cuda")
for _ in range(iters):
    chf.filter_async(xy, ws, out, cnt)
torch.cuda.synchronize()
print(dist, n, "survivors", int(cnt.item()))
