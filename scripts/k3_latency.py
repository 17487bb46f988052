#!/usr/bin/env python
"""Latency of K3 (combine + octagon build, one CTA) -- the octagon build that
K1's last CTA, K5 and K6 also run: CUDA events over back-to-back launches."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_2303_10581_b200 as chf  # noqa: E402
import synth  # noqa: E402

xy = synth.points("normal", 100_000, seed=0, device="cuda")
ws = chf.Workspace(xy.shape[0])
rec = torch.zeros(24, dtype=torch.int64, device="cuda")
chf.extremes8_async(xy, ws, ext_out=rec)
torch.cuda.synchronize()
for world in (1, 8):
    allr = rec.repeat(world)
    for _ in range(50):
        chf.combine8(allr, world, ws)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(1000):
        chf.combine8(allr, world, ws)
    e1.record()
    torch.cuda.synchronize()
    print(f"k3_combine8 world={world}: {e0.elapsed_time(e1):.1f} us per launch (back-to-back, incl. launch)")
