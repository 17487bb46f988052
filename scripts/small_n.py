#!/usr/bin/env python
"""Latency of one filter step at small n (the C1 regime): K5 (one CTA, one
launch, ``filter_async``) against K1 + K2 (``extremes8_async`` +
``filter_compact``), CUDA events over many back-to-back steps.

    python scripts/small_n.py [--sizes 1e3 1e4 6e4] [--out profiles/r01_small_n.txt]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2303_10581_b200 as chf  # noqa: E402
import synth  # noqa: E402


def time_us(fn, iters):
    for _ in range(20):
        fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(iters):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / iters


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", nargs="+", type=float, default=[1e2, 1e3, 4e3, 1e4, 3e4, 65536])
    ap.add_argument("--dists", nargs="+", default=["normal", "circle"])
    ap.add_argument("--iters", type=int, default=500)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    lines = ["# one filter step at small n, 1x B200, us per step (CUDA events, back-to-back, inputs resident)",
             f"{'workload':16s} {'step us':>9s} {'K1+K2 us':>9s} {'graph us':>9s}  (graph: ch_graph_launch of the "
             f"ch_filter_async step; K5 for n <= 2048, K6 for n <= 32768, else K1 + K2)"]
    print(lines[0], flush=True)
    for dist in a.dists:
        for nf in a.sizes:
            n = int(nf)
            xy = synth.points(dist, n, seed=0, device="cuda")
            ws, ws2 = chf.Workspace(n), chf.Workspace(n)
            out = torch.empty(n, dtype=torch.int64, device="cuda")
            out2 = torch.empty(n, dtype=torch.int64, device="cuda")
            cnt = torch.empty(1, dtype=torch.int64, device="cuda")

            def k5():
                chf.filter_async(xy, ws, out, cnt)

            def k12():
                chf.extremes8_async(xy, ws2)
                chf.filter_compact(xy, ws2, out=out2)

            ws3 = chf.Workspace(n)
            out3 = torch.empty(n, dtype=torch.int64, device="cuda")
            g = chf.FilterGraph(xy, ws3, out3, cnt)
            t5, t12, tg = time_us(k5, a.iters), time_us(k12, a.iters), time_us(g.launch, a.iters)
            c5, c12, cg = chf.read_result(ws).count, chf.read_result(ws2).count, chf.read_result(ws3).count
            assert c5 == c12 == cg and torch.equal(out[:c5], out2[:c12]) and torch.equal(out[:c5], out3[:cg])
            lines.append(f"{dist + '_' + format(n, '.0e'):16s} {t5:9.2f} {t12:9.2f} {tg:9.2f}")
            print(lines[-1], flush=True)
    if a.out:
        open(a.out, "w").write("\n".join(lines) + "\n")


if __name__ == "__main__":
    main()
