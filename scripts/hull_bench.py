#!/usr/bin/env python
"""Row a8 / f1: time the hull stage (Algorithm 1 line 4) separately
from the filter, device hull (f1) vs host monotone chain, on the BASELINE
configs.  Hull ids of the two paths are asserted equal.

    python scripts/hull_bench.py [--sizes 1e8] [--out profiles/r01_hull.txt]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2303_10581_b200 as chf  # noqa: E402
import synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", nargs="+", type=float, default=[1e8])
    ap.add_argument("--dists", nargs="+", default=["normal", "circle", "displaced"])
    ap.add_argument("--host-max", type=float, default=1e8, help="largest survivor count for the host path")
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "hull_bench.txt"))
    a = ap.parse_args()
    rows = []
    for nf in a.sizes:
        n = int(nf)
        for dist in a.dists:
            xy = synth.points(dist, n, seed=0, device="cuda")
            ws = chf.Workspace(n, hull=True)
            hull, surv, st = chf.hull_end_to_end(xy, ws)           # warm-up (allocator, modules)
            t0 = time.perf_counter()
            hull, surv, st = chf.hull_end_to_end(xy, ws)
            wall_dev = (time.perf_counter() - t0) * 1e3
            row = {"workload": f"{dist}_{n:.0e}", "n": n, "survivors": int(st.n_survivors), "hull": int(st.n_hull),
                   "ms_filter": st.ms_filter, "ms_hull_device": st.ms_hull + st.ms_gather, "ms_total_device": wall_dev}
            # the hull kept on the device (ch_hull_gpu_async), CUDA events
            tmp = torch.empty(int(chf._lib.load().ch_hull_gpu_temp_bytes(surv.shape[0])), dtype=torch.uint8,
                              device="cuda")
            chf.hull_gpu_async(xy, surv, tmp)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            hd, hc = chf.hull_gpu_async(xy, surv, tmp)
            e1.record()
            torch.cuda.synchronize()
            row["ms_hull_on_device"] = e0.elapsed_time(e1)
            assert int(hc.item()) == len(hull)
            del tmp, hd
            if st.n_survivors <= a.host_max:
                t0 = time.perf_counter()
                hull_h, _, sth = chf.hull_end_to_end(xy, ws, host_hull=True)
                row["ms_hull_host"] = sth.ms_hull + sth.ms_gather
                row["ms_total_host"] = (time.perf_counter() - t0) * 1e3
                assert np.array_equal(hull, hull_h), "device and host hulls differ"
                row["device_equals_host"] = True
            rows.append(row)
            print(json.dumps(row), flush=True)
            del xy, ws, surv
            torch.cuda.empty_cache()
    lines = ["# hull stage (a8 / f1), 1x B200: filter (K1+K2) and hull timed separately; device hull vs host chain",
             "# dev hull ms: ch_hull_end_to_end's hull stage incl. the id copy to pinned host memory; "
             "on-device ms: ch_hull_gpu_async (ids stay on the device), CUDA events",
             f"{'workload':16s} {'survivors':>11s} {'hull':>10s} {'filter ms':>10s} {'dev hull ms':>12s} "
             f"{'on-device ms':>13s} {'host hull ms':>13s}  equal"]
    for r in rows:
        lines.append(f"{r['workload']:16s} {r['survivors']:11d} {r['hull']:10d} {r['ms_filter']:10.3f} "
                     f"{r['ms_hull_device']:12.2f} {r['ms_hull_on_device']:13.2f} "
                     f"{r.get('ms_hull_host', float('nan')):13.2f}  {r.get('device_equals_host', '-')}")
    open(a.out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
