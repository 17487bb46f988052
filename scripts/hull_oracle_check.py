#!/usr/bin/env python
"""One full comparison of the device hull (f1) with the oracle's exact hull
on a large input (the 1e8-point circle, ~1e8 hull vertices).

    python scripts/hull_oracle_check.py [--dist circle] [--n 1e8]
"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_2303_10581_b200 as chf  # noqa: E402
import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--dist", default="circle")
ap.add_argument("--n", type=float, default=1e8)
a = ap.parse_args()
n = int(a.n)
xy = synth.points(a.dist, n, seed=0, device="cuda")
surv = chf.filter(xy)
t0 = time.perf_counter()
got = chf.hull_gpu(xy, surv)
t_dev = time.perf_counter() - t0
xy_h, surv_h = xy.cpu().numpy(), surv.cpu().numpy()
del xy
torch.cuda.empty_cache()
t0 = time.perf_counter()
want_surv, _ = oracle.filter_compact(xy_h)
t_of = time.perf_counter() - t0
t0 = time.perf_counter()
want = oracle.hull(xy_h, want_surv)
t_oh = time.perf_counter() - t0
print(f"{a.dist}_{n:.0e}: survivors {len(surv_h)} (oracle {len(want_surv)}, equal {np.array_equal(surv_h, want_surv)}); "
      f"hull vertices {len(got)} (oracle {len(want)}), equal {np.array_equal(got, want)}; "
      f"device hull {t_dev * 1e3:.1f} ms incl. copy to host; oracle filter {t_of:.1f} s, oracle hull {t_oh:.1f} s")
assert np.array_equal(surv_h, want_surv) and np.array_equal(got, want)
