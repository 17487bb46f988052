"""Device hull timing on skewed inputs (quantised keys crowded into few
digit buckets) against a uniform one: ch_hull_gpu_async, CUDA events."""
import sys; sys.path.insert(0, ".")
import numpy as np, torch, paper_2303_10581_b200 as chf

def t(xy, name):
    d = torch.tensor(xy, device="cuda")
    ids = torch.arange(len(xy), dtype=torch.int64, device="cuda")
    tmp = torch.empty(int(chf._lib.load().ch_hull_gpu_temp_bytes(len(xy))), dtype=torch.uint8, device="cuda")
    chf.hull_gpu_async(d, ids, tmp); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); h, c = chf.hull_gpu_async(d, ids, tmp); e1.record(); torch.cuda.synchronize()
    print(f"{name:28s} n={len(xy):9d} hull={int(c.item()):8d} {e0.elapsed_time(e1):8.2f} ms", flush=True)

rng = np.random.default_rng(0)
n = 10_000_000
th = rng.random(n) * 2 * np.pi
t(np.stack([np.cos(th), np.sin(th)], 1), "circle")
x = rng.random(n) * 1e-6; x[0] = 1.0
t(np.stack([x, rng.random(n)], 1), "x in [0,1e-6] + outlier")
x = np.round(rng.random(n) * 255) / 255.0
t(np.stack([x, rng.random(n)], 1), "256 distinct x")
x = np.full(n, 0.5); x[:1000] = rng.random(1000)
t(np.stack([x, rng.random(n)], 1), "one x value (+1000 others)")
