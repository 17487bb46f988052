import sys; sys.path.insert(0, ".")
import numpy as np, torch, paper_2303_10581_b200 as chf
rng = np.random.default_rng(0); n = 10_000_000
x = np.full(n, 0.5); x[:1000] = rng.random(1000)
d = torch.tensor(np.stack([x, rng.random(n)], 1), device="cuda")
ids = torch.arange(n, dtype=torch.int64, device="cuda")
tmp = torch.empty(int(chf._lib.load().ch_hull_gpu_temp_bytes(n)), dtype=torch.uint8, device="cuda")
chf.hull_gpu_async(d, ids, tmp); torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart(); chf.hull_gpu_async(d, ids, tmp); torch.cuda.synchronize(); torch.cuda.cudart().cudaProfilerStop()
