"""ncu helper: ch_hull_gpu (with the second filtering round) on the survivors
of a 1e8 set, one profiled call after a warm-up.
    python scripts/hull_prof_sync.py [dist]"""
import sys; sys.path.insert(0, ".")
import torch, paper_2303_10581_b200 as chf, synth
dist = sys.argv[1] if len(sys.argv) > 1 else "displaced"
xy = synth.points(dist, 100_000_000, seed=0, device="cuda")
surv = chf.filter(xy)
chf.hull_gpu(xy, surv); torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
chf.hull_gpu(xy, surv); torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
