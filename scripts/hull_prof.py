import sys; sys.path.insert(0, ".")
import torch, paper_2303_10581_b200 as chf, synth
xy = synth.points("circle", 100_000_000, seed=0, device="cuda")
surv = chf.filter(xy)
tmp = torch.empty(int(chf._lib.load().ch_hull_gpu_temp_bytes(surv.shape[0])), dtype=torch.uint8, device="cuda")
chf.hull_gpu_async(xy, surv, tmp); torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
chf.hull_gpu_async(xy, surv, tmp); torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
