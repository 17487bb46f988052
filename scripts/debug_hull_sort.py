"""Debug: run the device hull on one set and check the scratch's sorted points
(P at offset o_P) are in x order; report the first violation."""
import sys; sys.path.insert(0, ".")
import numpy as np, torch, ctypes
import paper_2303_10581_b200 as chf, synth, oracle
sys.path.insert(0, "tests")
from test_gpu_parity import _quantum_cluster_sets

def r256(b): return (b + 255) & ~255

def check(name, xy):
    lib = chf._lib.load()
    n = len(xy); m = n
    d = torch.tensor(xy, device="cuda")
    ids = torch.arange(n, dtype=torch.int64, device="cuda")
    tb = int(lib.ch_hull_gpu_temp_bytes(m))
    tmp = torch.zeros(tb, dtype=torch.uint8, device="cuda")
    out = np.zeros(m, dtype=np.int64); h = ctypes.c_int64(0)
    st = lib.ch_hull_gpu(chf._ptr(d), n, chf._ptr(ids), m, out.ctypes.data_as(ctypes.c_void_p), ctypes.byref(h),
                         chf._ptr(tmp), tb, chf._stream(None))
    torch.cuda.synchronize()
    oP = 4 * r256(8 * m)
    P = tmp[oP: oP + 16 * m].view(torch.float64).view(m, 2).cpu().numpy()
    bad = np.nonzero(np.diff(P[:, 0]) < 0)[0]
    want = oracle.hull(xy)
    ok = st == 0 and np.array_equal(out[: h.value], want)
    print(name, "status", st, "hull ok", ok, "nh", h.value, len(want), "unsorted at", bad[:10], flush=True)
    if len(bad):
        i = bad[0]
        print("  P around:", P[max(0, i - 3): i + 4].tolist())

which = sys.argv[1] if len(sys.argv) > 1 else "all"
for name, xy in _quantum_cluster_sets():
    if which in ("all", name):
        check(name, xy)
if which in ("all", "circle"):
    xy = synth.points("circle", int(float(sys.argv[2]) if len(sys.argv) > 2 else 1e7), seed=0, device="cuda").cpu().numpy()
    check("circle", xy)
