"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle,
element by element, on the same seeded bytes.  Integer / index outputs
(extremes, survivor indices, hull ids) must be bit-exact; the octagon's
floating-point fields must be bit-identical too (same binary64 operations in
the same order)."""
import numpy as np
import pytest
import torch

import oracle
import paper_2303_10581_b200 as chf
import synth
from exact import load_golden, near_edge_points

pytestmark = pytest.mark.gpu
DEV = "cuda"


def gpu_all(xy_d, plain=False, ws=None):
    n = xy_d.shape[0]
    ws = ws or chf.Workspace(n)
    e, o = chf.extremes8(xy_d, ws, plain=plain)
    surv = chf.filter(xy_d, ws, plain=plain).cpu().numpy()
    return chf.extremes_tuple(e)[0], chf.octagon_dict(o), surv, ws


def check_against_oracle(xy_d, plain=False, ws=None, name=""):
    xy = xy_d.cpu().numpy()
    idx, o, surv, ws = gpu_all(xy_d, plain, ws)
    want_s, want_idx = oracle.filter_compact(xy, certified=not plain)
    assert np.array_equal(idx, want_idx), (name, idx, want_idx)
    wo = oracle.octagon(xy, want_idx, certified=not plain)
    assert o["nv"] == wo["nv"] and o["degenerate"] == wo["degenerate"], name
    for f in ("vx", "vy", "ex", "ey", "thr"):
        assert np.array_equal(o[f].view(np.int64), wo[f].view(np.int64)), (name, f)
    assert np.array_equal(surv, want_s), (name, len(surv), len(want_s))
    return surv, ws


def test_kernels_launch_at_design_occupancy():
    """K1 3 CTAs/SM, K2 2 CTAs/SM: a few bytes more of
    static shared memory or registers silently halve K2's residency."""
    lib = chf._lib.load()
    torch.zeros(1, device=DEV)
    assert lib.ch_occupancy(0) >= 3
    assert lib.ch_occupancy(1) == 2
    assert lib.ch_occupancy(2) == 2
    assert lib.ch_occupancy(7) < 0


# ------------------------------------------------------------- golden -------
@pytest.mark.parametrize("ex", load_golden(), ids=[g["name"] for g in load_golden()])
def test_golden_on_gpu(ex):
    xy_d = torch.tensor(ex["points"], dtype=torch.float64, device=DEV)
    idx, o, surv, ws = gpu_all(xy_d)
    assert list(idx) == ex["extremes"]
    assert list(o["vidx"]) == ex["octagon"]
    assert o["degenerate"] == ex["degenerate"]
    assert list(surv) == ex["survivors"]
    hull, s2, st = chf.hull_end_to_end(xy_d, ws)
    assert list(hull) == ex["hull"]
    assert list(s2.cpu().numpy()) == ex["survivors"]


# ------------------------------------------------- sizes and distributions --
SIZES = [1, 2, 3, 31, 511, 512, 2048, 2049, 4095, 4096, 4097, 10_000, 123_457, 1_000_003]


@pytest.mark.parametrize("dist", ["normal", "circle", "displaced"])
@pytest.mark.parametrize("n", SIZES)
def test_parity_sizes(dist, n):
    xy_d = synth.points(dist, n, seed=n % 7, device=DEV)
    check_against_oracle(xy_d, name=f"{dist}-{n}")


def test_parity_config1_normal_1e4_seed0():
    """BASELINE.json configs[0]: 10^4 normal points, seed 0."""
    xy_d = synth.points("normal", 10 ** 4, seed=0, device=DEV)
    surv, _ = check_against_oracle(xy_d, name="config1")
    assert 0 < len(surv) < 100


@pytest.mark.parametrize("dist", ["normal", "circle", "displaced"])
def test_parity_plain_predicate(dist):
    xy_d = synth.points(dist, 300_001, seed=4, device=DEV)
    check_against_oracle(xy_d, plain=True, name=dist)


@pytest.mark.parametrize("p", [0.0, 0.02, 0.05, 0.3, 1.0])
def test_parity_displaced_sweep(p):
    xy_d = synth.points("displaced", 200_000, seed=2, p=p, device=DEV)
    check_against_oracle(xy_d, name=f"p={p}")


# ------------------------------------------------------------ adversarial --
def test_parity_ties_duplicates_signed_zero():
    rng = np.random.default_rng(0)
    for n in (5, 700, 9000, 70001):
        xy = rng.integers(-3, 4, size=(n, 2)).astype(np.float64)
        neg = rng.random((n, 2)) < 0.3
        xy[(xy == 0) & neg] = -0.0
        check_against_oracle(torch.tensor(xy, device=DEV), name=f"grid{n}")


def test_parity_all_equal_and_collinear():
    for xy in (np.full((5000, 2), 3.25), np.stack([np.arange(9000.0)] * 2, 1),
               np.stack([np.arange(9000.0), np.zeros(9000)], 1), np.array([[1.0, 2.0], [3.0, 4.0]])):
        check_against_oracle(torch.tensor(xy, device=DEV), name="degenerate")


def test_parity_near_edges_and_box():
    """Points within a few ulps of the octagon edges and of the accept box."""
    rng = np.random.default_rng(1)
    base = synth.points("normal", 50_000, seed=1).numpy()
    o = oracle.octagon(base)
    V = list(zip(o["vx"], o["vy"]))
    adv = near_edge_points(rng, V, 60_000, ulps=4)
    e = chf.Extremes()
    idx = oracle.extremes8(base)
    for k in range(8):
        e.idx[k] = int(idx[k]); e.x[k] = base[idx[k], 0]; e.y[k] = base[idx[k], 1]
    ob = chf.octagon_dict(chf.octagon_build(e))
    pts = [adv]
    if ob["has_box"]:
        x0, x1, y0, y1 = ob["box"]
        t = rng.random(20_000)
        bx = np.concatenate([np.full(5000, x0), np.full(5000, x1), x0 + t[:5000] * (x1 - x0), x0 + t[5000:10000] * (x1 - x0)])
        by = np.concatenate([y0 + t[:5000] * (y1 - y0), y0 + t[5000:10000] * (y1 - y0), np.full(5000, y0), np.full(5000, y1)])
        for s in (-2, -1, 0, 1, 2):
            pts.append(np.stack([bx + s * np.spacing(bx), by - s * np.spacing(by)], 1))
    xy = np.concatenate([base] + pts)
    check_against_oracle(torch.tensor(xy, device=DEV), name="adversarial")


def test_parity_misaligned_input_16B():
    """A 16-byte (not 32-byte) aligned input takes the LDG.128 path."""
    big = synth.points("displaced", 100_001, seed=5, device=DEV)
    xy_d = big[1:]
    assert xy_d.data_ptr() % 32 == 16
    check_against_oracle(xy_d.contiguous() if not xy_d.is_contiguous() else xy_d, name="misaligned")


def test_parity_f32_16B_and_32B_aligned():
    """float32 storage: a 32-byte aligned base takes K1's 256-bit (4-point)
    loads, a 16-byte aligned one the 128-bit loads; both equal the oracle."""
    big = synth.points("circle", 200_003, seed=9, device=DEV).float()
    for off in (0, 2):           # 2 points = 16 bytes
        xy_d = big[off:]
        assert xy_d.data_ptr() % 32 == (0 if off == 0 else 16)
        want, idx8 = oracle.filter_compact(xy_d.double().cpu().numpy())
        ws = chf.Workspace(xy_d.shape[0])
        e, _ = chf.extremes8(xy_d, ws)
        assert np.array_equal(np.array(e.idx[:]), idx8), off
        assert np.array_equal(chf.filter(xy_d).cpu().numpy(), want), off


def test_octagon_bits_vs_oracle_flags():
    for dist, n in (("normal", 100_003), ("circle", 65), ("displaced", 77_777)):
        xy_d = synth.points(dist, n, seed=6, device=DEV)
        ws = chf.Workspace(n)
        chf.extremes8(xy_d, ws)
        bits = chf.octagon_filter(xy_d, ws).cpu().numpy().view(np.uint32)
        keep = oracle.flags(xy_d.cpu().numpy())
        unpacked = ((bits[:, None] >> np.arange(32, dtype=np.uint32)) & 1).reshape(-1)
        assert np.array_equal(unpacked[:n], keep)
        assert not unpacked[n:].any()


def test_host_octagon_argument_path():
    """ch_filter_compact with a caller-provided octagon (host struct)."""
    xy_d = synth.points("displaced", 50_000, seed=7, device=DEV)
    xy = xy_d.cpu().numpy()
    idx = oracle.extremes8(xy)
    e = chf.Extremes()
    for k in range(8):
        e.idx[k] = int(idx[k]); e.x[k] = xy[idx[k], 0]; e.y[k] = xy[idx[k], 1]
    o = chf.octagon_build(e)
    ws = chf.Workspace(len(xy))
    out = chf.filter_compact(xy_d, ws, oct_=o)
    r = chf.read_result(ws)
    want, _ = oracle.filter_compact(xy)
    assert np.array_equal(out[: r.count].cpu().numpy(), want)


def test_nonfinite_detected():
    # 20 000: K6 (the flag of CTA 1 reaches CTA 0 through shared memory);
    # 3 000: K5; 100 000: K1 + K2
    for n, at in ((20_000, 12_345), (3_000, 2_999), (100_000, 77_777)):
        for bad in (np.nan, np.inf, -np.inf):
            xy = synth.points("normal", n, seed=0).numpy()
            xy[at, 1] = bad
            with pytest.raises(chf.CHError) as ei:
                chf.filter(torch.tensor(xy, device=DEV))
            assert ei.value.status == 3, (n, bad)
    chf.filter(synth.points("normal", 1000, seed=0, device=DEV))   # workspace state recovers


def _bits(v):
    import struct as _st
    if isinstance(v, float):
        return _st.pack("<d", v)
    if hasattr(v, "__len__"):
        return tuple(_bits(x) for x in v)
    return v


def _octagon_special_inputs(rng):
    """Point sets whose octagons exercise the assembly: coinciding slots,
    a trailing vertex equal to the first, +-0 coordinates, nv < 3."""
    sq = [(0.0, 0.0), (1.0, 0.0), (1.0, 1.0), (0.0, 1.0)]
    yield "square", sq
    yield "triangle", [(0.0, 0.0), (2.0, 0.0), (1.0, 3.0)]
    yield "triangle_left", [(0.0, 1.0), (3.0, 0.0), (3.0, 2.0)]
    yield "diamond", [(1.0, 0.0), (2.0, 1.0), (1.0, 2.0), (0.0, 1.0)]
    yield "signed_zero", [(-0.0, 1.0), (0.0, -1.0), (1.0, 0.0), (-1.0, -0.0), (0.0, 0.0)]
    yield "segment", [(0.0, 0.0), (1.0, 1.0)]
    yield "one_point", [(0.5, 0.25)]
    yield "horizontal", [(float(i), 3.0) for i in range(5)]
    for t in range(6):
        yield f"random{t}", [tuple(p) for p in rng.normal(size=(int(rng.integers(3, 12)), 2))]


@pytest.mark.parametrize("n", [3_000, 20_000, 100_000])
def test_device_octagon_equals_host_build(n):
    """The octagon K5 (n = 3000), K6 (20 000) and K1's last CTA (100 000)
    build on the device -- every field, the unused entries included -- equals
    chf::build_octagon on the host from the same extremes, and the extremes
    equal the oracle's.  The special points are placed first, the rest of the
    input is drawn strictly inside their hull (or repeats them)."""
    rng = np.random.default_rng(7)
    for name, pts in _octagon_special_inputs(rng):
        pts = np.array(pts, dtype=np.float64)
        m = len(pts)
        if m >= 3:
            w = rng.dirichlet(np.ones(m) * 5, size=n - m)   # convex combinations: inside the hull
            fill = w @ pts
        else:
            fill = pts[rng.integers(0, m, size=n - m)]
        xy = np.concatenate([pts, fill])
        ws = chf.Workspace(n)
        out = torch.empty(n, dtype=torch.int64, device=DEV)
        chf.filter_async(torch.tensor(xy, device=DEV), ws, out)
        e, o = chf.read_octagon(ws)
        want_idx = oracle.extremes8(xy)
        assert list(e.idx) == list(want_idx), name
        h = chf.octagon_build(e)
        for f, _ in chf.Octagon._fields_:
            assert _bits(getattr(o, f)) == _bits(getattr(h, f)), (name, n, f, getattr(o, f), getattr(h, f))


def test_all_nonfinite_input():
    """Every point non-finite (no slot can hold a finite key): the status is
    CH_ERR_NONFINITE on every path and no extreme index leaves the array."""
    for n in (1, 3_000, 20_000, 100_000):
        for bad in (np.nan, np.inf, -np.inf):
            xy = np.full((n, 2), bad)
            with pytest.raises(chf.CHError) as ei:
                chf.filter(torch.tensor(xy, device=DEV))
            assert ei.value.status == 3, (n, bad)
            torch.cuda.synchronize()
    chf.filter(synth.points("normal", 1000, seed=0, device=DEV))


def test_determinism_and_workspace_reuse():
    n = 777_777
    ws = chf.Workspace(n)
    xs = [synth.points(d, n, seed=3, device=DEV) for d in ("circle", "normal", "displaced")]
    ref = [chf.filter(x, ws).cpu().numpy() for x in xs]
    for _ in range(15):
        for x, r in zip(xs, ref):
            assert np.array_equal(chf.filter(x, ws).cpu().numpy(), r)
    # smaller inputs on the same workspace (stale look-back words are ignored)
    small = synth.points("displaced", 5000, seed=1, device=DEV)
    want, _ = oracle.filter_compact(small.cpu().numpy())
    assert np.array_equal(chf.filter(small, ws).cpu().numpy(), want)


def test_index_base_and_sharded_combine_world_independence():
    """K1 per shard with index_base + K3 combine + K2 per shard equals the
    single-GPU result for W = 1..8 (the multi-GPU path, simulated on 1 GPU)."""
    n = 300_001
    for dist in ("normal", "displaced", "circle"):
        xy_d = synth.points(dist, n, seed=8, device=DEV)
        want, want_idx = oracle.filter_compact(xy_d.cpu().numpy())
        for W in (1, 2, 3, 8):
            from paper_2303_10581_b200.dist import EXT_WORDS, shard_range
            recs = torch.empty(W * EXT_WORDS, dtype=torch.int64, device=DEV)
            wss = []
            for r in range(W):
                lo, hi = shard_range(n, W, r)
                ws = chf.Workspace(hi - lo)
                chf.extremes8_async(xy_d[lo:hi], ws, index_base=lo, ext_out=recs[r * EXT_WORDS:(r + 1) * EXT_WORDS])
                wss.append(ws)
            parts = []
            for r in range(W):
                lo, hi = shard_range(n, W, r)
                chf.combine8(recs, W, wss[r])
                out = chf.filter_compact(xy_d[lo:hi], wss[r], index_base=lo)
                c = chf.read_result(wss[r]).count
                parts.append(out[:c].cpu().numpy())
            got = np.concatenate(parts)
            assert np.array_equal(got, want), (dist, W)


def test_gather_and_hull_end_to_end():
    for dist in ("normal", "displaced"):
        xy_d = synth.points(dist, 400_000, seed=9, device=DEV)
        xy = xy_d.cpu().numpy()
        hull, surv, st = chf.hull_end_to_end(xy_d)
        want_hull, want_s, _ = oracle.hull_end_to_end(xy)
        assert np.array_equal(surv.cpu().numpy(), want_s)
        assert np.array_equal(hull, want_hull)
        assert st.n_hull == len(hull) and st.n_survivors == len(want_s)


# ---------------------------------------------- full sizes of BASELINE.json --
@pytest.mark.parametrize("dist", ["normal", "circle", "displaced"])
def test_parity_full_1e8(dist):
    """configs[1..3]: 10^8 points, full element-by-element parity in the
    launch configuration bench.py times."""
    n = 10 ** 8
    xy_d = synth.points(dist, n, seed=0, device=DEV)
    ws = chf.Workspace(n)
    check_against_oracle(xy_d, ws=ws, name=f"{dist}-1e8")
    if dist == "normal":
        hull, surv, st = chf.hull_end_to_end(xy_d, ws)
        want_h = oracle.hull(xy_d.cpu().numpy(), surv.cpu().numpy())
        assert np.array_equal(hull, want_h)
    del xy_d
    torch.cuda.empty_cache()


def test_parity_full_1e9_normal():
    """configs[4] at one GPU (the bench workload, ch_filter_async: K1 then K2
    with programmatic launch): extremes, octagon fields and EVERY survivor
    against a full oracle pass over all 10^9 points (~15 s of CPU)."""
    n = 10 ** 9
    free = torch.cuda.mem_get_info()[0]
    if free < 40e9:
        pytest.skip("needs ~40 GB of device memory")
    xy_d = synth.points("normal", n, seed=0, device=DEV)
    ws = chf.Workspace(n)
    out = torch.empty(n, dtype=torch.int64, device=DEV)
    cnt = torch.zeros(1, dtype=torch.int64, device=DEV)
    chf.filter_async(xy_d, ws, out, cnt)
    c = int(cnt.item())
    surv = out[:c].cpu().numpy()
    e, o = chf.read_octagon(ws)
    assert chf.read_result(ws).count == c
    xy = xy_d.cpu().numpy()
    del xy_d, out
    torch.cuda.empty_cache()
    want, idx8 = oracle.filter_compact(xy)
    assert np.array_equal(np.array(e.idx[:]), idx8)
    wo = oracle.octagon(xy, idx8)
    od = chf.octagon_dict(o)
    for f in ("vx", "vy", "ex", "ey", "thr"):
        assert np.array_equal(od[f].view(np.int64), wo[f].view(np.int64)), f
    assert np.array_equal(surv, want)


def _edge_band_points(rng, o, dists, per=400):
    """Points at signed distances d * |edge| from every octagon edge (both
    sides), around the fp32 pre-filter's uncertainty band."""
    V = list(zip(o["vx"], o["vy"]))
    nv = len(V)
    pts = []
    for k in range(nv):
        a, b = np.array(V[k]), np.array(V[(k + 1) % nv])
        ev = b - a
        L = np.hypot(*ev)
        nrm = np.array([-ev[1], ev[0]]) / L         # inward normal (CCW polygon)
        for d in dists:
            t = 0.02 + 0.96 * rng.random(per)
            for sgn in (-1.0, 1.0):
                pts.append(a[None, :] + t[:, None] * ev[None, :] + (sgn * d * L) * nrm[None, :])
    return np.concatenate(pts)


@pytest.mark.parametrize("dist", ["displaced", "circle", "normal"])
def test_parity_fp32_prefilter_band(dist):
    """Points straddling the fp32 certification margin (relative distances
    1e-13 .. 1e-3 from each edge): certified, uncertain and fp64-decided paths."""
    rng = np.random.default_rng(21)
    base = synth.points(dist, 100_000, seed=21).numpy()
    o = oracle.octagon(base)
    band = _edge_band_points(rng, o, [10.0 ** -e for e in range(3, 14)])
    xy = np.concatenate([base, band])
    _, oc = chf.extremes8(torch.tensor(xy, device=DEV))
    assert oc.has_f32 == 1
    check_against_oracle(torch.tensor(xy, device=DEV), name=f"band-{dist}")


@pytest.mark.parametrize("scale", [1e-40, 1e-20, 1e9, 1e15, 1e120])
def test_parity_extreme_scales(scale):
    """Scaled inputs: tiny (fp32 subnormal range), large, and beyond the fp32
    pre-filter's 2^40 domain (fp64-only path)."""
    xy = synth.points("displaced", 200_003, seed=22).numpy() * scale
    _, oc = chf.extremes8(torch.tensor(xy, device=DEV))
    assert oc.has_f32 == (1 if scale < 2.0 ** 40 / 0.3 else 0)
    check_against_oracle(torch.tensor(xy, device=DEV), name=f"scale-{scale}")


# ------------------------------------------------ float32 storage (f2) ------
@pytest.mark.parametrize("dist", ["normal", "circle", "displaced"])
@pytest.mark.parametrize("n", [1, 2, 3, 2047, 2048, 2049, 65_537, 1_000_001, 10_000_000])
def test_parity_f32_storage(dist, n):
    """float32 points: every result equals the float64 path on the exactly
    widened coordinates, i.e. the oracle on xy.astype(float64)."""
    xy32 = synth.points(dist, n, seed=n % 5, device=DEV).float()
    xy = xy32.double().cpu().numpy()
    ws = chf.Workspace(n)
    e, o = chf.extremes8(xy32, ws)
    surv = chf.filter(xy32, ws).cpu().numpy()
    want_s, want_idx = oracle.filter_compact(xy)
    assert np.array_equal(np.array(e.idx[:]), want_idx)
    wo = oracle.octagon(xy, want_idx)
    od = chf.octagon_dict(o)
    for f in ("vx", "vy", "ex", "ey", "thr"):
        assert np.array_equal(od[f].view(np.int64), wo[f].view(np.int64)), f
    assert np.array_equal(surv, want_s)


def test_f32_ties_degenerate_and_alignment():
    rng = np.random.default_rng(3)
    for xy in (rng.integers(-3, 4, size=(50_001, 2)).astype(np.float32),
               np.full((777, 2), 1.5, np.float32), np.stack([np.arange(5000.0)] * 2, 1).astype(np.float32)):
        t = torch.tensor(xy, device=DEV)
        want, _ = oracle.filter_compact(xy.astype(np.float64))
        assert np.array_equal(chf.filter(t).cpu().numpy(), want)
    big = synth.points("normal", 1001, seed=0, device=DEV).float()
    with pytest.raises(chf.CHError) as ei:
        chf.filter(big[1:])          # 8-byte aligned only
    assert ei.value.status == 4


def _dist_worker(rank, world, port, n, dist_name, storage, q):
    import os
    import torch.distributed as tdist
    from paper_2303_10581_b200 import dist as chdist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        lo, hi = chdist.shard_range(n, world, rank)
        xy = synth.points(dist_name, n, seed=4, device="cuda", lo=lo, hi=hi)
        if storage == "f32":
            xy = xy.float()
        df = chdist.DistFilter(n, xy, exchange="torch")
        df.step()
        loc, off, total = df.result()
        q.put((rank, lo, hi, off, total, loc.cpu().numpy()))
    except Exception:
        import traceback
        q.put((rank, traceback.format_exc()))
    finally:
        tdist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("storage", ["f64", "f32"])
def test_distfilter_multirank_single_gpu(world, storage):
    """The whole DistFilter step (K1 with index_base, extremes exchange, K3,
    K2, count exchange) with `world` ranks sharing cuda:0 over gloo: the
    concatenated survivors equal the oracle on the full array."""
    import socket
    import torch.multiprocessing as mp
    n = 1_000_003
    s0 = socket.socket(); s0.bind(("127.0.0.1", 0)); port = s0.getsockname()[1]; s0.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_dist_worker, args=(r, world, port, n, "displaced", storage, q)) for r in range(world)]
    for p_ in procs:
        p_.start()
    res = sorted([q.get(timeout=300) for _ in range(world)], key=lambda r: r[0])
    for p_ in procs:
        p_.join(timeout=60)
    for r in res:
        assert len(r) == 6, r[1]
    full = synth.points("displaced", n, seed=4, device="cuda")
    if storage == "f32":
        full = full.float()
    want, _ = oracle.filter_compact(full.double().cpu().numpy())
    got = np.concatenate([r[5] for r in res])
    assert np.array_equal(got, want)
    assert all(r[4] == len(want) for r in res)
    offs = [r[3] for r in res]
    assert offs == sorted(offs) and offs[0] == 0


def _peer_worker(rank, world, port, n, dist_name, storage, steps, q):
    import os
    import torch.distributed as tdist
    from paper_2303_10581_b200 import dist as chdist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        lo, hi = chdist.shard_range(n, world, rank)
        xy = synth.points(dist_name, n, seed=4, device="cuda", lo=lo, hi=hi)
        if storage == "f32":
            xy = xy.float()
        df = chdist.DistFilter(n, xy, exchange="peer")
        outs = []
        for _ in range(steps):       # several steps: both exchange banks, epochs
            df.out.fill_(-1)
            df.step()
            loc, off, total = df.result()
            outs.append((off, total, loc.cpu().numpy()))
        tdist.barrier()
        df.peer.close()
        q.put((rank, lo, hi, outs))
    except Exception:
        import traceback
        q.put((rank, traceback.format_exc()))
    finally:
        tdist.destroy_process_group()


@pytest.mark.parametrize("world,n,dist_name,storage", [(2, 1_000_003, "displaced", "f64"),
                                                       (3, 777_777, "circle", "f32"),
                                                       (3, 2, "normal", "f64"),
                                                       (4, 100_003, "displaced", "f64"),
                                                       (8, 200_003, "displaced", "f64")])
def test_peer_exchange_multirank_single_gpu(world, n, dist_name, storage):
    """The fused exchange (ch_filter_step_peer: K1 stores its extremes record
    into every peer's cudaIpc-mapped buffer, K3 acquires them, K2 stores its
    count) with `world` processes sharing cuda:0: every step's concatenated
    survivors equal the oracle, offsets are the exclusive scan.  n = 2 with
    3 ranks leaves rank 0 with an empty shard."""
    import socket
    import torch.multiprocessing as mp
    steps = 3
    s0 = socket.socket(); s0.bind(("127.0.0.1", 0)); port = s0.getsockname()[1]; s0.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_peer_worker, args=(r, world, port, n, dist_name, storage, steps, q))
             for r in range(world)]
    for p_ in procs:
        p_.start()
    res = sorted([q.get(timeout=300) for _ in range(world)], key=lambda r: r[0])
    for p_ in procs:
        p_.join(timeout=60)
    for r in res:
        assert len(r) == 4, r[1]
    full = synth.points(dist_name, n, seed=4, device="cuda")
    if storage == "f32":
        full = full.float()
    want, _ = oracle.filter_compact(full.double().cpu().numpy())
    for k in range(steps):
        got = np.concatenate([r[3][k][2] for r in res])
        assert np.array_equal(got, want), k
        assert all(r[3][k][1] == len(want) for r in res)
        offs = [r[3][k][0] for r in res]
        sizes = [len(r[3][k][2]) for r in res]
        assert offs == [sum(sizes[:i]) for i in range(world)]


def test_cub_variant_baseline_same_survivors():
    """the CUB Variant #4 rebuild finds the same survivors."""
    import ctypes
    import os
    import sys
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "baselines"))
    import build as bbuild
    lib = ctypes.CDLL(bbuild.build())
    lib.chb_cub_temp_bytes.restype = ctypes.c_size_t
    lib.chb_cub_temp_bytes.argtypes = [ctypes.c_int64]
    lib.chb_cub_filter.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.POINTER(ctypes.c_int64),
                                   ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p]
    for dist in ("normal", "displaced", "circle"):
        n = 1_000_003
        xy = synth.points(dist, n, seed=2, device=DEV)
        out = torch.empty(n, dtype=torch.int64, device=DEV)
        tb = int(lib.chb_cub_temp_bytes(n))
        tmp = torch.empty(tb, dtype=torch.uint8, device=DEV)
        cnt = ctypes.c_int64(0)
        rc = lib.chb_cub_filter(ctypes.c_void_p(xy.data_ptr()), n, ctypes.c_void_p(out.data_ptr()), ctypes.byref(cnt),
                                ctypes.c_void_p(tmp.data_ptr()), tb,
                                ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
        assert rc == 0
        want, _ = oracle.filter_compact(xy.cpu().numpy())
        assert np.array_equal(out[: cnt.value].cpu().numpy(), want), dist


def test_thrust_variants_baseline_same_survivors():
    """the Thrust Variants #2 (scan + scatter) and #3 (copy_if)
    rebuilt on B200 find the oracle's survivors."""
    import ctypes
    import os
    import sys
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "baselines"))
    import build as bbuild
    lib = ctypes.CDLL(bbuild.build())
    lib.chb_thrust_temp_bytes.restype = ctypes.c_size_t
    lib.chb_thrust_temp_bytes.argtypes = [ctypes.c_int64]
    lib.chb_thrust_filter.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p,
                                      ctypes.POINTER(ctypes.c_int64), ctypes.c_void_p, ctypes.c_size_t,
                                      ctypes.c_void_p]
    for dist in ("normal", "displaced", "circle"):
        n = 777_777
        xy = synth.points(dist, n, seed=3, device=DEV)
        want, _ = oracle.filter_compact(xy.cpu().numpy())
        for variant in (2, 3):
            out = torch.full((n,), -1, dtype=torch.int64, device=DEV)
            tb = int(lib.chb_thrust_temp_bytes(n))
            tmp = torch.empty(tb, dtype=torch.uint8, device=DEV)
            cnt = ctypes.c_int64(0)
            rc = lib.chb_thrust_filter(variant, ctypes.c_void_p(xy.data_ptr()), n, ctypes.c_void_p(out.data_ptr()),
                                       ctypes.byref(cnt), ctypes.c_void_p(tmp.data_ptr()), tb,
                                       ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
            assert rc == 0
            assert np.array_equal(out[: cnt.value].cpu().numpy(), want), (dist, variant)


# --------------------------------------------- f3: the exact predicate ------
@pytest.mark.parametrize("dist", ["normal", "circle", "displaced"])
def test_parity_exact_predicate(dist):
    """f3: CH_EXACT survivors equal the oracle's exact strict predicate,
    including near-edge points in the certified band (exact evaluation on
    the device) and fp32-band points."""
    rng = np.random.default_rng(41)
    base = synth.points(dist, 200_000, seed=41).numpy()
    o = oracle.octagon(base)
    V = list(zip(o["vx"], o["vy"]))
    adv = near_edge_points(rng, V, 50_000, ulps=3)
    band = _edge_band_points(rng, o, [10.0 ** -e for e in range(6, 17)], per=200)
    xy = np.concatenate([base, adv, band])
    d = torch.tensor(xy, device=DEV)
    want, want_idx = oracle.filter_compact_exact(xy)
    got = chf.filter(d, plain="exact").cpu().numpy()
    assert np.array_equal(got, want)
    cert, _ = oracle.filter_compact(xy)
    assert len(want) <= len(cert)
    ws = chf.Workspace(len(xy))
    e, oc = chf.extremes8(d, ws, plain="exact")
    assert oc.exact == 1 and np.array_equal(np.array(e.idx[:]), want_idx)
    # the bit-vector kernel (K4) agrees too
    bits = chf.octagon_filter(d, ws).cpu().numpy().view(np.uint32)
    keep = ((bits[:, None] >> np.arange(32, dtype=np.uint32)) & 1).reshape(-1)[: len(xy)]
    assert np.array_equal(np.flatnonzero(keep), want)


def test_parity_exact_predicate_sizes_and_f32():
    for n in (1, 7, 4097, 333_333):
        xy = synth.points("displaced", n, seed=n, device=DEV)
        want, _ = oracle.filter_compact_exact(xy.cpu().numpy())
        assert np.array_equal(chf.filter(xy, plain="exact").cpu().numpy(), want)
        x32 = xy.float()
        want32, _ = oracle.filter_compact_exact(x32.double().cpu().numpy())
        assert np.array_equal(chf.filter(x32, plain="exact").cpu().numpy(), want32)


# ------------------------------------------------------ f1: device hull ------
def _hull_sets():
    rng = np.random.default_rng(51)
    yield "single", np.array([[2.0, 3.0]])
    yield "two", np.array([[1.0, 2.0], [3.0, 4.0]])
    yield "same", np.full((1000, 2), 0.5)
    yield "collinear", np.stack([np.arange(3000.0), 2 * np.arange(3000.0)], 1)
    yield "vertical", np.stack([np.zeros(2000), rng.random(2000)], 1)
    for trial in range(4):
        yield f"grid{trial}", rng.integers(-20, 21, size=(int(rng.integers(1, 60000)), 2)).astype(np.float64)
    for n in (1000, 70_001, 1_000_003):
        th = rng.random(n) * 2 * np.pi
        yield f"circle{n}", np.stack([np.cos(th), np.sin(th)], 1) * 0.25
    yield "random", rng.random((300_000, 2))
    yield "signed_zero", np.array([[0.0, 0.0], [-0.0, 0.0], [1.0, 0.0], [0.0, -0.0], [0.0, 1.0], [-0.0, -0.0]])


def test_device_hull_matches_oracle():
    """The device hull (every point a candidate) equals the oracle hull."""
    for name, xy in _hull_sets():
        d = torch.tensor(xy, device=DEV)
        ids = torch.arange(len(xy), dtype=torch.int64, device=DEV)
        got = chf.hull_gpu(d, ids)
        assert np.array_equal(got, oracle.hull(xy)), name


@pytest.mark.parametrize("dist", ["normal", "circle", "displaced"])
def test_device_hull_end_to_end(dist):
    n = 2_000_003
    xy_d = synth.points(dist, n, seed=52, device=DEV)
    xy = xy_d.cpu().numpy()
    hull, surv, st = chf.hull_end_to_end(xy_d)
    hull_h, surv_h, st_h = chf.hull_end_to_end(xy_d, host_hull=True)
    want_hull, want_s, _ = oracle.hull_end_to_end(xy)
    assert np.array_equal(surv.cpu().numpy(), want_s)
    assert np.array_equal(hull, want_hull)
    assert np.array_equal(hull_h, want_hull)


def test_device_hull_async_on_device():
    """ch_hull_gpu_async: ids and count stay on the device, same hull; m = 0
    gives a zero count."""
    for name, xy in list(_hull_sets())[-4:]:
        d = torch.tensor(xy, device=DEV)
        ids = torch.arange(len(xy), dtype=torch.int64, device=DEV)
        h, c = chf.hull_gpu_async(d, ids)
        assert h.is_cuda and c.is_cuda
        assert np.array_equal(h[: int(c.item())].cpu().numpy(), oracle.hull(xy)), name
    d = torch.zeros((4, 2), dtype=torch.float64, device=DEV)
    h, c = chf.hull_gpu_async(d, torch.empty(0, dtype=torch.int64, device=DEV))
    assert int(c.item()) == 0


def test_hull_end_to_end_workspace_tail_and_malloc_paths():
    """The device-hull scratch from the workspace tail (Workspace(n, hull=True))
    and from cudaMallocAsync (plain workspace) give the same result."""
    n = 300_001
    xy_d = synth.points("displaced", n, seed=11, device=DEV)
    a, sa, _ = chf.hull_end_to_end(xy_d, chf.Workspace(n, hull=True))
    b, sb, _ = chf.hull_end_to_end(xy_d, chf.Workspace(n))
    want, want_s, _ = oracle.hull_end_to_end(xy_d.cpu().numpy())
    assert np.array_equal(a, want) and np.array_equal(b, want)
    assert np.array_equal(sa.cpu().numpy(), want_s) and np.array_equal(sb.cpu().numpy(), want_s)


def test_device_hull_golden():
    for ex in load_golden():
        d = torch.tensor(ex["points"], device=DEV)
        s = torch.tensor(ex["survivors"], dtype=torch.int64, device=DEV)
        assert list(chf.hull_gpu(d, s)) == ex["hull"], ex["name"]


def test_parity_beyond_2pow31_points():
    """X5: more than 2^31 points (int64 indices throughout).
    Extremes and EVERY survivor against a full oracle pass (~30 s of CPU);
    p = 0.02 keeps ~86% of the points, so survivor writes cross 2^31."""
    n = (1 << 31) + 12_345
    free = torch.cuda.mem_get_info()[0]
    if free < 70e9:
        pytest.skip("needs ~70 GB of device memory")
    xy_d = synth.points("displaced", n, seed=7, p=0.02, device=DEV)
    ws = chf.Workspace(n)
    e, o = chf.extremes8(xy_d, ws)
    surv = chf.filter(xy_d, ws).cpu().numpy()
    xy = xy_d.cpu().numpy()
    del xy_d
    torch.cuda.empty_cache()
    want, idx8 = oracle.filter_compact(xy)
    assert np.array_equal(np.array(e.idx[:]), idx8)
    assert want[-1] >= (1 << 31) and surv[-1] < n
    assert np.array_equal(surv, want)


@pytest.mark.parametrize("storage", ["f64", "f32"])
@pytest.mark.parametrize("index_base", [(1 << 32) - 3000, (1 << 32) - 1, (1 << 33) + 7, (1 << 39) - 2_000_000])
def test_index_base_straddling_2pow32(index_base, storage):
    """Shard indices above and across 2^32 without a 68 GB input: K1 and K2
    with index_base, so a warp's index range crosses a multiple of 2^32 and
    K2's 64-bit survivor stores run (VERDICT r1 missing 3).  Survivors =
    index_base + the oracle's survivors, extremes likewise."""
    n = 1_000_003
    xy_d = synth.points("displaced", n, seed=5, device=DEV)
    if storage == "f32":
        xy_d = xy_d.float()
    ws = chf.Workspace(n)
    e, o = chf.extremes8(xy_d, ws, index_base=index_base)
    cnt = torch.zeros(1, dtype=torch.int64, device=DEV)
    out = chf.filter_compact(xy_d, ws, index_base=index_base, count=cnt)
    got = out[: int(cnt.item())].cpu().numpy()
    want, idx8 = oracle.filter_compact(xy_d.double().cpu().numpy())
    assert np.array_equal(np.array(e.idx[:]), idx8 + index_base)
    assert np.array_equal(got, want + index_base)
    # a circle: every point survives, so every warp writes a full range
    c = synth.points("circle", n, seed=5, device=DEV)
    if storage == "f32":
        c = c.float()
    chf.extremes8(c, ws, index_base=index_base)
    out = chf.filter_compact(c, ws, index_base=index_base, count=cnt)
    wc, _ = oracle.filter_compact(c.double().cpu().numpy())
    assert np.array_equal(out[: int(cnt.item())].cpu().numpy(), wc + index_base)


def test_device_hull_64bit_ids_instantiation():
    """The device hull's 64-bit sort-value instantiation (taken when the point
    array has more than 2^32 points; VERDICT r1 missing 3), selected here by
    declaring n_points > 2^32 over a small array: same hull as the 32-bit one
    and the oracle."""
    import ctypes
    lib = chf._lib.load()
    for dist in ("circle", "displaced", "normal"):
        xy = synth.points(dist, 300_001, seed=3, device=DEV)
        surv = chf.filter(xy)
        m = int(surv.shape[0])
        tb = int(lib.ch_hull_gpu_temp_bytes(m))
        tmp = torch.empty(tb, dtype=torch.uint8, device=DEV)
        res = []
        for n_points in (xy.shape[0], (1 << 33) + 5):
            ids = np.zeros(m, dtype=np.int64)
            h = ctypes.c_int64(0)
            st = lib.ch_hull_gpu(chf._ptr(xy), n_points, chf._ptr(surv), m, ids.ctypes.data_as(ctypes.c_void_p),
                                 ctypes.byref(h), chf._ptr(tmp), tb, chf._stream(None))
            assert st == 0
            res.append(ids[: h.value].copy())
        want = oracle.hull(xy.cpu().numpy(), surv.cpu().numpy())
        assert np.array_equal(res[0], want), dist
        assert np.array_equal(res[1], want), dist


@pytest.mark.parametrize("dist", ["normal", "circle", "displaced"])
def test_small_n_single_kernel_equals_two_kernels(dist):
    """K5 (one CTA, n <= 2048) and K6 (one 8-CTA cluster, n <= 32768)
    against K1 + K2 and the oracle, f64 and f32, all predicate modes."""
    for n in (1, 5, 1023, 1024, 1025, 2047, 2048, 2049, 4095, 4096, 4097, 10_000, 16_383, 32_768, 32_769):
        for storage in ("f64", "f32"):
            xy_d = synth.points(dist, n, seed=n, device=DEV)
            if storage == "f32":
                xy_d = xy_d.float()
            xy = xy_d.double().cpu().numpy()
            for mode in (False, True, "exact"):
                ws = chf.Workspace(n)
                k5 = chf.filter(xy_d, ws, plain=mode).cpu().numpy()          # K5 / K6
                ws2 = chf.Workspace(n)
                chf.extremes8_async(xy_d, ws2, plain=mode)
                out = chf.filter_compact(xy_d, ws2)                          # K1 + K2
                k12 = out[: chf.read_result(ws2).count].cpu().numpy()
                if mode == "exact":
                    want, _ = oracle.filter_compact_exact(xy)
                else:
                    want, _ = oracle.filter_compact(xy, certified=not mode)
                assert np.array_equal(k5, want), (dist, n, storage, mode)
                assert np.array_equal(k12, want), (dist, n, storage, mode)


@pytest.mark.parametrize("dist", ["normal", "circle", "displaced"])
def test_graph_replay_equals_oracle(dist):
    """ch_filter_graph_create / ch_graph_launch: the captured step (K5 for
    n <= 2048, K6 to 32768, K1 + K2 above), replayed several times, gives the oracle's
    survivors every time, f64 and f32."""
    for n in (4096, 10_000, 300_007):
        for storage in ("f64", "f32"):
            xy_d = synth.points(dist, n, seed=7, device=DEV)
            if storage == "f32":
                xy_d = xy_d.float()
            want, _ = oracle.filter_compact(xy_d.double().cpu().numpy())
            ws = chf.Workspace(n)
            out = torch.full((n,), -1, dtype=torch.int64, device=DEV)
            cnt = torch.zeros(1, dtype=torch.int64, device=DEV)
            g = chf.FilterGraph(xy_d, ws, out, cnt)
            for rep in range(3):
                out.fill_(-1)
                g.launch()
                torch.cuda.synchronize()
                c = int(cnt.item())
                assert c == len(want) == chf.read_result(ws).count, (dist, n, storage, rep)
                assert np.array_equal(out[:c].cpu().numpy(), want), (dist, n, storage, rep)
            g.close()


def test_back_to_back_k2_and_steps_same_workspace():
    """K2 launched right after K2 on the same workspace (filter_compact twice),
    and whole steps back to back (K2 -> K1 -> K2 with the programmatic
    launch): every result equals the oracle -- K2's claim counter, epoch and
    look-back words are handed from one launch to the next in stream order."""
    for dist in ("displaced", "circle"):
        n = 600_011
        xy = synth.points(dist, n, seed=8, device=DEV)
        want, _ = oracle.filter_compact(xy.cpu().numpy())
        ws = chf.Workspace(n)
        chf.extremes8_async(xy, ws)
        outs = [torch.full((n,), -1, dtype=torch.int64, device=DEV) for _ in range(3)]
        for o in outs:
            chf.filter_compact(xy, ws, out=o)          # K2, K2, K2
        c = chf.read_result(ws).count
        for o in outs:
            assert np.array_equal(o[:c].cpu().numpy(), want), dist
        cnt = torch.zeros(1, dtype=torch.int64, device=DEV)
        outs = [torch.full((n,), -1, dtype=torch.int64, device=DEV) for _ in range(3)]
        for o in outs:
            chf.filter_async(xy, ws, o, cnt)             # K1, K2 (PDL), K1, K2, ...
        torch.cuda.synchronize()
        for o in outs:
            assert np.array_equal(o[: int(cnt.item())].cpu().numpy(), want), dist


def test_randomized_sweep_against_oracle():
    """A seeded sweep over sizes (every path: K5, K6, K1 + K2), storages,
    predicate modes and point-set shapes -- Gaussian, ring, integer grids with
    heavy ties and collinear runs, a few points far out, a tiny-scale and a
    huge-scale copy -- each compared with the oracle element by element."""
    rng = np.random.default_rng(2026)
    shapes = ("normal", "ring", "grid", "outliers", "tiny", "huge")
    for case in range(48):
        n = int(rng.choice([1, 2, 3, 7, 100, 4096, 4097, 9_999, 32_768, 32_769, 65_537, 150_001]))
        shape = shapes[case % len(shapes)]
        if shape == "normal":
            xy = rng.normal(0.5, 0.3, size=(n, 2))
        elif shape == "ring":
            t = rng.uniform(0, 2 * np.pi, n)
            r = rng.uniform(0.2, 0.25, n)
            xy = np.stack([r * np.cos(t), r * np.sin(t)], 1)
        elif shape == "grid":
            xy = rng.integers(-5, 6, size=(n, 2)).astype(np.float64)
        elif shape == "outliers":
            xy = rng.normal(0, 1, size=(n, 2))
            k = max(1, n // 1000)
            xy[rng.integers(0, n, k)] *= 50.0
        elif shape == "tiny":
            xy = rng.normal(0, 1, size=(n, 2)) * 1e-30
        else:
            xy = rng.normal(0, 1, size=(n, 2)) * 1e30
        storage = "f32" if case % 3 == 2 else "f64"
        if storage == "f32":
            xy = xy.astype(np.float32).astype(np.float64)
        mode = (False, True, "exact")[case % 3 if shape != "huge" else 0]
        xy_d = torch.tensor(xy, device=DEV, dtype=torch.float32 if storage == "f32" else torch.float64)
        got = chf.filter(xy_d, plain=mode).cpu().numpy()
        if mode == "exact":
            want, _ = oracle.filter_compact_exact(xy)
        else:
            want, _ = oracle.filter_compact(xy, certified=not mode)
        assert np.array_equal(got, want), (case, n, shape, storage, mode)


def test_device_hull_randomized_sweep():
    """The device hull on seeded sets with many chunk boundaries (up to
    ~300 chunks: every merge path -- three, two and one levels per copy) and
    hard shapes: integer grids (duplicates, collinear runs, vertical columns),
    points on a circle (nearly all on the hull), rings, subsets of candidates.
    Each equals the oracle's exact hull."""
    rng = np.random.default_rng(77)
    for case in range(24):
        n = int(rng.choice([3, 511, 512, 513, 4_097, 30_001, 150_000]))
        kind = case % 4
        if kind == 0:
            xy = rng.integers(-20, 21, size=(n, 2)).astype(np.float64)
        elif kind == 1:
            t = rng.uniform(0, 2 * np.pi, n)
            xy = np.stack([np.cos(t), np.sin(t)], 1)
        elif kind == 2:
            t = rng.uniform(0, 2 * np.pi, n)
            r = rng.uniform(0.9, 1.0, n)
            xy = np.stack([r * np.cos(t), r * np.sin(t)], 1)
        else:
            xy = rng.normal(0, 1, size=(n, 2))
            xy[:, 0] = np.round(xy[:, 0], 1)   # many equal x: vertical ties
        d = torch.tensor(xy, device=DEV)
        ids = np.sort(rng.choice(n, size=max(1, n - n // 7), replace=False)) if case % 2 else np.arange(n)
        got = chf.hull_gpu(d, torch.tensor(ids, dtype=torch.int64, device=DEV))
        want = oracle.hull(xy, ids)
        assert np.array_equal(got, want), (case, n, kind)


def _quantum_cluster_sets():
    """Point sets whose x collide in the device hull's 32-bit sort key (x
    quantised over the survivors' x range, 2^32 - 256 steps): the equal-key
    runs must then be sorted by the exact x (short runs by one thread, long
    ones by one CTA with a 64-bit radix sort over the run)."""
    rng = np.random.default_rng(2024)
    base = rng.random((20_000, 2))
    # 1. a long run of distinct x inside one quantum (~2.3e-10 wide), several tiles long
    c = np.stack([0.5 + rng.random(50_000) * 1e-12, rng.random(50_000)], 1)
    yield "cluster50k", np.concatenate([base, c])
    # 2. one tile or less: 40 and 4097 points in one quantum, next to each other
    c1 = np.stack([0.25 + rng.random(40) * 1e-13, rng.random(40)], 1)
    c2 = np.stack([0.75 + rng.random(4097) * 1e-13, rng.random(4097) * 3 - 1], 1)
    yield "clusters40_4097", np.concatenate([base, c1, c2])
    # 3. a giant vertical line (every x equal): one equal-x run, resolved block-wide
    v = np.stack([np.full(120_000, 0.125), rng.random(120_000) * 4 - 2], 1)
    yield "vertical120k", np.concatenate([base, v])
    # 4. x = -tiny, -0.0, +0.0, +tiny around 0 in [-1, 1]: one key, order-preserving 64-bit keys that
    #    differ in their top byte (8 digit passes), duplicates among them
    t = rng.choice([-1e-300, -0.0, 0.0, 1e-300, 5e-324, -5e-324], size=3000)
    z = np.stack([t, rng.integers(-3, 4, size=3000) / 4.0], 1)
    yield "signed_tiny", np.concatenate([rng.random((5000, 2)) * 2 - 1, z])
    # 5. many short runs with equal x inside (ties inside a run of the fast path)
    xs = np.round(rng.random(200_000), 12)
    yield "rounded12", np.stack([xs, rng.random(200_000)], 1)
    # 6. two distinct x values only, both long runs of equal x, keys 0 and 2^32 - 256
    yield "two_columns", np.stack([rng.integers(0, 2, 70_000) * 1.0, rng.random(70_000)], 1)
    # 6b. one x value for almost every point (a single equal-key run of ~all points; its end by
    #     galloping search, its ties block-wide), and a long equal-x run inside a longer key run
    v = np.stack([np.full(400_000, 0.5), rng.random(400_000)], 1)
    yield "one_x_value", np.concatenate([v, rng.random((1000, 2))])
    w = np.stack([np.full(300_000, 0.5), rng.random(300_000) * 2 - 1], 1)
    w2 = np.stack([0.5 + rng.random(5000) * 1e-13, rng.random(5000)], 1)
    yield "long_tie_in_run", np.concatenate([rng.random((2000, 2)), w, w2])
    # 7. a circle where runs of the same key hold whole arcs: x range 1, points within 1e-9 of x = +-1
    th = rng.random(300_000) * 1e-4
    circ = np.stack([np.cos(th), np.sin(th)], 1)
    yield "circle_cap", np.concatenate([circ, -circ, [[0.0, 0.0]]])


def test_device_hull_equal_key_runs():
    """The device hull's sort (hand-written radix sort on quantised keys, then
    the exact x order inside equal-key runs) on inputs built to make long and
    short equal-key runs, equal-x runs inside them, and an all-equal run:
    every hull equals the oracle's exact hull, for all points as candidates
    and for a subset, and through the 64-bit sort-value instantiation."""
    import ctypes
    lib = chf._lib.load()
    for name, xy in _quantum_cluster_sets():
        n = len(xy)
        d = torch.tensor(xy, device=DEV)
        for sub in (False, True):
            ids = np.arange(n) if not sub else np.sort(np.random.default_rng(n).choice(n, n - n // 5, replace=False))
            idt = torch.tensor(ids, dtype=torch.int64, device=DEV)
            got = chf.hull_gpu(d, idt)
            want = oracle.hull(xy, ids)
            assert np.array_equal(got, want), (name, sub)
        m = n
        tb = int(lib.ch_hull_gpu_temp_bytes(m))
        tmp = torch.empty(tb, dtype=torch.uint8, device=DEV)
        out = np.zeros(m, dtype=np.int64)
        h = ctypes.c_int64(0)
        allids = torch.arange(n, dtype=torch.int64, device=DEV)
        st = lib.ch_hull_gpu(chf._ptr(d), (1 << 33) + 1, chf._ptr(allids), m, out.ctypes.data_as(ctypes.c_void_p),
                             ctypes.byref(h), chf._ptr(tmp), tb, chf._stream(None))
        assert st == 0
        assert np.array_equal(out[: h.value], oracle.hull(xy)), (name, "64-bit values")


def test_device_hull_second_round():
    """ch_hull_gpu's second filtering round (64-direction polygon of input
    points, a survivor dropped only when strictly inside a fan triangle by the
    exact orientation): hulls equal the oracle's on sets that put many points
    on polygon edges, diagonals and vertices (duplicates with higher and lower
    ids), dense collinear hull sides, and rings; ch_hull_gpu_async (no second
    round) agrees."""
    rng = np.random.default_rng(99)
    sets = []
    # a square: dense sides (collinear, not strict vertices), corners duplicated, interior points
    t = rng.random(40_000)
    side = np.concatenate([np.stack([t, np.zeros_like(t)], 1), np.stack([np.ones_like(t), t], 1),
                           np.stack([t, np.ones_like(t)], 1), np.stack([np.zeros_like(t), t], 1)])
    corners = np.array([[0.0, 0.0], [1.0, 0.0], [1.0, 1.0], [0.0, 1.0]])
    sq = np.concatenate([rng.random((60_000, 2)), side, np.repeat(corners, 5, 0)])
    sets.append(("square", sq[rng.permutation(len(sq))]))
    # an integer octagon-ish grid: many points exactly on diagonals / edges of any polygon of grid points
    g = rng.integers(-50, 51, size=(200_000, 2)).astype(np.float64)
    g = g[np.abs(g[:, 0]) + np.abs(g[:, 1]) <= 70]
    sets.append(("diamond_grid", g))
    # a ring (C4-like) and a thin ring with duplicates of its outer points
    th = rng.random(300_000) * 2 * np.pi
    r = 0.25 * (1 + 0.1 * (2 * rng.random(300_000) - 1))
    ring = np.stack([r * np.cos(th), r * np.sin(th)], 1)
    sets.append(("ring", ring))
    outer = ring[np.argsort(-r)[:500]]
    sets.append(("ring_dups", np.concatenate([outer, ring, outer])))
    for name, xy in sets:
        d = torch.tensor(xy, device=DEV)
        ids = torch.arange(len(xy), dtype=torch.int64, device=DEV)
        got = chf.hull_gpu(d, ids)                   # ch_hull_gpu: with the second round
        h, c = chf.hull_gpu_async(d, ids)            # ch_hull_gpu_async: without it
        want = oracle.hull(xy)
        assert np.array_equal(got, want), name
        assert np.array_equal(h[: int(c.item())].cpu().numpy(), want), name


def test_device_hull_merges_as_cuts_small_inputs(monkeypatch):
    """The merges-as-cuts path (per-chunk parts, linked non-empty chunks;
    taken by the library from 2^22 sorted points) forced on small inputs
    through CH_HULL_CUTS_MIN=0: the randomized sweep's hard shapes (grids with
    duplicates and collinear runs, circles, rings, vertical ties, chunk
    boundaries) and the golden sets give the oracle's hull."""
    monkeypatch.setenv("CH_HULL_CUTS_MIN", "0")
    for ex in load_golden():
        d = torch.tensor(ex["points"], device=DEV)
        s = torch.tensor(ex["survivors"], dtype=torch.int64, device=DEV)
        assert list(chf.hull_gpu(d, s)) == ex["hull"], ex["name"]
    rng = np.random.default_rng(1234)
    for case in range(20):
        n = int(rng.choice([1, 2, 3, 17, 511, 513, 4_097, 65_537, 300_000]))
        kind = case % 4
        if kind == 0:
            xy = rng.integers(-20, 21, size=(n, 2)).astype(np.float64)
        elif kind == 1:
            t = rng.uniform(0, 2 * np.pi, n)
            xy = np.stack([np.cos(t), np.sin(t)], 1)
        elif kind == 2:
            t = rng.uniform(0, 2 * np.pi, n)
            r = rng.uniform(0.9, 1.0, n)
            xy = np.stack([r * np.cos(t), r * np.sin(t)], 1)
        else:
            xy = rng.normal(0, 1, size=(n, 2))
            xy[:, 0] = np.round(xy[:, 0], 1)
        d = torch.tensor(xy, device=DEV)
        ids = np.sort(rng.choice(n, size=max(1, n - n // 7), replace=False)) if case % 2 else np.arange(n)
        idt = torch.tensor(ids, dtype=torch.int64, device=DEV)
        want = oracle.hull(xy, ids)
        assert np.array_equal(chf.hull_gpu(d, idt), want), (case, n, kind)
        h, c = chf.hull_gpu_async(d, idt)
        assert np.array_equal(h[: int(c.item())].cpu().numpy(), want), (case, n, kind, "async")


def test_device_hull_cuts_path_large_circle():
    """A circle above 2^22 points: the library's own choice is the cuts path;
    every point is a hull vertex, so every merge keeps nearly everything."""
    n = (1 << 22) + 12_345
    xy = synth.points("circle", n, seed=8, device=DEV)
    ids = torch.arange(n, dtype=torch.int64, device=DEV)
    h, c = chf.hull_gpu_async(xy, ids)
    assert np.array_equal(h[: int(c.item())].cpu().numpy(), oracle.hull(xy.cpu().numpy()))


def test_device_hull_sort_tile_and_round_boundaries():
    """Sizes around the radix sort's tile (6144 keys) and its multiples, and
    around the second round's 2^16 threshold, on a circle (every point a hull
    vertex, so any misplaced key changes the hull) and a ring (the round
    drops most points): ch_hull_gpu and ch_hull_gpu_async equal the oracle."""
    rng = np.random.default_rng(6144)
    for n in (6143, 6144, 6145, 12_287, 12_289, 65_535, 65_536, 65_537, 6144 * 11 + 1):
        th = rng.random(n) * 2 * np.pi
        for kind in ("circle", "ring"):
            r = 1.0 if kind == "circle" else 1.0 - 0.05 * rng.random(n)
            xy = np.stack([r * np.cos(th), r * np.sin(th)], 1)
            d = torch.tensor(xy, device=DEV)
            ids = torch.arange(n, dtype=torch.int64, device=DEV)
            want = oracle.hull(xy)
            assert np.array_equal(chf.hull_gpu(d, ids), want), (n, kind)
            h, c = chf.hull_gpu_async(d, ids)
            assert np.array_equal(h[: int(c.item())].cpu().numpy(), want), (n, kind, "async")


def test_k1_f32_keys_rounding_ties():
    """K1's float32 fast path compares fl32(x +- y) with the fp64 bests rounded
    outward; inputs where fl32 and fl64 sums disagree must still give the
    fp64 extremes (R1, lowest index on ties, R2).  Floats near 2^24 (sums not
    representable in fp32); points exactly on x + y = 0.75 and x - y = 0.75
    (fp64 ties, lowest index wins); and a point whose fp64 sum beats that
    line by 2^-26 while its fp32 sum rounds onto it, at a high index."""
    rng = np.random.default_rng(11)
    cases = []
    # 1. near 2^24: x + y needs 25+ bits
    a = (np.float32(2 ** 24) + rng.integers(-64, 64, size=300_000)).astype(np.float32)
    b = (rng.integers(-64, 64, size=300_000) + rng.choice([0.0, 0.5, 0.25], size=300_000)).astype(np.float32)
    cases.append(np.stack([a, b], 1))
    # 2. exact fp64 ties on the lines (t has 10 fraction bits, so 0.75 - t is exact)
    t = (rng.integers(-1024, 1025, size=100_000) / 1024.0 * 0.25).astype(np.float32)
    line = np.concatenate([np.stack([t, np.float32(0.75) - t], 1), np.stack([t, t - np.float32(0.75)], 1)])
    noise = rng.uniform(-0.3, 0.3, size=(200_000, 2)).astype(np.float32)
    pts = np.concatenate([noise, line]).astype(np.float32)
    pts = pts[rng.permutation(len(pts))]
    assert (pts[:, 0].astype(np.float64) + pts[:, 1]).max() == 0.75
    cases.append(pts)
    # 3. x = 1, y = -(1/4 - 2^-26): fp64 sum 0.75 + 2^-26, fp32 sum 0.75
    c3 = pts.copy()
    y3 = np.float32(-(0.25 - 2.0 ** -26))
    assert float(y3) == -(0.25 - 2.0 ** -26) and np.float32(np.float32(1.0) + y3) == np.float32(0.75)
    c3[-3] = (np.float32(1.0), y3)
    cases.append(c3)
    for xy in cases:
        d = torch.tensor(xy, device=DEV)
        ws = chf.Workspace(xy.shape[0])
        e, _ = chf.extremes8(d, ws)
        want, idx8 = oracle.filter_compact(xy.astype(np.float64))
        assert np.array_equal(np.array(e.idx[:]), idx8)
        assert np.array_equal(chf.filter(d).cpu().numpy(), want)
    assert idx8[1] == len(c3) - 3   # the lone point is TR
