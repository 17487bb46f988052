"""C-ABI tests that need no GPU: the library loads, exports every symbol the
header declares, validates arguments before touching CUDA, and its pure-host
calls (octagon assembly, exact hull) agree with the oracle."""
import ctypes
import os
import re

import numpy as np
import pytest

import oracle
import paper_2303_10581_b200 as chf
import synth
from exact import jarvis_hull, load_golden, orient_exact

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "chfilter.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(ch_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    lib = chf._lib.load()
    names = declared_functions()
    assert len(names) >= 15
    for name in names:
        assert hasattr(lib, name), name
        assert name in chf._lib.SIGNATURES, name
    assert lib.ch_abi_version() == chf._lib.ABI_VERSION == 3


def test_library_is_sm100a():
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", chf._lib.lib_path()], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_status_strings_and_workspace_size():
    lib = chf._lib.load()
    assert lib.ch_status_str(0) == b"CH_OK"
    assert lib.ch_status_str(3) == b"CH_ERR_NONFINITE"
    a, b = lib.ch_workspace_bytes(1), lib.ch_workspace_bytes(10 ** 9)
    assert a % 4096 == 0 and b % 4096 == 0 and b > a
    assert b < 16 * 10 ** 9 // 1000        # << the input (one status word per 4096-point tile)


def test_argument_validation_without_gpu():
    lib = chf._lib.load()
    P = ctypes.c_void_p
    ws = P(1 << 20)        # never dereferenced: validation fails first
    nbytes = lib.ch_workspace_bytes(100)
    st = lib.ch_extremes8(P(1 << 20), 0, 0, 0, None, None, None, ws, nbytes, None)
    assert st == 2                                            # EMPTY
    st = lib.ch_extremes8(P((1 << 20) + 8), 100, 0, 0, None, None, None, ws, nbytes, None)
    assert st == 4                                            # MISALIGNED
    st = lib.ch_extremes8(P(1 << 20), 100, 0, 0, None, None, None, None, nbytes, None)
    assert st == 5                                            # WORKSPACE
    st = lib.ch_filter_compact(P(1 << 20), 10 ** 8, 0, None, P(1 << 21), None, ws, nbytes, None)
    assert st == 5                                            # workspace too small for n
    st = lib.ch_filter_compact(P(1 << 20), 100, 0, None, None, None, ws, nbytes, None)
    assert st == 1                                            # NULL survivors
    assert b"NULL" in lib.ch_last_error()
    assert lib.ch_read_octagon(None, None, None, None) == 1   # NULL workspace


@pytest.mark.parametrize("ex", load_golden(), ids=[g["name"] for g in load_golden()])
def test_host_octagon_build_matches_oracle_golden(ex):
    xy = ex["points"]
    idx = oracle.extremes8(xy)
    e = chf.Extremes()
    for k in range(8):
        e.idx[k] = int(idx[k]); e.x[k] = xy[idx[k], 0]; e.y[k] = xy[idx[k], 1]
    o = chf.octagon_dict(chf.octagon_build(e))
    want = oracle.octagon(xy, idx)
    assert list(o["vidx"]) == ex["octagon"] == list(want["vidx"])
    assert o["degenerate"] == want["degenerate"]
    for f in ("vx", "vy", "ex", "ey", "thr"):
        assert np.array_equal(o[f], want[f]), f


@pytest.mark.parametrize("dist", ["normal", "circle", "displaced"])
@pytest.mark.parametrize("plain", [False, True])
def test_host_octagon_build_bitwise_vs_oracle(dist, plain):
    xy = synth.points(dist, 100000, seed=3).numpy()
    idx = oracle.extremes8(xy)
    e = chf.Extremes()
    for k in range(8):
        e.idx[k] = int(idx[k]); e.x[k] = xy[idx[k], 0]; e.y[k] = xy[idx[k], 1]
    oc = chf.octagon_build(e, plain=plain)
    o = chf.octagon_dict(oc)
    want = oracle.octagon(xy, idx, certified=not plain)
    for f in ("vx", "vy", "ex", "ey", "thr"):
        assert np.array_equal(o[f].view(np.int64), want[f].view(np.int64)), f
    # the early-accept box only contains points the oracle discards
    if o["has_box"]:
        x0, x1, y0, y1 = o["box"]
        inb = (xy[:, 0] >= x0) & (xy[:, 0] <= x1) & (xy[:, 1] >= y0) & (xy[:, 1] <= y1)
        keep = oracle.flags(xy, certified=not plain)
        assert inb.sum() > 0 or dist == "circle"
        assert np.all(keep[inb] == 0)


def test_host_hull_matches_oracle_and_jarvis():
    rng = np.random.default_rng(5)
    for trial in range(40):
        n = int(rng.integers(1, 150))
        if trial % 2:
            xy = rng.integers(-4, 5, size=(n, 2)).astype(np.float64)
        else:
            th = rng.random(n) * 2 * np.pi
            xy = np.stack([np.cos(th), np.sin(th)], 1)
        ids = np.arange(n, dtype=np.int64) + 1000
        got = chf.hull_points(xy, ids)
        assert list(got - 1000) == list(oracle.hull(xy)) == jarvis_hull(xy)


def test_host_hull_golden():
    for ex in load_golden():
        xy = ex["points"]
        s = np.array(ex["survivors"], dtype=np.int64)
        assert list(chf.hull_points(xy[s], s)) == ex["hull"], ex["name"]


def test_host_orient_exact():
    rng = np.random.default_rng(8)
    for _ in range(2000):
        a, b = rng.random(2), rng.random(2)
        c = a + rng.random() * (b - a)
        c[0] = np.nextafter(c[0], [-np.inf, np.inf][rng.integers(2)])
        assert chf.orient_sign(a, b, c) == orient_exact(a, b, c)


def test_caller_octagon_is_validated_before_any_cuda_call():
    """a caller-supplied octagon with nv outside [0, 8] or an
    inconsistent `degenerate` flag is rejected on the host (the kernels index
    eight edge slots); pointers are never dereferenced."""
    lib = chf._lib.load()
    P = ctypes.c_void_p
    ws = P(1 << 20)
    nbytes = lib.ch_workspace_bytes(100)
    base = oracle.octagon(np.array([[0, 0], [2, 0], [2, 2], [0, 2], [1, 1]], dtype=np.float64))
    e = chf.Extremes()
    for k, i in enumerate([1, 2, 2, 3, 0, 0, 0, 1]):
        e.idx[k] = i
    pts = [(0, 0), (2, 0), (2, 2), (0, 2)]
    for k, i in enumerate([1, 2, 2, 3, 0, 0, 0, 1]):
        e.x[k], e.y[k] = pts[i]
    o = chf.octagon_build(e)
    assert o.nv == base["nv"] == 4
    for nv, deg in ((9, 0), (-1, 1), (4, 1), (2, 0)):
        bad = chf.Octagon.from_buffer_copy(o)
        bad.nv, bad.degenerate = nv, deg
        st = lib.ch_filter_compact(P(1 << 20), 100, 0, ctypes.byref(bad), P(1 << 21), None, ws, nbytes, None)
        assert st == 1, (nv, deg)
        st = lib.ch_octagon_filter(P(1 << 20), 100, ctypes.byref(bad), P(1 << 21), ws, nbytes, None)
        assert st == 1, (nv, deg)


def test_host_orient_exact_tiny_magnitudes():
    """products of coordinate differences below ~2^-969 underflow;
    the exact stage scales the differences by a power of two (sign-preserving,
    the determinant is bilinear).  Expected signs follow from scale invariance:
    det((1,1),(1,1+2^-52)) = 2^-52 > 0 at every scale s."""
    for s in (2.0 ** -300, 2.0 ** -540, 2.0 ** -600, 2.0 ** -1000):
        a, b, c = (0.0, 0.0), (s, s), (s, s * (1 + 2.0 ** -52))
        assert chf.orient_sign(a, b, c) == 1, s
        assert chf.orient_sign(a, c, b) == -1, s
        assert chf.orient_sign(a, b, (2 * s, 2 * s)) == 0, s


def test_host_hull_golden_scaled_tiny():
    """The golden hulls are invariant under scaling by a power of two; at
    2^-540 every product of coordinate differences underflows."""
    for s in (2.0 ** -470, 2.0 ** -540, 2.0 ** -700):
        for ex in load_golden():
            xy = np.array(ex["points"], dtype=np.float64) * s
            sv = np.array(ex["survivors"], dtype=np.int64)
            assert list(chf.hull_points(xy[sv], sv)) == ex["hull"], (ex["name"], s)
