"""Pins for the CPU oracle (CPU only).  Each test checks the oracle against
something other than itself: hand-worked values (tests/golden), numpy
library routines, exact rational arithmetic, brute force (Jarvis march,
literal Manhattan minimisation), closed forms and invariants."""
from fractions import Fraction as F

import numpy as np
import pytest

import oracle
import synth
from exact import (det_exact, jarvis_hull, load_golden, manhattan_corner_argmin,
                   near_edge_points, orient_exact, strictly_inside_exact)

GOLDEN = load_golden()


# ---------------------------------------------------------------- golden ----
@pytest.mark.parametrize("ex", GOLDEN, ids=[g["name"] for g in GOLDEN])
def test_golden_worked_examples(ex):
    xy = ex["points"]
    assert list(oracle.extremes8(xy)) == ex["extremes"]
    o = oracle.octagon(xy)
    assert list(o["vidx"]) == ex["octagon"]
    assert o["degenerate"] == ex["degenerate"]
    surv, idx8 = oracle.filter_compact(xy)
    assert list(surv) == ex["survivors"]
    assert list(oracle.hull(xy, surv)) == ex["hull"]
    assert list(oracle.hull(xy)) == ex["hull"]           # filtering never changes the hull
    assert jarvis_hull(xy) == ex["hull"]                # independent brute force agrees


def test_spec_point_strictly_inside_square():
    # square polygon, (1,1) inside, (2,1) on an edge (kept), (3,3) outside.
    sq = np.array([(0, 0), (2, 0), (2, 2), (0, 2), (1, 1), (2, 1), (3, 3)], dtype=np.float64)
    o = oracle.octagon(sq[:4])
    keep = oracle.flags(sq, oct_=o)
    assert list(keep[4:]) == [0, 1, 1]
    assert list(oracle.flags(sq[:5])) == [1, 1, 1, 1, 0]


def test_spec_compaction_examples():
    # S:223 (scan of [1,1,1,1,0]).
    assert list(oracle.compact([1, 1, 1, 1, 0])) == [0, 1, 2, 3]
    assert list(oracle.compact([0, 0, 0])) == []
    assert list(oracle.compact([1, 1, 1])) == [0, 1, 2]
    assert list(oracle.compact([0, 1, 0, 1], index_base=100)) == [101, 103]


def test_admission():
    with pytest.raises(ValueError):
        oracle.filter_compact(np.zeros((0, 2)))
    for bad in (np.nan, np.inf, -np.inf):
        xy = np.array([(0.0, 0.0), (1.0, bad), (2.0, 2.0)])
        assert oracle.admit(xy) == oracle.NONFINITE
        with pytest.raises(ValueError):
            oracle.filter_compact(xy)
    assert oracle.admit(np.array([(1e308, -1e308)])) == oracle.OK


# -------------------------------------------------------------- extremes ----
def _datasets(n, seed):
    rng = np.random.default_rng(seed)
    yield "normal", synth.points("normal", n, seed=seed).numpy()
    yield "circle", synth.points("circle", n, seed=seed).numpy()
    yield "displaced", synth.points("displaced", n, seed=seed, p=0.1).numpy()
    g = rng.integers(-8, 9, size=(n, 2)).astype(np.float64)   # heavy ties
    g[rng.random(n) < 0.1] *= -0.0                               # signed zeros
    yield "grid", g


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_extremes_vs_numpy_first_occurrence(seed):
    """numpy argmax/argmin return the first occurrence = lowest index (a library routine)."""
    for name, xy in _datasets(20000, seed):
        x, y = xy[:, 0], xy[:, 1]
        s, d = x + y, x - y
        want = [np.argmax(x), np.argmax(s), np.argmax(y), np.argmin(d),
                np.argmin(x), np.argmin(s), np.argmin(y), np.argmax(d)]
        assert list(oracle.extremes8(xy)) == [int(w) for w in want], name


def test_extremes_vs_literal_manhattan_corners():
    """corners minimise the Manhattan distance to the bbox corners.  On
    integer coordinates fl(x+y) is exact, so the +-x+-y keys must pick exactly
    the indices of a literal (exact, brute-force) Manhattan minimisation."""
    rng = np.random.default_rng(7)
    for _ in range(20):
        n = int(rng.integers(1, 200))
        xy = rng.integers(-50, 51, size=(n, 2)).astype(np.float64)
        assert list(oracle.extremes8(xy)) == manhattan_corner_argmin(xy)


def test_extremes_self_concatenation_invariance():
    """duplicating the set never changes the chosen (lowest) indices."""
    for name, xy in _datasets(5000, 3):
        a = oracle.extremes8(xy)
        b = oracle.extremes8(np.concatenate([xy, xy]))
        assert list(a) == list(b), name


def test_extremes_optimality():
    """S:176 support-direction optimality, checked exactly on the rounded keys."""
    for name, xy in _datasets(5000, 4):
        idx = oracle.extremes8(xy)
        x, y = xy[:, 0], xy[:, 1]
        keys = [x, x + y, y, -(x - y), -x, -(x + y), -y, x - y]
        for k in range(8):
            assert keys[k][idx[k]] == keys[k].max(), (name, k)
            assert np.flatnonzero(keys[k] == keys[k].max())[0] == idx[k]


# --------------------------------------------------------------- octagon ----
@pytest.mark.parametrize("dist", ["normal", "circle", "displaced"])
def test_octagon_vertices_ccw_convex(dist):
    xy = synth.points(dist, 50000, seed=5).numpy()
    o = oracle.octagon(xy)
    nv = o["nv"]
    assert 3 <= nv <= 8 and not o["degenerate"]   # one point may be extreme in two directions
    V = list(zip(o["vx"], o["vy"]))
    for k in range(nv):
        assert orient_exact(V[k], V[(k + 1) % nv], V[(k + 2) % nv]) >= 0
    # vertices are the support points, consecutive duplicates removed
    idx = oracle.extremes8(xy)
    dedup = []
    for i in idx:
        if not dedup or tuple(xy[i]) != tuple(xy[dedup[-1]]):
            dedup.append(int(i))
    while len(dedup) > 1 and tuple(xy[dedup[-1]]) == tuple(xy[dedup[0]]):
        dedup.pop()
    assert list(o["vidx"]) == dedup
    # edge vectors: ex = fl(bx - ax), ey = fl(by - ay)
    for k in range(nv):
        assert o["ex"][k] == V[(k + 1) % nv][0] - V[k][0]
        assert o["ey"][k] == V[(k + 1) % nv][1] - V[k][1]


def test_threshold_scale_and_bound():
    """T_k = 8 eps S_k exactly (a power-of-two scaling); and T_k exceeds
    Shewchuk's orient2d bound (3 + 16 eps) eps (|l| + |r|) for every point in
    the bounding box (checked at the box corners, where |l| + |r| is largest)."""
    xy = synth.points("normal", 20000, seed=9).numpy()
    o = oracle.octagon(xy)
    xmin, xmax, ymin, ymax = o["bbox"]
    eps = F(1, 2 ** 53)
    for k in range(o["nv"]):
        ax, ay = o["vx"][k], o["vy"][k]
        X = max(xmax - ax, ax - xmin)
        Y = max(ymax - ay, ay - ymin)
        S = abs(o["ex"][k]) * Y + abs(o["ey"][k]) * X
        assert o["thr"][k] == S * 2.0 ** -50
        bound = (3 + 16 * eps) * eps * (abs(F(o["ex"][k])) * F(Y) + abs(F(o["ey"][k])) * F(X))
        assert F(o["thr"][k]) > bound * (1 + 4 * eps)
    assert np.all(oracle.octagon(xy, certified=False)["thr"] == 0.0)


# ---------------------------------------------------------------- filter ----
def _safety_check(xy, certified=True):
    surv, _ = oracle.filter_compact(xy, certified)
    o = oracle.octagon(xy, certified=certified)
    V = list(zip(o["vx"], o["vy"]))
    keep = np.zeros(len(xy), bool)
    keep[surv] = True
    # every discarded point is exactly strictly inside the octagon
    for i in np.flatnonzero(~keep):
        assert strictly_inside_exact(V, xy[i]), i
    # every strict hull vertex survives, and the hull is unchanged
    hull_all = jarvis_hull(xy)
    assert set(hull_all) <= set(surv.tolist())
    assert list(oracle.hull(xy, surv)) == hull_all
    return surv


@pytest.mark.parametrize("dist", ["normal", "circle", "displaced"])
@pytest.mark.parametrize("seed", [0, 1])
def test_filter_safety_exact(dist, seed):
    """P:124 'All points inside the polygon ... are guaranteed not to belong to
    the convex hull': discarded => exactly strictly inside; hull unchanged."""
    xy = synth.points(dist, 400, seed=seed).numpy()
    _safety_check(xy)


def test_filter_safety_adversarial_near_edges():
    """Points within +-3 ulps of octagon edges.  The
    certified predicate never discards a point that is not exactly inside."""
    rng = np.random.default_rng(11)
    base = synth.points("normal", 2000, seed=11).numpy()
    o = oracle.octagon(base)
    V = list(zip(o["vx"], o["vy"]))
    adv = near_edge_points(rng, V, 3000)
    xy = np.concatenate([base, adv])
    o2 = oracle.octagon(xy)
    assert list(o2["vidx"]) == list(o["vidx"])       # adversarial points do not move the octagon
    keep = oracle.flags(xy)
    for i in np.flatnonzero(keep == 0):
        assert strictly_inside_exact(V, xy[i])


def test_plain_predicate_is_unsafe_certified_is_not():
    """Reading #4 (DESIGN R4): the plain fp64 test (T = 0) can discard points
    that are exactly on/outside an edge; the certified test never does."""
    rng = np.random.default_rng(12)
    V = [(0.22508822294500092, 0.06835271525859574), (0.0791090718368002, 0.28086546201638074)]
    # SURVEY App. B.4 counter-example: exact det < 0 but the plain fp64 D > 0.
    a, b = V
    p = (0.08296056976764533, 0.2752585489866622)
    assert det_exact(a, b, p) < 0
    D = (b[0] - a[0]) * (p[1] - a[1]) - (b[1] - a[1]) * (p[0] - a[0])
    assert D > 0
    base = synth.points("circle", 3000, seed=12).numpy()
    o = oracle.octagon(base)
    VV = list(zip(o["vx"], o["vy"]))
    adv = near_edge_points(rng, VV, 20000)
    xy = np.concatenate([base, adv])
    plain = oracle.flags(xy, certified=False)
    cert = oracle.flags(xy, certified=True)
    bad_plain = sum(1 for i in np.flatnonzero(plain == 0) if not strictly_inside_exact(VV, xy[i]))
    bad_cert = sum(1 for i in np.flatnonzero(cert == 0) if not strictly_inside_exact(VV, xy[i]))
    assert bad_cert == 0
    assert bad_plain > 0
    assert np.all(cert >= plain)        # certified keeps a superset


def test_filter_decision_bracketed_by_exact_margins():
    """Both directions of the predicate against exact arithmetic:
    exact det_k <= 0 on some edge => kept;
    exact det_k > 2^-45 S_k on every edge => discarded (T_k = 2^-50 S_k and the
    fp64 error of D_k is < 4 eps S_k, so D_k > T_k)."""
    rng = np.random.default_rng(13)
    base = synth.points("displaced", 3000, seed=13).numpy()
    o = oracle.octagon(base)
    V = list(zip(o["vx"], o["vy"]))
    # points at controlled relative distances inside each edge
    pts = []
    xmin, xmax, ymin, ymax = o["bbox"]
    for k in range(8):
        a, b = V[k], V[(k + 1) % 8]
        ex, ey = b[0] - a[0], b[1] - a[1]
        L = (ex * ex + ey * ey) ** 0.5
        nx, ny = -ey / L, ex / L                     # inward normal
        for e in range(30, 56):
            t = 0.05 + 0.9 * rng.random()
            h = 2.0 ** -e
            pts.append((a[0] + t * ex + nx * h, a[1] + t * ey + ny * h))
            pts.append((a[0] + t * ex - nx * h, a[1] + t * ey - ny * h))
    xy = np.concatenate([base, np.array(pts)])
    o2 = oracle.octagon(xy)
    assert list(o2["vidx"]) == list(o["vidx"])
    keep = oracle.flags(xy)
    S = [F(t) * 2 ** 50 for t in o2["thr"]]
    n_low = n_high = 0
    for i in range(len(base), len(xy)):
        dets = [det_exact(V[k], V[(k + 1) % 8], xy[i]) for k in range(8)]
        if min(dets) <= 0:
            assert keep[i] == 1
            n_low += 1
        elif all(dets[k] > S[k] * F(1, 2 ** 45) for k in range(8)):
            assert keep[i] == 0
            n_high += 1
    assert n_low > 100 and n_high > 100


@pytest.mark.parametrize("seed", [0, 1])
def test_circle_closed_form_all_survive(seed):
    """P:259 'all points are part of a circumference ... no point is
    filtered': every circumference point survives (s = n)."""
    xy = synth.points("circle", 200000, seed=seed).numpy()
    for cert in (True, False):
        surv, _ = oracle.filter_compact(xy, cert)
        assert len(surv) == len(xy)


def test_normal_discards_most():
    """filtered_hull discards > 99% of a normal set."""
    xy = synth.points("normal", 10 ** 6, seed=0).numpy()
    surv, _ = oracle.filter_compact(xy)
    assert len(surv) < 0.01 * len(xy)
    assert len(surv) > 8


def test_displaced_survivor_ratio_reading():
    """Reading R11: rho ~ U[r(1-p), r(1+p)] at p = 0.1 keeps about 28.3% of the
    points (the paper's Table 1 is context only, parity unpinned)."""
    xy = synth.points("displaced", 10 ** 6, seed=0, p=0.1).numpy()
    surv, _ = oracle.filter_compact(xy)
    assert 0.27 < len(surv) / len(xy) < 0.30


def test_compaction_matches_flatnonzero_and_tile_recombination():
    """segment-local scan + global scan of segment totals
    (segment[pos] + global[pos / num_segment]) equals the flat scan."""
    rng = np.random.default_rng(2)
    keep = (rng.random(100003) < 0.3).astype(np.uint8)
    got = oracle.compact(keep)
    assert np.array_equal(got, np.flatnonzero(keep))
    seg = 256
    pad = np.concatenate([keep, np.zeros(-len(keep) % seg, np.uint8)]).reshape(-1, seg).astype(np.int64)
    local = np.cumsum(pad, axis=1) - pad
    glob = np.concatenate([[0], np.cumsum(pad.sum(axis=1))[:-1]])
    recombined = (local + glob[:, None]).reshape(-1)[: len(keep)]
    flat = np.cumsum(keep.astype(np.int64)) - keep
    assert np.array_equal(recombined, flat)
    assert np.array_equal(got, np.flatnonzero(keep))
    assert np.array_equal(flat[got], np.arange(len(got)))


# ------------------------------------------------------------ orientation ----
def test_orient_sign_vs_exact_rational():
    rng = np.random.default_rng(3)
    for _ in range(3000):
        a, b = rng.random(2), rng.random(2)
        t = rng.random()
        c = a + t * (b - a)
        c = np.array([np.nextafter(c[0], np.inf * rng.choice([-1, 1])), c[1]])
        if rng.random() < 0.3:
            c = rng.random(2)
        want = orient_exact(a, b, c)
        assert oracle.orient_sign(a, b, c) == want
        assert oracle.orient_sign(a, c, b) == -want      # antisymmetry
    # SPEC S:66-69
    assert oracle.orient_sign((0, 0), (1, 0), (0, 1)) == 1
    assert oracle.orient_sign((0, 0), (1, 0), (2, 0)) == 0
    assert oracle.orient_sign((0, 0), (0, 1), (1, 1)) == -1


# ------------------------------------------------------------------- hull ----
def test_hull_vs_jarvis_random():
    rng = np.random.default_rng(4)
    for trial in range(60):
        n = int(rng.integers(1, 120))
        if trial % 3 == 0:
            xy = rng.integers(-5, 6, size=(n, 2)).astype(np.float64)   # collinear + duplicates
        elif trial % 3 == 1:
            xy = rng.random((n, 2))
        else:
            th = rng.random(n) * 2 * np.pi
            xy = np.stack([np.cos(th), np.sin(th)], 1)
        assert list(oracle.hull(xy)) == jarvis_hull(xy), trial


def test_hull_spec_examples():
    assert list(oracle.hull([(0, 0), (4, 0), (0, 3)])) == [0, 1, 2]
    th = np.arange(200) * (2 * np.pi / 200)
    xy = np.stack([np.cos(th), np.sin(th)], 1)
    h = oracle.hull(xy)
    assert len(h) == jarvis_hull(xy).__len__()
    assert list(h) == jarvis_hull(xy)


def test_hull_idempotent():
    """hull(hull(S)) == hull(S)."""
    xy = synth.points("displaced", 3000, seed=6).numpy()
    h = oracle.hull(xy)
    assert list(oracle.hull(xy, h)) == list(h)


# -------------------------------------------------- f3: exact predicate ----
@pytest.mark.parametrize("dist", ["normal", "displaced", "circle"])
def test_exact_predicate_matches_rational_definition(dist):
    """f3: discard iff the exact orientation (Fraction) is > 0
    on every octagon edge; the certified survivors are a superset."""
    rng = np.random.default_rng(31)
    base = synth.points(dist, 3000, seed=31).numpy()
    o = oracle.octagon(base)
    V = list(zip(o["vx"], o["vy"]))
    adv = near_edge_points(rng, V, 3000, ulps=3)
    xy = np.concatenate([base, adv])
    assert list(oracle.octagon(xy)["vidx"]) == list(o["vidx"])
    surv_x, _ = oracle.filter_compact_exact(xy)
    keep_x = np.zeros(len(xy), bool)
    keep_x[surv_x] = True
    for i in range(len(xy)):
        assert keep_x[i] == (not strictly_inside_exact(V, xy[i])), i
    surv_c, _ = oracle.filter_compact(xy)
    assert set(surv_x.tolist()) <= set(surv_c.tolist())
    assert list(oracle.hull(xy, surv_x)) == list(oracle.hull(xy))


def test_exact_predicate_golden():
    for ex in load_golden():
        surv, _ = oracle.filter_compact_exact(ex["points"])
        assert list(surv) == ex["survivors"], ex["name"]
