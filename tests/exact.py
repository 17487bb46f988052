"""Exact-rational helpers used to pin the oracle (and, through it, the CUDA
path) to mathematics rather than to itself.  Nothing here is imported by the
oracle or by the product; everything uses ``fractions.Fraction`` (exact for
every finite binary64 value) and textbook algorithms different from the
oracle's (Jarvis march instead of Andrew's monotone chain, brute-force
Manhattan distances instead of x+y keys).
"""
from __future__ import annotations

import os
from fractions import Fraction as F

import numpy as np

SLOTS = ("R", "TR", "T", "TL", "L", "BL", "B", "BR")


def orient_exact(a, b, c) -> int:
    """sign((b - a) x (c - a)) in exact rational arithmetic."""
    ax, ay, bx, by, cx, cy = (F(float(v)) for v in (*a, *b, *c))
    det = (bx - ax) * (cy - ay) - (by - ay) * (cx - ax)
    return (det > 0) - (det < 0)


def det_exact(a, b, p) -> F:
    ax, ay, bx, by, px, py = (F(float(v)) for v in (*a, *b, *p))
    return (bx - ax) * (py - ay) - (by - ay) * (px - ax)


def unique_lowest(pts) -> dict:
    """coordinate tuple -> lowest index having it (numeric ==, so -0.0 == 0.0)."""
    seen = {}
    for i, (x, y) in enumerate(pts):
        key = (float(x) + 0.0, float(y) + 0.0)  # +0.0 folds -0.0 into 0.0
        if key not in seen:
            seen[key] = i
    return seen


def jarvis_hull(pts, idx=None) -> list:
    """Strict CCW convex hull by gift wrapping with exact predicates.
    Returns input indices starting at the lexicographic minimum; duplicate
    coordinates resolve to the lowest index; collinear boundary points are
    excluded."""
    pts = [(float(x), float(y)) for x, y in pts]
    if idx is None:
        idx = list(range(len(pts)))
    cand = {}
    for i in idx:
        key = (pts[i][0] + 0.0, pts[i][1] + 0.0)
        if key not in cand or i < cand[key]:
            cand[key] = i
    keys = sorted(cand.keys())
    if len(keys) == 0:
        return []
    if len(keys) == 1:
        return [cand[keys[0]]]
    start = keys[0]
    hull = [start]
    cur = start
    while True:
        nxt = None
        for q in keys:
            if q == cur:
                continue
            if nxt is None:
                nxt = q
                continue
            o = orient_exact(cur, nxt, q)
            if o < 0:  # q is to the right of cur->nxt: wrap tighter
                nxt = q
            elif o == 0:  # collinear: keep the farthest (strict hull)
                d1 = (F(nxt[0]) - F(cur[0])) ** 2 + (F(nxt[1]) - F(cur[1])) ** 2
                d2 = (F(q[0]) - F(cur[0])) ** 2 + (F(q[1]) - F(cur[1])) ** 2
                if d2 > d1:
                    nxt = q
        if nxt == start:
            break
        hull.append(nxt)
        cur = nxt
        if len(hull) > len(keys) + 1:
            raise RuntimeError("jarvis did not close")
    return [cand[k] for k in hull]


def strictly_inside_exact(verts, p) -> bool:
    """p strictly left of every directed edge of the closed cycle verts."""
    nv = len(verts)
    return all(det_exact(verts[k], verts[(k + 1) % nv], p) > 0 for k in range(nv))


def manhattan_corner_argmin(pts) -> list:
    """Slot indices by literally minimising the Manhattan distance to each
    bounding-box corner, exact, lowest index on ties; extremes
    of x / y by exact argmax / argmin.  Returns order R,TR,T,TL,L,BL,B,BR."""
    P = [(F(float(x)), F(float(y))) for x, y in pts]
    xs = [p[0] for p in P]
    ys = [p[1] for p in P]
    xmin, xmax, ymin, ymax = min(xs), max(xs), min(ys), max(ys)

    def argmin(f):
        best, bi = None, -1
        for i, p in enumerate(P):
            v = f(p)
            if best is None or v < best:
                best, bi = v, i
        return bi

    def man(c):
        return lambda p: abs(p[0] - c[0]) + abs(p[1] - c[1])

    return [
        argmin(lambda p: -p[0]),           # R
        argmin(man((xmax, ymax))),         # TR
        argmin(lambda p: -p[1]),           # T
        argmin(man((xmin, ymax))),         # TL
        argmin(lambda p: p[0]),            # L
        argmin(man((xmin, ymin))),         # BL
        argmin(lambda p: p[1]),            # B
        argmin(man((xmax, ymin))),         # BR
    ]


def load_golden(name: str = "worked_examples.txt") -> list:
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", name)
    blocks, cur = [], {}
    with open(path) as f:
        for line in f:
            line = line.rstrip("\n")
            if line.startswith("#"):
                continue
            if not line.strip():
                if cur:
                    blocks.append(cur)
                    cur = {}
                continue
            k, v = line.split(":", 1)
            cur[k.strip()] = v.strip()
    if cur:
        blocks.append(cur)
    out = []
    for b in blocks:
        pts = [tuple(float(t) for t in pair.split()) for pair in b["points"].split(";")]
        ints = lambda s: [int(t) for t in s.split()]  # noqa: E731
        out.append({
            "name": b["name"], "cite": b["cite"],
            "points": np.array(pts, dtype=np.float64),
            "extremes": ints(b["extremes"]), "octagon": ints(b["octagon"]),
            "degenerate": bool(int(b["degenerate"])),
            "survivors": ints(b["survivors"]), "hull": ints(b["hull"]),
        })
    return out


def near_edge_points(rng, verts, m, ulps=3):
    """Points within +-ulps of the segment between consecutive vertices
    (the adversarial set of SURVEY App. B.4)."""
    nv = len(verts)
    out = []
    for _ in range(m):
        k = int(rng.integers(nv))
        a, b = verts[k], verts[(k + 1) % nv]
        t = rng.random()
        x = a[0] + t * (b[0] - a[0])
        y = a[1] + t * (b[1] - a[1])
        for _ in range(int(rng.integers(0, ulps + 1))):
            x = np.nextafter(x, np.inf if rng.random() < 0.5 else -np.inf)
        for _ in range(int(rng.integers(0, ulps + 1))):
            y = np.nextafter(y, np.inf if rng.random() < 0.5 else -np.inf)
        out.append((x, y))
    return np.array(out, dtype=np.float64).reshape(-1, 2)
