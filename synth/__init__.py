"""Seeded synthetic inputs shared by the oracle-side tests and the CUDA path.

This module holds none of the filter's arithmetic: it only draws points from
the three study-case distributions of PAPER.md section 5:

* ``normal``    -- x, y i.i.d. N(mu = 0.5, sigma^2 = 0.1)          (DESIGN R9)
* ``circle``    -- r = 0.25 centred at the origin, theta ~ U[0,2pi) (DESIGN R10)
* ``displaced`` -- radius rho ~ U[r(1-p), r(1+p)], theta ~ U[0,2pi) (DESIGN R11)

Points are produced in fixed chunks of ``CHUNK`` points, chunk ``c`` drawn
from a fresh ``torch.Generator`` seeded with ``seed * 2**20 + c`` on the
target device.  A rank that owns global points [lo, hi) generates exactly the
chunks that overlap that range, so the global array does not depend on the
world size (DESIGN R12).  The same call on "cpu" and "cuda" gives different
(but equally distributed) bytes; every test draws once and feeds the same
bytes to the oracle and to the CUDA library.
"""
from __future__ import annotations

import math

import torch

CHUNK = 1 << 22
R_CIRCLE = 0.25
MU, VAR = 0.5, 0.1
DISTS = ("normal", "circle", "displaced")


def _gen(seed: int, chunk: int, device) -> torch.Generator:
    g = torch.Generator(device=device)
    g.manual_seed((int(seed) * (1 << 20) + int(chunk)) & ((1 << 63) - 1))
    return g


def _chunk(dist: str, seed: int, c: int, p: float, device) -> torch.Tensor:
    g = _gen(seed, c, device)
    if dist == "normal":
        z = torch.randn(CHUNK, 2, dtype=torch.float64, device=device, generator=g)
        return z.mul_(math.sqrt(VAR)).add_(MU)
    u = torch.rand(CHUNK, 2, dtype=torch.float64, device=device, generator=g)
    theta = u[:, 0] * (2.0 * math.pi)
    if dist == "circle":
        rho = torch.full_like(theta, R_CIRCLE)
    elif dist == "displaced":
        rho = R_CIRCLE * (1.0 - p) + (2.0 * R_CIRCLE * p) * u[:, 1]
    else:
        raise ValueError(f"unknown distribution {dist!r}")
    return torch.stack((rho * torch.cos(theta), rho * torch.sin(theta)), dim=1)


def points(dist: str, n: int, seed: int = 0, p: float = 0.1, device="cpu",
           lo: int = 0, hi: int | None = None, out: torch.Tensor | None = None) -> torch.Tensor:
    """Global points [lo, hi) of the n-point set ``dist``/``seed`` as a
    contiguous float64 tensor of shape [hi - lo, 2] (AoS: x at 2i, y at 2i+1)."""
    if hi is None:
        hi = n
    if not (0 <= lo <= hi <= n):
        raise ValueError("bad range")
    m = hi - lo
    if out is None:
        out = torch.empty(m, 2, dtype=torch.float64, device=device)
    c0, c1 = lo // CHUNK, (hi + CHUNK - 1) // CHUNK
    for c in range(c0, c1):
        a, b = max(lo, c * CHUNK), min(hi, (c + 1) * CHUNK)
        blk = _chunk(dist, seed, c, p, out.device)
        out[a - lo: b - lo].copy_(blk[a - c * CHUNK: b - c * CHUNK])
    return out


def shard_range(n: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous shard [floor(r n / W), floor((r+1) n / W)) (DESIGN R14)."""
    return (rank * n) // world, ((rank + 1) * n) // world
