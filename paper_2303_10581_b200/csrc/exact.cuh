// exact.cuh -- exact orientation sign for the device (and host) paths of the
// product: f3's exact strict predicate and the GPU hull.
//
// orient_sign(a, b, p) = sign((bx - ax)(py - ay) - (by - ay)(px - ax)).
// Stage 1: fp64 with Shewchuk's bound (3 + 16 eps) eps (|l| + |r|) (valid for
// any inputs without over/underflow).  Stage 2: the four differences split
// exactly (two_diff), the two products expanded into eight exact product
// terms (two_prod via FMA), summed into a non-overlapping expansion
// (Grow-Expansion with zero elimination); the sign is that of the largest
// component.  Same arithmetic on host and device (explicitly rounded ops).
#pragma once

#include "octagon.cuh"

#ifdef __CUDA_ARCH__
#define CH_FMA(a, b, c) __fma_rn((a), (b), (c))
#else
#include <cmath>
#define CH_FMA(a, b, c) std::fma((a), (b), (c))
#endif

namespace chf {

CH_HD void two_sum(double a, double b, double &s, double &e)
{
    s = CH_ADD(a, b);
    const double bb = CH_SUB(s, a);
    e = CH_ADD(CH_SUB(a, CH_SUB(s, bb)), CH_SUB(b, bb));
}
CH_HD void two_diff(double a, double b, double &s, double &e)
{
    s = CH_SUB(a, b);
    const double bb = CH_SUB(a, s);
    e = CH_ADD(CH_SUB(a, CH_ADD(s, bb)), CH_SUB(bb, b));
}
CH_HD void two_prod(double a, double b, double &p, double &e)
{
    p = CH_MUL(a, b);
    e = CH_FMA(a, b, -p);
}
// h[0..len) non-overlapping, increasing magnitude; add b; zero elimination.
CH_HD int expansion_grow(double *h, int len, double b)
{
    double q = b;
    int o = 0;
    for (int i = 0; i < len; i++) {
        double s, e;
        two_sum(q, h[i], s, e);
        q = s;
        if (e != 0.0)
            h[o++] = e;
    }
    if (q != 0.0 || o == 0)
        h[o++] = q;
    return o;
}

// Exact sign of (bx-ax)(py-ay) - (by-ay)(px-ax) (stage 2 only).
CH_HD int orient_sign_exact_stage(double ax, double ay, double bx, double by, double px, double py)
{
    double p1, p0, q1, q0, r1, r0, s1, s0;
    two_diff(bx, ax, p1, p0);
    two_diff(py, ay, q1, q0);
    two_diff(by, ay, r1, r0);
    two_diff(px, ax, s1, s0);
    const double pa[4] = {p1, p1, p0, p0}, qa[4] = {q1, q0, q1, q0};
    const double ra[4] = {r1, r1, r0, r0}, sa[4] = {s1, s0, s1, s0};
    double h[34];
    int len = 0;
    for (int t = 0; t < 4; t++) {
        double p, e;
        two_prod(pa[t], qa[t], p, e);
        len = expansion_grow(h, len, p);
        len = expansion_grow(h, len, e);
        two_prod(ra[t], sa[t], p, e);
        len = expansion_grow(h, len, -p);
        len = expansion_grow(h, len, -e);
    }
    for (int i = len - 1; i >= 0; i--)
        if (h[i] != 0.0)
            return (h[i] > 0.0) - (h[i] < 0.0);
    return 0;
}

// Adaptive: fp64 filter first, exact stage only when uncertain.
CH_HD int orient_sign(double ax, double ay, double bx, double by, double px, double py)
{
    const double l = CH_MUL(CH_SUB(bx, ax), CH_SUB(py, ay));
    const double r = CH_MUL(CH_SUB(by, ay), CH_SUB(px, ax));
    const double det = CH_SUB(l, r);
    const double eb = CH_MUL((3.0 + 16.0 * 0x1p-53) * 0x1p-53, CH_ADD(dabs(l), dabs(r)));
    if (det > eb)
        return 1;
    if (-det > eb)
        return -1;
    return orient_sign_exact_stage(ax, ay, bx, by, px, py);
}

} // namespace chf
