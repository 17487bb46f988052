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
//
// Underflow: two_prod is exact only while a product stays above
// about 2^-969, and Shewchuk's bound assumes no underflow.  So stage 1 decides
// only when |l| + |r| >= 2^-900, and stage 2 first scales the eight exact
// difference components by one power of two (the determinant is bilinear, so
// its sign is unchanged) so that the largest lies in [2^479, 2^480).  Stage 2
// is then exact whenever the nonzero components span at most 2^963, e.g. for
// every input whose coordinates are all tiny (|x| ~ 1e-160 and below).
#pragma once

#include "octagon.cuh"

#ifdef __CUDA_ARCH__
#define CH_FMA(a, b, c) __fma_rn((a), (b), (c))
#define CH_ILOGB(a) ilogb(a)
#define CH_LDEXP(a, e) ldexp((a), (e))
#else
#include <cmath>
#define CH_FMA(a, b, c) std::fma((a), (b), (c))
#define CH_ILOGB(a) std::ilogb(a)
#define CH_LDEXP(a, e) std::ldexp((a), (e))
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
    // scale every component by 2^(479 - ilogb(max)): exact (a power of two,
    // no overflow), sign-preserving (bilinear determinant)
    const double m = dmax(dmax(dmax(dabs(p1), dabs(q1)), dmax(dabs(r1), dabs(s1))),
                          dmax(dmax(dabs(p0), dabs(q0)), dmax(dabs(r0), dabs(s0))));
    if (m == 0.0)
        return 0;
    if (m < 0x1p479) {
        const int sh = 479 - CH_ILOGB(m);
        p1 = CH_LDEXP(p1, sh), p0 = CH_LDEXP(p0, sh), q1 = CH_LDEXP(q1, sh), q0 = CH_LDEXP(q0, sh);
        r1 = CH_LDEXP(r1, sh), r0 = CH_LDEXP(r0, sh), s1 = CH_LDEXP(s1, sh), s0 = CH_LDEXP(s0, sh);
    }
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
    const double sum = CH_ADD(dabs(l), dabs(r));
    const double eb = CH_MUL((3.0 + 16.0 * 0x1p-53) * 0x1p-53, sum);
    if (sum >= 0x1p-900) { // (below: the products may have underflowed)
        if (det > eb)
            return 1;
        if (-det > eb)
            return -1;
    }
    return orient_sign_exact_stage(ax, ay, bx, by, px, py);
}

} // namespace chf
