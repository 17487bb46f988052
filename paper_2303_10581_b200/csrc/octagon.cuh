// octagon.cuh -- octagon assembly and the edge predicate (product code).
//
// Compiled for the device (sm_100a, inside K1's last CTA and K3) and for the
// host (ch_octagon_build), from this one definition.  Every floating-point
// step uses explicitly rounded operations (device: __d*_rn intrinsics, which
// are never contracted into DFMA; host: plain operators compiled with
// -ffp-contract=off), so both evaluate binary64 RNE in the stated order.
//
// Paper: P:124 ("The polygon is formed by the four extreme points ... and the
// four points that, according to the Manhattan distance, are closest to the
// corners ... in a counterclockwise fashion"), P:174 (Algorithm 1 line 1),
// P:145 (the inside test).  Readings R1-R6 of DESIGN.md.
#pragma once

#include <stdint.h>

#include "../../include/chfilter.h"

#ifdef __CUDA_ARCH__
#define CH_HD __host__ __device__ __forceinline__
#define CH_ADD(a, b) __dadd_rn((a), (b))
#define CH_SUB(a, b) __dsub_rn((a), (b))
#define CH_MUL(a, b) __dmul_rn((a), (b))
#define CH_INF (__longlong_as_double(0x7ff0000000000000LL))
#define CH_F32(v) __double2float_rn(v)
#define CH_NEXTF(a, b) nextafterf((a), (b))
#define CH_D2LL(v) __double_as_longlong(v)
#define CH_LL2D(v) __longlong_as_double(v)
#else
#define CH_HD inline
#define CH_ADD(a, b) ((a) + (b))
#define CH_SUB(a, b) ((a) - (b))
#define CH_MUL(a, b) ((a) * (b))
#define CH_INF (__builtin_inf())
#define CH_F32(v) ((float)(v))
#define CH_NEXTF(a, b) __builtin_nextafterf((a), (b))
#define CH_D2LL(v) chf_d2ll(v)
#define CH_LL2D(v) chf_ll2d(v)
#include <string.h>
static inline long long chf_d2ll(double v) { long long r; memcpy(&r, &v, 8); return r; }
static inline double chf_ll2d(long long v) { double r; memcpy(&r, &v, 8); return r; }
#endif

namespace chf {

// Edge predicate value D_k(x, y) = fl( fl(ex * fl(y - ay)) - fl(ey * fl(x - ax)) ).
// (P:145 inside test written as an orientation; DESIGN R4.)
CH_HD double edge_det(double ax, double ay, double ex, double ey, double x, double y)
{
    double dy = CH_SUB(y, ay);
    double dx = CH_SUB(x, ax);
    double l = CH_MUL(ex, dy);
    double r = CH_MUL(ey, dx);
    return CH_SUB(l, r);
}

CH_HD double dabs(double v) { return v < 0.0 ? -v : v; }
CH_HD double dmax(double a, double b) { return a > b ? a : b; }
CH_HD double dmin(double a, double b) { return a < b ? a : b; }

// Box validity: D_k is non-decreasing or non-increasing in x and in y
// separately (every RNE operation is monotone in each argument), so on a
// closed axis box its minimum is attained at one of the four corners.  If
// every corner satisfies D_k > T_k for every edge (box_corner_ok below),
// every point of the box does, i.e. the box only ever discards points the
// oracle discards.

// The smallest fp32 value >= v, i.e. v rounded toward +inf (host: round to
// nearest, then one step up if it fell below; device: the directed-rounding
// conversion, one instruction, the same function), and likewise down.
CH_HD float f32_up(double v)
{
#ifdef __CUDA_ARCH__
    return __double2float_ru(v);
#else
    float f = CH_F32(v);
    return ((double)f < v) ? CH_NEXTF(f, __builtin_huge_valf()) : f;
#endif
}
CH_HD float f32_down(double v)
{
#ifdef __CUDA_ARCH__
    return __double2float_rd(v);
#else
    float f = CH_F32(v);
    return ((double)f > v) ? CH_NEXTF(f, -__builtin_huge_valf()) : f;
#endif
}

// fp32 certification of the edge predicate,
// computed per edge in octagon_edge().
// Edge k is first scaled by sigma = 2^s (s = -ilogb(max(|ex|, |ey|)), clamped
// to [-100, 100]), exactly: ex' = sigma ex, ey' = sigma ey, T' = sigma T,
// S' = sigma S.  For a point inside the bounding box let
// E' = a x + b y + c exactly, with a = -ey', b = ex', c = ey' ax - ex' ay, so
// E' = sigma (ex (y - ay) - ey (x - ax)).  Then (eps = 2^-53, u = 2^-24):
//   |sigma D_k - E'| <= 3.001 eps S'                     (five fp64 roundings)
//   v = fma32(fl32(a), fl32(x), fma32(fl32(b), fl32(y), cin))
//   |v - (a x + b y + cin)| <= 4.001 u (|a| Xm + |b| Ym + |cin|)
// (Xm, Ym: largest |x|, |y| in the box).  cin is rounded DOWN from
// fl(c) - T' - M with M = 8 u (B0 + C + |T'|) + 4 eps S' + 2^-100,
// B0 = |a| Xm + |b| Ym, C = |ey' ax| + |ex' ay| (>= |c| and bounding fl(c)'s
// error by 3 eps C).  So c - T' - cin >= M - 3 eps C, which exceeds
// 4.001 u (B0 + |cin|) + 3.001 eps S', and v >= 0 implies E' - T' >
// 3.001 eps S', i.e. D_k > T_k (inside certificate).  The 2^-100 slack
// covers fp32 subnormal roundings (|a|, |b| < 2 after scaling) and sigma
// times the fp64 ones (|s| <= 100).
// Keep certificate from the SAME value v: sigma D_k <= v + (fl(c) - cin)
// + 3 eps C + 4.001 u (B0 + |cin|) + 3.001 eps S', so v < -dk with
// dk >= (fl(c) - cin - T'') + 3 eps C + 4.001 u (B0 + |cin|) + 3.001 eps S'
// implies D_k < T'' / sigma, where T'' = T' (certified, plain: the point is
// kept) or -T' (exact mode: the exact orientation is negative, R4's bound).
// dk is evaluated in fp64 with 5 u, 4 eps S', an extra 16 eps (C + |T'| +
// |cin|) for the fp64 roundings of the sum, 2^-100, a factor 1 + 2^-20, and
// rounded UP to fp32.  The scaling makes |a|, |b| of every edge comparable,
// so one bound f32_delta = max_k dk serves all edges: with
// G = min_k v_k, "G >= 0" proves the point is discarded and
// "G + f32_delta < 0" proves it is kept (v_k = G < -f32_delta <= -dk_k for
// the minimising k).  Enabled only when the box lies within [-2^40, 2^40]^2
// (no fp32 overflow).
CH_HD bool f32_domain_ok(const ch_octagon &o)
{
    const double Xm = dmax(dabs(o.bbox[0]), dabs(o.bbox[1]));
    const double Ym = dmax(dabs(o.bbox[2]), dabs(o.bbox[3]));
    return !o.degenerate && Xm <= 0x1p40 && Ym <= 0x1p40;
}

// Edge k of an octagon whose vertices and bbox are set: ex, ey, S_k, T_k (R4)
// from the vertices and the bbox only.
CH_HD void edge_core(const ch_octagon &o, int k, double &ex, double &ey, double &S, double &T)
{
    const int k1 = (k + 1 == o.nv) ? 0 : k + 1;
    const double ax = o.vx[k], ay = o.vy[k];
    ex = CH_SUB(o.vx[k1], ax);
    ey = CH_SUB(o.vy[k1], ay);
    const double X = dmax(CH_SUB(o.bbox[1], ax), CH_SUB(ax, o.bbox[0]));
    const double Y = dmax(CH_SUB(o.bbox[3], ay), CH_SUB(ay, o.bbox[2]));
    S = CH_ADD(CH_MUL(dabs(ex), Y), CH_MUL(dabs(ey), X));
    T = o.plain ? 0.0 : CH_MUL(S, 0x1p-50); // exact power-of-two scaling
}

// 2^s with s = -(binary exponent of m), clamped to [-100, 100]; 1 for
// m == 0.  From the exponent field (a subnormal m reads as 2^-1023, then
// clamps), so host and device agree exactly.
CH_HD double edge_scale(double m)
{
    if (!(m > 0.0))
        return 1.0;
    int e = (int)((CH_D2LL(m) >> 52) & 0x7ff) - 1023;
    e = e < -100 ? -100 : (e > 100 ? 100 : e);
    return CH_LL2D((long long)(1023 - e) << 52);
}

CH_HD void octagon_edge(ch_octagon &o, int k)
{
    const double ax = o.vx[k], ay = o.vy[k];
    double ex, ey, S, T;
    edge_core(o, k, ex, ey, S, T);
    o.ex[k] = ex;
    o.ey[k] = ey;
    o.thr[k] = T;
    // fp32 certificate constants (used only if f32_domain_ok), on the edge
    // scaled by sigma (exact power-of-two products)
    const double sg = edge_scale(dmax(dabs(ex), dabs(ey)));
    const double sex = CH_MUL(ex, sg), sey = CH_MUL(ey, sg), sT = CH_MUL(T, sg), sS = CH_MUL(S, sg);
    const double Xm = dmax(dabs(o.bbox[0]), dabs(o.bbox[1]));
    const double Ym = dmax(dabs(o.bbox[2]), dabs(o.bbox[3]));
    const double c = CH_SUB(CH_MUL(sey, ax), CH_MUL(sex, ay));
    const double C = CH_ADD(dabs(CH_MUL(sey, ax)), dabs(CH_MUL(sex, ay)));
    const double B0 = CH_ADD(CH_MUL(dabs(sey), Xm), CH_MUL(dabs(sex), Ym));
    // 1 + 2^-20 absorbs the roundings of these fp64 bound computations
    const double M = CH_MUL(CH_ADD(CH_ADD(CH_MUL(CH_ADD(CH_ADD(B0, C), dabs(sT)), 8.0 * 0x1p-24),
                                          CH_MUL(sS, 4.0 * 0x1p-53)),
                                   0x1p-100),
                            1.0 + 0x1p-20);
    const float cin = f32_down(CH_SUB(CH_SUB(c, sT), M));
    o.f32_a[k] = CH_F32(-sey);
    o.f32_b[k] = CH_F32(sex);
    o.f32_c[k] = cin;
    const double acin = dabs((double)cin);
    const double d1 = CH_SUB(CH_SUB(c, (double)cin), o.exact ? -sT : sT);
    const double err = CH_ADD(CH_ADD(CH_ADD(CH_MUL(C, 3.0 * 0x1p-53), CH_MUL(CH_ADD(B0, acin), 5.0 * 0x1p-24)),
                                     CH_MUL(sS, 4.0 * 0x1p-53)),
                              CH_MUL(CH_ADD(CH_ADD(C, dabs(sT)), acin), 16.0 * 0x1p-53));
    o.f32_dk[k] = f32_up(CH_MUL(CH_ADD(CH_ADD(dmax(d1, 0.0), err), 0x1p-100), 1.0 + 0x1p-20));
}

// The common keep bound (after every edge is set).
CH_HD void octagon_f32_delta(ch_octagon &o)
{
    float d = 0.0f;
    for (int k = 0; k < o.nv; k++)
        d = o.f32_dk[k] > d ? o.f32_dk[k] : d;
    o.f32_delta = d;
}

// Octagon assembly (DESIGN R5), vertex part: cycle [R,TR,T,TL,L,BL,B,BR];
// drop a vertex equal (numeric ==) to the last kept one, then trailing
// vertices equal to the first; nv < 3 => degenerate (every point survives,
// R6).  Also the bbox, the octant centre and the guessed-edge table.
CH_HD void octagon_vertices(const ch_extremes &e, int flags, ch_octagon &o)
{
    o.nv = 0;
    o.degenerate = 0;
    o.has_box = 0;
    o.plain = (flags & CH_PLAIN) ? 1 : 0;
    o.exact = (!o.plain && (flags & CH_EXACT)) ? 1 : 0;
    int slot_vertex[8];
    for (int k = 0; k < 8; k++) {
        o.vidx[k] = -1;
        o.vx[k] = o.vy[k] = o.ex[k] = o.ey[k] = o.thr[k] = 0.0;
        o.guess_edge[k] = 0;
        o.f32_a[k] = o.f32_b[k] = o.f32_c[k] = o.f32_dk[k] = 0.0f;
    }
    o.has_f32 = 0;
    o.f32_delta = 0.0f;
    for (int k = 0; k < 8; k++) {
        double x = e.x[k], y = e.y[k];
        if (!(o.nv > 0 && x == o.vx[o.nv - 1] && y == o.vy[o.nv - 1])) {
            o.vidx[o.nv] = e.idx[k];
            o.vx[o.nv] = x;
            o.vy[o.nv] = y;
            o.nv++;
        }
        slot_vertex[k] = o.nv - 1;
    }
    while (o.nv > 1 && o.vx[o.nv - 1] == o.vx[0] && o.vy[o.nv - 1] == o.vy[0]) {
        o.vidx[o.nv - 1] = -1;
        o.nv--;
    }
    o.bbox[0] = e.x[4]; // xmin (L)
    o.bbox[1] = e.x[0]; // xmax (R)
    o.bbox[2] = e.y[6]; // ymin (B)
    o.bbox[3] = e.y[2]; // ymax (T)
    o.box[0] = CH_INF;
    o.box[1] = -CH_INF;
    o.box[2] = CH_INF;
    o.box[3] = -CH_INF;
    o.cx = CH_MUL(0.5, CH_ADD(o.bbox[0], o.bbox[1]));
    o.cy = CH_MUL(0.5, CH_ADD(o.bbox[2], o.bbox[3]));
    if (o.nv < 3) {
        o.degenerate = 1;
        return;
    }
    // Octant k of (x - cx, y - cy) lies between slot directions k and k+1;
    // test first the edge leaving slot k's kept vertex (speed hint only).
    for (int k = 0; k < 8; k++)
        o.guess_edge[k] = slot_vertex[k] < o.nv ? slot_vertex[k] : 0;
}

// Early-accept box candidate t (t < 7): the box spanned by the corner
// vertices, shrunk toward its centre by shrink[t] of its size on each side.
constexpr int BOX_CANDIDATES = 7;
CH_HD bool box_candidate(const ch_extremes &e, int t, double b[4])
{
    const double x0 = dmax(e.x[3], e.x[5]), x1 = dmin(e.x[1], e.x[7]);
    const double y0 = dmax(e.y[5], e.y[7]), y1 = dmin(e.y[1], e.y[3]);
    if (!(x0 < x1 && y0 < y1))
        return false;
    // shrink factors 0, 2^-40, 2^-24, 2^-12, 2^-6, 2^-3, 2^-2 (a select chain:
    // a table indexed at run time would live in local memory on the device)
    const double shrink = t == 0 ? 0.0 : t == 1 ? 0x1p-40 : t == 2 ? 0x1p-24 : t == 3 ? 0x1p-12
                        : t == 4 ? 0x1p-6 : t == 5 ? 0x1p-3 : 0x1p-2;
    const double wx = CH_MUL(CH_SUB(x1, x0), shrink);
    const double wy = CH_MUL(CH_SUB(y1, y0), shrink);
    b[0] = CH_ADD(x0, wx);
    b[1] = CH_SUB(x1, wx);
    b[2] = CH_ADD(y0, wy);
    b[3] = CH_SUB(y1, wy);
    return b[0] <= b[1] && b[2] <= b[3];
}

// One corner of a candidate box against one edge: D_k(corner) > T_k.
CH_HD bool box_corner_ok(const ch_octagon &o, int k, const double b[4], int corner)
{
    const double x = (corner & 1) ? b[1] : b[0];
    const double y = (corner & 2) ? b[3] : b[2];
    return edge_det(o.vx[k], o.vy[k], o.ex[k], o.ey[k], x, y) > o.thr[k];
}

// The same test with the edge recomputed (edge_core: the same operations, so
// the same values as o.ex / o.ey / o.thr): lets the device validate the box
// while other threads are still storing the edges.
CH_HD bool box_corner_ok_core(const ch_octagon &o, int k, const double b[4], int corner)
{
    const double x = (corner & 1) ? b[1] : b[0];
    const double y = (corner & 2) ? b[3] : b[2];
    double ex, ey, S, T;
    edge_core(o, k, ex, ey, S, T);
    return edge_det(o.vx[k], o.vy[k], ex, ey, x, y) > T;
}

// Serial assembly (host, and tests): vertices, every edge, the fp32 domain
// flag, then the first valid accept-box candidate.  The device builds the
// same octagon with one thread per edge / per (candidate, edge, corner).
CH_HD void build_octagon(const ch_extremes &e, int flags, ch_octagon &o)
{
    octagon_vertices(e, flags, o);
    if (o.degenerate)
        return;
    for (int k = 0; k < o.nv; k++)
        octagon_edge(o, k);
    octagon_f32_delta(o);
    o.has_f32 = f32_domain_ok(o) ? 1 : 0;
    for (int t = 0; t < BOX_CANDIDATES; t++) {
        double b[4];
        if (!box_candidate(e, t, b))
            continue;
        bool ok = true;
        for (int k = 0; k < o.nv && ok; k++)
            for (int c = 0; c < 4 && ok; c++)
                ok = box_corner_ok(o, k, b, c);
        if (ok) {
            o.box[0] = b[0];
            o.box[1] = b[1];
            o.box[2] = b[2];
            o.box[3] = b[3];
            o.has_box = 1;
            break;
        }
    }
}

// Slot keys (DESIGN R1): 0 R max x, 1 TR max x+y, 2 T max y, 3 TL min x-y,
// 4 L min x, 5 BL min x+y, 6 B min y, 7 BR max x-y.  is_max[k] tells the
// direction; "better" = better key, then lower global index (R2).
CH_HD double slot_key(int k, double x, double y)
{
    switch (k & 3) {
    case 0: return x;
    case 1: return CH_ADD(x, y);
    case 2: return y;
    default: return CH_SUB(x, y);
    }
}
CH_HD bool slot_is_max(int k) { return k == 0 || k == 1 || k == 2 || k == 7; }
CH_HD bool slot_better(int k, double v, int64_t i, double w, int64_t j)
{
    if (slot_is_max(k)) {
        if (v > w) return true;
        if (v < w) return false;
    } else {
        if (v < w) return true;
        if (v > w) return false;
    }
    return i < j; // equal keys (incl. -0.0 == +0.0): lowest index
}

} // namespace chf
