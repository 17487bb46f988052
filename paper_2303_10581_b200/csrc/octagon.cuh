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
#else
#define CH_HD inline
#define CH_ADD(a, b) ((a) + (b))
#define CH_SUB(a, b) ((a) - (b))
#define CH_MUL(a, b) ((a) * (b))
#define CH_INF (__builtin_inf())
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
// every corner satisfies D_k > T_k for every edge, every point of the box
// does, i.e. the box only ever discards points the oracle discards.
CH_HD bool box_valid(const ch_octagon &o, double x0, double x1, double y0, double y1)
{
    if (!(x0 <= x1) || !(y0 <= y1))
        return false;
    for (int k = 0; k < o.nv; k++) {
        double cxs[2] = {x0, x1};
        double cys[2] = {y0, y1};
        for (int i = 0; i < 2; i++)
            for (int j = 0; j < 2; j++) {
                double D = edge_det(o.vx[k], o.vy[k], o.ex[k], o.ey[k], cxs[i], cys[j]);
                if (!(D > o.thr[k]))
                    return false;
            }
    }
    return true;
}

// Octagon assembly (DESIGN R5): cycle [R,TR,T,TL,L,BL,B,BR]; drop a vertex
// equal (numeric ==) to the last kept one, then trailing vertices equal to
// the first; nv < 3 => degenerate (every point survives, R6).  Certified
// threshold T_k = 2^-50 fl(fl(|ex| Y) + fl(|ey| X)) (R4; proof in DESIGN.md).
CH_HD void build_octagon(const ch_extremes &e, int flags, ch_octagon &o)
{
    o.nv = 0;
    o.degenerate = 0;
    o.has_box = 0;
    o.plain = (flags & CH_PLAIN) ? 1 : 0;
    int slot_vertex[8];
    for (int k = 0; k < 8; k++) {
        o.vidx[k] = -1;
        o.vx[k] = o.vy[k] = o.ex[k] = o.ey[k] = o.thr[k] = 0.0;
        o.guess_edge[k] = 0;
    }
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
    for (int k = 0; k < o.nv; k++) {
        int k1 = (k + 1 == o.nv) ? 0 : k + 1;
        double ax = o.vx[k], ay = o.vy[k];
        o.ex[k] = CH_SUB(o.vx[k1], ax);
        o.ey[k] = CH_SUB(o.vy[k1], ay);
        if (o.plain) {
            o.thr[k] = 0.0;
        } else {
            double X = dmax(CH_SUB(o.bbox[1], ax), CH_SUB(ax, o.bbox[0]));
            double Y = dmax(CH_SUB(o.bbox[3], ay), CH_SUB(ay, o.bbox[2]));
            double S = CH_ADD(CH_MUL(dabs(o.ex[k]), Y), CH_MUL(dabs(o.ey[k]), X));
            o.thr[k] = CH_MUL(S, 0x1p-50); // exact power-of-two scaling (RNE if subnormal)
        }
    }
    // Octant k of (x - cx, y - cy) lies between slot directions k and k+1;
    // test first the edge leaving slot k's kept vertex (speed hint only).
    for (int k = 0; k < 8; k++)
        o.guess_edge[k] = slot_vertex[k] < o.nv ? slot_vertex[k] : 0;

    // Early-accept box from the corner vertices, validated (and shrunk
    // toward the centre until valid) with box_valid().
    double x0 = dmax(e.x[3], e.x[5]), x1 = dmin(e.x[1], e.x[7]);
    double y0 = dmax(e.y[5], e.y[7]), y1 = dmin(e.y[1], e.y[3]);
    if (x0 < x1 && y0 < y1) {
        const double shrink[7] = {0.0, 0x1p-40, 0x1p-24, 0x1p-12, 0x1p-6, 0x1p-3, 0x1p-2};
        for (int t = 0; t < 7; t++) {
            double wx = CH_MUL(CH_SUB(x1, x0), shrink[t]);
            double wy = CH_MUL(CH_SUB(y1, y0), shrink[t]);
            double bx0 = CH_ADD(x0, wx), bx1 = CH_SUB(x1, wx);
            double by0 = CH_ADD(y0, wy), by1 = CH_SUB(y1, wy);
            if (box_valid(o, bx0, bx1, by0, by1)) {
                o.box[0] = bx0;
                o.box[1] = bx1;
                o.box[2] = by0;
                o.box[3] = by1;
                o.has_box = 1;
                break;
            }
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
