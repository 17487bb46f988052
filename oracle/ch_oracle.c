/*
 * oracle/ch_oracle.c -- TEST INFRASTRUCTURE, NOT PRODUCT CODE.
 *
 * A plain, slow, sequential CPU oracle for the convex-hull pre-filter of
 * Carrasco, Ferrada, Navarro, Hitschfeld, "An Evaluation of GPU Filters for
 * Accelerating the 2D Convex Hull" (arXiv 2303.10581).  Citations "P:<line>"
 * refer to /root/reference/PAPER.md, "S:<line>" to SPEC.md, "SURVEY 8(c).k"
 * to the numbered oracle steps / readings of /root/repo/SURVEY.md section 8(c),
 * "DESIGN R<k>" to the readings listed in DESIGN.md.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library.  It shares no code, header,
 * table or helper with the CUDA path (paper_2303_10581_b200/csrc); neither
 * includes or links the other.
 *
 * Build (see oracle/__init__.py): gcc -O2 -ffp-contract=off -fno-fast-math
 *   -fPIC -shared  ->  binary64, round-to-nearest-even, no FMA contraction,
 *   no flush-to-zero.  Every floating-point expression below is evaluated
 *   exactly in the order written.
 *
 * Every function follows the plain definition in the paper's order:
 *   Algorithm 1: findingPolygon -> buildingFilter ->
 *   compactingFilteredPoints -> convexHull_algorithm.
 *
 * Pins: see tests/test_oracle_*.py (hand examples, exact rational signs,
 * brute-force hulls, numpy argmax/argmin, closed forms).  No function here is
 * "parity unpinned".
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define OR_OK 0
#define OR_EMPTY 2
#define OR_NONFINITE 3

/* ------------------------------------------------------------------------ */
/* a1  Admission: n >= 1 and every coordinate finite.  */
/* ------------------------------------------------------------------------ */
int oracle_admit(const double *xy, int64_t n)
{
    if (n < 1)
        return OR_EMPTY;
    for (int64_t i = 0; i < 2 * n; i++)
        if (!isfinite(xy[i]))
            return OR_NONFINITE;
    return OR_OK;
}

/* ------------------------------------------------------------------------ */
/* a2  Eight extremes ("the four extreme points ... and the four points */
/* that, according to the Manhattan distance, are closest to the corners";   */
/* P:185).  Corner c_tr minimises the Manhattan distance   */
/* (xmax-x)+(ymax-y) = const-(x+y), i.e. maximises x+y; likewise    */
/* c_tl <-> min (x-y), c_bl <-> min (x+y), c_br <-> max (x-y).  Keys are the  */
/* rounded fl(x+y), fl(x-y) (SURVEY 8(c) reading #1).                        */
/* Slot order (counter-clockwise): R, TR, T, TL, L, BL, B, BR. */
/* Ties: strict comparison in increasing i keeps the lowest index (reading   */
/* #2).  Numeric comparison, so -0.0 == +0.0.                                */
/* ------------------------------------------------------------------------ */
void oracle_extremes8(const double *xy, int64_t n, int64_t idx[8])
{
    double best[8];
    for (int k = 0; k < 8; k++) {
        idx[k] = 0;
    }
    {
        double x = xy[0], y = xy[1];
        double s = x + y, d = x - y;
        best[0] = x; best[1] = s; best[2] = y; best[3] = d;
        best[4] = x; best[5] = s; best[6] = y; best[7] = d;
    }
    for (int64_t i = 1; i < n; i++) {
        double x = xy[2 * i], y = xy[2 * i + 1];
        double s = x + y;
        double d = x - y;
        if (x > best[0]) { best[0] = x; idx[0] = i; } /* R  : max x   */
        if (s > best[1]) { best[1] = s; idx[1] = i; } /* TR : max x+y */
        if (y > best[2]) { best[2] = y; idx[2] = i; } /* T  : max y   */
        if (d < best[3]) { best[3] = d; idx[3] = i; } /* TL : min x-y */
        if (x < best[4]) { best[4] = x; idx[4] = i; } /* L  : min x   */
        if (s < best[5]) { best[5] = s; idx[5] = i; } /* BL : min x+y */
        if (y < best[6]) { best[6] = y; idx[6] = i; } /* B  : min y   */
        if (d > best[7]) { best[7] = d; idx[7] = i; } /* BR : max x-y */
    }
}

/* ------------------------------------------------------------------------ */
/* a3  Octagon ("counterclockwise"; S:145-153 without the       */
/* convexity repair, SURVEY 8(c).3 and reading #5).                          */
/* ------------------------------------------------------------------------ */
typedef struct {
    int32_t nv;          /* kept vertices (<= 8)                          */
    int32_t degenerate;  /* nv < 3: every point survives (reading #6)     */
    int64_t vidx[8];     /* input index of each kept vertex               */
    double vx[8], vy[8]; /* kept vertex coordinates                       */
    double ex[8], ey[8]; /* edge k: b - a, a = v[k], b = v[(k+1) % nv]     */
    double thr[8];       /* T_k (0 for the plain predicate)               */
    double xmin, xmax, ymin, ymax; /* bounding box from the extremes      */
} oracle_octagon;

void oracle_octagon_build(const double *xy, const int64_t idx8[8], int certified,
                          oracle_octagon *o)
{
    memset(o, 0, sizeof(*o));
    /* Cycle V = [R,TR,T,TL,L,BL,B,BR]; keep a vertex only if its (x,y)
     * differs from the last kept vertex. */
    for (int k = 0; k < 8; k++) {
        double x = xy[2 * idx8[k]], y = xy[2 * idx8[k] + 1];
        if (o->nv > 0 && x == o->vx[o->nv - 1] && y == o->vy[o->nv - 1])
            continue;
        o->vidx[o->nv] = idx8[k];
        o->vx[o->nv] = x;
        o->vy[o->nv] = y;
        o->nv++;
    }
    /* Then drop trailing vertices equal to the first. */
    while (o->nv > 1 && o->vx[o->nv - 1] == o->vx[0] && o->vy[o->nv - 1] == o->vy[0])
        o->nv--;

    o->xmin = xy[2 * idx8[4]]; /* L */
    o->xmax = xy[2 * idx8[0]]; /* R */
    o->ymin = xy[2 * idx8[6] + 1]; /* B */
    o->ymax = xy[2 * idx8[2] + 1]; /* T */

    if (o->nv < 3) {
        o->degenerate = 1;
        return;
    }
    for (int k = 0; k < o->nv; k++) {
        int k1 = (k + 1) % o->nv;
        double ax = o->vx[k], ay = o->vy[k];
        o->ex[k] = o->vx[k1] - ax;
        o->ey[k] = o->vy[k1] - ay;
        if (certified) {
            /* T_k = 8 eps S_k (eps = 2^-53), S_k = |ex| Y + |ey| X with
             * X, Y the largest |x - ax|, |y - ay| over the bounding box.
             * Proof (SURVEY 8(c) "Why the certified threshold is safe"):
             * for every input point |fl(y-ay)| <= Y, |fl(x-ax)| <= X by
             * monotone rounding, so fl(|l|+|r|) <= S; Shewchuk's orient2d
             * bound (3+16 eps) eps fl(|l|+|r|) < T; hence D > T implies the
             * exact orientation is > 0. */
            double X1 = o->xmax - ax, X2 = ax - o->xmin;
            double Y1 = o->ymax - ay, Y2 = ay - o->ymin;
            double X = X1 > X2 ? X1 : X2;
            double Y = Y1 > Y2 ? Y1 : Y2;
            double S = fabs(o->ex[k]) * Y + fabs(o->ey[k]) * X;
            o->thr[k] = ldexp(S, -50);
        } else {
            o->thr[k] = 0.0;
        }
    }
}

/* ------------------------------------------------------------------------ */
/* a5  Octagon test ("checks if it lies within the polygon"; S:155-   */
/* 168).  Discard iff for every edge k                        */
/*   D_k = fl( fl(ex_k * fl(y - ay_k)) - fl(ey_k * fl(x - ax_k)) ) > T_k.    */
/* Boundary and uncertain points are kept (reading #3).                      */
/* ------------------------------------------------------------------------ */
int oracle_discard(const oracle_octagon *o, double x, double y)
{
    if (o->degenerate)
        return 0;
    for (int k = 0; k < o->nv; k++) {
        double dy = y - o->vy[k];
        double dx = x - o->vx[k];
        double l = o->ex[k] * dy;
        double r = o->ey[k] * dx;
        double D = l - r;
        if (!(D > o->thr[k]))
            return 0;
    }
    return 1;
}

/* keep[i] = 1 for a survivor (the paper's bit_vector_flag). */
void oracle_flags(const double *xy, int64_t n, const oracle_octagon *o, uint8_t *keep)
{
    for (int64_t i = 0; i < n; i++)
        keep[i] = (uint8_t)!oracle_discard(o, xy[2 * i], xy[2 * i + 1]);
}

/* ------------------------------------------------------------------------ */
/* a6  Compaction (P:147, P:193-199 filter / scan / scatter):     */
/* the increasing list of survivor indices, plus their count.                */
/* ------------------------------------------------------------------------ */
int64_t oracle_compact(const uint8_t *keep, int64_t n, int64_t index_base, int64_t *out)
{
    int64_t c = 0;
    for (int64_t i = 0; i < n; i++)
        if (keep[i])
            out[c++] = index_base + i;
    return c;
}

/* Algorithm 1 lines 1-3 in one call. Returns the status. */
int oracle_filter_compact(const double *xy, int64_t n, int certified,
                          int64_t idx8_out[8], oracle_octagon *oct_out,
                          int64_t *survivors, int64_t *count)
{
    int st = oracle_admit(xy, n);
    if (st != OR_OK)
        return st;
    int64_t idx8[8];
    oracle_extremes8(xy, n, idx8);
    oracle_octagon oct;
    oracle_octagon_build(xy, idx8, certified, &oct);
    int64_t c = 0;
    for (int64_t i = 0; i < n; i++)
        if (!oracle_discard(&oct, xy[2 * i], xy[2 * i + 1]))
            survivors[c++] = i;
    *count = c;
    if (idx8_out)
        memcpy(idx8_out, idx8, sizeof(idx8));
    if (oct_out)
        *oct_out = oct;
    return OR_OK;
}

/* ------------------------------------------------------------------------ */
/* Exact orientation sign: sign of (b-a) x (c-a), evaluated as an  */
/* exact sum of the six products                                             */
/*   bx*cy - bx*ay - ax*cy - by*cx + by*ax + ay*cx                           */
/* each split exactly into two doubles (product + fma error term), summed    */
/* into a non-overlapping expansion (Shewchuk 1997, Grow-Expansion with zero */
/* elimination).  The sign of a non-overlapping expansion is the sign of its */
/* largest (last) component.  Exact provided no product over/underflows      */
/* (|coordinates| in [2^-480, 2^480] or zero).                               */
/* ------------------------------------------------------------------------ */
static void two_sum(double a, double b, double *s, double *e)
{
    double x = a + b;
    double bv = x - a;
    double av = x - bv;
    double br = b - bv;
    double ar = a - av;
    *s = x;
    *e = ar + br;
}

static int grow(double *h, int hlen, double b)
{
    double q = b;
    int out = 0;
    for (int i = 0; i < hlen; i++) {
        double s, e;
        two_sum(q, h[i], &s, &e);
        q = s;
        if (e != 0.0)
            h[out++] = e;
    }
    if (q != 0.0 || out == 0)
        h[out++] = q;
    return out;
}

int oracle_orient_sign(double ax, double ay, double bx, double by, double cx, double cy)
{
    double f[6][2] = {{bx, cy}, {-bx, ay}, {-ax, cy}, {-by, cx}, {by, ax}, {ay, cx}};
    double h[16];
    int hlen = 0;
    for (int t = 0; t < 6; t++) {
        double p = f[t][0] * f[t][1];
        double e = fma(f[t][0], f[t][1], -p);
        hlen = grow(h, hlen, p);
        hlen = grow(h, hlen, e);
    }
    double top = 0.0;
    for (int i = hlen - 1; i >= 0; i--)
        if (h[i] != 0.0) { top = h[i]; break; }
    return (top > 0.0) - (top < 0.0);
}

/* ------------------------------------------------------------------------ */
/* f3  The exact strict predicate: point p is   */
/* discarded iff orient(v_k, v_{k+1}, p) > 0 exactly on every edge of the     */
/* octagon (the same vertex cycle, R5).  Maximal hull-safe discard.          */
/* ------------------------------------------------------------------------ */
int oracle_orient_sign(double ax, double ay, double bx, double by, double cx, double cy);

int oracle_discard_exact(const oracle_octagon *o, double x, double y)
{
    if (o->degenerate)
        return 0;
    for (int k = 0; k < o->nv; k++) {
        int k1 = (k + 1) % o->nv;
        if (oracle_orient_sign(o->vx[k], o->vy[k], o->vx[k1], o->vy[k1], x, y) <= 0)
            return 0;
    }
    return 1;
}

int oracle_filter_compact_exact(const double *xy, int64_t n, int64_t idx8_out[8], int64_t *survivors,
                                int64_t *count)
{
    int st = oracle_admit(xy, n);
    if (st != OR_OK)
        return st;
    int64_t idx8[8];
    oracle_extremes8(xy, n, idx8);
    oracle_octagon oct;
    oracle_octagon_build(xy, idx8, 1, &oct);
    int64_t c = 0;
    for (int64_t i = 0; i < n; i++)
        if (!oracle_discard_exact(&oct, xy[2 * i], xy[2 * i + 1]))
            survivors[c++] = i;
    *count = c;
    if (idx8_out)
        memcpy(idx8_out, idx8, sizeof(idx8));
    return OR_OK;
}

/* ------------------------------------------------------------------------ */
/* a8  Hull of the candidates ("connected to any existing convex   */
/* hull implementation").  Andrew's monotone    */
/* chain with the exact sign above: sort by (x, y, index), drop duplicate    */
/* coordinates keeping the lowest index, pop while the turn is <= 0 (strict  */
/* hull, collinear points excluded).  Output counter-clockwise starting at   */
/* the lexicographic minimum (reading #8).                                   */
/* ------------------------------------------------------------------------ */
typedef struct {
    double x, y;
    int64_t i;
} or_pt;

static int cmp_pt(const void *pa, const void *pb)
{
    const or_pt *a = (const or_pt *)pa, *b = (const or_pt *)pb;
    if (a->x < b->x) return -1;
    if (a->x > b->x) return 1;
    if (a->y < b->y) return -1;
    if (a->y > b->y) return 1;
    return (a->i > b->i) - (a->i < b->i);
}

/* in: m candidate indices into xy (any order).  out: capacity >= m + 1. */
int64_t oracle_hull(const double *xy, const int64_t *in, int64_t m, int64_t *out)
{
    if (m <= 0)
        return 0;
    or_pt *p = (or_pt *)malloc((size_t)m * sizeof(or_pt));
    for (int64_t j = 0; j < m; j++) {
        p[j].x = xy[2 * in[j]];
        p[j].y = xy[2 * in[j] + 1];
        p[j].i = in[j];
    }
    qsort(p, (size_t)m, sizeof(or_pt), cmp_pt);
    int64_t u = 0; /* unique coordinates, lowest index first */
    for (int64_t j = 0; j < m; j++)
        if (u == 0 || p[j].x != p[u - 1].x || p[j].y != p[u - 1].y)
            p[u++] = p[j];
    if (u == 1) {
        out[0] = p[0].i;
        free(p);
        return 1;
    }
    or_pt *h = (or_pt *)malloc((size_t)(2 * u + 1) * sizeof(or_pt));
    int64_t k = 0;
    for (int64_t j = 0; j < u; j++) { /* lower chain */
        while (k >= 2 && oracle_orient_sign(h[k - 2].x, h[k - 2].y, h[k - 1].x, h[k - 1].y,
                                            p[j].x, p[j].y) <= 0)
            k--;
        h[k++] = p[j];
    }
    int64_t lower = k + 1;
    for (int64_t j = u - 2; j >= 0; j--) { /* upper chain */
        while (k >= lower && oracle_orient_sign(h[k - 2].x, h[k - 2].y, h[k - 1].x, h[k - 1].y,
                                                p[j].x, p[j].y) <= 0)
            k--;
        h[k++] = p[j];
    }
    k--; /* the last point repeats the first */
    for (int64_t j = 0; j < k; j++)
        out[j] = h[j].i;
    free(h);
    free(p);
    return k;
}
