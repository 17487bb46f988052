// hull.cpp -- Algorithm 1 line 4 ("connected to any existing convex
// hull implementation"): exact strict convex hull of the filter's
// survivors on the host.  The paper hands the survivors to CGAL on the CPU
// (P:151); CGAL is a comparison system we do not ship, so this is
// Andrew's monotone chain with an adaptive exact orientation predicate
// (DESIGN R8: strict hull, CCW from the lexicographic minimum, duplicates ->
// lowest id, collinear points excluded).  Compiled with -ffp-contract=off.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <numeric>
#include <vector>

namespace chh {

// Knuth two-sum / two-diff and an FMA-based exact product.
static inline void two_sum(double a, double b, double &s, double &e)
{
    s = a + b;
    double bb = s - a;
    e = (a - (s - bb)) + (b - bb);
}
static inline void two_diff(double a, double b, double &s, double &e)
{
    s = a - b;
    double bb = a - s;
    e = (a - (s + bb)) + (bb - b);
}
static inline void two_prod(double a, double b, double &p, double &e)
{
    p = a * b;
    e = std::fma(a, b, -p);
}

// Add b into the non-overlapping expansion h[0..len) (increasing magnitude),
// dropping zero components; returns the new length.
static inline int expansion_add(double *h, int len, double b)
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

// sign((b - a) x (c - a)).  Stage 1: fp64 with Shewchuk's first error bound
// (3 + 16 eps) eps (|l| + |r|).  Stage 2 (rare): the differences are split
// exactly (two_diff), so det = (p1 + p0)(q1 + q0) - (r1 + r0)(s1 + s0) is a
// sum of eight exact products, accumulated exactly.
static int orient_sign(double ax, double ay, double bx, double by, double cx, double cy)
{
    double l = (bx - ax) * (cy - ay);
    double r = (by - ay) * (cx - ax);
    double det = l - r;
    const double eps = 0x1p-53;
    const double bound = (3.0 + 16.0 * eps) * eps;
    double sum = std::fabs(l) + std::fabs(r);
    if (std::fabs(det) > bound * sum)
        return (det > 0) - (det < 0);
    if (l == 0.0 && r == 0.0)
        return 0;
    double p1, p0, q1, q0, r1, r0, s1, s0;
    two_diff(bx, ax, p1, p0);
    two_diff(cy, ay, q1, q0);
    two_diff(by, ay, r1, r0);
    two_diff(cx, ax, s1, s0);
    double h[40];
    int len = 0;
    const double pf[4][2] = {{p1, q1}, {p1, q0}, {p0, q1}, {p0, q0}};
    const double nf[4][2] = {{r1, s1}, {r1, s0}, {r0, s1}, {r0, s0}};
    for (int t = 0; t < 4; t++) {
        double p, e;
        two_prod(pf[t][0], pf[t][1], p, e);
        len = expansion_add(h, len, p);
        len = expansion_add(h, len, e);
        two_prod(nf[t][0], nf[t][1], p, e);
        len = expansion_add(h, len, -p);
        len = expansion_add(h, len, -e);
    }
    for (int i = len - 1; i >= 0; i--)
        if (h[i] != 0.0)
            return (h[i] > 0) - (h[i] < 0);
    return 0;
}

} // namespace chh

extern "C" int ch_internal_orient_sign(double ax, double ay, double bx, double by, double cx, double cy)
{
    return chh::orient_sign(ax, ay, bx, by, cx, cy);
}

// m points (pts[2j], pts[2j+1]) with ids ids[j]; writes the hull ids.
extern "C" int64_t ch_internal_hull(const double *pts, const int64_t *ids, int64_t m, int64_t *hull)
{
    if (m <= 0)
        return 0;
    std::vector<int64_t> ord((size_t)m);
    std::iota(ord.begin(), ord.end(), (int64_t)0);
    std::sort(ord.begin(), ord.end(), [&](int64_t a, int64_t b) {
        double ax = pts[2 * a], bx = pts[2 * b];
        if (ax != bx) return ax < bx;
        double ay = pts[2 * a + 1], by = pts[2 * b + 1];
        if (ay != by) return ay < by;
        return ids[a] < ids[b];
    });
    // unique coordinates; the first of each run has the lowest id
    size_t u = 0;
    for (size_t j = 0; j < ord.size(); j++) {
        int64_t q = ord[j];
        if (u > 0) {
            int64_t p = ord[u - 1];
            if (pts[2 * p] == pts[2 * q] && pts[2 * p + 1] == pts[2 * q + 1])
                continue;
        }
        ord[u++] = q;
    }
    if (u == 1) {
        hull[0] = ids[ord[0]];
        return 1;
    }
    std::vector<int64_t> st;
    st.reserve(2 * u + 1);
    auto turn = [&](int64_t a, int64_t b, int64_t c) {
        return chh::orient_sign(pts[2 * a], pts[2 * a + 1], pts[2 * b], pts[2 * b + 1],
                                pts[2 * c], pts[2 * c + 1]);
    };
    for (size_t j = 0; j < u; j++) {
        while (st.size() >= 2 && turn(st[st.size() - 2], st.back(), ord[j]) <= 0)
            st.pop_back();
        st.push_back(ord[j]);
    }
    size_t lower = st.size() + 1;
    for (size_t j = u - 1; j-- > 0;) {
        while (st.size() >= lower && turn(st[st.size() - 2], st.back(), ord[j]) <= 0)
            st.pop_back();
        st.push_back(ord[j]);
    }
    st.pop_back();
    for (size_t j = 0; j < st.size(); j++)
        hull[j] = ids[st[j]];
    return (int64_t)st.size();
}
