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

#include "exact.cuh"

// The exact orientation is exact.cuh's chf::orient_sign (the same
// adaptive predicate the device hull and CH_EXACT use), compiled for the host.
namespace chh {
static inline int orient_sign(double ax, double ay, double bx, double by, double cx, double cy)
{
    return chf::orient_sign(ax, ay, bx, by, cx, cy);
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
