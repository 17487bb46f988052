// hull_gpu.cu -- SURVEY 8(f) f1: Algorithm 1 line 4 (the
// paper's future work P:432 "a complete parallel convex hull ... avoiding
// unnecessary data copying between the device and host") on the device.
//
// The exact strict hull of the survivors (DESIGN R8: CCW from the
// lexicographic minimum, duplicates -> lowest id, collinear points excluded),
// identical to the host monotone chain and the oracle:
//   1. sort the survivors by x (one radix sort on order-preserving 64-bit
//      keys, -0.0 folded into +0.0), then resolve every run of equal x in
//      place (k_ties): only the run's lowest point (min y, then lowest id)
//      and highest point (max y, then lowest id) can be strict hull
//      vertices -- the points between them lie inside a vertical segment --
//      so the run becomes [low, low, ..., low, high], which is sorted by
//      (x, y) and whose copies the chains skip as duplicates;
//   2. lower and upper chains: one thread per chunk of HG_CHUNK sorted points
//      runs Andrew's monotone chain (pop while the exact turn is <= 0,
//      chf::orient_sign; a point equal to its sorted predecessor is skipped,
//      so the lowest id survives); the upper chain is the same routine on the
//      reversed order;
//   3. a tree of merges: adjacent x-separated chains A, B are joined at their
//      bridge (two-pointer walk with the same exact turn test; the result is
//      the unique strict lower chain of A u B), then copied in parallel;
//   4. lower[0..-1) + upper[0..-1) mapped back to ids.
// Chain positions (indices into the sorted points) are 32-bit words when
// m < 2^32, else 64-bit; the merge copies index groups with shifts (the
// group span is a power of two).
#include <cuda_runtime.h>

#include <cub/cub.cuh>

#include <algorithm>
#include <cstdint>
#include <vector>

#include "../../include/chfilter.h"
#include "exact.cuh"

namespace {

constexpr long long HG_CHUNK = 512;
constexpr int HG_THREADS = 128;

__device__ __forceinline__ unsigned long long okey(double d)
{
    d = __dadd_rn(d, 0.0); // -0.0 -> +0.0 (numeric equality, R2)
    const unsigned long long u = (unsigned long long)__double_as_longlong(d);
    return (u & 0x8000000000000000ull) ? ~u : (u | 0x8000000000000000ull);
}

template <typename V>
__global__ void k_xkeys(const double *__restrict__ xy, const long long *__restrict__ surv, long long m,
                        unsigned long long *__restrict__ key, V *__restrict__ val)
{
    for (long long j = (long long)blockIdx.x * blockDim.x + threadIdx.x; j < m; j += (long long)gridDim.x * blockDim.x) {
        const long long id = surv ? surv[j] : j; // NULL: every point of xy, in order
        key[j] = okey(xy[2 * id]);
        val[j] = (V)id;
    }
}

// Runs of equal x (numeric ==) in the x-sorted points: the thread at a run's
// head scans it for the lowest point (min y, ties: lowest sort value) and the
// highest (max y, ties: lowest sort value) and rewrites the run as [low, ...,
// low, high].  Only those two can be strict hull vertices (every other point
// of the run lies on the segment between them or equals one of them), the
// result is sorted by (x, y), and the chains skip the copies (a point equal
// to its sorted predecessor).  One thread per run: linear in the run length.
template <typename V>
__global__ void k_ties(double2 *__restrict__ P, V *__restrict__ val, long long m)
{
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (long long)gridDim.x * blockDim.x) {
        const double x = P[i].x;
        if ((i > 0 && P[i - 1].x == x) || i + 1 >= m || P[i + 1].x != x)
            continue; // not the head of a run of >= 2
        double2 lo = P[i], hi = lo;
        V vlo = val[i], vhi = vlo;
        long long e = i + 1;
        for (; e < m; e++) {
            const double2 q = P[e];
            if (q.x != x)
                break;
            const V vq = val[e];
            if (q.y < lo.y || (q.y == lo.y && vq < vlo)) {
                lo = q;
                vlo = vq;
            }
            if (q.y > hi.y || (q.y == hi.y && vq < vhi)) {
                hi = q;
                vhi = vq;
            }
        }
        for (long long k = i; k < e - 1; k++) {
            P[k] = lo;
            val[k] = vlo;
        }
        P[e - 1] = hi;
        val[e - 1] = vhi;
    }
}

template <typename V>
__global__ void k_points(const double *__restrict__ xy, const V *__restrict__ val, long long m,
                         double2 *__restrict__ P)
{
    for (long long j = (long long)blockIdx.x * blockDim.x + threadIdx.x; j < m; j += (long long)gridDim.x * blockDim.x) {
        const long long id = (long long)val[j];
        P[j] = make_double2(xy[2 * id], xy[2 * id + 1]);
    }
}

struct Seq {
    const double2 *P;
    long long m;
    int rev; // 0: lower chain (increasing order), 1: upper chain (reversed)
    __device__ __forceinline__ long long fwd(long long r) const { return rev ? m - 1 - r : r; }
    __device__ __forceinline__ double2 at(long long r) const { return P[fwd(r)]; }
    // equal to its sorted predecessor (so only the lowest id of a run is used)
    __device__ __forceinline__ bool dup(long long r) const
    {
        const long long f = fwd(r);
        return f > 0 && P[f].x == P[f - 1].x && P[f].y == P[f - 1].y;
    }
};

__device__ __forceinline__ int turn(const double2 &a, const double2 &b, const double2 &c)
{
    return chf::orient_sign(a.x, a.y, b.x, b.y, c.x, c.y);
}

// Andrew's monotone chain over one chunk; the stack lives in pos[start..].
template <typename I>
__global__ void k_chunk_chain(Seq s, long long nchunks, I *__restrict__ pos, long long *__restrict__ len)
{
    const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= nchunks)
        return;
    const long long start = t * HG_CHUNK, end = min(start + HG_CHUNK, s.m);
    long long top = 0;
    double2 p1 = make_double2(0, 0), p2 = make_double2(0, 0); // stack[top-1], stack[top-2]
    // One new point per step, loaded a step ahead: the next point in
    // traversal order, which in the upper chain's (reversed) order is also
    // the sorted predecessor P[f - 1] the duplicate test needs; in the lower
    // chain's order the predecessor is the previous point, kept in a register.
    const long long f0 = s.fwd(start);
    double2 cur = s.P[f0];
    double2 pred = (!s.rev && f0 > 0) ? s.P[f0 - 1] : make_double2(0, 0);
    for (long long r = start; r < end; r++) {
        const long long f = s.fwd(r);
        const bool have_nx = s.rev ? f > 0 : r + 1 < end;
        const double2 nx = have_nx ? s.P[s.rev ? f - 1 : f + 1] : cur;
        const double2 pd = s.rev ? nx : pred;
        const bool dup = f > 0 && cur.x == pd.x && cur.y == pd.y;
        if (!dup) {
            while (top >= 2 && turn(p2, p1, cur) <= 0) {
                top--;
                p1 = p2;
                if (top >= 2)
                    p2 = s.at(pos[start + top - 2]);
            }
            pos[start + top] = (I)r;
            top++;
            p2 = p1;
            p1 = cur;
        }
        pred = cur;
        cur = nx;
    }
    len[t] = top;
}

// Chain access for the merges.  Mat: the chains as stored (the chain of the
// group starting at chunk L is pos[L HG_CHUNK ...]).  Merged: the chains of
// the groups one merge level up, not materialised: group L (2w chunks) is
// A[0..i] ++ B[j..] of its two halves (i, j of its pair p = L / 2w).
template <typename I> struct Mat {
    using Idx = I;
    const I *pos;
    __device__ __forceinline__ I at(long long L, long long q) const { return pos[L * HG_CHUNK + q]; }
};
template <typename Inner> struct Merged {
    using Idx = typename Inner::Idx;
    Inner in;             // the chains one level down
    const long long *bi, *bj;
    long long w;          // chunks per half
    int lg2w;             // log2(2 w)
    __device__ __forceinline__ Idx at(long long L, long long q) const
    {
        const long long p = L >> lg2w, i = bi[p];
        return q <= i ? in.at(L, q) : in.at(L + w, bj[p] + (q - i - 1));
    }
};

// Bridge of the chains of groups L = 2pW and R = (2p+1)W (W chunks each).
template <typename I, typename Acc>
__global__ void k_bridge(Seq s, long long nchunks, long long W, const Acc acc, const long long *__restrict__ len,
                         long long *__restrict__ bi, long long *__restrict__ bj, long long *__restrict__ len_out)
{
    const long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const long long L = 2 * p * W, R = L + W;
    if (L >= nchunks)
        return;
    const long long la = len[L];
    const long long lb = R < nchunks ? len[R] : 0;
    long long i = la - 1, j = 0;
    if (la > 0 && lb > 0) {
        while (true) {
            bool changed = false;
            while (i > 0 && turn(s.at(acc.at(L, i - 1)), s.at(acc.at(L, i)), s.at(acc.at(R, j))) <= 0) {
                i--;
                changed = true;
            }
            while (j < lb - 1 && turn(s.at(acc.at(L, i)), s.at(acc.at(R, j)), s.at(acc.at(R, j + 1))) <= 0) {
                j++;
                changed = true;
            }
            if (!changed)
                break;
        }
    }
    bi[p] = i;
    bj[p] = j;
    len_out[L] = (i + 1) + (lb - j);
}

// Parallel copy of every merged chain (groups of 2W chunks): A[0..i] then
// B[j..], A and B read through `acc`.  The group span 2 W HG_CHUNK is a power
// of two: group and offset by shift and mask.
template <typename I, typename Acc>
__global__ void k_merge_copy(long long m_cap, long long nchunks, long long W, int span_log2, const Acc acc,
                             const long long *__restrict__ len_out, const long long *__restrict__ bi,
                             const long long *__restrict__ bj, I *__restrict__ pos_out)
{
    const long long mask = (1ll << span_log2) - 1;
    for (long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x; g < m_cap; g += (long long)gridDim.x * blockDim.x) {
        const long long p = g >> span_log2, q = g & mask;
        const long long L = 2 * p * W;
        if (L >= nchunks || q >= len_out[L])
            continue;
        const long long i = bi[p];
        pos_out[g] = q <= i ? acc.at(L, q) : acc.at(L + W, bj[p] + (q - i - 1));
    }
}

// lower[0 .. nl-1) then upper[0 .. nu-1) (each excludes its last point,
// which is the other's first); upper positions are in reversed order.  The
// chain lengths are read on the device, so nothing waits for the host.
template <typename I, typename V>
__global__ void k_assemble(long long m, const I *__restrict__ low, const long long *__restrict__ d_nl,
                           const I *__restrict__ up, const long long *__restrict__ d_nu,
                           const V *__restrict__ val, const long long *__restrict__ idmap, long long *__restrict__ out,
                           long long *__restrict__ d_nh)
{
    // idmap (nullable): the output id of sort value v is idmap[v]
    auto id = [&](V v) { return idmap ? idmap[(long long)v] : (long long)v; };
    const long long nl = *d_nl, nu = *d_nu;
    if (nl <= 1) {
        // a single distinct point: the lowest id among all survivors
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            out[0] = id(val[low[0]]);
            *d_nh = 1;
        }
        return;
    }
    const long long a = nl - 1, total = a + (nu - 1);
    if (blockIdx.x == 0 && threadIdx.x == 0)
        *d_nh = total;
    for (long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x; g < total; g += (long long)gridDim.x * blockDim.x)
        out[g] = g < a ? id(val[low[g]]) : id(val[m - 1 - (long long)up[g - a]]);
}

// One thread per item (the bridges: not grid-stride).
unsigned blocks_for(long long items, int threads) { return (unsigned)std::max<long long>(1, (items + threads - 1) / threads); }

int grid_for(long long work, int threads)
{
    long long b = (work + threads - 1) / threads;
    return (int)std::max<long long>(1, std::min<long long>(b, 148LL * 16));
}

} // namespace

// One chain (lower: rev = 0, upper: rev = 1) of the m sorted points P; the
// result positions are in the returned buffer (pos_a or pos_b), the length in
// the returned device word (len_a[0] or len_b[0]).  Asynchronous.
template <typename I>
static I *chain_gpu(const double2 *P, long long m, int rev, I *pos_a, I *pos_b, long long *len_a, long long *len_b,
                    long long *bi, long long *bj, long long *bi2, long long *bj2, long long *bi3, long long *bj3,
                    long long *len_m, long long *len_m2, const long long **d_len, cudaStream_t st)
{
    const long long nchunks = (m + HG_CHUNK - 1) / HG_CHUNK;
    const long long m_cap = nchunks * HG_CHUNK;
    Seq s{P, m, rev};
    k_chunk_chain<I><<<(unsigned)((nchunks + HG_THREADS - 1) / HG_THREADS), HG_THREADS, 0, st>>>(s, nchunks, pos_a,
                                                                                                  len_a);
    static_assert((HG_CHUNK & (HG_CHUNK - 1)) == 0, "chunk size is a power of two");
    int lgw = 0, lgc = 0; // log2 w, log2 HG_CHUNK
    while ((1ll << lgc) < HG_CHUNK)
        lgc++;
    // Up to three merge levels per copy: each level's bridges read the chains
    // of the level below through Merged (not materialised), then one copy
    // materialises them -- a third of the copies of one level at a time.
    for (long long w = 1; w < nchunks;) {
        const long long np1 = (nchunks + 2 * w - 1) / (2 * w);
        const Mat<I> m0{pos_a};
        if (2 * w >= nchunks) {
            k_bridge<I><<<blocks_for(np1, HG_THREADS), HG_THREADS, 0, st>>>(s, nchunks, w, m0, len_a, bi, bj, len_b);
            k_merge_copy<I><<<grid_for(m_cap, 256), 256, 0, st>>>(m_cap, nchunks, w, lgw + 1 + lgc, m0, len_b, bi,
                                                                  bj, pos_b);
            w *= 2;
            lgw += 1;
        } else {
            k_bridge<I><<<blocks_for(np1, HG_THREADS), HG_THREADS, 0, st>>>(s, nchunks, w, m0, len_a, bi, bj, len_m);
            const Merged<Mat<I>> m1{m0, bi, bj, w, lgw + 1};
            const long long np2 = (nchunks + 4 * w - 1) / (4 * w);
            if (4 * w >= nchunks) {
                k_bridge<I><<<blocks_for(np2, HG_THREADS), HG_THREADS, 0, st>>>(s, nchunks, 2 * w, m1, len_m, bi2, bj2,
                                                                              len_b);
                k_merge_copy<I><<<grid_for(m_cap, 256), 256, 0, st>>>(m_cap, nchunks, 2 * w, lgw + 2 + lgc, m1, len_b,
                                                                      bi2, bj2, pos_b);
                w *= 4;
                lgw += 2;
            } else {
                k_bridge<I><<<blocks_for(np2, HG_THREADS), HG_THREADS, 0, st>>>(s, nchunks, 2 * w, m1, len_m, bi2, bj2,
                                                                              len_m2);
                const Merged<Merged<Mat<I>>> m2{m1, bi2, bj2, 2 * w, lgw + 2};
                const long long np3 = (nchunks + 8 * w - 1) / (8 * w);
                k_bridge<I><<<blocks_for(np3, HG_THREADS), HG_THREADS, 0, st>>>(s, nchunks, 4 * w, m2, len_m2, bi3, bj3,
                                                                              len_b);
                k_merge_copy<I><<<grid_for(m_cap, 256), 256, 0, st>>>(m_cap, nchunks, 4 * w, lgw + 3 + lgc, m2, len_b,
                                                                      bi3, bj3, pos_b);
                w *= 8;
                lgw += 3;
            }
        }
        std::swap(pos_a, pos_b);
        std::swap(len_a, len_b);
    }
    *d_len = len_a;
    return pos_a;
}

// Scratch layout of ch_hull_gpu_async for m survivors (all 256-B aligned).
struct HullTmp {
    size_t sort_tmp = 0, total = 0;
    size_t o_k0, o_k1, o_v0, o_v1, o_P, o_pa, o_pb, o_pc, o_pd, o_la, o_lb, o_lc, o_ld, o_bi, o_bj, o_out;
    size_t o_bi2, o_bj2, o_lm, o_bi3, o_bj3, o_lm2;
    explicit HullTmp(long long m)
    {
        if (m < 1)
            m = 1;
        const size_t nchunks = (size_t)((m + HG_CHUNK - 1) / HG_CHUNK), cap = nchunks * HG_CHUNK;
        const size_t isz = m < (1ll << 32) ? 4 : 8; // chain position width
        cub::DoubleBuffer<unsigned long long> kb(nullptr, nullptr);
        cub::DoubleBuffer<long long> vb(nullptr, nullptr);
        cub::DeviceRadixSort::SortPairs(nullptr, sort_tmp, kb, vb, (int64_t)m);
        size_t p = 0;
        auto take = [&](size_t b) { const size_t o = p; p += (b + 255) & ~(size_t)255; return o; };
        take(sort_tmp);
        o_k0 = take((size_t)m * 8); o_k1 = take((size_t)m * 8);
        o_v0 = take((size_t)m * 8); o_v1 = take((size_t)m * 8);
        o_P = take((size_t)m * 16);
        o_pa = take(cap * isz); o_pb = take(cap * isz); o_pc = take(cap * isz); o_pd = take(cap * isz);
        o_la = take(nchunks * 8 + 8); o_lb = take(nchunks * 8 + 8);
        o_lc = take(nchunks * 8 + 8); o_ld = take(nchunks * 8 + 8);
        o_bi = take(nchunks * 8 + 8); o_bj = take(nchunks * 8 + 8);
        o_bi2 = take(nchunks * 8 + 8); o_bj2 = take(nchunks * 8 + 8); o_lm = take(nchunks * 8 + 8);
        o_bi3 = take(nchunks * 8 + 8); o_bj3 = take(nchunks * 8 + 8); o_lm2 = take(nchunks * 8 + 8);
        o_out = take((size_t)m * 8 + 8);
        total = p;
    }
};

// The pipeline with sort values (survivor ids) of type V.
template <typename V>
// surv == NULL: the hull of d_xy[0..m) itself; idmap (nullable) maps the
// resulting point positions / ids to output ids.
static ch_status hull_async(const double *d_xy, const long long *surv, long long m, long long *d_hull,
                            long long *d_n_hull, void *d_tmp, const HullTmp &L, cudaStream_t st,
                            const long long *idmap = nullptr)
{
    char *b = (char *)d_tmp;
    auto *k0 = (unsigned long long *)(b + L.o_k0), *k1 = (unsigned long long *)(b + L.o_k1);
    auto *v0 = (V *)(b + L.o_v0), *v1 = (V *)(b + L.o_v1);
    auto *P = (double2 *)(b + L.o_P);
    auto *pa = b + L.o_pa, *pb = b + L.o_pb, *pc = b + L.o_pc, *pd = b + L.o_pd;
    auto *la = (long long *)(b + L.o_la), *lb = (long long *)(b + L.o_lb);
    auto *lc = (long long *)(b + L.o_lc), *ld = (long long *)(b + L.o_ld);
    auto *bi = (long long *)(b + L.o_bi), *bj = (long long *)(b + L.o_bj);
    auto *bi2 = (long long *)(b + L.o_bi2), *bj2 = (long long *)(b + L.o_bj2), *lm = (long long *)(b + L.o_lm);
    auto *bi3 = (long long *)(b + L.o_bi3), *bj3 = (long long *)(b + L.o_bj3), *lm2 = (long long *)(b + L.o_lm2);

    const int g = grid_for(m, 256);
    k_xkeys<V><<<g, 256, 0, st>>>(d_xy, surv, m, k0, v0);
    cub::DoubleBuffer<unsigned long long> kb(k0, k1);
    cub::DoubleBuffer<V> vb(v0, v1);
    size_t tb = L.sort_tmp;
    if (cub::DeviceRadixSort::SortPairs(d_tmp, tb, kb, vb, (int64_t)m, 0, 64, st) != cudaSuccess)
        return CH_ERR_CUDA;
    V *val = vb.Current();
    k_points<V><<<g, 256, 0, st>>>(d_xy, val, m, P);
    k_ties<V><<<g, 256, 0, st>>>(P, val, m); // equal x: the run's lowest and highest points

    auto chains = [&](auto tag) {
        using I = decltype(tag);
        const long long *d_hl, *d_hu;
        const I *low = chain_gpu<I>(P, m, 0, (I *)pa, (I *)pb, la, lb, bi, bj, bi2, bj2, bi3, bj3, lm, lm2, &d_hl, st);
        const I *up = chain_gpu<I>(P, m, 1, (I *)pc, (I *)pd, lc, ld, bi, bj, bi2, bj2, bi3, bj3, lm, lm2, &d_hu, st);
        k_assemble<I, V><<<grid_for(m, 256), 256, 0, st>>>(m, low, d_hl, up, d_hu, val, idmap, d_hull, d_n_hull);
    };
    if (m < (1ll << 32))
        chains((unsigned)0);
    else
        chains((long long)0);
    return cudaGetLastError() == cudaSuccess ? CH_OK : CH_ERR_CUDA;
}

extern "C" {

// Device scratch for ch_hull_gpu / ch_hull_gpu_async on m survivors.
size_t ch_hull_gpu_temp_bytes(int64_t m)
{
    return HullTmp(m).total;
}

// The device hull, asynchronous: hull ids to d_hull (device, capacity m), the
// count to *d_n_hull (device).  No host synchronization.
ch_status ch_hull_gpu_async(const double *d_xy, int64_t n_points, const int64_t *d_surv, int64_t m,
                            int64_t *d_hull, int64_t *d_n_hull, void *d_tmp, size_t tmp_bytes, void *stream)
{
    cudaStream_t st = (cudaStream_t)stream;
    if (m < 0 || n_points < 0 || !d_n_hull || (m > 0 && (!d_xy || !d_surv || !d_hull || !d_tmp)))
        return CH_ERR_INVALID_ARG;
    if (m == 0)
        return cudaMemsetAsync(d_n_hull, 0, sizeof(int64_t), st) == cudaSuccess ? CH_OK : CH_ERR_CUDA;
    const HullTmp L(m);
    if (tmp_bytes < L.total)
        return CH_ERR_WORKSPACE;
    // ids fit 32 bits when the point array does: the sorts then move 12, not
    // 16, bytes per element and pass
    return n_points <= (1ll << 32) ? hull_async<unsigned>(d_xy, (const long long *)d_surv, m, (long long *)d_hull,
                                                           (long long *)d_n_hull, d_tmp, L, st)
                                   : hull_async<unsigned long long>(d_xy, (const long long *)d_surv, m,
                                                                    (long long *)d_hull, (long long *)d_n_hull, d_tmp,
                                                                    L, st);
}

// The hull of m points given by their coordinates d_pts (e.g. survivors
// gathered from every rank, in increasing id order) and ids d_ids.  Same
// canonical form; duplicates resolve to the lowest position, which is the
// lowest id when d_ids is increasing.  Asynchronous like ch_hull_gpu_async.
ch_status ch_hull_gpu_pts_async(const double *d_pts, const int64_t *d_ids, int64_t m, int64_t *d_hull,
                                int64_t *d_n_hull, void *d_tmp, size_t tmp_bytes, void *stream)
{
    cudaStream_t st = (cudaStream_t)stream;
    if (m < 0 || !d_n_hull || (m > 0 && (!d_pts || !d_ids || !d_hull || !d_tmp)))
        return CH_ERR_INVALID_ARG;
    if (m == 0)
        return cudaMemsetAsync(d_n_hull, 0, sizeof(int64_t), st) == cudaSuccess ? CH_OK : CH_ERR_CUDA;
    const HullTmp L(m);
    if (tmp_bytes < L.total)
        return CH_ERR_WORKSPACE;
    return m <= (1ll << 32) ? hull_async<unsigned>(d_pts, nullptr, m, (long long *)d_hull, (long long *)d_n_hull,
                                                    d_tmp, L, st, (const long long *)d_ids)
                            : hull_async<unsigned long long>(d_pts, nullptr, m, (long long *)d_hull,
                                                             (long long *)d_n_hull, d_tmp, L, st,
                                                             (const long long *)d_ids);
}

// The device hull with the ids copied to h_hull (host, capacity m).
// Synchronizes `stream`.
ch_status ch_hull_gpu(const double *d_xy, int64_t n_points, const int64_t *d_surv, int64_t m, int64_t *h_hull,
                      int64_t *h_n_hull, void *d_tmp, size_t tmp_bytes, void *stream)
{
    cudaStream_t st = (cudaStream_t)stream;
    if (!h_n_hull || (m > 0 && (!d_xy || !d_surv || !h_hull || !d_tmp)))
        return CH_ERR_INVALID_ARG;
    if (m <= 0) {
        *h_n_hull = 0;
        return m == 0 ? CH_OK : CH_ERR_INVALID_ARG;
    }
    const HullTmp L(m);
    if (tmp_bytes < L.total)
        return CH_ERR_WORKSPACE;
    int64_t *d_out = (int64_t *)((char *)d_tmp + L.o_out);
    int64_t *d_nh = d_out + m; // the word after the ids (o_out holds m + 1 words)
    ch_status s = ch_hull_gpu_async(d_xy, n_points, d_surv, m, d_out, d_nh, d_tmp, tmp_bytes, stream);
    if (s != CH_OK)
        return s;
    int64_t nh = 0;
    cudaMemcpyAsync(&nh, d_nh, sizeof(nh), cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    cudaMemcpyAsync(h_hull, d_out, (size_t)nh * 8, cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    if (cudaGetLastError() != cudaSuccess)
        return CH_ERR_CUDA;
    *h_n_hull = nh;
    return CH_OK;
}

} // extern "C"
