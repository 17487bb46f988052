// hull_gpu.cu -- SURVEY 8(f) f1: Algorithm 1 line 4 (the
// paper's future work P:432 "a complete parallel convex hull ... avoiding
// unnecessary data copying between the device and host") on the device.
//
// The exact strict hull of the survivors (DESIGN R8: CCW from the
// lexicographic minimum, duplicates -> lowest id, collinear points excluded),
// identical to the host monotone chain and the oracle:
//   1. sort the survivors by (x, y) with two stable radix sorts (y, then x) on
//      order-preserving 64-bit keys (-0.0 folded into +0.0); equal points
//      keep increasing-id order;
//   2. lower and upper chains: one thread per chunk of HG_CHUNK sorted points
//      runs Andrew's monotone chain (pop while the exact turn is <= 0,
//      chf::orient_sign; a point equal to its sorted predecessor is skipped,
//      so the lowest id survives); the upper chain is the same routine on the
//      reversed order;
//   3. a tree of merges: adjacent x-separated chains A, B are joined at their
//      bridge (two-pointer walk with the same exact turn test; the result is
//      the unique strict lower chain of A u B), then copied in parallel;
//   4. lower[0..-1) + upper[0..-1) mapped back to ids.
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

__global__ void k_ykeys(const double *__restrict__ xy, const long long *__restrict__ surv, long long m,
                        unsigned long long *__restrict__ key, long long *__restrict__ val)
{
    for (long long j = (long long)blockIdx.x * blockDim.x + threadIdx.x; j < m; j += (long long)gridDim.x * blockDim.x) {
        const long long id = surv[j];
        key[j] = okey(xy[2 * id + 1]);
        val[j] = id;
    }
}

__global__ void k_xkeys(const double *__restrict__ xy, const long long *__restrict__ val, long long m,
                        unsigned long long *__restrict__ key)
{
    for (long long j = (long long)blockIdx.x * blockDim.x + threadIdx.x; j < m; j += (long long)gridDim.x * blockDim.x)
        key[j] = okey(xy[2 * val[j]]);
}

__global__ void k_points(const double *__restrict__ xy, const long long *__restrict__ val, long long m,
                         double2 *__restrict__ P)
{
    for (long long j = (long long)blockIdx.x * blockDim.x + threadIdx.x; j < m; j += (long long)gridDim.x * blockDim.x) {
        const long long id = val[j];
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
__global__ void k_chunk_chain(Seq s, long long nchunks, long long *__restrict__ pos, long long *__restrict__ len)
{
    const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= nchunks)
        return;
    const long long start = t * HG_CHUNK, end = min(start + HG_CHUNK, s.m);
    long long top = 0;
    double2 p1 = make_double2(0, 0), p2 = make_double2(0, 0); // stack[top-1], stack[top-2]
    for (long long r = start; r < end; r++) {
        if (s.dup(r))
            continue;
        const double2 pr = s.at(r);
        while (top >= 2 && turn(p2, p1, pr) <= 0) {
            top--;
            p1 = p2;
            if (top >= 2)
                p2 = s.at(pos[start + top - 2]);
        }
        pos[start + top] = r;
        top++;
        p2 = p1;
        p1 = pr;
    }
    len[t] = top;
}

// Bridge of the chains of chunk groups L = 2pw and R = (2p+1)w.
__global__ void k_bridge(Seq s, long long nchunks, long long w, const long long *__restrict__ pos,
                         const long long *__restrict__ len, long long *__restrict__ bi, long long *__restrict__ bj,
                         long long *__restrict__ len_out)
{
    const long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const long long L = 2 * p * w, R = L + w;
    if (L >= nchunks)
        return;
    const long long la = len[L];
    const long long lb = R < nchunks ? len[R] : 0;
    long long i = la - 1, j = 0;
    if (la > 0 && lb > 0) {
        const long long *A = pos + L * HG_CHUNK, *B = pos + R * HG_CHUNK;
        while (true) {
            bool changed = false;
            while (i > 0 && turn(s.at(A[i - 1]), s.at(A[i]), s.at(B[j])) <= 0) {
                i--;
                changed = true;
            }
            while (j < lb - 1 && turn(s.at(A[i]), s.at(B[j]), s.at(B[j + 1])) <= 0) {
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

// Parallel copy of every merged chain: A[0..i] then B[j..].
__global__ void k_merge_copy(long long m_cap, long long nchunks, long long w, const long long *__restrict__ pos_in,
                             const long long *__restrict__ len_out, const long long *__restrict__ bi,
                             const long long *__restrict__ bj, long long *__restrict__ pos_out)
{
    const long long span = 2 * w * HG_CHUNK;
    for (long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x; g < m_cap; g += (long long)gridDim.x * blockDim.x) {
        const long long p = g / span, q = g - p * span;
        const long long L = 2 * p * w;
        if (L >= nchunks || q >= len_out[L])
            continue;
        const long long i = bi[p];
        pos_out[g] = q <= i ? pos_in[L * HG_CHUNK + q] : pos_in[(L + w) * HG_CHUNK + bj[p] + (q - i - 1)];
    }
}

__global__ void k_assemble(long long m, const long long *__restrict__ low, long long nl, const long long *__restrict__ up,
                           long long nu, const long long *__restrict__ val, long long *__restrict__ out)
{
    // lower[0 .. nl-1) then upper[0 .. nu-1) (each excludes its last point,
    // which is the other's first); upper positions are in reversed order
    const long long a = nl - 1, total = a + (nu - 1);
    for (long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x; g < total; g += (long long)gridDim.x * blockDim.x)
        out[g] = g < a ? val[low[g]] : val[m - 1 - up[g - a]];
}

int grid_for(long long work, int threads)
{
    long long b = (work + threads - 1) / threads;
    return (int)std::max<long long>(1, std::min<long long>(b, 148LL * 16));
}

} // namespace

// One chain (lower: rev = 0, upper: rev = 1) of the m sorted points P; the
// result positions are in pos_a (returned pointer) with length *h.
static long long *chain_gpu(const double2 *P, long long m, int rev, long long *pos_a, long long *pos_b, long long *len_a,
                            long long *len_b, long long *bi, long long *bj, long long *h, cudaStream_t st)
{
    const long long nchunks = (m + HG_CHUNK - 1) / HG_CHUNK;
    const long long m_cap = nchunks * HG_CHUNK;
    Seq s{P, m, rev};
    k_chunk_chain<<<(unsigned)((nchunks + HG_THREADS - 1) / HG_THREADS), HG_THREADS, 0, st>>>(s, nchunks, pos_a, len_a);
    for (long long w = 1; w < nchunks; w *= 2) {
        const long long npairs = (nchunks + 2 * w - 1) / (2 * w);
        k_bridge<<<(unsigned)((npairs + HG_THREADS - 1) / HG_THREADS), HG_THREADS, 0, st>>>(s, nchunks, w, pos_a, len_a,
                                                                                             bi, bj, len_b);
        k_merge_copy<<<grid_for(m_cap, 256), 256, 0, st>>>(m_cap, nchunks, w, pos_a, len_b, bi, bj, pos_b);
        std::swap(pos_a, pos_b);
        std::swap(len_a, len_b);
    }
    cudaMemcpyAsync(h, len_a, sizeof(long long), cudaMemcpyDeviceToHost, st);
    return pos_a;
}

extern "C" {

// Device scratch for ch_hull_gpu on m survivors.
size_t ch_hull_gpu_temp_bytes(int64_t m)
{
    if (m < 1)
        m = 1;
    const size_t nchunks = (size_t)((m + HG_CHUNK - 1) / HG_CHUNK);
    const size_t cap = nchunks * HG_CHUNK;
    size_t sort_tmp = 0;
    cub::DoubleBuffer<unsigned long long> kb(nullptr, nullptr);
    cub::DoubleBuffer<long long> vb(nullptr, nullptr);
    cub::DeviceRadixSort::SortPairs(nullptr, sort_tmp, kb, vb, (int64_t)m);
    auto al = [](size_t b) { return (b + 255) & ~(size_t)255; };
    return al(sort_tmp) + 4 * al((size_t)m * 8)   // keys x2, vals x2
           + al((size_t)m * 16)                     // sorted points
           + 4 * al(cap * 8)                        // chain positions: 2 per chain
           + 4 * al(nchunks * 8 + 8)                // lengths x2, bridges x2
           + al((size_t)m * 8 + 8);                 // assembled hull
}

// Exact strict hull of the m survivors d_surv (indices into d_xy) on the
// device; hull ids are written to h_hull (host, capacity m) and the count to
// *h_n_hull.  Synchronizes `stream`.
ch_status ch_hull_gpu(const double *d_xy, const int64_t *d_surv, int64_t m, int64_t *h_hull, int64_t *h_n_hull,
                      void *d_tmp, size_t tmp_bytes, void *stream)
{
    cudaStream_t st = (cudaStream_t)stream;
    if (!h_n_hull || (m > 0 && (!d_xy || !d_surv || !h_hull || !d_tmp)))
        return CH_ERR_INVALID_ARG;
    if (m == 0) {
        *h_n_hull = 0;
        return CH_OK;
    }
    if (tmp_bytes < ch_hull_gpu_temp_bytes(m))
        return CH_ERR_WORKSPACE;
    const long long nchunks = (m + HG_CHUNK - 1) / HG_CHUNK;
    const size_t cap = (size_t)nchunks * HG_CHUNK;
    size_t sort_tmp = 0;
    {
        cub::DoubleBuffer<unsigned long long> kb(nullptr, nullptr);
        cub::DoubleBuffer<long long> vb(nullptr, nullptr);
        cub::DeviceRadixSort::SortPairs(nullptr, sort_tmp, kb, vb, (int64_t)m);
    }
    auto al = [](size_t b) { return (b + 255) & ~(size_t)255; };
    char *p = (char *)d_tmp;
    void *tmp = p; p += al(sort_tmp);
    auto *k0 = (unsigned long long *)p; p += al((size_t)m * 8);
    auto *k1 = (unsigned long long *)p; p += al((size_t)m * 8);
    auto *v0 = (long long *)p; p += al((size_t)m * 8);
    auto *v1 = (long long *)p; p += al((size_t)m * 8);
    auto *P = (double2 *)p; p += al((size_t)m * 16);
    auto *pa = (long long *)p; p += al(cap * 8);
    auto *pb = (long long *)p; p += al(cap * 8);
    auto *pc = (long long *)p; p += al(cap * 8);
    auto *pd = (long long *)p; p += al(cap * 8);
    auto *la = (long long *)p; p += al((size_t)nchunks * 8 + 8);
    auto *lb = (long long *)p; p += al((size_t)nchunks * 8 + 8);
    auto *bi = (long long *)p; p += al((size_t)nchunks * 8 + 8);
    auto *bj = (long long *)p; p += al((size_t)nchunks * 8 + 8);
    auto *out = (long long *)p;

    const int g = grid_for(m, 256);
    k_ykeys<<<g, 256, 0, st>>>(d_xy, (const long long *)d_surv, m, k0, v0);
    cub::DoubleBuffer<unsigned long long> kb(k0, k1);
    cub::DoubleBuffer<long long> vb(v0, v1);
    size_t tb = sort_tmp;
    if (cub::DeviceRadixSort::SortPairs(tmp, tb, kb, vb, (int64_t)m, 0, 64, st) != cudaSuccess)
        return CH_ERR_CUDA;
    // x keys in the y-sorted order, then a stable sort by x
    k_xkeys<<<g, 256, 0, st>>>(d_xy, vb.Current(), m, kb.Alternate());
    kb.selector ^= 1;
    tb = sort_tmp;
    if (cub::DeviceRadixSort::SortPairs(tmp, tb, kb, vb, (int64_t)m, 0, 64, st) != cudaSuccess)
        return CH_ERR_CUDA;
    const long long *val = vb.Current();
    k_points<<<g, 256, 0, st>>>(d_xy, val, m, P);

    long long hl = 0, hu = 0;
    long long *low_keep = chain_gpu(P, m, 0, pa, pb, la, lb, bi, bj, &hl, st);
    cudaStreamSynchronize(st); // hl is read below; la/lb/bi/bj are reused
    long long *up = chain_gpu(P, m, 1, pc, pd, la, lb, bi, bj, &hu, st);
    cudaStreamSynchronize(st);
    if (cudaGetLastError() != cudaSuccess)
        return CH_ERR_CUDA;
    long long nh;
    if (hl <= 1) {
        // a single distinct point: the lowest id among all survivors
        nh = 1;
        k_assemble<<<1, 1, 0, st>>>(m, low_keep, 2, up, 1, val, out); // out[0] = val[low[0]]
    } else {
        nh = (hl - 1) + (hu - 1);
        k_assemble<<<grid_for(nh, 256), 256, 0, st>>>(m, low_keep, hl, up, hu, val, out);
    }
    cudaMemcpyAsync(h_hull, out, (size_t)nh * 8, cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    if (cudaGetLastError() != cudaSuccess)
        return CH_ERR_CUDA;
    *h_n_hull = nh;
    return CH_OK;
}

} // extern "C"
