// hull_gpu.cu -- SURVEY 8(f) f1: Algorithm 1 line 4 (the
// paper's future work P:432 "a complete parallel convex hull ... avoiding
// unnecessary data copying between the device and host") on the device.
//
// The exact strict hull of the survivors (DESIGN R8: CCW from the
// lexicographic minimum, duplicates -> lowest id, collinear points excluded),
// identical to the host monotone chain and the oracle:
//   1. sort the survivors by x: a hand-written LSD radix sort (radix_sort.cuh,
//      four 8-bit onesweep passes) on 32-bit keys that quantise x linearly
//      and monotonically over the survivors' x range, then every run of equal
//      keys sorted by x exactly (a thread per short run, a CTA per long one,
//      which runs the same radix ranking on the 64-bit order-preserving keys
//      of x, -0.0 folded into +0.0); in the same step every run of equal x is
//      resolved: only the run's lowest point (min y, then lowest id) and
//      highest point (max y, then lowest id) can be strict hull vertices --
//      the points between them lie inside a vertical segment -- so the run
//      becomes [low, low, ..., low, high], which is sorted by (x, y) and
//      whose copies the chains skip as duplicates;
//   2. lower and upper chains: one thread per chunk of 2^chunk_log2(m) sorted points
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


#include <algorithm>
#include <cstdlib>
#include <cmath>
#include <string>
#include <cstdint>
#include <vector>

#include "../../include/chfilter.h"
#include "exact.cuh"
#include "internal.h"
#include "radix_sort.cuh"

namespace {

// Points per chunk chain: a power of two from 16 (few survivors: enough
// threads for the serial walks) to 512 (many: fewer merge levels).
constexpr int HG_LGC_MIN = 4, HG_LGC_MAX = 9;
constexpr long long HG_FLAT_M = 1ll << 22; // fewer sorted points: every merge level materialised
inline int chunk_log2(long long m)
{
    int lgc = HG_LGC_MIN;
    while (lgc < HG_LGC_MAX && (m >> (lgc + 16)) > 0) // ~2^16 chunks or more before it doubles
        lgc++;
    return lgc;
}
// With the count on the device (the asynchronous second round), chunks are
// sized for m >> HG_DEV_SHIFT so a heavily reduced set still gives enough
// threads.
#ifndef HG_DEV_SHIFT
#define HG_DEV_SHIFT 2 // (A/B: 0 / 1 / 2 / 3 / 4 / 6 -> 1e8 displaced 2.33 / 1.92 / 1.80 / 1.86 / 2.06 / 2.31 ms)
#endif
inline int chunk_log2_dev(long long m) { return chunk_log2(m >> HG_DEV_SHIFT > 0 ? m >> HG_DEV_SHIFT : 1); }
constexpr int HG_THREADS = 128;

__device__ __forceinline__ unsigned long long okey(double d)
{
    d = __dadd_rn(d, 0.0); // -0.0 -> +0.0 (numeric equality, R2)
    const unsigned long long u = (unsigned long long)__double_as_longlong(d);
    return (u & 0x8000000000000000ull) ? ~u : (u | 0x8000000000000000ull);
}

__device__ __forceinline__ double okey_inv(unsigned long long k)
{
    return __longlong_as_double((long long)((k & 0x8000000000000000ull) ? (k & 0x7fffffffffffffffull) : ~k));
}

__device__ __forceinline__ unsigned long long shfl_xor64(unsigned long long v, int o)
{
    return __shfl_xor_sync(0xffffffffu, v, o);
}

// Sort values (survivor ids, or positions when surv == NULL) and their x to X,
// plus min / max of x as order-preserving keys (mm[0] min, mm[1] max; the
// caller sets them to ~0 and 0).
template <typename V>
__global__ void k_gather_x(const double *__restrict__ xy, const long long *__restrict__ surv, long long m,
                           double *__restrict__ X, V *__restrict__ val, unsigned long long *__restrict__ mm,
                           const long long *__restrict__ dm, const long long *__restrict__ kept,
                           const unsigned long long *__restrict__ use_kept)
{
    // (dm: the count is on the device; use_kept: the ids come from `kept`)
    if (dm)
        m = *dm;
    if (use_kept && *use_kept)
        surv = kept;
    unsigned long long lo = ~0ull, hi = 0;
    for (long long j = (long long)blockIdx.x * blockDim.x + threadIdx.x; j < m; j += (long long)gridDim.x * blockDim.x) {
        const long long id = surv ? surv[j] : j; // NULL: every point of xy, in order
        const double x = xy[2 * id];
        X[j] = x;
        val[j] = (V)id;
        const unsigned long long o = okey(x);
        lo = o < lo ? o : lo;
        hi = o > hi ? o : hi;
    }
    for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long a = shfl_xor64(lo, o), b = shfl_xor64(hi, o);
        lo = a < lo ? a : lo;
        hi = b > hi ? b : hi;
    }
    // one atomic pair per block (per warp, ~m/16 atomics on two words serialise)
    __shared__ unsigned long long s_lo[32], s_hi[32];
    const int w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    if ((threadIdx.x & 31) == 0) {
        s_lo[w] = lo;
        s_hi[w] = hi;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int i = 1; i < nw; i++) {
            lo = s_lo[i] < lo ? s_lo[i] : lo;
            hi = s_hi[i] > hi ? s_hi[i] : hi;
        }
        atomicMin(&mm[0], lo);
        atomicMax(&mm[1], hi);
    }
}

// The 32-bit sort key: x quantised linearly over [lo, hi] of the survivors,
// floor((x/2 - lo/2) * (2^32 - 256) / (hi/2 - lo/2)), every operation rounded
// to nearest (monotone), so x1 < x2 implies key1 <= key2 and key1 < key2
// implies x1 < x2: sorting by the key puts the points in x order up to runs
// of equal keys, which k_fix_runs / k_fix_big then sort by x exactly.  The
// halves keep hi/2 - lo/2 finite; equal x (also -0.0 / +0.0) gives equal keys.
struct Quant {
    double h_lo, s;
};
__device__ __forceinline__ Quant quant_params(const unsigned long long *mm)
{
    const double lo = okey_inv(mm[0]), hi = okey_inv(mm[1]);
    const double h_lo = __dmul_rn(lo, 0.5);
    const double d = __dsub_rn(__dmul_rn(hi, 0.5), h_lo);
    const double s = d > 0.0 ? fmin(__ddiv_rn(4294967040.0, d), 1.7976931348623157e308) : 0.0;
    return {h_lo, s};
}
__device__ __forceinline__ unsigned quant(double x, const Quant &q)
{
    const double t = __dmul_rn(__dsub_rn(__dmul_rn(x, 0.5), q.h_lo), q.s);
    return (unsigned)fmin(floor(t), 4294967295.0);
}

// Keys from X, and the 256-bin histogram of each of the four 8-bit digits
// (hist[4][256], zeroed by the caller).  HG_KH_ITEMS loads in flight per
// thread; plain shared-memory atomics (lanes of a warp collide only on equal
// digits).
constexpr int HG_KH_ITEMS = 8;
__global__ void __launch_bounds__(256) k_keys_hist(const double *__restrict__ X, long long m,
                                                   const unsigned long long *__restrict__ mm, unsigned *__restrict__ key,
                                                   unsigned long long *__restrict__ hist, const long long *__restrict__ dm)
{
    if (dm)
        m = *dm;
    __shared__ unsigned h[4][chrs::RS_BINS];
    for (int b = threadIdx.x; b < 4 * chrs::RS_BINS; b += blockDim.x)
        (&h[0][0])[b] = 0;
    __syncthreads();
    const Quant q = quant_params(mm);
    const long long stride = (long long)gridDim.x * blockDim.x * HG_KH_ITEMS;
    for (long long j0 = (long long)blockIdx.x * blockDim.x * HG_KH_ITEMS + threadIdx.x; j0 < m; j0 += stride) {
        double x[HG_KH_ITEMS];
#pragma unroll
        for (int u = 0; u < HG_KH_ITEMS; u++) {
            const long long j = j0 + (long long)u * blockDim.x;
            x[u] = j < m ? X[j] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < HG_KH_ITEMS; u++) {
            const long long j = j0 + (long long)u * blockDim.x;
            if (j < m) {
                const unsigned k = quant(x[u], q);
                key[j] = k;
#pragma unroll
                for (int p = 0; p < 4; p++)
                    atomicAdd(&h[p][(k >> (8 * p)) & 255u], 1u);
            }
        }
    }
    __syncthreads();
    for (int b = threadIdx.x; b < 4 * chrs::RS_BINS; b += blockDim.x) {
        const unsigned c = (&h[0][0])[b];
        if (c)
            atomicAdd(&hist[b], (unsigned long long)c);
    }
}

template <typename V>
__global__ void k_points(const double *__restrict__ xy, const V *__restrict__ val, long long m,
                         double2 *__restrict__ P, const long long *__restrict__ dm)
{
    if (dm)
        m = *dm;
    const double2 *__restrict__ xy2 = reinterpret_cast<const double2 *>(xy);
    for (long long j = (long long)blockIdx.x * blockDim.x + threadIdx.x; j < m; j += (long long)gridDim.x * blockDim.x)
        P[j] = xy2[(long long)val[j]];
}

// Runs of equal x (numeric ==) inside [a, e), which is sorted by x: each run
// of >= 2 becomes [low, ..., low, high] -- low = min y (ties: lowest sort
// value), high = max y (ties: lowest sort value).  Only those two can be
// strict hull vertices (every other point of the run lies on the segment
// between them or equals one of them); the result is sorted by (x, y) and the
// chains skip the copies (a point equal to its sorted predecessor).
template <typename V> __device__ __forceinline__ void ties_local(double2 *p, V *v, int L)
{
    for (int i = 0; i < L;) {
        int e = i + 1;
        double2 lo = p[i], hi = lo;
        V vlo = v[i], vhi = vlo;
        for (; e < L && p[e].x == p[i].x; e++) {
            const double2 q = p[e];
            const V vq = v[e];
            if (q.y < lo.y || (q.y == lo.y && vq < vlo)) {
                lo = q;
                vlo = vq;
            }
            if (q.y > hi.y || (q.y == hi.y && vq < vhi)) {
                hi = q;
                vhi = vq;
            }
        }
        if (e - i >= 2) {
            for (int k = i; k < e - 1; k++) {
                p[k] = lo;
                v[k] = vlo;
            }
            p[e - 1] = hi;
            v[e - 1] = vhi;
        }
        i = e;
    }
}
template <typename V> __device__ void ties_global(double2 *P, V *val, long long i, long long e)
{
    double2 lo = P[i], hi = lo;
    V vlo = val[i], vhi = vlo;
    for (long long k = i + 1; k < e; k++) {
        const double2 q = P[k];
        const V vq = val[k];
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

// The end of a run in sorted data: the first e in [lo, hi) with !same(e)
// (hi if none), given same(lo - 1) and a monotone same (true, then false):
// galloping then binary search, O(log run length) probes instead of a
// serial scan (a single run can hold every point).
template <typename F> __device__ __forceinline__ long long run_end(long long lo, long long hi, F same)
{
    long long step = 1, ok = lo - 1; // same(ok) holds
    while (true) {
        const long long p = ok + step;
        if (p >= hi || !same(p)) {
            hi = p < hi ? p : hi;
            break;
        }
        ok = p;
        step *= 2;
    }
    while (hi - ok > 1) { // same(ok), !same(hi) (or hi the bound)
        const long long mid = ok + (hi - ok) / 2;
        if (same(mid))
            ok = mid;
        else
            hi = mid;
    }
    return hi;
}

// Runs of equal 32-bit key in the key-sorted points.  A run of at most
// HG_SMALL_RUN is sorted by x (insertion sort) and its equal-x runs resolved
// (ties_local) by the thread at its head; a longer one is queued for
// k_fix_big (runs[2 r] = start, runs[2 r + 1] = length).
constexpr int HG_SMALL_RUN = 32;
constexpr int HG_FIX_W = 4; // k_fix_runs: 32-key windows per warp iteration
constexpr long long HG_TIE_SERIAL = 256; // k_fix_big: longer equal-x runs are reduced block-wide
// The run of equal keys headed at i (i is a head of a run of >= 2): sorted
// by x and its equal-x runs resolved here when short (ties_local), else
// queued for k_fix_big as (start, length).
template <typename V>
__device__ __forceinline__ void fix_run(long long i, const unsigned *__restrict__ key, double2 *__restrict__ P,
                                        V *__restrict__ val, long long m, long long *__restrict__ runs,
                                        unsigned long long *__restrict__ nruns)
{
    const unsigned k = key[i];
    long long e = i + 2;
    while (e < m && e - i <= HG_SMALL_RUN && key[e] == k)
        e++;
    if (e - i > HG_SMALL_RUN) {
        e = run_end(e, m, [&](long long q) { return key[q] == k; });
        const unsigned long long r = atomicAdd(nruns, 1ull);
        runs[2 * r] = i;
        runs[2 * r + 1] = e - i;
        return;
    }
    const int L = (int)(e - i);
    if (L == 2) { // the common case, in registers
        double2 p0 = P[i], p1 = P[i + 1];
        V v0 = val[i], v1 = val[i + 1];
        if (p1.x < p0.x || (p1.x == p0.x && (p1.y < p0.y || (p1.y == p0.y && v1 < v0)))) {
            const double2 tp = p0;
            p0 = p1;
            p1 = tp;
            const V tv = v0;
            v0 = v1;
            v1 = tv;
        }
        // equal x: [low, high] is the (x, y, value) order, except for
        // equal points, where high takes the lowest value too
        if (p1.x == p0.x && p1.y == p0.y)
            v1 = v0;
        P[i] = p0;
        P[i + 1] = p1;
        val[i] = v0;
        val[i + 1] = v1;
        return;
    }
    double2 p[HG_SMALL_RUN];
    V v[HG_SMALL_RUN];
    for (int t = 0; t < L; t++) { // insertion sort by x (equal x in any order)
        const double2 q = P[i + t];
        const V vq = val[i + t];
        int u = t;
        for (; u > 0 && p[u - 1].x > q.x; u--) {
            p[u] = p[u - 1];
            v[u] = v[u - 1];
        }
        p[u] = q;
        v[u] = vq;
    }
    ties_local(p, v, L);
    for (int t = 0; t < L; t++) {
        P[i + t] = p[t];
        val[i + t] = v[t];
    }
}

template <typename V>
__global__ void k_fix_runs(const unsigned *__restrict__ key, double2 *__restrict__ P, V *__restrict__ val, long long m,
                           long long *__restrict__ runs, unsigned long long *__restrict__ nruns,
                           const long long *__restrict__ dm)
{
    if (dm)
        m = *dm;
    // warps walk 32-key windows, HG_FIX_W windows' loads in flight; the
    // neighbours come by shuffles (the window's edge lanes load theirs)
    const int lane = threadIdx.x & 31;
    const long long nwarps = ((long long)gridDim.x * blockDim.x) >> 5;
    const long long w0 = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    for (long long wb = w0 * 32; wb < m; wb += nwarps * 32 * HG_FIX_W) {
        unsigned kc[HG_FIX_W], kp[HG_FIX_W], kn[HG_FIX_W];
#pragma unroll
        for (int u = 0; u < HG_FIX_W; u++) {
            const long long i = wb + (long long)u * nwarps * 32 + lane;
            kc[u] = i < m ? key[i] : 0u;
            kp[u] = (lane == 0 && i > 0 && i - 1 < m) ? key[i - 1] : 0u;
            kn[u] = (lane == 31 && i + 1 < m) ? key[i + 1] : 0u;
        }
        unsigned heads = 0;
#pragma unroll
        for (int u = 0; u < HG_FIX_W; u++) {
            const long long i = wb + (long long)u * nwarps * 32 + lane;
            const unsigned up = __shfl_up_sync(0xffffffffu, kc[u], 1), dn = __shfl_down_sync(0xffffffffu, kc[u], 1);
            const unsigned prv = lane == 0 ? kp[u] : up, nxt = lane == 31 ? kn[u] : dn;
            // the head of a run of >= 2 equal keys
            const bool h = i < m && !(i > 0 && prv == kc[u]) && i + 1 < m && nxt == kc[u];
            heads |= (h ? 1u : 0u) << u;
        }
        for (int wu = 0; wu < HG_FIX_W; wu++)
            if ((heads >> wu) & 1u)
                fix_run(wb + (long long)wu * nwarps * 32 + lane, key, P, val, m, runs, nruns);
    }
}

// One run of equal x, [a, a + L), reduced block-wide to [low, ..., low,
// high] (ties_local's rule); the candidates go through the tile's shared
// arrays.  Every thread of the CTA; ends with a barrier.
template <typename V>
__device__ void ties_block(double2 *__restrict__ P, V *__restrict__ val, long long a, long long L,
                           chrs::TileSmem<unsigned long long, unsigned> &s)
{
    double2 plo = P[a], phi = plo;
    V vlo = val[a], vhi = vlo;
    for (long long t = threadIdx.x; t < L; t += blockDim.x) {
        const double2 q = P[a + t];
        const V vq = val[a + t];
        if (q.y < plo.y || (q.y == plo.y && vq < vlo)) {
            plo = q;
            vlo = vq;
        }
        if (q.y > phi.y || (q.y == phi.y && vq < vhi)) {
            phi = q;
            vhi = vq;
        }
    }
    double2 (*s_p)[chrs::RS_THREADS] = reinterpret_cast<double2 (*)[chrs::RS_THREADS]>(s.key);
    V (*s_v)[chrs::RS_THREADS] = reinterpret_cast<V (*)[chrs::RS_THREADS]>(s.val);
    __syncthreads(); // (s.key / s.val may hold the caller's data until here)
    s_p[0][threadIdx.x] = plo;
    s_v[0][threadIdx.x] = vlo;
    s_p[1][threadIdx.x] = phi;
    s_v[1][threadIdx.x] = vhi;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int u = 1; u < chrs::RS_THREADS; u++) {
            const double2 q = s_p[0][u];
            const V vq = s_v[0][u];
            if (q.y < plo.y || (q.y == plo.y && vq < vlo)) {
                plo = q;
                vlo = vq;
            }
            const double2 q2 = s_p[1][u];
            const V vq2 = s_v[1][u];
            if (q2.y > phi.y || (q2.y == phi.y && vq2 < vhi)) {
                phi = q2;
                vhi = vq2;
            }
        }
        s_p[0][0] = plo;
        s_v[0][0] = vlo;
        s_p[1][0] = phi;
        s_v[1][0] = vhi;
    }
    __syncthreads();
    plo = s_p[0][0];
    vlo = s_v[0][0];
    phi = s_p[1][0];
    vhi = s_v[1][0];
    for (long long t = threadIdx.x; t < L - 1; t += blockDim.x) {
        P[a + t] = plo;
        val[a + t] = vlo;
    }
    if (threadIdx.x == 0) {
        P[a + L - 1] = phi;
        val[a + L - 1] = vhi;
    }
    __syncthreads();
}

// The long runs, one CTA per run (grid-stride over the queue): 64-bit
// order-preserving keys of x, a single-CTA LSD sort over the digits where the
// run's keys differ (chrs::cta_sort_pass), the points and values permuted by
// the sorted positions (through ka/kb, free by now), then the equal-x runs.
// A run whose x are all equal is one equal-x run (a block-wide lowest/highest
// point).  Scratch at the run's own positions [a, a + L): ka, kb (8-byte
// words), ia, ib (32-bit positions; a run is shorter than 2^32).
template <typename V>
__global__ void __launch_bounds__(chrs::RS_THREADS) k_fix_big(double2 *__restrict__ P, V *__restrict__ val,
                                                            const long long *__restrict__ runs,
                                                            const unsigned long long *__restrict__ nruns,
                                                            unsigned long long *ka, unsigned long long *kb,
                                                            unsigned *ia, unsigned *ib)
{
    using S = chrs::TileSmem<unsigned long long, unsigned>;
    extern __shared__ __align__(16) unsigned char fb_smem[];
    S &s = *reinterpret_cast<S *>(fb_smem);
    const long long nr = (long long)*nruns;
    for (long long r = blockIdx.x; r < nr; r += gridDim.x) {
        const long long a = runs[2 * r], L = runs[2 * r + 1];
        unsigned long long lo = ~0ull, hi = 0;
        for (long long t = threadIdx.x; t < L; t += blockDim.x) { // (read-only: an all-equal run needs no keys)
            const unsigned long long o = okey(P[a + t].x);
            lo = o < lo ? o : lo;
            hi = o > hi ? o : hi;
        }
        for (int o = 16; o > 0; o >>= 1) {
            const unsigned long long x0 = shfl_xor64(lo, o), x1 = shfl_xor64(hi, o);
            lo = x0 < lo ? x0 : lo;
            hi = x1 > hi ? x1 : hi;
        }
        if (threadIdx.x == 0) {
            s.lo = ~0ull;
            s.hi = 0;
        }
        __syncthreads();
        if ((threadIdx.x & 31) == 0) {
            atomicMin(&s.lo, lo);
            atomicMax(&s.hi, hi);
        }
        __syncthreads();
        lo = s.lo;
        hi = s.hi;
        __syncthreads();
        if (lo == hi) { // one equal-x run: lowest and highest point, block-wide
            ties_block(P, val, a, L, s);
            continue;
        }
        for (long long t = threadIdx.x; t < L; t += blockDim.x) {
            ka[a + t] = okey(P[a + t].x);
            ia[a + t] = (unsigned)t;
        }
        __syncthreads();
        // LSD passes over the bytes below the highest differing bit
        const int top = 63 - __clzll((long long)(lo ^ hi));
        unsigned long long *kin = ka, *kout = kb;
        unsigned *iin = ia, *iout = ib;
        for (int shift = 0; shift <= top; shift += 8) {
            if (chrs::cta_sort_pass<unsigned long long, unsigned>(s, kin, kout, iin, iout, a, L, shift)) {
                unsigned long long *tk = kin;
                kin = kout;
                kout = tk;
                unsigned *ti = iin;
                iin = iout;
                iout = ti;
            }
            __syncthreads();
        }
        // permute: positions iin[a + t] (run-relative) in x order, staged in
        // the run's own 8-byte words of ka / kb (free now)
        double *tx = reinterpret_cast<double *>(ka + a), *ty = reinterpret_cast<double *>(kb + a);
        const unsigned *srt = iin + a;
        for (long long t = threadIdx.x; t < L; t += blockDim.x) {
            const double2 q = P[a + srt[t]];
            tx[t] = q.x;
            ty[t] = q.y;
        }
        __syncthreads();
        for (long long t = threadIdx.x; t < L; t += blockDim.x)
            P[a + t] = make_double2(tx[t], ty[t]);
        __syncthreads();
        V *tv = reinterpret_cast<V *>(ka + a); // sizeof(V) <= 8
        for (long long t = threadIdx.x; t < L; t += blockDim.x)
            tv[t] = val[a + srt[t]];
        __syncthreads();
        for (long long t = threadIdx.x; t < L; t += blockDim.x)
            val[a + t] = tv[t];
        __syncthreads();
        // equal-x runs inside the sorted run: one thread per run head (its
        // end by galloping search); runs longer than HG_TIE_SERIAL are
        // listed and reduced block-wide
        if (threadIdx.x == 0)
            s.tile = 0; // (the count of listed long runs)
        __syncthreads();
        long long *longs = reinterpret_cast<long long *>(s.gofs); // up to RS_BINS / 2 (start, end) pairs
        for (long long t = threadIdx.x; t < L; t += blockDim.x) {
            const double x = P[a + t].x;
            if ((t > 0 && P[a + t - 1].x == x) || t + 1 >= L || P[a + t + 1].x != x)
                continue;
            const long long e = run_end(t + 2, L, [&](long long q) { return P[a + q].x == x; });
            if (e - t > HG_TIE_SERIAL) {
                const unsigned long long slot = atomicAdd(&s.tile, 1ull);
                if (slot < chrs::RS_BINS / 2) {
                    longs[2 * slot] = a + t;
                    longs[2 * slot + 1] = a + e;
                    continue;
                }
            }
            ties_global(P, val, a + t, a + e); // short, or the list is full
        }
        __syncthreads();
        const long long nlong = (long long)min(s.tile, (unsigned long long)(chrs::RS_BINS / 2));
        for (long long r2 = 0; r2 < nlong; r2++) {
            const long long b0 = longs[2 * r2], b1 = longs[2 * r2 + 1];
            ties_block(P, val, b0, b1 - b0, s);
        }
        __syncthreads();
    }
}

// ------------------------------------------------ second filtering round --
// Before the sort (ch_hull_gpu only: it synchronizes anyway), the survivors
// are filtered once more, Akl-Toussaint style with HG_DIRS directions instead
// of the octagon's 8: the approximate extremes of a strided sample in HG_DIRS
// directions (fp32 dot products; any input points will do) form a polygon
// V[0..nv) of input points, and a survivor p is discarded only if it lies
// STRICTLY inside a fan triangle (V[0], V[j], V[j+1]), decided by the exact
// orientation sign (chf::orient_sign) on all three edges.  Strictly inside a
// triangle of input points is strictly inside their hull, so p is neither a
// hull vertex nor on the hull boundary: the hull of the rest is the hull of
// the survivors, whatever the polygon looks like (the fp64 binary search for j
// only picks the triangle to test).  On ring-like survivors (C4) this removes
// most of them; on a circle (every survivor a hull vertex) nothing, and the
// original list is used.
constexpr int HG_DIRS = 64;
constexpr long long HG_REFINE_MIN = 1ll << 16; // fewer survivors: no second round
constexpr long long HG_SAMPLE = 1ll << 18;     // sample the direction extremes are taken over
struct Dirs {
    float u[HG_DIRS][2];
};
struct RefinePoly { // device scratch
    double2 v[HG_DIRS];
    int nv;
};

// best[k] = max over the sample of (orderable fp32 u_k . p) << 32 | sample
// index (zeroed by the caller).  Thread t of a 64-thread group owns direction
// t % 64; the group's threads read the same point (one broadcast load).
__global__ void __launch_bounds__(256) k_dir_extremes(const double *__restrict__ xy, const long long *__restrict__ surv,
                                                      long long stride, long long nsample, const Dirs D,
                                                      unsigned long long *__restrict__ best)
{
    const int k = threadIdx.x % HG_DIRS;
    const long long g = ((long long)blockIdx.x * blockDim.x + threadIdx.x) / HG_DIRS;
    const long long ng = (long long)gridDim.x * blockDim.x / HG_DIRS;
    const float ux = D.u[k][0], uy = D.u[k][1];
    unsigned long long b = 0;
    for (long long s0 = g; s0 < nsample; s0 += 4 * ng) { // four points' loads in flight
        long long id[4];
#pragma unroll
        for (int u = 0; u < 4; u++) {
            const long long s = s0 + u * ng;
            id[u] = s < nsample ? (surv ? surv[s * stride] : s * stride) : -1;
        }
        double2 q[4];
#pragma unroll
        for (int u = 0; u < 4; u++)
            q[u] = id[u] >= 0 ? reinterpret_cast<const double2 *>(xy)[id[u]] : make_double2(0, 0);
#pragma unroll
        for (int u = 0; u < 4; u++) {
            if (id[u] < 0)
                continue;
            const float d = __fmaf_rn(ux, (float)q[u].x, __fmul_rn(uy, (float)q[u].y));
            const unsigned bits = __float_as_uint(d);
            const unsigned ok = (bits & 0x80000000u) ? ~bits : (bits | 0x80000000u);
            const unsigned long long key = ((unsigned long long)ok << 32) | (unsigned long long)(s0 + u * ng);
            b = key > b ? key : b;
        }
    }
    atomicMax(&best[k], b);
}

// The polygon: the extremes in direction order (counterclockwise), equal
// consecutive points dropped (also across the wrap); nv < 3 -> no polygon.
__global__ void k_refine_poly(const double *__restrict__ xy, const long long *__restrict__ surv, long long stride,
                              const unsigned long long *__restrict__ best, RefinePoly *poly)
{
    __shared__ double2 e[HG_DIRS];
    for (int k = threadIdx.x; k < HG_DIRS; k += blockDim.x) { // the extreme points, loaded in parallel
        const long long pos = (long long)(best[k] & 0xffffffffull) * stride;
        const long long id = surv ? surv[pos] : pos;
        e[k] = reinterpret_cast<const double2 *>(xy)[id];
    }
    __syncthreads();
    if (threadIdx.x != 0)
        return;
    int nv = 0;
    for (int k = 0; k < HG_DIRS; k++) {
        const double2 q = e[k];
        if (nv > 0 && q.x == poly->v[nv - 1].x && q.y == poly->v[nv - 1].y)
            continue;
        poly->v[nv++] = q;
    }
    while (nv > 1 && poly->v[nv - 1].x == poly->v[0].x && poly->v[nv - 1].y == poly->v[0].y)
        nv--;
    poly->nv = nv >= 3 ? nv : 0;
}

// Strictly inside p's fan triangle of the polygon V[0..nv) (nv >= 3)?  The
// triangle is picked by a binary search on the fp64 (inexact) side of
// V0 -> V[mid]; the decision is the exact orientation on its three edges.
__device__ __forceinline__ bool refine_inside(const double2 *V, int nv, double2 p)
{
    int lo = 1, hi = nv - 1;
    const double2 a = V[0];
    while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        const double2 b = V[mid];
        const double o = __dsub_rn(__dmul_rn(__dsub_rn(b.x, a.x), __dsub_rn(p.y, a.y)),
                                   __dmul_rn(__dsub_rn(b.y, a.y), __dsub_rn(p.x, a.x)));
        if (o >= 0.0)
            lo = mid;
        else
            hi = mid;
    }
    const double2 b = V[lo], c = V[lo + 1];
    return chf::orient_sign(a.x, a.y, b.x, b.y, p.x, p.y) > 0 && chf::orient_sign(b.x, b.y, c.x, c.y, p.x, p.y) > 0 &&
           chf::orient_sign(c.x, c.y, a.x, a.y, p.x, p.y) > 0;
}

// The round's expected yield: how many of the sample points it would drop.
__global__ void __launch_bounds__(256) k_refine_probe(const double *__restrict__ xy,
                                                      const long long *__restrict__ surv, long long stride,
                                                      long long nsample, const RefinePoly *__restrict__ poly,
                                                      unsigned long long *__restrict__ ndrop)
{
    __shared__ double2 V[HG_DIRS];
    if (threadIdx.x < HG_DIRS)
        V[threadIdx.x] = poly->v[threadIdx.x];
    __syncthreads();
    const int nv = poly->nv;
    unsigned c = 0;
    if (nv >= 3)
        for (long long s = (long long)blockIdx.x * blockDim.x + threadIdx.x; s < nsample;
             s += (long long)gridDim.x * blockDim.x) {
            const long long pos = s * stride;
            const long long id = surv ? surv[pos] : pos;
            c += refine_inside(V, nv, reinterpret_cast<const double2 *>(xy)[id]) ? 1u : 0u;
        }
    for (int o = 16; o > 0; o >>= 1)
        c += __shfl_xor_sync(0xffffffffu, c, o);
    if ((threadIdx.x & 31) == 0 && c)
        atomicAdd(ndrop, (unsigned long long)c);
}

// Keeps every survivor not strictly inside its fan triangle: kept[] gets
// their ids, tile by tile (HG_RF_ITEMS x 256 survivors, one atomic per tile
// for the tile's place; the order across tiles is arbitrary -- the hull
// pipeline does not depend on it), *nkept the count.
constexpr int HG_RF_ITEMS = 16;
__global__ void __launch_bounds__(256) k_refine_filter(const double *__restrict__ xy, const long long *__restrict__ surv,
                                                       long long m, const RefinePoly *__restrict__ poly,
                                                       long long *__restrict__ kept,
                                                       unsigned long long *__restrict__ nkept,
                                                       const unsigned long long *__restrict__ ndrop, long long nsample)
{
    // (ndrop: the asynchronous round -- the probe's yield decides on the device)
    if (ndrop && 4 * *ndrop < (unsigned long long)nsample)
        return;
    __shared__ double2 V[HG_DIRS];
    __shared__ int s_wcnt[HG_RF_ITEMS][8];
    __shared__ unsigned long long s_base;
    if (threadIdx.x < HG_DIRS)
        V[threadIdx.x] = poly->v[threadIdx.x];
    __syncthreads();
    const int nv = poly->nv;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const unsigned lt = chrs::lanemask_lt();
    constexpr long long TILE = 256LL * HG_RF_ITEMS;
    for (long long t0 = (long long)blockIdx.x * TILE; t0 < m; t0 += (long long)gridDim.x * TILE) {
        unsigned bal[HG_RF_ITEMS];
        long long ids[HG_RF_ITEMS];
#pragma unroll
        for (int i = 0; i < HG_RF_ITEMS; i++) {
            const long long j = t0 + 256LL * i + threadIdx.x;
            bool keep = false;
            ids[i] = 0;
            if (j < m) {
                ids[i] = surv ? surv[j] : j;
                keep = nv < 3 || !refine_inside(V, nv, reinterpret_cast<const double2 *>(xy)[ids[i]]);
            }
            bal[i] = __ballot_sync(0xffffffffu, keep);
            if (lane == 0)
                s_wcnt[i][w] = __popc(bal[i]);
        }
        __syncthreads();
        if (threadIdx.x == 0) { // the tile's exclusive prefix over (item, warp), in place, and its place
            int run = 0;
            for (int i = 0; i < HG_RF_ITEMS; i++)
                for (int ww = 0; ww < 8; ww++) {
                    const int c = s_wcnt[i][ww];
                    s_wcnt[i][ww] = run;
                    run += c;
                }
            s_base = run ? atomicAdd(nkept, (unsigned long long)run) : 0ull;
        }
        __syncthreads();
        const unsigned long long base = s_base;
#pragma unroll
        for (int i = 0; i < HG_RF_ITEMS; i++)
            if ((bal[i] >> lane) & 1u)
                kept[base + s_wcnt[i][w] + __popc(bal[i] & lt)] = ids[i];
        __syncthreads(); // s_wcnt / s_base are rewritten by the next tile
    }
}

// The asynchronous round's outcome on the device: use the kept list when the
// probe found the round worth it and it kept fewer than m (and some) points;
// *dm = the count the pipeline then sorts.
__global__ void k_refine_finish(long long m, long long nsample, const unsigned long long *__restrict__ ndrop,
                                const unsigned long long *__restrict__ nkept, unsigned long long *__restrict__ use,
                                long long *__restrict__ dm)
{
    const unsigned long long nk = *nkept;
    const bool u = 4 * *ndrop >= (unsigned long long)nsample && nk > 0 && (long long)nk < m;
    *use = u ? 1ull : 0ull;
    *dm = u ? (long long)nk : m;
}

// ------------------------------------------------------------ small m --
// At most HG_SMALL_M points: the whole hull in one CTA (one launch instead
// of the pipeline's ~40, whose launch latency is the cost there).  The
// points, padded to a power of two with +inf, are sorted by (x, y, id) with
// a bitonic network in shared memory; the first point of each run of equal
// (x, y) -- the lowest id -- stands for the run; one thread runs Andrew's
// lower chain and another the upper chain, popping while the exact turn
// (chf::orient_sign) is <= 0.  The same canonical hull as the pipeline
// (DESIGN R8).  surv (nullable: position i) selects the points; idmap
// (nullable) gives position i's output id.
constexpr int HG_SMALL_M = 1024;
__global__ void __launch_bounds__(512) k_small_hull(const double *__restrict__ xy, const long long *__restrict__ surv,
                                                    const long long *__restrict__ idmap, long long m,
                                                    long long *__restrict__ out, long long *__restrict__ d_nh)
{
    __shared__ double sx[HG_SMALL_M], sy[HG_SMALL_M];
    __shared__ long long sid[HG_SMALL_M];
    __shared__ int lst[HG_SMALL_M], ust[HG_SMALL_M];
    __shared__ int s_nl, s_nu;
    const int n = (int)m;
    int n2 = 1;
    while (n2 < n)
        n2 <<= 1;
    for (int i = threadIdx.x; i < n2; i += blockDim.x) {
        if (i < n) {
            const long long id = surv ? surv[i] : i;
            const double2 q = reinterpret_cast<const double2 *>(xy)[id];
            sx[i] = q.x;
            sy[i] = q.y;
            sid[i] = idmap ? idmap[i] : id;
        } else {
            sx[i] = sy[i] = CH_INF;
            sid[i] = 0x7fffffffffffffffll;
        }
    }
    __syncthreads();
    auto less = [&](int a, int b) {
        return sx[a] < sx[b] || (sx[a] == sx[b] && (sy[a] < sy[b] || (sy[a] == sy[b] && sid[a] < sid[b])));
    };
    for (int k = 2; k <= n2; k <<= 1)
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int i = threadIdx.x; i < n2; i += blockDim.x) {
                const int l = i ^ j;
                if (l > i) {
                    const bool up = (i & k) == 0;
                    if (up ? less(l, i) : less(i, l)) {
                        const double tx = sx[i], ty = sy[i];
                        const long long td = sid[i];
                        sx[i] = sx[l];
                        sy[i] = sy[l];
                        sid[i] = sid[l];
                        sx[l] = tx;
                        sy[l] = ty;
                        sid[l] = td;
                    }
                }
            }
            __syncthreads();
        }
    // the first point of each run of equal (x, y) stands for the run
    auto first = [&](int i) { return i == 0 || !(sx[i] == sx[i - 1] && sy[i] == sy[i - 1]); };
    auto turn_le0 = [&](int a, int b, int c) {
        return chf::orient_sign(sx[a], sy[a], sx[b], sy[b], sx[c], sy[c]) <= 0;
    };
    if (threadIdx.x == 0) { // lower chain, left to right
        int k = 0;
        for (int i = 0; i < n; i++) {
            if (!first(i))
                continue;
            while (k >= 2 && turn_le0(lst[k - 2], lst[k - 1], i))
                k--;
            lst[k++] = i;
        }
        s_nl = k;
    } else if (threadIdx.x == 32) { // upper chain, right to left (another warp)
        int k = 0;
        for (int i = n - 1; i >= 0; i--) {
            if (!first(i))
                continue;
            while (k >= 2 && turn_le0(ust[k - 2], ust[k - 1], i))
                k--;
            ust[k++] = i;
        }
        s_nu = k;
    }
    __syncthreads();
    const int nl = s_nl, nu = s_nu;
    if (nl <= 1) { // one distinct point
        if (threadIdx.x == 0) {
            out[0] = sid[lst[0]];
            *d_nh = 1;
        }
        return;
    }
    const int a = nl - 1, total = a + nu - 1;
    for (int g = threadIdx.x; g < total; g += blockDim.x)
        out[g] = g < a ? sid[lst[g]] : sid[ust[g - a]];
    if (threadIdx.x == 0)
        *d_nh = total;
}

struct Seq {
    const double2 *P;
    long long m;
    int rev; // 0: lower chain (increasing order), 1: upper chain (reversed)
    int lgc; // log2 of the chunk size
    const long long *dm; // nullable: m is on the device (the kernels read it first)
    __device__ __forceinline__ long long fwd(long long r) const { return rev ? m - 1 - r : r; }
    __device__ __forceinline__ double2 at(long long r) const { return P[fwd(r)]; }
};

__device__ __forceinline__ int turn(const double2 &a, const double2 &b, const double2 &c)
{
    return chf::orient_sign(a.x, a.y, b.x, b.y, c.x, c.y);
}

// Andrew's monotone chain over one chunk; the stack lives in pos[start..].
// Points are loaded HG_PF steps ahead of their turn
// (a shift register): q[0] is the current point in traversal order, q[1] the
// next -- in the upper chain's (reversed) order also the sorted predecessor
// P[f - 1] the duplicate test needs, so the reversed walk loads one point
// past its chunk; in the lower chain's order the predecessor is the previous
// point, kept in a register.
#ifndef HG_PF
#define HG_PF 4
#endif

template <typename I>
__global__ void k_chunk_chain(Seq s, long long nchunks, I *__restrict__ pos, long long *__restrict__ len)
{
    if (s.dm)
        s.m = *s.dm;
    const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= nchunks)
        return;
    const long long start = t << s.lgc, end = min(start + (1ll << s.lgc), s.m);
    // the last traversal index loaded: the chunk's, or one past it (reversed walk)
    const long long lend = s.rev ? min(end, s.m - 1) : end - 1;
    auto ld = [&](long long rr) { return rr <= lend ? s.at(rr) : make_double2(0, 0); };
    long long top = 0;
    double2 p1 = make_double2(0, 0), p2 = make_double2(0, 0); // stack[top-1], stack[top-2]
    double2 p3 = make_double2(0, 0);                          // stack[top-3] when have3
    bool have3 = false;
    double2 q[HG_PF + 1];
#pragma unroll
    for (int k = 0; k <= HG_PF; k++)
        q[k] = ld(start + k);
    const long long f0 = s.fwd(start);
    double2 pred = (!s.rev && f0 > 0) ? s.P[f0 - 1] : make_double2(0, 0);
    for (long long r = start; r < end; r++) {
        const double2 cur = q[0];
#pragma unroll
        for (int k = 0; k < HG_PF; k++)
            q[k] = q[k + 1];
        q[HG_PF] = ld(r + HG_PF + 1);
        const long long f = s.fwd(r);
        const double2 pd = s.rev ? q[0] : pred;
        const bool dup = f > 0 && cur.x == pd.x && cur.y == pd.y;
        if (!dup) {
            while (top >= 2 && turn(p2, p1, cur) <= 0) {
                top--;
                p1 = p2;
                if (top >= 2) {
                    // stack[top-2]: the cached third entry when valid (a
                    // single pop, the common case), else reloaded
                    p2 = have3 ? p3 : s.at(pos[start + top - 2]);
                    have3 = false;
                }
            }
            pos[start + top] = (I)r;
            top++;
            p3 = p2;
            have3 = top >= 3;
            p2 = p1;
            p1 = cur;
        }
        pred = cur;
    }
    len[t] = top;
}

// Chain access for the merges.  Mat: the chains as stored (the chain of the
// group starting at chunk L is pos[L << lgc ...]).  Merged: the chains of
// the groups one merge level up, not materialised: group L (2w chunks) is
// A[0..i] ++ B[j..] of its two halves (i, j of its pair p = L / 2w).
template <typename I> struct Mat {
    using Idx = I;
    const I *pos;
    int lgc;
    __device__ __forceinline__ I at(long long L, long long q) const { return pos[(L << lgc) + q]; }
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
// B[j..], A and B read through `acc`.  The group span 2 W 2^lgc is a power
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

// ---------------------------------------------- merges without copies --
// (HG_RANGES) Each chunk c keeps the surviving part of its own chain,
// pos[(c << lgc) + lo[c] .. + hi[c]); a group's chain is the concatenation of
// its chunks' parts, so a merge only moves the cut points: the bridge walk
// steps (chunk, slot) cursors over non-empty chunks, then one thread per
// chunk applies the cut (A keeps up to (cA, sA), B from (cB, sB)).  After the
// last level one scan of the part lengths places every part in the output.
#ifndef HG_RANGES
#define HG_RANGES 1
#endif
// nx / pv: links between a group's non-empty chunks (a cut links A's last
// kept chunk to B's first, skipping the emptied ones); head / tail: a group's
// first and last non-empty chunk (-1: empty), indexed by the group's first
// chunk -- so a bridge walk never scans emptied chunks.
struct Ranges {
    int *lo, *hi, *nx, *pv;
};

template <typename I>
__global__ void k_ranges_init(long long nchunks, const long long *__restrict__ len, Ranges R, int *__restrict__ head,
                              int *__restrict__ tail)
{
    for (long long c = (long long)blockIdx.x * blockDim.x + threadIdx.x; c < nchunks; c += (long long)gridDim.x * blockDim.x) {
        const int l = (int)len[c];
        R.lo[c] = 0;
        R.hi[c] = l;
        R.nx[c] = (int)c + 1;
        R.pv[c] = (int)c - 1;
        head[c] = tail[c] = l > 0 ? (int)c : -1;
    }
}

// Bridge of groups A = chunks [L, L + W) and B = [L + W, L + 2W) (clipped to
// nchunks): the same two-pointer walk as k_bridge (i moves back while the turn
// A[i-1], A[i], B[j] is <= 0, j forward while A[i], B[j], B[j+1] is), on
// cursors.  Writes the cut (cA, sA + 1, cB, sB); cA = -1: one side is empty,
// nothing to cut.
template <typename I>
__global__ void k_bridge_r(Seq s, long long nchunks, long long W, const I *__restrict__ pos, const Ranges R,
                           int *__restrict__ head, int *__restrict__ tail, long long *__restrict__ cutA,
                           long long *__restrict__ cutB, int *__restrict__ cutS)
{
    if (s.dm)
        s.m = *s.dm;
    const long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const long long L = 2 * p * W, M = L + W;
    if (L >= nchunks)
        return;
    const long long bend = min(M + W, nchunks);
    const long long np = (nchunks + 2 * W - 1) / (2 * W);
    long long cA = tail[L];
    long long cB = M < nchunks ? head[M] : -1;
    if (cA < 0 || cB < 0) { // one side empty: the group is the other side, uncut
        cutA[p] = -1;
        if (cA < 0 && cB >= 0) {
            head[L] = head[M];
            tail[L] = tail[M];
        }
        return;
    }
    const int lgc = s.lgc;
    int sA = R.hi[cA] - 1, loA = R.lo[cA];
    int sB = R.lo[cB], hiB = R.hi[cB];
    auto pt = [&](long long c, int sl) { return s.at((long long)pos[(c << lgc) + sl]); };
    double2 pA = pt(cA, sA), pB = pt(cB, sB);
    while (true) {
        bool changed = false;
        while (true) { // i > 0 and turn(A[i-1], A[i], B[j]) <= 0: i--
            long long pc = cA;
            int ps = sA - 1, plo = loA;
            if (sA == loA) {
                pc = R.pv[cA];
                while (pc >= L && R.hi[pc] == R.lo[pc]) // (chunks empty from the start)
                    pc = R.pv[pc];
                if (pc < L)
                    break;
                ps = R.hi[pc] - 1;
                plo = R.lo[pc];
            }
            const double2 q = pt(pc, ps);
            if (turn(q, pA, pB) > 0)
                break;
            cA = pc;
            sA = ps;
            loA = plo;
            pA = q;
            changed = true;
        }
        while (true) { // j < lb - 1 and turn(A[i], B[j], B[j+1]) <= 0: j++
            long long nc = cB;
            int ns = sB + 1, nhi = hiB;
            if (ns == hiB) {
                nc = R.nx[cB];
                while (nc < bend && R.hi[nc] == R.lo[nc])
                    nc = R.nx[nc];
                if (nc >= bend)
                    break;
                ns = R.lo[nc];
                nhi = R.hi[nc];
            }
            const double2 q = pt(nc, ns);
            if (turn(pA, pB, q) > 0)
                break;
            cB = nc;
            sB = ns;
            hiB = nhi;
            pB = q;
            changed = true;
        }
        if (!changed)
            break;
    }
    cutA[p] = cA;
    cutB[p] = cB;
    cutS[p] = sA + 1;  // A's new end slot in chunk cA
    cutS[np + p] = sB; // B's new start slot in chunk cB
    R.nx[cA] = (int)cB;
    R.pv[cB] = (int)cA;
    tail[L] = tail[M]; // head[L] stays: A keeps its first element
}

__global__ void k_cut(long long nchunks, long long W, int lg2w, const long long *__restrict__ cutA,
                      const long long *__restrict__ cutB, const int *__restrict__ cutS, Ranges R)
{
    const long long np = (nchunks + 2 * W - 1) / (2 * W);
    for (long long c = (long long)blockIdx.x * blockDim.x + threadIdx.x; c < nchunks; c += (long long)gridDim.x * blockDim.x) {
        const long long p = c >> lg2w;
        const long long ca = cutA[p];
        if (ca < 0)
            continue;
        if (c < (p << lg2w) + W) { // in A
            if (c > ca)
                R.hi[c] = R.lo[c];
            else if (c == ca)
                R.hi[c] = cutS[p];
        } else {                   // in B
            const long long cb = cutB[p];
            if (c < cb)
                R.lo[c] = R.hi[c];
            else if (c == cb)
                R.lo[c] = cutS[np + p];
        }
    }
}

// Exclusive scan of the part lengths hi - lo of both chains (blockIdx.y):
// HG_SCAN_B lengths per block, block sums, then the offsets; tot[y] = the
// chain's length.
constexpr int HG_SCAN_B = 1024;
__global__ void __launch_bounds__(HG_SCAN_B) k_scan_sums(long long nchunks, const Ranges R0, const Ranges R1,
                                                         long long *__restrict__ bsum)
{
    const Ranges R = blockIdx.y ? R1 : R0;
    const long long c = (long long)blockIdx.x * HG_SCAN_B + threadIdx.x;
    int v = c < nchunks ? R.hi[c] - R.lo[c] : 0;
    __shared__ int ws[HG_SCAN_B / 32];
    for (int o = 16; o > 0; o >>= 1)
        v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0)
        ws[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
        long long t = 0;
        for (int i = 0; i < HG_SCAN_B / 32; i++)
            t += ws[i];
        bsum[blockIdx.y * gridDim.x + blockIdx.x] = t;
    }
}
__global__ void k_scan_bsums(int nb, long long *__restrict__ bsum, long long *__restrict__ tot)
{
    // one thread per chain: the block sums are few (nchunks / 1024)
    if (threadIdx.x >= 2)
        return;
    long long *b = bsum + (long long)threadIdx.x * nb, run = 0;
    for (int i = 0; i < nb; i++) {
        const long long t = b[i];
        b[i] = run;
        run += t;
    }
    tot[threadIdx.x] = run;
}
__global__ void __launch_bounds__(HG_SCAN_B) k_scan_offsets(long long nchunks, const Ranges R0, const Ranges R1,
                                                            const long long *__restrict__ bsum, long long *__restrict__ pre0,
                                                            long long *__restrict__ pre1)
{
    const Ranges R = blockIdx.y ? R1 : R0;
    long long *pre = blockIdx.y ? pre1 : pre0;
    const long long c = (long long)blockIdx.x * HG_SCAN_B + threadIdx.x;
    const int v = c < nchunks ? R.hi[c] - R.lo[c] : 0;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    int inc = v;
    for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o)
            inc += t;
    }
    __shared__ int ws[HG_SCAN_B / 32];
    if (lane == 31)
        ws[w] = inc;
    __syncthreads();
    int base = 0;
    for (int i = 0; i < w; i++)
        base += ws[i];
    if (c < nchunks)
        pre[c] = bsum[blockIdx.y * gridDim.x + blockIdx.x] + base + inc - v;
}

// lower[0 .. nl-1) then upper[0 .. nu-1) (as k_assemble), read from the
// chunks' parts: slot sl of chunk c is element pre[c] + sl - lo[c] of its chain.
template <typename I, typename V>
__global__ void k_assemble_r(long long m, int lgc, long long nchunks, const I *__restrict__ pl, const Ranges Rl,
                             const long long *__restrict__ prel, const I *__restrict__ pu, const Ranges Ru,
                             const long long *__restrict__ preu, const long long *__restrict__ tot,
                             const V *__restrict__ val, const long long *__restrict__ idmap, long long *__restrict__ out,
                             long long *__restrict__ d_nh, const long long *__restrict__ dm)
{
    if (dm)
        m = *dm;
    auto id = [&](V v) { return idmap ? idmap[(long long)v] : (long long)v; };
    const long long nl = tot[0], nu = tot[1];
    const long long a = nl - 1, total = nl <= 1 ? 1 : a + (nu - 1);
    if (blockIdx.x == 0 && threadIdx.x == 0)
        *d_nh = total;
    // one warp per chunk: its parts' bounds and offsets once, then 32 slots
    // at a time (coalesced reads of the positions and writes of the ids)
    const int lane = threadIdx.x & 31;
    const long long nwarps = ((long long)gridDim.x * blockDim.x) >> 5;
    for (long long c = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5; c < nchunks; c += nwarps) {
        const long long base = c << lgc;
        const int lol = Rl.lo[c], hil = Rl.hi[c];
        const long long pl0 = prel[c] - lol;
        for (int sl = lol + lane; sl < hil; sl += 32) {
            const long long e = pl0 + sl;
            if (nl <= 1 ? e == 0 : e < a) // (nl <= 1: a single distinct point, the lowest id)
                out[e] = id(val[(long long)pl[base + sl]]);
        }
        if (nl > 1) {
            const int lou = Ru.lo[c], hiu = Ru.hi[c];
            const long long pu0 = preu[c] - lou;
            for (int sl = lou + lane; sl < hiu; sl += 32) {
                const long long e = pu0 + sl;
                if (e < nu - 1)
                    out[a + e] = id(val[m - 1 - (long long)pu[base + sl]]);
            }
        }
    }
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
    const int lgc = chunk_log2(m); // log2 of the chunk size
    const long long nchunks = (m + (1ll << lgc) - 1) >> lgc;
    const long long m_cap = nchunks << lgc;
    Seq s{P, m, rev, lgc};
    k_chunk_chain<I><<<(unsigned)((nchunks + HG_THREADS - 1) / HG_THREADS), HG_THREADS, 0, st>>>(s, nchunks, pos_a,
                                                                                                  len_a);
    int lgw = 0; // log2 w
    // Up to three merge levels per copy (m >= HG_FLAT_M): each level's bridges read the chains
    // of the level below through Merged (not materialised), then one copy
    // materialises them -- a third of the copies of one level at a time.
    for (long long w = 1; w < nchunks;) {
        const long long np1 = (nchunks + 2 * w - 1) / (2 * w);
        const Mat<I> m0{pos_a, lgc};
        // few points: one merge level per copy (the copies are cheap, and the
        // bridge walks -- serial, latency-bound -- then read flat chains)
        if (2 * w >= nchunks || m < HG_FLAT_M) {
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

// One chain with HG_RANGES: chunk chains into pos, parts initialised, the
// merge levels as cuts.  The parts stay in (pos, R).  Asynchronous.
template <typename I>
static void chain_gpu_ranges(const double2 *P, long long m, int rev, I *pos, Ranges R, long long *len_tmp,
                             int *head, int *tail, long long *cutA, long long *cutB, int *cutS, int lgc,
                             const long long *dm, cudaStream_t st)
{
    const long long nchunks = (m + (1ll << lgc) - 1) >> lgc;
    Seq s{P, m, rev, lgc, dm};
    k_chunk_chain<I><<<(unsigned)((nchunks + HG_THREADS - 1) / HG_THREADS), HG_THREADS, 0, st>>>(s, nchunks, pos,
                                                                                                  len_tmp);
    k_ranges_init<I><<<grid_for(nchunks, 256), 256, 0, st>>>(nchunks, len_tmp, R, head, tail);
    int lgw = 0;
    for (long long w = 1; w < nchunks; w *= 2, lgw++) {
        const long long np = (nchunks + 2 * w - 1) / (2 * w);
        k_bridge_r<I><<<blocks_for(np, HG_THREADS), HG_THREADS, 0, st>>>(s, nchunks, w, pos, R, head, tail, cutA,
                                                                        cutB, cutS);
        k_cut<<<grid_for(nchunks, 256), 256, 0, st>>>(nchunks, w, lgw + 1, cutA, cutB, cutS, R);
    }
}

// Scratch layout of ch_hull_gpu_async for m survivors (all 256-B aligned).
// The radix sort's control block (status words, histograms, tickets, min /
// max, the long-run count) is contiguous so one memset clears it.
struct HullTmp {
    size_t total = 0;
    size_t o_k0, o_k1, o_v0, o_v1, o_P, o_pa, o_pb, o_pc, o_pd, o_la, o_lb, o_lc, o_ld, o_bi, o_bj, o_out;
    size_t o_bi2, o_bj2, o_lm, o_bi3, o_bj3, o_lm2, o_runs, o_ctl, ctl_bytes;
    size_t o_hist, o_tk, o_mm, o_nruns; // inside the control block
    long long ntiles;
    explicit HullTmp(long long m)
    {
        if (m < 1)
            m = 1;
        // chunk arrays for the smaller of the two chunk sizes (chunk_log2,
        // chunk_log2_dev); positions for the larger capacity
        const int lgc = chunk_log2_dev(m), lgc1 = chunk_log2(m);
        const size_t nchunks = (size_t)((m + (1ll << lgc) - 1) >> lgc);
        const size_t cap = std::max(nchunks << lgc, (size_t)((m + (1ll << lgc1) - 1) >> lgc1) << lgc1);
        const size_t isz = m < (1ll << 32) ? 4 : 8; // chain position width
        ntiles = (m + chrs::RS_TILE - 1) / chrs::RS_TILE;
        size_t p = 0;
        auto take = [&](size_t b) { const size_t o = p; p += (b + 255) & ~(size_t)255; return o; };
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
        o_runs = take(((size_t)m / (HG_SMALL_RUN + 1) + 1) * 16);
        // control block: status | hist[4][256] | tickets[4] | mm[2] | nruns
        const size_t st = (size_t)ntiles * chrs::RS_BINS * 8;
        o_hist = st;
        o_tk = o_hist + 4 * chrs::RS_BINS * 8;
        o_mm = o_tk + 4 * 8;
        o_nruns = o_mm + 2 * 8;
        ctl_bytes = o_nruns + 8;
        o_ctl = take(ctl_bytes);
        total = p;
    }
};

template <typename F> static void set_smem(F *f, size_t bytes)
{
    if (bytes > 48 * 1024)
        cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
}

// The pipeline with sort values (survivor ids) of type V.
template <typename V>
// surv == NULL: the hull of d_xy[0..m) itself; idmap (nullable) maps the
// resulting point positions / ids to output ids.
static ch_status hull_async(const double *d_xy, const long long *surv, long long m, long long *d_hull,
                            long long *d_n_hull, void *d_tmp, const HullTmp &L, cudaStream_t st,
                            const long long *idmap = nullptr, const long long *dm = nullptr,
                            const long long *kept = nullptr, const unsigned long long *use_kept = nullptr)
{
    // dm (nullable): the count is *dm <= m, known on the device only (the
    // launches are sized for m); use_kept: the ids come from `kept`
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

    auto *ctl = (unsigned char *)(b + L.o_ctl);
    auto *status = (unsigned long long *)ctl;
    auto *hist = (unsigned long long *)(ctl + L.o_hist);
    auto *tk = (unsigned long long *)(ctl + L.o_tk);
    auto *mm = (unsigned long long *)(ctl + L.o_mm);
    auto *nruns = (unsigned long long *)(ctl + L.o_nruns);
    auto *runs = (long long *)(b + L.o_runs);
    if (cudaMemsetAsync(ctl, 0, L.ctl_bytes, st) != cudaSuccess || cudaMemsetAsync(mm, 0xff, 8, st) != cudaSuccess)
        return chi::fail(CH_ERR_CUDA, "device hull: memset");

    // 1. x and the sort values, min / max of x; 2. 32-bit keys + histograms
    const int g = grid_for(m, 256);
    double *X = (double *)k0;
    auto *keyA = (unsigned *)k1, *keyB = (unsigned *)k0;
    k_gather_x<V><<<g, 256, 0, st>>>(d_xy, surv, m, X, v0, mm, dm, kept, use_kept);
    k_keys_hist<<<std::min(g, 148 * 4), 256, 0, st>>>(X, m, mm, keyA, hist, dm);
    // 3. four stable 8-bit passes (keys k1 -> k0 -> k1 -> k0 -> k1, values v0 -> v1 -> ... -> v0)
    const size_t smem = sizeof(chrs::TileSmem<unsigned, V>);
    auto pass_kernel = m <= 0xffffffffll ? chrs::k_rs_pass<unsigned, V, unsigned> : chrs::k_rs_pass<unsigned, V, long long>;
    set_smem(pass_kernel, smem);
    unsigned *kin = keyA, *kout = keyB;
    V *vin = v0, *vout = v1;
    for (int pass = 0; pass < 4; pass++) {
        pass_kernel<<<(unsigned)L.ntiles, chrs::RS_THREADS, smem, st>>>(kin, kout, vin, vout, m, 8 * pass, pass,
                                                                     hist + pass * chrs::RS_BINS, status, tk + pass,
                                                                     dm);
        std::swap(kin, kout);
        std::swap(vin, vout);
    }
    V *val = vin; // == v0
    // 4. the points in key order; runs of equal key sorted by x exactly, equal x resolved
    k_points<V><<<g, 256, 0, st>>>(d_xy, val, m, P, dm);
    k_fix_runs<V><<<g, 256, 0, st>>>(kin, P, val, m, runs, nruns, dm);
    const size_t fsmem = sizeof(chrs::TileSmem<unsigned long long, unsigned>);
    set_smem(k_fix_big<V>, fsmem);
    k_fix_big<V><<<148 * 2, chrs::RS_THREADS, fsmem, st>>>(P, val, runs, nruns, (unsigned long long *)k0,
                                                          (unsigned long long *)k1, (unsigned *)v1,
                                                          (unsigned *)v1 + m);

    // merges as cuts (m >= cuts_min) or by copies (fewer points: flat levels
    // are cheaper than cursor walks); CH_HULL_CUTS_MIN overrides the
    // threshold (tests run both paths on small inputs)
    long long cuts_min = HG_FLAT_M;
    if (const char *e = getenv("CH_HULL_CUTS_MIN"))
        cuts_min = atoll(e);
    auto chains = [&](auto tag) {
        using I = decltype(tag);
#if HG_RANGES
      if (m >= cuts_min || dm) { // (the device count: only the cuts handle empty chunks)
        // lower parts in (pa, la/lb as lo/hi + links), upper in (pc, lc/ld);
        // cuts in bi / bj / bi2, group heads / tails in bi3, chunk lengths
        // then block sums in bj3, offsets in lm / lm2, totals in bj2
        const int lgc = dm ? chunk_log2_dev(m) : chunk_log2(m);
        const long long nchunks = (m + (1ll << lgc) - 1) >> lgc;
        // (la..ld hold 2 nchunks + 2 ints each: lo or hi, then a link array)
        const Ranges Rl{(int *)la, (int *)lb, (int *)la + nchunks, (int *)lb + nchunks};
        const Ranges Ru{(int *)lc, (int *)ld, (int *)lc + nchunks, (int *)ld + nchunks};
        int *head = (int *)bi3, *tail = (int *)bi3 + nchunks;
        chain_gpu_ranges<I>(P, m, 0, (I *)pa, Rl, bj3, head, tail, bi, bj, (int *)bi2, lgc, dm, st);
        chain_gpu_ranges<I>(P, m, 1, (I *)pc, Ru, bj3, head, tail, bi, bj, (int *)bi2, lgc, dm, st);
        const unsigned nb = (unsigned)((nchunks + HG_SCAN_B - 1) / HG_SCAN_B);
        k_scan_sums<<<dim3(nb, 2), HG_SCAN_B, 0, st>>>(nchunks, Rl, Ru, bj3);
        k_scan_bsums<<<1, 32, 0, st>>>((int)nb, bj3, bj2);
        k_scan_offsets<<<dim3(nb, 2), HG_SCAN_B, 0, st>>>(nchunks, Rl, Ru, bj3, lm, lm2);
        k_assemble_r<I, V><<<grid_for(nchunks * 32, 256), 256, 0, st>>>(m, lgc, nchunks, (const I *)pa, Rl, lm,
                                                                          (const I *)pc, Ru, lm2, bj2, val, idmap,
                                                                          d_hull, d_n_hull, dm);
        return;
      }
#endif
        const long long *d_hl, *d_hu;
        const I *low = chain_gpu<I>(P, m, 0, (I *)pa, (I *)pb, la, lb, bi, bj, bi2, bj2, bi3, bj3, lm, lm2, &d_hl, st);
        const I *up = chain_gpu<I>(P, m, 1, (I *)pc, (I *)pd, lc, ld, bi, bj, bi2, bj2, bi3, bj3, lm, lm2, &d_hu, st);
        k_assemble<I, V><<<grid_for(m, 256), 256, 0, st>>>(m, low, d_hl, up, d_hu, val, idmap, d_hull, d_n_hull);
    };
    if (m < (1ll << 32))
        chains((unsigned)0);
    else
        chains((long long)0);
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? CH_OK : chi::fail(CH_ERR_CUDA, std::string("device hull: ") + cudaGetErrorString(e));
}

// (the second round's scratch follows the pipeline's: the kept ids, then
// the polygon, the direction extremes, the kept count and the probe's count)
static size_t refine_offset(int64_t m) { return (HullTmp(m).total + 255) & ~(size_t)255; }
static size_t refine_bytes(int64_t m)
{
    return ((size_t)(m < 1 ? 1 : m) * 8 + 255) / 256 * 256 + sizeof(RefinePoly) + HG_DIRS * 8 + 32 + 256;
}
// The second filtering round (k_refine_filter) on survivors surv[0..m) of
// d_xy (surv NULL: every point), when they are many and the scratch
// (ch_hull_gpu_temp_bytes(m)) has room: *surv_out / *m_out = the kept ids
// (in the scratch, past HullTmp(m)) and their count, else surv / m.
// Synchronizes `st`.
static ch_status refine_round(const double *d_xy, const long long *surv, long long m, void *d_tmp, size_t tmp_bytes,
                              cudaStream_t st, const long long **surv_out, int64_t *m_out)
{
    *surv_out = surv;
    *m_out = m;
    if (!(m >= HG_REFINE_MIN && tmp_bytes >= refine_offset(m) + refine_bytes(m)))
        return CH_OK;
    char *rb = (char *)d_tmp + refine_offset(m);
    auto *kept = (long long *)rb;
    auto *poly = (RefinePoly *)(rb + ((size_t)m * 8 + 255) / 256 * 256);
    auto *best = (unsigned long long *)(poly + 1);
    auto *nkept = best + HG_DIRS;
    Dirs D;
    for (int k = 0; k < HG_DIRS; k++) {
        const double th = 2.0 * 3.14159265358979323846 * k / HG_DIRS;
        D.u[k][0] = (float)std::cos(th);
        D.u[k][1] = (float)std::sin(th);
    }
    const long long stride = m > HG_SAMPLE ? m / HG_SAMPLE : 1;
    const long long nsample = (m + stride - 1) / stride;
    if (cudaMemsetAsync(best, 0, (HG_DIRS + 2) * 8, st) != cudaSuccess)
        return chi::fail(CH_ERR_CUDA, "device hull: memset");
    k_dir_extremes<<<148 * 4, 256, 0, st>>>(d_xy, surv, stride, nsample, D, best);
    k_refine_poly<<<1, HG_DIRS, 0, st>>>(d_xy, surv, stride, best, poly);
    // the yield on the sample decides whether the full round pays (a
    // circle: nothing to drop, every survivor is a hull vertex)
    k_refine_probe<<<grid_for(nsample, 256), 256, 0, st>>>(d_xy, surv, stride, nsample, poly, nkept + 1);
    unsigned long long ndrop = 0;
    cudaMemcpyAsync(&ndrop, nkept + 1, 8, cudaMemcpyDeviceToHost, st);
    if (cudaStreamSynchronize(st) != cudaSuccess)
        return chi::fail(CH_ERR_CUDA, std::string("device hull (second round): ") +
                                          cudaGetErrorString(cudaGetLastError()));
    if (4 * ndrop < (unsigned long long)nsample) // < 25% of the sample dropped
        return CH_OK;
    const long long tiles = (m + 256LL * HG_RF_ITEMS - 1) / (256LL * HG_RF_ITEMS);
    k_refine_filter<<<(unsigned)std::min<long long>(tiles, 148 * 8), 256, 0, st>>>(d_xy, surv, m, poly, kept, nkept,
                                                                                   nullptr, 0);
    unsigned long long nk = 0;
    cudaMemcpyAsync(&nk, nkept, 8, cudaMemcpyDeviceToHost, st);
    if (cudaStreamSynchronize(st) != cudaSuccess)
        return chi::fail(CH_ERR_CUDA, std::string("device hull (second round): ") +
                                          cudaGetErrorString(cudaGetLastError()));
    if ((long long)nk < m && nk > 0) {
        *surv_out = kept;
        *m_out = (int64_t)nk;
    }
    return CH_OK;
}

// The second round without a host synchronization (ch_hull_gpu_async): the
// probe's yield is read by k_refine_filter and k_refine_finish on the
// device, which leave *dm (the count) and *use (the kept list or `surv`) for
// the pipeline.  False when m or the scratch is too small.
static bool refine_round_async(const double *d_xy, const long long *surv, long long m, void *d_tmp, size_t tmp_bytes,
                               cudaStream_t st, const long long **kept_out, const long long **dm_out,
                               const unsigned long long **use_out)
{
    if (!(m >= HG_REFINE_MIN && tmp_bytes >= refine_offset(m) + refine_bytes(m)))
        return false;
    char *rb = (char *)d_tmp + refine_offset(m);
    auto *kept = (long long *)rb;
    auto *poly = (RefinePoly *)(rb + ((size_t)m * 8 + 255) / 256 * 256);
    auto *best = (unsigned long long *)(poly + 1);
    auto *nkept = best + HG_DIRS; // nkept[0] kept, [1] the probe's drops, [2] use, [3] dm
    Dirs D;
    for (int k = 0; k < HG_DIRS; k++) {
        const double th = 2.0 * 3.14159265358979323846 * k / HG_DIRS;
        D.u[k][0] = (float)std::cos(th);
        D.u[k][1] = (float)std::sin(th);
    }
    const long long stride = m > HG_SAMPLE ? m / HG_SAMPLE : 1;
    const long long nsample = (m + stride - 1) / stride;
    if (cudaMemsetAsync(best, 0, (HG_DIRS + 4) * 8, st) != cudaSuccess)
        return false;
    k_dir_extremes<<<148 * 4, 256, 0, st>>>(d_xy, surv, stride, nsample, D, best);
    k_refine_poly<<<1, HG_DIRS, 0, st>>>(d_xy, surv, stride, best, poly);
    k_refine_probe<<<grid_for(nsample, 256), 256, 0, st>>>(d_xy, surv, stride, nsample, poly, nkept + 1);
    const long long tiles = (m + 256LL * HG_RF_ITEMS - 1) / (256LL * HG_RF_ITEMS);
    k_refine_filter<<<(unsigned)std::min<long long>(tiles, 148 * 8), 256, 0, st>>>(d_xy, surv, m, poly, kept, nkept,
                                                                                   nkept + 1, nsample);
    k_refine_finish<<<1, 1, 0, st>>>(m, nsample, nkept + 1, nkept, nkept + 2, (long long *)(nkept + 3));
    *kept_out = kept;
    *use_out = nkept + 2;
    *dm_out = (const long long *)(nkept + 3);
    return true;
}

extern "C" {

// Device scratch for ch_hull_gpu / ch_hull_gpu_async on m survivors.
size_t ch_hull_gpu_temp_bytes(int64_t m)
{
    return refine_offset(m) + refine_bytes(m);
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
    if (m <= HG_SMALL_M) { // one CTA, one launch
        k_small_hull<<<1, 512, 0, st>>>(d_xy, (const long long *)d_surv, nullptr, m, (long long *)d_hull,
                                        (long long *)d_n_hull);
        const cudaError_t e = cudaGetLastError();
        return e == cudaSuccess ? CH_OK : chi::fail(CH_ERR_CUDA, std::string("device hull: ") + cudaGetErrorString(e));
    }
    // the second filtering round, decided on the device (no host
    // synchronization) when the scratch has room for it
    const long long *kept = nullptr, *dm = nullptr;
    const unsigned long long *use = nullptr;
    refine_round_async(d_xy, (const long long *)d_surv, m, d_tmp, tmp_bytes, st, &kept, &dm, &use);
    // ids fit 32 bits when the point array does: the sorts then move 12, not
    // 16, bytes per element and pass
    return n_points <= (1ll << 32) ? hull_async<unsigned>(d_xy, (const long long *)d_surv, m, (long long *)d_hull,
                                                           (long long *)d_n_hull, d_tmp, L, st, nullptr, dm, kept, use)
                                   : hull_async<unsigned long long>(d_xy, (const long long *)d_surv, m,
                                                                    (long long *)d_hull, (long long *)d_n_hull, d_tmp,
                                                                    L, st, nullptr, dm, kept, use);
}

} // extern "C"

// The root's hull stage of ch_hull_end_to_end_dist: ch_hull_gpu_pts_async
// preceded by the second filtering round (so it synchronizes `stream`).
ch_status chi::hull_pts_refined(const double *d_pts, const int64_t *d_ids, int64_t m, int64_t *d_hull,
                                int64_t *d_n_hull, void *d_tmp, size_t tmp_bytes, cudaStream_t st)
{
    if (m <= 0 || !d_pts || !d_ids || !d_tmp)
        return ch_hull_gpu_pts_async(d_pts, d_ids, m, d_hull, d_n_hull, d_tmp, tmp_bytes, st);
    const long long *kept = nullptr;
    int64_t m2 = m;
    ch_status s = refine_round(d_pts, nullptr, m, d_tmp, tmp_bytes, st, &kept, &m2);
    if (s != CH_OK || kept == nullptr)
        return s != CH_OK ? s : ch_hull_gpu_pts_async(d_pts, d_ids, m, d_hull, d_n_hull, d_tmp, tmp_bytes, st);
    // positions kept[0..m2) into d_pts; the ids through the idmap d_ids
    const HullTmp L2(m2);
    return m2 <= (1ll << 32) ? hull_async<unsigned>(d_pts, kept, m2, (long long *)d_hull, (long long *)d_n_hull, d_tmp,
                                                     L2, st, (const long long *)d_ids)
                             : hull_async<unsigned long long>(d_pts, kept, m2, (long long *)d_hull,
                                                              (long long *)d_n_hull, d_tmp, L2, st,
                                                              (const long long *)d_ids);
}

extern "C" {

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
    if (m <= HG_SMALL_M) { // one CTA, one launch (positions i, ids d_ids[i])
        k_small_hull<<<1, 512, 0, st>>>(d_pts, nullptr, (const long long *)d_ids, m, (long long *)d_hull,
                                        (long long *)d_n_hull);
        const cudaError_t e = cudaGetLastError();
        return e == cudaSuccess ? CH_OK : chi::fail(CH_ERR_CUDA, std::string("device hull: ") + cudaGetErrorString(e));
    }
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
    // the second filtering round (see k_refine_filter)
    const int64_t *surv = d_surv;
    int64_t m2 = m;
    ch_status s = refine_round(d_xy, (const long long *)d_surv, m, d_tmp, tmp_bytes, st, (const long long **)&surv, &m2);
    if (s != CH_OK)
        return s;
    const HullTmp L2(m2);
    int64_t *d_out = (int64_t *)((char *)d_tmp + L2.o_out);
    int64_t *d_nh = d_out + m2; // the word after the ids (o_out holds m + 1 words)
    s = ch_hull_gpu_async(d_xy, n_points, surv, m2, d_out, d_nh, d_tmp, L2.total, stream);
    if (s != CH_OK)
        return s;
    int64_t nh = 0;
    cudaMemcpyAsync(&nh, d_nh, sizeof(nh), cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    cudaMemcpyAsync(h_hull, d_out, (size_t)nh * 8, cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess)
        return chi::fail(CH_ERR_CUDA, std::string("ch_hull_gpu: ") + cudaGetErrorString(e));
    *h_n_hull = nh;
    return CH_OK;
}

} // extern "C"
