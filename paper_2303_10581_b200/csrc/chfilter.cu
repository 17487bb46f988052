// chfilter.cu -- B200 (sm_100a) kernels and the C ABI of include/chfilter.h.
//
// The hot path is two streaming kernels over the float64 AoS point array:
//   K1 k1_extremes8       one read of every point: the eight extremes (P:124,
//                         P:185), grid combine, octagon built by the last CTA.
//   K2 k2_filter_compact  the second and last read: octagon test fused
//                         with a single-pass decoupled look-back compaction
//                         (replaces the paper's filter/scan/scatter).
// plus K3 k3_combine8 (multi-GPU exchange), K4 k4_octagon_bits (the paper's
// bit vector) and a gather for the hull stage.
//
// Arithmetic follows DESIGN.md "Readings": binary64 RNE, explicit __d*_rn
// intrinsics (never contracted), built with -fmad=false as well.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <climits>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "../../include/chfilter.h"
#include "internal.h"
#include "octagon.cuh"
#include "exact.cuh"

extern "C" int64_t ch_internal_hull(const double *pts, const int64_t *ids, int64_t m, int64_t *hull);

namespace {

constexpr unsigned FULL = 0xffffffffu;

#ifndef CH_K1_UNROLL_F
#define CH_K1_UNROLL_F 4 // K1 wide loads (CH_K1_PPL_F points each) per thread per chunk, float32 storage
#endif
#ifndef CH_K1_PPL_F
#define CH_K1_PPL_F 4 // float32 points per K1 wide load: 2 (128 bits) or 4 (256 bits)
#endif
#ifndef CH_K1_MINB_F
#define CH_K1_MINB_F 3 // K1 CTAs per SM for float32 storage
#endif
#ifndef CH_K2_NP_D
#define CH_K2_NP_D 8 // K2 points per consumer thread per sub-tile, float64 storage
#endif
#ifndef CH_K2_NP_F
#define CH_K2_NP_F 16 // the same, float32 storage
#endif
#ifndef CH_K2_STAGES
#define CH_K2_STAGES 3 // K2 TMA ring depth
#endif
#ifndef CH_K2_STAGES_F
#define CH_K2_STAGES_F 3 // the same, float32 storage
#endif
#ifndef CH_K2_MINB
#define CH_K2_MINB 2 // K2 resident CTAs per SM the registers are sized for
#endif
#ifndef CH_K2_SUPERS
#define CH_K2_SUPERS 8 // K2 super-tiles per resident CTA the super-tile size aims for
#endif
#ifndef CH_K2_BOX
#define CH_K2_BOX 1 // K2 accept-box stage: 0 never (certificates only), 1 adaptive
#endif
#ifndef CH_CERT_H
#define CH_CERT_H 8 // points per consume_cert pass
#endif

// ----------------------------------------------------------------- layout --
constexpr int K1_THREADS = 256;
// Point storage: float64 AoS (16 B/pt, the default) or float32 AoS (8 B/pt,
// the paper's storage precision).  Float coordinates are widened to
// double exactly, so both run the same fp64 arithmetic.
template <typename T> struct PtTraits;
template <> struct PtTraits<double> {
    using V2 = double2;
    static constexpr int K1_UNROLL = 4; // wide loads (2 points each) per thread per chunk
    static constexpr int K1_PPL = 2;    // points per wide load (256 bits)
    static constexpr int K1_MINB = 3;   // K1 CTAs per SM the registers are sized for
    static constexpr int K2_NP = CH_K2_NP_D;     // points per consumer thread per sub-tile
    static constexpr int K2_STAGES = CH_K2_STAGES; // TMA ring depth (sub-tiles)
};
template <> struct PtTraits<float> {
    using V2 = float2;
    static constexpr int K1_UNROLL = CH_K1_UNROLL_F;
    static constexpr int K1_PPL = CH_K1_PPL_F;
    static constexpr int K1_MINB = CH_K1_MINB_F;
    static constexpr int K2_NP = CH_K2_NP_F;
    static constexpr int K2_STAGES = CH_K2_STAGES_F;
};
template <typename T> constexpr long long k1_chunk()
{
    return (long long)K1_THREADS * PtTraits<T>::K1_UNROLL * PtTraits<T>::K1_PPL;
}
constexpr int K1_MAX_CTAS = 2048;

constexpr int K2_CWARPS = 8;                                   // consumer (compute) warps per CTA
constexpr int K2_CTHREADS = K2_CWARPS * 32;
constexpr int K2_PROD_WARP = K2_CWARPS + 1;                    // TMA producer warp
constexpr int K2_THREADS = K2_CTHREADS + 64;
constexpr int K2_ENTRIES = 4 * K2_CTHREADS;                    // ballot words per super-tile (block scan: 4/thread)
constexpr int K2_SLOTS = K2_ENTRIES / K2_CWARPS;               // ballot words per consumer warp per super-tile
template <typename T> constexpr long long k2_sub() { return (long long)K2_CTHREADS * PtTraits<T>::K2_NP; }
template <typename T> constexpr int k2_groups() { return PtTraits<T>::K2_NP * K2_CWARPS; } // 32-point groups / sub-tile
template <typename T> constexpr int k2_maxsub() { return K2_ENTRIES / k2_groups<T>(); }   // sub-tiles / super-tile
template <typename T>
constexpr size_t k2_dsmem() // stages + bits[2] + scan[2]
{
    return (size_t)PtTraits<T>::K2_STAGES * k2_sub<T>() * sizeof(typename PtTraits<T>::V2) + 4 * K2_ENTRIES * 4;
}
constexpr int K2_BAR_BASE = 1;                                 // named barrier ids 1..5

constexpr int K4_THREADS = 256;

// Look-back status word: flag(2) | epoch(22) | value(40).
constexpr unsigned long long ST_A = 1ull, ST_P = 2ull;
constexpr int ST_EPOCH_BITS = 22;
constexpr unsigned long long ST_VALUE_MASK = (1ull << 40) - 1;
constexpr unsigned ST_EPOCH_MASK = (1u << ST_EPOCH_BITS) - 1;

struct Partial {
    double key[8];
    long long idx[8];
    int nonfinite;
    int pad[3];
};

struct WsHeader {
    unsigned k1_ticket;
    unsigned k2_claim;
    unsigned k2_exit;
    unsigned epoch;
    unsigned peer_timeout; // K3's wait for a peer's record timed out (CH_ERR_PEER)
    unsigned tag_valid;    // the octagon below was built from the points (tag_xy, tag_n, tag_base)
    unsigned pad_[2];
    long long tag_xy, tag_n, tag_base;
    ch_result result;
    ch_extremes ext;
    ch_octagon oct;
};
static_assert(sizeof(WsHeader) <= 4096, "header too large");
constexpr size_t WS_HEADER = 4096;
constexpr size_t WS_PARTIALS = (size_t)K1_MAX_CTAS * sizeof(Partial);

inline long long ntiles_of(long long n) { return (n + k2_sub<double>() - 1) / k2_sub<double>(); } // >= super-tiles

// ------------------------------------------------------------ PTX helpers --
__device__ __forceinline__ void ld256(const double *p, double &a, double &b, double &c, double &d)
{
    asm volatile("ld.global.nc.L1::no_allocate.v4.f64 {%0,%1,%2,%3}, [%4];"
                 : "=d"(a), "=d"(b), "=d"(c), "=d"(d)
                 : "l"(p));
}
__device__ __forceinline__ void ld128(const double *p, double &a, double &b)
{
    asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0,%1}, [%2];" : "=d"(a), "=d"(b) : "l"(p));
}
__device__ __forceinline__ void ld128f(const float *p, float &a, float &b, float &c, float &d)
{
    asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(a), "=f"(b), "=f"(c), "=f"(d)
                 : "l"(p));
}
__device__ __forceinline__ void ld256f(const float *p, float (&r)[8])
{
    asm volatile("ld.global.nc.L1::no_allocate.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=f"(r[0]), "=f"(r[1]), "=f"(r[2]), "=f"(r[3]), "=f"(r[4]), "=f"(r[5]), "=f"(r[6]), "=f"(r[7])
                 : "l"(p));
}
__device__ __forceinline__ void ld64f(const float *p, float &a, float &b)
{
    asm volatile("ld.global.nc.L1::no_allocate.v2.f32 {%0,%1}, [%2];" : "=f"(a), "=f"(b) : "l"(p));
}
// Two consecutive points in their storage type (widened at use).
template <typename T, bool VEC>
__device__ __forceinline__ void ld2raw(const T *p, T (&r)[4]);
template <>
__device__ __forceinline__ void ld2raw<double, true>(const double *p, double (&r)[4]) { ld256(p, r[0], r[1], r[2], r[3]); }
template <>
__device__ __forceinline__ void ld2raw<double, false>(const double *p, double (&r)[4])
{
    ld128(p, r[0], r[1]);
    ld128(p + 2, r[2], r[3]);
}
template <>
__device__ __forceinline__ void ld2raw<float, true>(const float *p, float (&r)[4]) { ld128f(p, r[0], r[1], r[2], r[3]); }
template <>
__device__ __forceinline__ void ld2raw<float, false>(const float *p, float (&r)[4])
{
    ld64f(p, r[0], r[1]);
    ld64f(p + 2, r[2], r[3]);
}
// One point in its storage type.
__device__ __forceinline__ void ld1raw(const double *xy, long long i, double &x, double &y) { ld128(xy + 2 * i, x, y); }
__device__ __forceinline__ void ld1raw(const float *xy, long long i, float &x, float &y) { ld64f(xy + 2 * i, x, y); }
// One point as doubles.
__device__ __forceinline__ void ld1pt(const double *xy, long long i, double &x, double &y) { ld128(xy + 2 * i, x, y); }
__device__ __forceinline__ void ld1pt(const float *xy, long long i, double &x, double &y)
{
    float fx, fy;
    ld64f(xy + 2 * i, fx, fy);
    x = fx, y = fy;
}
__device__ __forceinline__ unsigned long long ld_acquire(const unsigned long long *p)
{
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release(unsigned long long *p, unsigned long long v)
{
    asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned lanemask_lt()
{
    unsigned m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

// The workspace octagon's data tag: the octagon in the header was built from
// the points (xy, n, index_base) by K1 / K5 / K6 (or K3, from records whose
// bbox contains that shard's).  K2 trusts the fp32 certificates (whose error
// bound needs every point inside the octagon's bbox) only for those points.
__device__ __forceinline__ void set_tag(WsHeader *hdr, const void *xy, long long n, long long index_base)
{
    hdr->tag_xy = (long long)xy;
    hdr->tag_n = n;
    hdr->tag_base = index_base;
    hdr->tag_valid = 1;
}

// --------------------------------------------------- peer exchange (a4, a7) --
// Exchange buffer of one rank: [2 banks][CH_MAX_PEERS slots][PEER_SLOT words];
// slot s holds what rank s sent: words 0..23 its ch_extremes record, 24 the
// record's epoch flag, 25 its survivor count, 26 the count's epoch flag.
constexpr int PEER_SLOT = 32; // 256 B
constexpr int PEER_REC_FLAG = 24, PEER_CNT = 25, PEER_CNT_FLAG = 26;
constexpr size_t PEER_BUF_BYTES = 2ull * CH_MAX_PEERS * PEER_SLOT * 8;
struct PeerPush {
    unsigned long long *base[CH_MAX_PEERS]; // every rank's buffer, as mapped in this process
    int world, rank;                        // world == 0: no peer exchange
    unsigned long long epoch;               // step number (>= 1), bank = epoch & 1
    unsigned long long timeout_ns;          // K3's wait for a record (CH_PEER_TIMEOUT_MS, default 60 s)
    __device__ __forceinline__ unsigned long long *slot(int peer, int of) const
    {
        return base[peer] + ((size_t)(epoch & 1) * CH_MAX_PEERS + of) * PEER_SLOT;
    }
};
static_assert(sizeof(ch_extremes) == 24 * 8, "record = 24 words");

__device__ __forceinline__ void st_release_sys(unsigned long long *p, unsigned long long v)
{
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long *p)
{
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ unsigned long long globaltimer_ns()
{
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// Store one 24-word record into slot[rank] of every peer, then (after a
// system-scope fence) the epoch flag.  Called by every thread of one CTA;
// `rec` may be in shared or global memory.
__device__ void peer_push_record(const PeerPush &pp, const unsigned long long *rec)
{
    const int tid = threadIdx.x;
    for (int q = tid; q < 24 * pp.world; q += blockDim.x)
        pp.slot(q / 24, pp.rank)[q % 24] = rec[q % 24];
    __threadfence_system();
    __syncthreads();
    if (tid < pp.world)
        st_release_sys(pp.slot(tid, pp.rank) + PEER_REC_FLAG, pp.epoch);
}
// The survivor count into slot[rank] of every peer, then its flag.
__device__ void peer_push_count(const PeerPush &pp, long long count)
{
    for (int t = 0; t < pp.world; t++)
        pp.slot(t, pp.rank)[PEER_CNT] = (unsigned long long)count;
    __threadfence_system();
    for (int t = 0; t < pp.world; t++)
        st_release_sys(pp.slot(t, pp.rank) + PEER_CNT_FLAG, pp.epoch);
}

// ------------------------------------------------- TMA bulk copy + mbarrier --
__device__ __forceinline__ unsigned smem_u32(const void *p)
{
    return (unsigned)__cvta_generic_to_shared(p);
}
// One float from shared memory (volatile: not merged into an (x, y) pair
// load, so the value lands directly in its FFMA2 operand pair).
__device__ __forceinline__ float lds_f32(unsigned addr)
{
    float v;
    asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(addr));
    return v;
}
__device__ __forceinline__ void mbar_init(unsigned long long *bar, unsigned count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long *bar, unsigned bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long *bar)
{
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long *bar, unsigned parity)
{
    // try_wait with a suspend-time hint: the warp sleeps until the phase
    // completes (or the hint expires) instead of spinning on issue slots.
    unsigned ok = 0;
    while (true) {
#ifdef CH_NO_SUSPEND_HINT
        asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
                     " selp.u32 %0, 1, 0, p;\n}"
                     : "=r"(ok)
                     : "r"(smem_u32(bar)), "r"(parity)
                     : "memory");
#else
        asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n"
                     " selp.u32 %0, 1, 0, p;\n}"
                     : "=r"(ok)
                     : "r"(smem_u32(bar)), "r"(parity), "r"(1000000u)
                     : "memory");
#endif
        if (ok)
            break;
    }
}
// 1-D bulk copy global -> shared (TMA engine), completion counted on `bar`.
__device__ __forceinline__ void tma_load_1d(void *dst, const void *src, unsigned bytes, unsigned long long *bar)
{
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

// ===================================================================== K1 ==
// One pass over the points.  Each thread keeps running extremes (key, global
// index) for the 8 slots, walking indices downward.  Per point: 2 DADD (the
// x+y, x-y keys), 8 compares OR-ed into one predicate, and only if some key
// reaches its running best (rare after the first few chunks) a per-lane
// update with the exact (key, lowest index) rule.  Every K1_SHARE chunks the
// warp shares its best per slot (so thresholds tighten 32x).  Then warp
// shuffles, CTA partials, and an atomic ticket: the last CTA combines all
// partials (best key, then lowest index: order independent, R2) and builds
// the octagon.  Non-finite detection: acc += x*0 (exact 0 for finite x,
// NaN otherwise) via DFMA.
constexpr int K1_SHARE = 16;
struct Best {
    double v[8];
    long long i[8];
};

__device__ __forceinline__ void reduce_pair(int k, double &v, long long &i, double w, long long j);

__device__ __forceinline__ void k1_slow_update(Best &b, double x, double y, double s, double d, long long gi)
{
    const double key[8] = {x, s, y, d, x, s, y, d};
#pragma unroll
    for (int k = 0; k < 8; k++)
        reduce_pair(k, b.v[k], b.i[k], key[k], gi);
}

__device__ __forceinline__ void k1_update(Best &b, double x, double y, long long gi, double &acc)
{
    const double s = __dadd_rn(x, y);
    const double d = __dsub_rn(x, y);
    const bool t = (x >= b.v[0]) | (s >= b.v[1]) | (y >= b.v[2]) | (d <= b.v[3]) | (x <= b.v[4]) |
                   (s <= b.v[5]) | (y <= b.v[6]) | (d >= b.v[7]);
    if (t)
        k1_slow_update(b, x, y, s, d, gi);
    acc = __fma_rn(x, 0.0, acc);
    acc = __fma_rn(y, 0.0, acc);
}

// Float storage: the same filter on fp32 keys (no fp64 op on the fast path).
// x and y are floats, so x >= th[0] etc. are exact; s and d are compared as
// RN32 sums against the running fp64 best rounded outward (RD32 for a max
// slot, RU32 for a min slot): fl64(x + y) >= best implies fl32(x + y) >=
// RD32(best) (RN32 and RN64 are monotone and RD32(best) is a float <= best
// with no float in between), so every point the fp64 rule would consider
// still reaches k1_slow_update, which decides exactly as the fp64 path does.
__device__ __forceinline__ void k1_thresholds(const Best &b, float (&th)[8])
{
    th[0] = (float)b.v[0]; // x, y slots: floats (or +-inf) already
    th[1] = __double2float_rd(b.v[1]);
    th[2] = (float)b.v[2];
    th[3] = __double2float_ru(b.v[3]);
    th[4] = (float)b.v[4];
    th[5] = __double2float_ru(b.v[5]);
    th[6] = (float)b.v[6];
    th[7] = __double2float_rd(b.v[7]);
}
__device__ __forceinline__ void k1_update_f32(Best &b, float (&th)[8], float x, float y, long long gi, float &acc)
{
    const float s = __fadd_rn(x, y);
    const float d = __fsub_rn(x, y);
    const bool t = (x >= th[0]) | (s >= th[1]) | (y >= th[2]) | (d <= th[3]) | (x <= th[4]) | (s <= th[5]) |
                   (y <= th[6]) | (d >= th[7]);
    if (t) {
        const double xd = x, yd = y;
        k1_slow_update(b, xd, yd, __dadd_rn(xd, yd), __dsub_rn(xd, yd), gi);
        k1_thresholds(b, th);
    }
    acc = __fmaf_rn(x, 0.0f, acc);
    acc = __fmaf_rn(y, 0.0f, acc);
}

__device__ __forceinline__ void k1_warp_share(Best &b)
{
#pragma unroll
    for (int k = 0; k < 8; k++) {
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
            const double w = __shfl_xor_sync(FULL, b.v[k], off);
            const long long j = __shfl_xor_sync(FULL, b.i[k], off);
            reduce_pair(k, b.v[k], b.i[k], w, j);
        }
    }
}

__device__ __forceinline__ void reduce_pair(int k, double &v, long long &i, double w, long long j)
{
    if (chf::slot_better(k, w, j, v, i)) {
        v = w;
        i = j;
    }
}

// The same decision as reduce_pair (chf::slot_better: better key, else --
// equal or unordered -- the lower index), written as selects so that the
// eight keys' chains interleave (K5, K6).
template <int K>
__device__ __forceinline__ void reduce_pair_sel(double &v, long long &i, double w, long long j)
{
    const bool gt = chf::slot_is_max(K) ? (w > v) : (w < v);
    const bool lt = chf::slot_is_max(K) ? (w < v) : (w > v);
    const bool take = gt | (!lt & (j < i));
    v = take ? w : v;
    i = take ? j : i;
}
__device__ __forceinline__ void best_init(Best &b)
{
#pragma unroll
    for (int k = 0; k < 8; k++) {
        b.v[k] = chf::slot_is_max(k) ? -CH_INF : CH_INF;
        b.i[k] = LLONG_MAX;
    }
}
// One point into a thread's running extremes (points visited in increasing
// index order: equal keys keep the earlier, i.e. lower, index).
__device__ __forceinline__ void best_point(Best &b, double x, double y, long long gi)
{
    const double s = __dadd_rn(x, y), d = __dsub_rn(x, y);
    reduce_pair_sel<0>(b.v[0], b.i[0], x, gi);
    reduce_pair_sel<1>(b.v[1], b.i[1], s, gi);
    reduce_pair_sel<2>(b.v[2], b.i[2], y, gi);
    reduce_pair_sel<3>(b.v[3], b.i[3], d, gi);
    reduce_pair_sel<4>(b.v[4], b.i[4], x, gi);
    reduce_pair_sel<5>(b.v[5], b.i[5], s, gi);
    reduce_pair_sel<6>(b.v[6], b.i[6], y, gi);
    reduce_pair_sel<7>(b.v[7], b.i[7], d, gi);
}
// Max-oriented pairs (v, i): a min-slot key is carried negated (exact), so
// that one merge rule serves every key -- the larger value, else (equal or
// unordered) the lower index: chf::slot_better's decision on the original key.
__device__ __forceinline__ void max_merge(double &v, long long &i, double w, long long j)
{
    const bool take = (w > v) | (!(w < v) & (j < i));
    v = take ? w : v;
    i = take ? j : i;
}
__device__ __forceinline__ void max_xor(double &v, long long &i, int off)
{
    const double w = __shfl_xor_sync(FULL, v, off);
    const long long j = __shfl_xor_sync(FULL, i, off);
    max_merge(v, i, w, j);
}
// The key lane l holds after best_warp_rs: bits 4, 3, 2 of the lane.
__device__ __forceinline__ int rs_key(int lane) { return ((lane >> 4) & 1) * 4 + ((lane >> 3) & 1) * 2 + ((lane >> 2) & 1); }
// Reduce-scatter butterfly over the warp: each level a lane sends the half
// of its keys its partner keeps (16: four keys, 8: two, 4: one), then two
// plain levels; lane l ends with the warp's best for key rs_key(l)
// (max-oriented).  9 merges and 36 shuffles instead of 40 and 160.
__device__ __forceinline__ void best_warp_rs(const Best &b, double &ov, long long &oi)
{
    const int lane = threadIdx.x & 31;
    double v[8];
#pragma unroll
    for (int k = 0; k < 8; k++)
        v[k] = chf::slot_is_max(k) ? b.v[k] : -b.v[k];
    const bool h4 = lane & 16, h3 = lane & 8, h2 = lane & 4;
    double v4[4];
    long long i4[4];
#pragma unroll
    for (int j = 0; j < 4; j++) {
        v4[j] = h4 ? v[4 + j] : v[j];
        i4[j] = h4 ? b.i[4 + j] : b.i[j];
        const double w = __shfl_xor_sync(FULL, h4 ? v[j] : v[4 + j], 16);
        const long long jj = __shfl_xor_sync(FULL, h4 ? b.i[j] : b.i[4 + j], 16);
        max_merge(v4[j], i4[j], w, jj);
    }
    double v2[2];
    long long i2[2];
#pragma unroll
    for (int j = 0; j < 2; j++) {
        v2[j] = h3 ? v4[2 + j] : v4[j];
        i2[j] = h3 ? i4[2 + j] : i4[j];
        const double w = __shfl_xor_sync(FULL, h3 ? v4[j] : v4[2 + j], 8);
        const long long jj = __shfl_xor_sync(FULL, h3 ? i4[j] : i4[2 + j], 8);
        max_merge(v2[j], i2[j], w, jj);
    }
    ov = h2 ? v2[1] : v2[0];
    oi = h2 ? i2[1] : i2[0];
    {
        const double w = __shfl_xor_sync(FULL, h2 ? v2[0] : v2[1], 4);
        const long long jj = __shfl_xor_sync(FULL, h2 ? i2[0] : i2[1], 4);
        max_merge(ov, oi, w, jj);
    }
    max_xor(ov, oi, 2);
    max_xor(ov, oi, 1);
}
// Warp 0 combines R rows of 8 max-oriented pairs (s_v[r][k], s_i[r][k]):
// lane l takes key l & 7 of rows l >> 3, (l >> 3) + 4, ...; then two
// butterfly levels; lanes 0..7 end with key = lane.  Called by warp 0.
template <int R>
__device__ __forceinline__ void rows_combine(const double (*s_v)[8], const long long (*s_i)[8], double &ov,
                                             long long &oi)
{
    const int lane = threadIdx.x & 31, k = lane & 7;
    ov = -CH_INF;
    oi = LLONG_MAX;
#pragma unroll
    for (int r = lane >> 3; r < R; r += 4)
        max_merge(ov, oi, s_v[r][k], s_i[r][k]);
    max_xor(ov, oi, 8);
    max_xor(ov, oi, 16);
}

#ifdef CH_TRACE // developer build only (CH_NVCC_EXTRA=-DCH_TRACE): phase clocks of K5 / K6
__device__ long long g_trace[32];
#define CH_TR(k) do { if (threadIdx.x == 0 && blockIdx.x == 0) g_trace[k] = clock64(); } while (0)
#else
#define CH_TR(k) do { } while (0)
#endif

// chf::octagon_vertices on warp 0, lane k holding slot k: a slot is dropped
// iff it equals the previous SLOT (numeric ==; equal to the last kept vertex
// exactly when it equals the previous slot, == being transitive and a dropped
// slot equal to the kept one), and consecutive kept vertices differ, so at
// most one trailing vertex can equal the first.  Same fields as the serial
// function.  Called by the 32 lanes of one warp.
__device__ __forceinline__ void octagon_vertices_warp(const ch_extremes &e, int flags, ch_octagon &o /*shared*/)
{
    const int lane = threadIdx.x & 31;
    const int k = lane & 7;
    const double x = e.x[k], y = e.y[k];
    const double xp = __shfl_sync(FULL, x, (k + 7) & 7), yp = __shfl_sync(FULL, y, (k + 7) & 7);
    const bool keep = k == 0 || !(x == xp && y == yp);
    const unsigned mask = __ballot_sync(FULL, keep && lane < 8);
    const int nv0 = __popc(mask);
    const int last = 31 - __clz(mask);
    const double xl = __shfl_sync(FULL, x, last), yl = __shfl_sync(FULL, y, last);
    const double x0 = __shfl_sync(FULL, x, 0), y0 = __shfl_sync(FULL, y, 0);
    const int nv = nv0 - ((nv0 > 1 && xl == x0 && yl == y0) ? 1 : 0);
    const int degenerate = nv < 3;
    if (lane < 8) {
        const int pos = __popc(mask & ((1u << k) - 1u)); // kept vertices before slot k
        if (keep) { // (a dropped trailing vertex keeps its coordinates, index -1)
            o.vidx[pos] = pos < nv ? e.idx[k] : -1;
            o.vx[pos] = x;
            o.vy[pos] = y;
        }
        if (k >= nv0) {
            o.vidx[k] = -1;
            o.vx[k] = o.vy[k] = 0.0;
        }
        o.ex[k] = o.ey[k] = o.thr[k] = 0.0;
        o.f32_a[k] = o.f32_b[k] = o.f32_c[k] = o.f32_dk[k] = 0.0f;
        const int sv = __popc(mask & ((2u << k) - 1u)) - 1; // slot k's kept vertex
        o.guess_edge[k] = (!degenerate && sv < nv) ? sv : 0;
    }
    if (lane == 0) {
        o.nv = nv;
        o.degenerate = degenerate;
        o.has_box = 0;
        o.plain = (flags & CH_PLAIN) ? 1 : 0;
        o.exact = (!o.plain && (flags & CH_EXACT)) ? 1 : 0;
        o.has_f32 = 0;
        o.f32_delta = 0.0f;
        o.bbox[0] = e.x[4]; // xmin (L)
        o.bbox[1] = e.x[0]; // xmax (R)
        o.bbox[2] = e.y[6]; // ymin (B)
        o.bbox[3] = e.y[2]; // ymax (T)
        o.box[0] = CH_INF;
        o.box[1] = -CH_INF;
        o.box[2] = CH_INF;
        o.box[3] = -CH_INF;
        o.cx = __dmul_rn(0.5, __dadd_rn(o.bbox[0], o.bbox[1]));
        o.cy = __dmul_rn(0.5, __dadd_rn(o.bbox[2], o.bbox[3]));
    }
}

// The octagon (DESIGN R5, R4) built by a whole CTA from extremes in shared
// memory: warp 0 assembles the vertices (octagon_vertices_warp), one thread
// per edge computes ex, ey, T_k and the fp32 constants, one thread per (box
// candidate, edge, corner) validates the accept box, and warp 0 keeps the
// first candidate valid at every corner.  Same result as the serial
// chf::build_octagon (the host path).  Called by every thread of the CTA.
__device__ void build_octagon_cta(const ch_extremes &e, int flags, ch_octagon &o /*shared*/)
{
    __shared__ int s_bad[chf::BOX_CANDIDATES], s_cand[chf::BOX_CANDIDATES];
    __shared__ double s_box[chf::BOX_CANDIDATES][4];
    const int tid = threadIdx.x;
    if (tid < 32)
        octagon_vertices_warp(e, flags, o);
    if (tid < chf::BOX_CANDIDATES)
        s_bad[tid] = 0;
    __syncthreads();
    CH_TR(21);
    if (o.degenerate)
        return;
    // the edges (items BOX_CANDIDATES * 32 + k) and the box validation (one
    // item per candidate, edge and corner, recomputing its edge) side by side
    CH_TR(22);
    for (int q = tid; q < chf::BOX_CANDIDATES * 32 + 8; q += blockDim.x) {
        if (q >= chf::BOX_CANDIDATES * 32) {
            if (q - chf::BOX_CANDIDATES * 32 < o.nv)
                chf::octagon_edge(o, q - chf::BOX_CANDIDATES * 32);
            continue;
        }
        const int t = q >> 5, k = (q >> 2) & 7, corner = q & 3;
        double b[4];
        const bool cand = chf::box_candidate(e, t, b);
        if ((q & 31) == 0) { // one thread per candidate keeps it for the pick
            s_cand[t] = cand;
            s_box[t][0] = b[0];
            s_box[t][1] = b[1];
            s_box[t][2] = b[2];
            s_box[t][3] = b[3];
        }
        if (k < o.nv && (!cand || !chf::box_corner_ok_core(o, k, b, corner)))
            s_bad[t] = 1;
    }
    __syncthreads();
    CH_TR(23);
    if (tid < 32) { // the first candidate valid everywhere (lane t: candidate t)
        const bool ok = tid < chf::BOX_CANDIDATES && s_cand[tid] && !s_bad[tid];
        const unsigned okm = __ballot_sync(FULL, ok);
        if (okm && tid == __ffs(okm) - 1) {
            o.box[0] = s_box[tid][0];
            o.box[1] = s_box[tid][1];
            o.box[2] = s_box[tid][2];
            o.box[3] = s_box[tid][3];
            o.has_box = 1;
        }
    } else if (tid == 32) { // (another warp: runs alongside the pick)
        chf::octagon_f32_delta(o);
        o.has_f32 = chf::f32_domain_ok(o) ? 1 : 0;
    }
    __syncthreads();
    CH_TR(24);
}

template <typename T>
__device__ void k1_finalize(const T *__restrict__ xy, long long n, long long index_base, int flags,
                            WsHeader *hdr, const Partial *parts, int nparts, void *ext_out, const PeerPush &pp)
{
    // Called by every thread of the last CTA.
    __shared__ double s_v[K1_THREADS / 32][8];
    __shared__ long long s_i[K1_THREADS / 32][8];
    __shared__ int s_nf;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    double v[8];
    long long id[8];
    int nf = 0;
    for (int k = 0; k < 8; k++) {
        v[k] = chf::slot_is_max(k) ? -CH_INF : CH_INF;
        id[k] = LLONG_MAX;
    }
    for (int p = tid; p < nparts; p += K1_THREADS) {
        const Partial *q = parts + p;
        for (int k = 0; k < 8; k++)
            reduce_pair(k, v[k], id[k], __ldcg(&q->key[k]), __ldcg(&q->idx[k]));
        nf |= __ldcg(&q->nonfinite);
    }
    nf = __syncthreads_or(nf);
    for (int k = 0; k < 8; k++) {
        for (int off = 16; off > 0; off >>= 1) {
            double w = __shfl_xor_sync(FULL, v[k], off);
            long long j = __shfl_xor_sync(FULL, id[k], off);
            reduce_pair(k, v[k], id[k], w, j);
        }
        if (lane == 0) {
            s_v[warp][k] = v[k];
            s_i[warp][k] = id[k];
        }
    }
    if (tid == 0)
        s_nf = nf;
    __syncthreads();
    __shared__ ch_extremes s_e;
    __shared__ ch_octagon s_o;
    if (tid < 8) {
        const int k = tid;
        double bv = s_v[0][k];
        long long bi = s_i[0][k];
        for (int w = 1; w < K1_THREADS / 32; w++)
            reduce_pair(k, bv, bi, s_v[w][k], s_i[w][k]);
        // no finite candidate at all (every point NaN: the status will be
        // CH_ERR_NONFINITE): keep the sentinel, read nothing
        const long long loc = bi - index_base;
        const bool any = bi != LLONG_MAX;
        s_e.idx[k] = bi;
        s_e.x[k] = any ? (double)xy[2 * loc] : __longlong_as_double(0x7ff8000000000000LL);
        s_e.y[k] = any ? (double)xy[2 * loc + 1] : __longlong_as_double(0x7ff8000000000000LL);
    }
    __syncthreads();
    build_octagon_cta(s_e, flags, s_o);
    // publish (cooperative copies of the two structs)
    {
        const unsigned *src = (const unsigned *)&s_o;
        unsigned *dst = (unsigned *)&hdr->oct;
        for (int i = tid; i < (int)(sizeof(ch_octagon) / 4); i += K1_THREADS)
            dst[i] = src[i];
        const unsigned *se = (const unsigned *)&s_e;
        unsigned *de = (unsigned *)&hdr->ext;
        unsigned *dx = (unsigned *)ext_out;
        for (int i = tid; i < (int)(sizeof(ch_extremes) / 4); i += K1_THREADS) {
            de[i] = se[i];
            if (dx)
                dx[i] = se[i];
        }
    }
    if (tid == 0) {
        hdr->result.nonfinite = s_nf;
        hdr->result.degenerate = s_o.degenerate;
        hdr->peer_timeout = 0; // a new step
        set_tag(hdr, xy, n, index_base);
        hdr->k1_ticket = 0; // ready for the next call (stream order)
    }
    if (pp.world > 0) // a4 fused: this rank's record into every peer's buffer
        peer_push_record(pp, (const unsigned long long *)&s_e);
}

template <typename T, bool VEC>
__global__ void __launch_bounds__(K1_THREADS, PtTraits<T>::K1_MINB)
k1_extremes8(const T *__restrict__ xy, long long n, long long index_base, int flags,
             WsHeader *hdr, Partial *parts, void *ext_out, const PeerPush pp)
{
    constexpr int K1_UNROLL = PtTraits<T>::K1_UNROLL;
    constexpr long long K1_CHUNK = k1_chunk<T>();
    const int tid = threadIdx.x;
    Best b;
#pragma unroll
    for (int k = 0; k < 8; k++) {
        b.v[k] = chf::slot_is_max(k) ? -CH_INF : CH_INF;
        b.i[k] = LLONG_MAX;
    }
    double acc = 0.0;
    float accf = 0.0f;
    float th[8];
    k1_thresholds(b, th);
    const long long nchunks = (n + K1_CHUNK - 1) / K1_CHUNK;
    int it = 0;
    for (long long c = nchunks - 1 - blockIdx.x; c >= 0; c -= gridDim.x, it++) {
        const long long base = c * K1_CHUNK;
        const long long gbase = index_base + base + 2 * tid;
        if constexpr (sizeof(T) == 4) {
            constexpr int PPL = PtTraits<T>::K1_PPL;
            const long long gb = index_base + base + PPL * tid;
            if (base + K1_CHUNK <= n) {
                float v[K1_UNROLL][2 * PPL];
#pragma unroll
                for (int u = 0; u < K1_UNROLL; u++) {
                    const float *q = (const float *)xy + 2 * (base + PPL * ((long long)u * K1_THREADS + tid));
                    if constexpr (PPL == 4 && VEC) {
                        ld256f(q, *(float(*)[8]) & v[u][0]);
                    } else {
#pragma unroll
                        for (int h2 = 0; h2 < PPL / 2; h2++)
                            ld2raw<T, VEC>((const T *)q + 4 * h2, *(T(*)[4]) & v[u][4 * h2]);
                    }
                }
#pragma unroll
                for (int u = K1_UNROLL - 1; u >= 0; u--)
#pragma unroll
                    for (int h = PPL - 1; h >= 0; h--)
                        k1_update_f32(b, th, v[u][2 * h], v[u][2 * h + 1], gb + PPL * u * K1_THREADS + h, accf);
            } else {
                for (int u = K1_UNROLL - 1; u >= 0; u--) {
                    long long p = base + PPL * ((long long)u * K1_THREADS + tid);
                    for (int h = PPL - 1; h >= 0; h--) {
                        if (p + h < n) {
                            float x, y;
                            ld1raw(xy, p + h, x, y);
                            k1_update_f32(b, th, x, y, index_base + p + h, accf);
                        }
                    }
                }
            }
            if ((it & (K1_SHARE - 1)) == 0) {
                k1_warp_share(b);
                k1_thresholds(b, th);
            }
            continue;
        }
        if (base + K1_CHUNK <= n) {
            T v[K1_UNROLL][4];
#pragma unroll
            for (int u = 0; u < K1_UNROLL; u++)
                ld2raw<T, VEC>(xy + 2 * (base + 2 * ((long long)u * K1_THREADS + tid)), v[u]);
#pragma unroll
            for (int u = K1_UNROLL - 1; u >= 0; u--) {
                k1_update(b, (double)v[u][2], (double)v[u][3], gbase + 2 * u * K1_THREADS + 1, acc);
                k1_update(b, (double)v[u][0], (double)v[u][1], gbase + 2 * u * K1_THREADS, acc);
            }
        } else {
            for (int u = K1_UNROLL - 1; u >= 0; u--) {
                long long p = base + 2 * ((long long)u * K1_THREADS + tid);
                for (int h = 1; h >= 0; h--) {
                    if (p + h < n) {
                        double x, y;
                        ld1pt(xy, p + h, x, y);
                        k1_update(b, x, y, index_base + p + h, acc);
                    }
                }
            }
        }
        if ((it & (K1_SHARE - 1)) == 0)
            k1_warp_share(b); // uniform: every lane of the CTA runs the same iterations
    }
    // PDL: this CTA is done reading the points; K2 (launched with programmatic
    // stream serialization) may start its prologue and stream its first
    // sub-tiles while the reductions and the last CTA's octagon build finish
    // (K2's octagon readers wait with griddepcontrol.wait).
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    double v[8];
    long long id[8];
#pragma unroll
    for (int k = 0; k < 8; k++) {
        v[k] = b.v[k];
        id[k] = b.i[k];
    }
    __shared__ double s_v[K1_THREADS / 32][8];
    __shared__ long long s_i[K1_THREADS / 32][8];
    __shared__ bool s_last;
    const int lane = tid & 31, warp = tid >> 5;
#pragma unroll
    for (int k = 0; k < 8; k++) {
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
            double w = __shfl_xor_sync(FULL, v[k], off);
            long long j = __shfl_xor_sync(FULL, id[k], off);
            reduce_pair(k, v[k], id[k], w, j);
        }
        if (lane == 0) {
            s_v[warp][k] = v[k];
            s_i[warp][k] = id[k];
        }
    }
    int nf = __syncthreads_or(acc != acc || accf != accf);
    if (tid < 8) {
        const int k = tid;
        double bv = s_v[0][k];
        long long bi = s_i[0][k];
        for (int w = 1; w < K1_THREADS / 32; w++)
            reduce_pair(k, bv, bi, s_v[w][k], s_i[w][k]);
        parts[blockIdx.x].key[k] = bv;
        parts[blockIdx.x].idx[k] = bi;
        if (k == 0)
            parts[blockIdx.x].nonfinite = nf;
        __threadfence();
    }
    __syncthreads();
    if (tid == 0) {
        __threadfence();
        unsigned t = atomicAdd(&hdr->k1_ticket, 1u);
        s_last = (t == gridDim.x - 1);
    }
    __syncthreads();
    if (s_last) {
        __threadfence();
        k1_finalize(xy, n, index_base, flags, hdr, parts, gridDim.x, ext_out, pp);
    }
}

// ===================================================================== K3 ==
// The combine of a4, by one CTA: W per-rank records (max key, tie -> min
// global index; empty shards have idx -1) -> the global extremes and octagon
// in the workspace header, bit-identical to the 1-GPU K1.
__device__ void combine_records(const ch_extremes *all, int world, int flags, WsHeader *hdr)
{
    __shared__ ch_extremes s_e;
    __shared__ ch_octagon s_o;
    __shared__ double s_lb[4]; // the bbox of the octagon K1 built from this rank's shard
    const int tid = threadIdx.x;
    if (tid < 4)
        s_lb[tid] = hdr->oct.bbox[tid];
    if (tid < 8) {
        const int k = tid;
        double bv = chf::slot_is_max(k) ? -CH_INF : CH_INF;
        long long bi = LLONG_MAX;
        double bx = 0.0, by = 0.0;
        for (int r = 0; r < world; r++) {
            const long long i = all[r].idx[k];
            if (i < 0)
                continue; // empty shard
            const double x = all[r].x[k], y = all[r].y[k];
            const double key = chf::slot_key(k, x, y);
            if (chf::slot_better(k, key, i, bv, bi)) {
                bv = key;
                bi = i;
                bx = x;
                by = y;
            }
        }
        s_e.idx[k] = bi;
        s_e.x[k] = bx;
        s_e.y[k] = by;
    }
    __syncthreads();
    build_octagon_cta(s_e, flags, s_o);
    __syncthreads(); // s_lb read before the header is overwritten
    const unsigned *src = (const unsigned *)&s_o;
    unsigned *dst = (unsigned *)&hdr->oct;
    for (int i = tid; i < (int)(sizeof(ch_octagon) / 4); i += blockDim.x)
        dst[i] = src[i];
    const unsigned *se = (const unsigned *)&s_e;
    unsigned *de = (unsigned *)&hdr->ext;
    for (int i = tid; i < (int)(sizeof(ch_extremes) / 4); i += blockDim.x)
        de[i] = se[i];
    if (tid == 0) {
        hdr->result.degenerate = s_o.degenerate;
        // the shard's points lie in its own bbox; the fp32 certificates stay
        // valid for them iff that bbox lies in the combined one
        const bool inside = s_lb[0] >= s_o.bbox[0] && s_lb[1] <= s_o.bbox[1] && s_lb[2] >= s_o.bbox[2] &&
                            s_lb[3] <= s_o.bbox[3];
        if (!inside)
            hdr->tag_valid = 0;
    }
}

__global__ void __launch_bounds__(256) k3_combine8(const ch_extremes *__restrict__ all, int world, int flags,
                                                   WsHeader *hdr)
{
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); // K2's producer may start (PDL)
    if (threadIdx.x == 0)
        hdr->peer_timeout = 0;
    combine_records(all, world, flags, hdr);
}

// K3 of the fused exchange: acquire the W epoch flags of this rank's own
// exchange buffer (the peers' K1s store their records there), then combine.
// A wait longer than pp.timeout_ns (60 s unless CH_PEER_TIMEOUT_MS) sets
// hdr->peer_timeout (CH_ERR_PEER) and combines the records that arrived,
// the late ones as empty shards, rather than hanging.  Every K3 rewrites
// peer_timeout, so a late record fails only its own step.
__global__ void __launch_bounds__(256) k3_combine8_peer(const PeerPush pp, int flags, WsHeader *hdr)
{
    __shared__ ch_extremes s_all[CH_MAX_PEERS];
    __shared__ int s_late;
    const int tid = threadIdx.x;
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); // K2's producer streams while we wait (PDL)
    if (tid == 0)
        s_late = 0;
    __syncthreads();
    if (tid < pp.world) {
        const unsigned long long *slot = pp.slot(pp.rank, tid); // own buffer, sender tid
        const unsigned long long t0 = globaltimer_ns();
        while (ld_acquire_sys(slot + PEER_REC_FLAG) != pp.epoch) {
            if (globaltimer_ns() - t0 > pp.timeout_ns) {
                s_late = 1;
                break;
            }
            __nanosleep(100);
        }
        unsigned long long *dst = (unsigned long long *)&s_all[tid];
        const bool late = ld_acquire_sys(slot + PEER_REC_FLAG) != pp.epoch;
        // a record that did not arrive counts as an empty shard (idx -1): the
        // octagon is then built from input points of the other shards only
        // (still hull-safe), and the step reports CH_ERR_PEER
        for (int w = 0; w < 24; w++)
            dst[w] = late ? (w < 8 ? ~0ull : 0ull) : *(const volatile unsigned long long *)(slot + w);
    }
    __syncthreads();
    if (tid == 0)
        hdr->peer_timeout = s_late;
    combine_records(s_all, pp.world, flags, hdr);
}

// An empty shard's part of the exchange: its empty record (what = 0) or its
// zero count (what = 1).
__global__ void k_peer_push(const PeerPush pp, int what)
{
    if (what == 0) {
        __shared__ unsigned long long rec[24];
        if (threadIdx.x < 24)
            rec[threadIdx.x] = threadIdx.x < 8 ? ~0ull : 0ull; // idx = -1, x = y = 0
        __syncthreads();
        peer_push_record(pp, rec);
    } else if (threadIdx.x == 0) {
        peer_push_count(pp, 0);
    }
}

// ========================================================= octagon test ==
struct __align__(16) SEdge { // 48 B: lanes indexing different edges hit distinct banks
    double ax, ay, ex, ey, thr, pad;
};
struct SOct {
    SEdge e[8];
    float4 fab[8]; // {a, a, b, b}: edge k's (scaled) fp32 coefficients as FFMA2 operand pairs
    float2 fc[8];  // {c, c}; edges k >= nv: a = b = 0, c = 2^100 (never the minimum)
    unsigned long long fdelta; // {f32_delta, f32_delta}
    unsigned long long nbx0, bx1, nby0, by1; // float storage, as f32x2 pairs: (-boxf[0], -boxf[0]), (boxf[1], boxf[1]), ...
    double box[4];
    float boxf[4]; // float bounds with x >= boxf[0] <=> (double)x >= box[0], etc.
    double cx, cy;
    int nv, degenerate, has_f32, exact;
    int guess[8];
};

// f32_ok: the points being tested are the ones the octagon was built from
// (the data tag), so the fp32 certificates' bbox assumption holds.
__device__ __forceinline__ void load_soct(SOct &s, const ch_octagon *__restrict__ o, bool f32_ok = true)
{
    const int t = threadIdx.x;
    if (t < 8) {
        s.e[t].ax = o->vx[t];
        s.e[t].ay = o->vy[t];
        s.e[t].ex = o->ex[t];
        s.e[t].ey = o->ey[t];
        s.e[t].thr = o->thr[t];
        s.e[t].pad = 0.0;
        s.guess[t] = o->guess_edge[t];
        const bool used = t < o->nv;
        const float a = used ? o->f32_a[t] : 0.0f, b = used ? o->f32_b[t] : 0.0f;
        const float c = used ? o->f32_c[t] : 0x1p100f;
        s.fab[t] = make_float4(a, a, b, b);
        s.fc[t] = make_float2(c, c);
    } else if (t < 12) { // one float bound of the accept box each (threads 8..11)
        const int j = t - 8;
        const double bj = o->box[j];
        const float f = (j & 1) ? chf::f32_down(bj) : chf::f32_up(bj);
        s.box[j] = bj;
        s.boxf[j] = f;
        const float g = (j & 1) ? f : -f; // the x0 / y0 bounds are stored negated
        const unsigned long long d = ((unsigned long long)__float_as_uint(g) << 32) | __float_as_uint(g);
        if (j == 0)
            s.nbx0 = d;
        else if (j == 1)
            s.bx1 = d;
        else if (j == 2)
            s.nby0 = d;
        else
            s.by1 = d;
    } else if (t == 12) {
        s.cx = o->cx;
        s.cy = o->cy;
        s.nv = o->nv;
        s.degenerate = o->degenerate;
        s.has_f32 = f32_ok ? o->has_f32 : 0;
        s.exact = o->exact;
        s.fdelta = ((unsigned long long)__float_as_uint(o->f32_delta) << 32) | __float_as_uint(o->f32_delta);
    }
}

// The exact expansion stage, out of line: it is cold (exact mode, points
// within a few ulps of an edge), and inlining it into the unrolled loops
// made most of K2's code.
__device__ __noinline__ int exact_stage(double ax, double ay, double bx, double by, double x, double y)
{
    return chf::orient_sign_exact_stage(ax, ay, bx, by, x, y);
}

// One edge in fp64: true if the point is certainly "inside" for this edge.
// Certified / plain modes: D_k > T_k (the definition, R4).  Exact mode (f3):
// the exact orientation is > 0 -- decided by Shewchuk's per-point bound
// (3 + 16 eps) eps (|l| + |r|) on the same D_k, else by exact expansion
// arithmetic (chf::orient_sign_exact_stage).
__device__ __forceinline__ bool edge_inside(const SOct &s, int k, int exact, double x, double y)
{
    const SEdge &e = s.e[k];
    const double dy = __dsub_rn(y, e.ay), dx = __dsub_rn(x, e.ax);
    const double l = __dmul_rn(e.ex, dy), r = __dmul_rn(e.ey, dx);
    const double D = __dsub_rn(l, r);
    if (!exact)
        return D > e.thr;
    const double sum = __dadd_rn(fabs(l), fabs(r));
    const double eb = __dmul_rn((3.0 + 16.0 * 0x1p-53) * 0x1p-53, sum);
    if (sum >= 0x1p-900) { // (below: the products may have underflowed; exact_stage scales)
        if (D > eb)
            return true;
        if (-D > eb)
            return false;
    }
    const int k1 = k + 1 < s.nv ? k + 1 : 0; // the edge's end point: the next vertex
    return exact_stage(e.ax, e.ay, s.e[k1].ax, s.e[k1].ay, x, y) > 0;
}

// Survivor test, bit-identical to "not (forall k: D_k > T_k)" (R4): the
// accept box and the edge order are shortcuts that cannot change the result
// (box: proof at chf::box_corner_ok; order: a conjunction is order-free).
__device__ __forceinline__ bool keep_point(const SOct &s, double x, double y)
{
    if (x >= s.box[0] && x <= s.box[1] && y >= s.box[2] && y <= s.box[3])
        return false;
    const int nv = s.nv;
    double dx = __dsub_rn(x, s.cx), dy = __dsub_rn(y, s.cy);
    bool c = fabs(dx) >= fabs(dy);
    int oct = dy >= 0.0 ? (dx >= 0.0 ? (c ? 0 : 1) : (c ? 3 : 2))
                        : (dx < 0.0 ? (c ? 4 : 5) : (c ? 7 : 6));
    int g = s.guess[oct];
    for (int t = 0; t < nv; t++) {
        int off = (t & 1) ? ((t + 1) >> 1) : -(t >> 1);
        int k = g + off;
        k = k < 0 ? k + nv : (k >= nv ? k - nv : k);
        if (!edge_inside(s, k, s.exact, x, y))
            return true;
    }
    return false;
}

// Survivor mask for NP points of one thread (bit i = point i), bit-identical
// to "not (forall k: D_k > T_k)" for every valid point (R4), without the
// fp32 certificates: K5 and K6 (the small-input steps), and K2's path for
// caller-supplied octagons, degenerate or out-of-domain ones, and the
// partial last sub-tile (full sub-tiles of octagons built from the data take
// consume_cert).  Stages, each skipped
// when no lane of the warp needs it (warp-uniform branches):
//  1. the certified accept box (4 DSETP): inside => discarded (proof at
//     chf::box_corner_ok);
//  2. adaptively, the octant-guessed edge in fp64 (D_g <= T_g => kept, the
//     oracle's exists-k condition; a warp whose points it did not settle
//     skips it for the next 15 sub-tiles);
//  3. fp64 D_k on every edge for every undecided point.
template <typename C, int NP>
__device__ __forceinline__ unsigned classify(const SOct &s, const C (&px)[NP], const C (&py)[NP],
                                             unsigned valid, int &guess_mode, int np = NP)
{
    // np (warp-uniform): only points [0, np) can be valid; the rest are skipped
    static_assert(NP <= 32, "one mask bit per point");
    unsigned und = 0;
#pragma unroll
    for (int i = 0; i < NP; i++) {
        bool inbox;
        if constexpr (sizeof(C) == 4) // float storage: the same test on float bounds
            inbox = px[i] >= s.boxf[0] && px[i] <= s.boxf[1] && py[i] >= s.boxf[2] && py[i] <= s.boxf[3];
        else
            inbox = px[i] >= s.box[0] && px[i] <= s.box[1] && py[i] >= s.box[2] && py[i] <= s.box[3];
        und |= (inbox ? 0u : 1u) << i;
    }
    und &= valid;
    if (!__any_sync(FULL, und))
        return 0u;
    const int nv = s.nv;
    unsigned keep = 0;
    if (guess_mode <= 0) {
        // 2'. the guessed edge of the point's octant: D_g <= T_g => kept
#pragma unroll
        for (int i = 0; i < NP; i++) {
            if (i >= np)
                break;
            double dx = __dsub_rn((double)px[i], s.cx), dy = __dsub_rn((double)py[i], s.cy);
            bool c = fabs(dx) >= fabs(dy);
            int oct = dy >= 0.0 ? (dx >= 0.0 ? (c ? 0 : 1) : (c ? 3 : 2))
                                : (dx < 0.0 ? (c ? 4 : 5) : (c ? 7 : 6));
            const SEdge &e = s.e[s.guess[oct]];
            double D = chf::edge_det(e.ax, e.ay, e.ex, e.ey, (double)px[i], (double)py[i]);
            // exact mode: only D < -T_k proves the exact orientation negative
            keep |= ((s.exact ? D < -e.thr : !(D > e.thr)) ? 1u : 0u) << i;
        }
        keep &= und;
        und &= ~keep;
        if (!__any_sync(FULL, und))
            return keep;
        guess_mode = 16; // the next stage was needed anyway: skip 2' for a while
    }
    guess_mode--;
    unsigned disc = und;
    if (!s.exact) {
        for (int k = 0; k < nv; k++) {
            const double ax = s.e[k].ax, ay = s.e[k].ay, ex = s.e[k].ex, ey = s.e[k].ey, thr = s.e[k].thr;
#pragma unroll
            for (int i = 0; i < NP; i++) {
                if (i >= np)
                    break;
                double D = chf::edge_det(ax, ay, ex, ey, (double)px[i], (double)py[i]);
                disc &= ~((D > thr ? 0u : 1u) << i);
            }
        }
    } else {
        for (int k = 0; k < nv; k++) {
#pragma unroll
            for (int i = 0; i < NP; i++)
                if ((disc >> i) & 1u)
                    disc &= ~((edge_inside(s, k, 1, (double)px[i], (double)py[i]) ? 0u : 1u) << i);
        }
    }
    return keep | (und & ~disc);
}

// Two fp32 lanes in one 64-bit register pair (low word = first point): the
// operand form of the sm_100 paired FP32 instructions.  Keeping the pairs as
// b64 values makes the register allocator hold each pair once instead of
// re-packing it for every FFMA2.
typedef unsigned long long f32x2;
__device__ __forceinline__ f32x2 pk2(float lo, float hi)
{
    f32x2 r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
    return r;
}
__device__ __forceinline__ f32x2 ffma2(f32x2 a, f32x2 b, f32x2 c) // each half: one RN fma
{
    f32x2 d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
    return d;
}
__device__ __forceinline__ f32x2 fmul2(f32x2 a, f32x2 b)
{
    f32x2 d;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}
__device__ __forceinline__ f32x2 fadd2(f32x2 a, f32x2 b)
{
    f32x2 d;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}

__device__ __forceinline__ void unpk2(f32x2 v, float &lo, float &hi)
{
    asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
}
__device__ __forceinline__ float fmin3(float a, float b, float c) // FMNMX3 (sm_100)
{
    float d;
    asm("min.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
    return d;
}
__device__ __forceinline__ bool sign_lo(f32x2 v) { return (int)(unsigned)v < 0; }
__device__ __forceinline__ bool sign_hi(f32x2 v) { return (int)(unsigned)(v >> 32) < 0; }

// G = min over the 8 edge slots of the certificate values v_k =
// fma(a_k, x, fma(b_k, y, c_k)) (scaled edges, chf::octagon_edge), two
// points per FFMA2 and two edges per FMNMX3; the unused slots (k >= nv) give
// 2^100.  glo / ghi: G of points 2q and 2q + 1.
template <int NQ>
__device__ __forceinline__ void cert_min(const SOct &s, const f32x2 (&X)[NQ], const f32x2 (&Y)[NQ],
                                         float (&glo)[NQ], float (&ghi)[NQ])
{
#pragma unroll
    for (int k = 0; k < 8; k += 2) {
        const f32x2 *e0 = (const f32x2 *)&s.fab[k], *e1 = (const f32x2 *)&s.fab[k + 1];
        const f32x2 a0 = e0[0], b0 = e0[1], a1 = e1[0], b1 = e1[1];
        const f32x2 c0 = *(const f32x2 *)&s.fc[k], c1 = *(const f32x2 *)&s.fc[k + 1];
#pragma unroll
        for (int q = 0; q < NQ; q++) {
            float l0, h0, l1, h1;
            unpk2(ffma2(a0, X[q], ffma2(b0, Y[q], c0)), l0, h0);
            unpk2(ffma2(a1, X[q], ffma2(b1, Y[q], c1)), l1, h1);
            if (k == 0) {
                glo[q] = fminf(l0, l1);
                ghi[q] = fminf(h0, h1);
            } else {
                glo[q] = fmin3(glo[q], l0, l1);
                ghi[q] = fmin3(ghi[q], h0, h1);
            }
        }
    }
}

// The min-certificate (chf::octagon_edge) on points held
// in registers (K5, K6): slots [0, np) of this thread (np warp-uniform),
// `valid` the slots holding a point.  Survivor mask, bit-identical to
// "not (forall k: D_k > T_k)" (R4): G >= +0 discards, G + f32_delta < 0
// keeps, the rest (the ~1e-7 band) is decided in fp64 on every edge.
template <int NP>
__device__ __forceinline__ unsigned cert_classify(const SOct &s, const double (&px)[NP], const double (&py)[NP],
                                                  unsigned valid, int np)
{
    static_assert(NP % 2 == 0, "point pairs");
    constexpr int HQ = NP / 2;
    f32x2 X[HQ], Y[HQ];
    float glo[HQ], ghi[HQ];
#pragma unroll
    for (int q = 0; q < HQ; q++) {
        X[q] = pk2((float)px[2 * q], (float)px[2 * q + 1]);
        Y[q] = pk2((float)py[2 * q], (float)py[2 * q + 1]);
        glo[q] = ghi[q] = 0.0f;
    }
#pragma unroll
    for (int k = 0; k < 8; k += 2) {
        const f32x2 *e0 = (const f32x2 *)&s.fab[k], *e1 = (const f32x2 *)&s.fab[k + 1];
        const f32x2 a0 = e0[0], b0 = e0[1], a1 = e1[0], b1 = e1[1];
        const f32x2 c0 = *(const f32x2 *)&s.fc[k], c1 = *(const f32x2 *)&s.fc[k + 1];
#pragma unroll
        for (int q = 0; q < HQ; q++) {
            if (2 * q >= np)
                break;
            float l0, h0, l1, h1;
            unpk2(ffma2(a0, X[q], ffma2(b0, Y[q], c0)), l0, h0);
            unpk2(ffma2(a1, X[q], ffma2(b1, Y[q], c1)), l1, h1);
            if (k == 0) {
                glo[q] = fminf(l0, l1);
                ghi[q] = fminf(h0, h1);
            } else {
                glo[q] = fmin3(glo[q], l0, l1);
                ghi[q] = fmin3(ghi[q], h0, h1);
            }
        }
    }
    float dl, dh;
    unpk2(s.fdelta, dl, dh);
    unsigned keep = 0, band = 0;
#pragma unroll
    for (int i = 0; i < NP; i++) {
        const float G = (i & 1) ? ghi[i / 2] : glo[i / 2];
        const bool neg = (int)__float_as_uint(G) < 0;                    // not certified inside
        const bool kc = (int)__float_as_uint(__fadd_rn(G, dl)) < 0;     // certified kept
        keep |= (kc ? 1u : 0u) << i;
        band |= (neg && !kc ? 1u : 0u) << i;
    }
    keep &= valid;
    band &= valid;
    if (__any_sync(FULL, band)) {
#pragma unroll
        for (int i = 0; i < NP; i++) {
            if ((band >> i) & 1u) {
                bool kf = false;
                for (int k = 0; k < s.nv && !kf; k++)
                    kf = !edge_inside(s, k, s.exact, px[i], py[i]);
                keep |= (kf ? 1u : 0u) << i;
            }
        }
    }
    return keep;
}

// One full sub-tile of a consumer warp for has_f32 octagons, read straight
// from the TMA stage (held until the caller releases it).  Writes, for each
// point slot u, the warp ballot of "point u of this lane survives" to
// mw[u] (lane 0; the warp's slots are contiguous, 16-byte aligned), bit-identical to "not (forall k: D_k > T_k)"
// (R4).  Every stage is a certificate proven on its own (box:
// chf::box_corner_ok; fp32: chf::octagon_edge), so the order cannot change a
// result.  Per-point state is a sign bit; the warp-uniform skips are one
// vote per pass:
//  1. the accept box: inside => discarded.  A pass whose points are all
//     inside is done (normal data);
//  2. G = min_k v_k over the scaled edges: G >= +0 => discarded (inside
//     every edge), G + f32_delta < 0 => kept (outside some edge);
//  3. fp64 D_k on every edge for the points in neither (the ~1e-7 band), the
//     coordinates re-read from the stage.
template <typename T, int NP, bool USE_BOX>
__device__ __forceinline__ void consume_cert(const SOct &s, const typename PtTraits<T>::V2 *sp, unsigned *mw,
                                             int &box_mode)
{
    constexpr int H = CH_CERT_H < NP ? CH_CERT_H : NP; // points per pass (register budget)
    constexpr int HQ = H / 2;
    static_assert(H % 4 == 0 && NP % H == 0, "passes of whole 16-byte ballot stores");
    constexpr f32x2 SIGN2 = 0x8000000080000000ull;
    const int tid = threadIdx.x;
    const bool lane0 = (tid & 31) == 0;
#pragma unroll
    for (int h0 = 0; h0 < NP; h0 += H) {
        f32x2 X[HQ], Y[HQ]; // x (resp. y) of points (2q, 2q + 1) of the pass
        f32x2 ob[HQ];       // sign bits: outside the accept box
        f32x2 anyout = 0;
        constexpr bool use_box = USE_BOX;
        // Outside the accept box <=> a sign bit among x - x0, x1 - x, y - y0,
        // y1 - y: an RNE difference has the sign of the exact one and is +0
        // when equal (the same decision as x >= x0 && ... on finite input).
        if constexpr (sizeof(T) == 8) {
#pragma unroll
            for (int q = 0; q < HQ; q++) {
                float fx[2], fy[2];
                unsigned o[2];
#pragma unroll
                for (int h = 0; h < 2; h++) {
                    const double2 v = sp[(h0 + 2 * q + h) * K2_CTHREADS + tid];
                    if (use_box) {
                        const double t0 = __dsub_rn(v.x, s.box[0]), t1 = __dsub_rn(s.box[1], v.x);
                        const double t2 = __dsub_rn(v.y, s.box[2]), t3 = __dsub_rn(s.box[3], v.y);
                        o[h] = (__double2hiint(t0) | __double2hiint(t1) | __double2hiint(t2) |
                                __double2hiint(t3)) & 0x80000000u;
                    } else {
                        o[h] = 0x80000000u;
                    }
                    fx[h] = (float)v.x;
                    fy[h] = (float)v.y;
                }
                X[q] = pk2(fx[0], fx[1]);
                Y[q] = pk2(fy[0], fy[1]);
                ob[q] = ((f32x2)o[1] << 32) | o[0];
                anyout |= ob[q];
            }
        } else {
            // float storage: each float loaded straight into its pair half;
            // the box on the pairs (exact for floats)
            const unsigned sa = smem_u32(sp) + 8u * tid;
            const f32x2 m1 = pk2(-1.f, -1.f), ONE2 = pk2(1.f, 1.f);
#pragma unroll
            for (int q = 0; q < HQ; q++) {
                const unsigned a0 = sa + 8u * (h0 + 2 * q) * K2_CTHREADS, a1 = a0 + 8u * K2_CTHREADS;
                // (x 1.0: exact; makes each pair one FMUL2 result, which the
                // register allocator then keeps whole)
                X[q] = fmul2(pk2(lds_f32(a0), lds_f32(a1)), ONE2);
                Y[q] = fmul2(pk2(lds_f32(a0 + 4), lds_f32(a1 + 4)), ONE2);
                if (use_box)
                    ob[q] = (fadd2(X[q], s.nbx0) | ffma2(m1, X[q], s.bx1) | fadd2(Y[q], s.nby0) |
                             ffma2(m1, Y[q], s.by1)) & SIGN2;
                else
                    ob[q] = SIGN2;
                anyout |= ob[q];
            }
        }
        if (use_box) {
            const int nout = __popc(__ballot_sync(FULL, anyout != 0ull));
            if (nout >= 8)
                box_mode = 64;
            if (nout == 0) {
#pragma unroll
                for (int i = 0; i < H; i += 4)
                    if (lane0)
                        *(uint4 *)&mw[h0 + i] = make_uint4(0u, 0u, 0u, 0u);
                continue;
            }
        }
        float glo[HQ], ghi[HQ];
        cert_min<HQ>(s, X, Y, glo, ghi);
        if constexpr (!USE_BOX) { // every point certified inside (G >= +0): all discarded
            unsigned neg = 0;
#pragma unroll
            for (int q = 0; q < HQ; q++)
                neg |= __float_as_uint(glo[q]) | __float_as_uint(ghi[q]);
            if (!__any_sync(FULL, (int)neg < 0)) {
#pragma unroll
                for (int i = 0; i < H; i += 4)
                    if (lane0)
                        *(uint4 *)&mw[h0 + i] = make_uint4(0u, 0u, 0u, 0u);
                continue;
            }
        }
        f32x2 keep[HQ], band = 0;
#pragma unroll
        for (int q = 0; q < HQ; q++) {
            const f32x2 G = pk2(glo[q], ghi[q]);
            const f32x2 t = fadd2(G, s.fdelta); // sign: G + delta < 0, certified kept
            keep[q] = ob[q] & t & SIGN2;
            ob[q] &= ~t & G & SIGN2; // the band: outside the box, neither certificate
            band |= ob[q];
        }
        if (__any_sync(FULL, band != 0ull)) {
            // 3. fp64 on every edge for the band points (rare)
#pragma unroll
            for (int i = 0; i < H; i++) {
                if ((i & 1) ? sign_hi(ob[i / 2]) : sign_lo(ob[i / 2])) {
                    double x, y;
                    if constexpr (sizeof(T) == 8) {
                        // re-read (volatile: the doubles must not stay live across the pass)
                        const volatile double *vp = (const volatile double *)(sp + (h0 + i) * K2_CTHREADS + tid);
                        x = vp[0];
                        y = vp[1];
                    } else {
                        const auto v = sp[(h0 + i) * K2_CTHREADS + tid];
                        x = v.x;
                        y = v.y;
                    }
                    bool kf = false;
                    for (int k = 0; k < s.nv && !kf; k++)
                        kf = !edge_inside(s, k, s.exact, x, y);
                    if (kf)
                        keep[i / 2] |= (i & 1) ? 0x8000000000000000ull : 0x80000000ull;
                }
            }
        }
#pragma unroll
        for (int i = 0; i < H; i += 4) { // four ballots, one 16-byte store (this warp's slots are contiguous)
            const unsigned m0 = __ballot_sync(FULL, sign_lo(keep[i / 2]));
            const unsigned m1 = __ballot_sync(FULL, sign_hi(keep[i / 2]));
            const unsigned m2 = __ballot_sync(FULL, sign_lo(keep[i / 2 + 1]));
            const unsigned m3 = __ballot_sync(FULL, sign_hi(keep[i / 2 + 1]));
            if (lane0)
                *(uint4 *)&mw[h0 + i] = make_uint4(m0, m1, m2, m3);
        }
    }
}

// Survivor stores of one 32-point group: lane l stores v (its point's global
// index) at pb[c + rank of l among the group's survivors] if bit l of the
// group's ballot m is set -- one predicated, coalesced warp store (m is
// warp-uniform, the bit test is per lane).
__device__ __forceinline__ void store_group(long long *pb, unsigned m, int c, long long v, unsigned lb, unsigned lt)
{
    long long *p = pb + (c + __popc(m & lt));
    asm volatile("{\n .reg .pred q;\n setp.ne.u32 q, %0, 0;\n @q st.global.s64 [%1], %2;\n}" ::"r"(m & lb), "l"(p),
                 "l"(v)
                 : "memory");
}

// The same with the index given as (lo, hi) 32-bit words (little endian).
__device__ __forceinline__ void store_group32(long long *pb, unsigned m, int c, unsigned lo, unsigned hi, unsigned lb,
                                              unsigned lt)
{
    long long *p = pb + (c + __popc(m & lt));
    asm volatile("{\n .reg .pred q;\n setp.ne.u32 q, %0, 0;\n @q st.global.v2.u32 [%1], {%2, %3};\n}" ::"r"(m & lb),
                 "l"(p), "r"(lo), "r"(hi)
                 : "memory");
}

// ===================================================================== K2 ==
// Persistent, warp-specialized CTAs: 8 consumer warps, 1 publisher warp and
// 1 TMA producer warp.  The producer claims "super-tiles" of `subs` x K2_SUB
// consecutive points with one atomic each (in increasing order, one claim
// ahead) and streams them as 32 KB sub-tiles through a K2_STAGES-deep ring
// in shared memory (cp.async.bulk + full/empty mbarriers), so loads stay in
// flight while the consumers compute.  Consumer thread t tests points
// u * 256 + t (u < K2_NP) of each sub-tile j; the results are ballot-ed per
// (sub-tile, u, warp) -- 32 consecutive points, group e = (j * K2_NP + u) *
// 8 + warp, so e order is index order -- into one of two shared-memory
// buffers.  At the end of a super-tile the consumers block-scan the group
// popcounts and publish the super-tile's aggregate (flag A) at once; the
// publisher warp then runs ONE decoupled look-back (Merrill & Garland) for
// it and publishes the inclusive prefix (flag P), while the consumers stream
// the next super-tile into the other buffer.  When a buffer comes round
// again, each consumer warp writes its own groups' survivors (int64 global
// indices, in index order) with predicated coalesced stores.  Claims are
// made in increasing order by running CTAs, so every predecessor of a
// claimed super-tile is owned by a running CTA: the look-back always makes
// progress.  Hand-offs use named barriers (bar.arrive / bar.sync):
// K2_BAR_BASE + b: consumers arrive, publisher syncs (buffer b full);
// K2_BAR_BASE + 2 + b: publisher arrives, consumers sync (buffer b's offset
// known); K2_BAR_BASE + 4: consumers only; K2_BAR_BASE + 5: consumers and
// publisher, once (the octagon is loaded).
constexpr unsigned TILE_DONE = 0xffffffffu;

__device__ __forceinline__ void bar_sync(int id, int nthreads)
{
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}
__device__ __forceinline__ void bar_arrive(int id, int nthreads)
{
    asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

template <typename T>
__global__ void __launch_bounds__(K2_THREADS, CH_K2_MINB)
k2_filter_compact(const T *__restrict__ xy, long long n, long long index_base,
                  const ch_octagon *__restrict__ oct, WsHeader *hdr,
                  unsigned long long *status, long long *__restrict__ out,
                  long long *d_count, unsigned nsuper, int subs, long long nstatus, const PeerPush pp)
{
    extern __shared__ __align__(128) unsigned char dsm[];
    using V2 = typename PtTraits<T>::V2;
    constexpr int K2_STAGES = PtTraits<T>::K2_STAGES;
    constexpr int K2_NP = PtTraits<T>::K2_NP;
    constexpr long long K2_SUB = k2_sub<T>();
    constexpr int K2_GROUPS = k2_groups<T>();
    V2 *stage = (V2 *)dsm;                                                        // [K2_STAGES][K2_SUB]
    unsigned *bits = (unsigned *)(dsm + (size_t)K2_STAGES * K2_SUB * sizeof(V2)); // [2][K2_ENTRIES]
    int *gscan = (int *)(bits + 2 * K2_ENTRIES);                            // [2][K2_ENTRIES]
    __shared__ SOct so;
    __shared__ __align__(8) unsigned long long s_full[K2_STAGES], s_empty[K2_STAGES];
    __shared__ unsigned s_desc_super[K2_STAGES];
    __shared__ int s_desc_j[K2_STAGES], s_desc_nsub[K2_STAGES], s_desc_copied[K2_STAGES];
    __shared__ int s_wsum[K2_CWARPS];
    __shared__ int s_total[2];
    __shared__ unsigned s_tile[2];
    __shared__ int s_nsub[2];
    __shared__ long long s_excl[2];
    __shared__ unsigned s_epoch;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const long long super_pts = (long long)subs * K2_SUB;
    const unsigned lt = lanemask_lt();

    if (tid == 0) {
        s_epoch = *(volatile unsigned *)&hdr->epoch;
        for (int st = 0; st < K2_STAGES; st++) {
            mbar_init(&s_full[st], 1);
            mbar_init(&s_empty[st], K2_CWARPS);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const unsigned epoch = s_epoch & ST_EPOCH_MASK;
    if (warp != K2_PROD_WARP) {
        // PDL: the octagon comes from the preceding kernel (K1's last CTA or
        // K3); everything that reads it or publishes results waits for that
        // grid here.  The producer only streams points, so it starts at once.
        asm volatile("griddepcontrol.wait;" ::: "memory");
        load_soct(so, oct,
                  hdr->tag_valid && hdr->tag_xy == (long long)xy && hdr->tag_n == n && hdr->tag_base == index_base);
        bar_sync(K2_BAR_BASE + 5, K2_CTHREADS + 32); // consumers + publisher: `so` is ready
    }

    if (warp == K2_PROD_WARP) {
        // ------------------------------------------------ TMA producer --
        // Streams this CTA's claimed super-tiles, sub-tile by sub-tile, into
        // the ring.  Claims are made in increasing order, each two sub-tiles
        // before the current super-tile ends.
        if (lane == 0) {
            __threadfence();
            unsigned p_super = atomicAdd(&hdr->k2_claim, 1u);
            unsigned p_next = TILE_DONE;
            bool next_claimed = false;
            int p_j = 0;
            int p_nsub = 0;
            if (p_super < nsuper)
                p_nsub = (int)min((long long)subs, (n - (long long)p_super * super_pts + K2_SUB - 1) / K2_SUB);
            for (unsigned seq = 0;; seq++) {
                const int st = (int)(seq % K2_STAGES);
                if (seq >= K2_STAGES)
                    mbar_wait(&s_empty[st], ((seq / K2_STAGES) - 1) & 1u); // consumers released it
                if (p_super >= nsuper) {
                    // End of stream.  (compute-sanitizer racecheck flags this
                    // store against the consumers' descriptor read: it does not
                    // model a phase completed by a tx-less arrive.  The arrive
                    // has release and try_wait acquire semantics, and the slot's
                    // previous readers released it through s_empty, exactly as
                    // for data stages.)
                    s_desc_super[st] = TILE_DONE;
                    mbar_expect_tx(&s_full[st], 0u);
                    break;
                }
                const long long base = (long long)p_super * super_pts + (long long)p_j * K2_SUB;
                const unsigned cnt = (unsigned)min(K2_SUB, n - base);
                // bulk copies move multiples of 16 bytes: an odd float tail
                // point is read from global memory by its consumer thread
                const unsigned copied = (cnt * (unsigned)sizeof(V2)) % 16u ? cnt - 1 : cnt;
                // Claim the next super-tile two sub-tiles before this one's
                // end (the atomic's latency hides behind them), not earlier:
                // super-tiles are then processed nearly in claim order, so a
                // look-back rarely waits on a predecessor that another CTA
                // claimed but has not started.
                if (!next_claimed && p_j >= p_nsub - 2) {
                    p_next = atomicAdd(&hdr->k2_claim, 1u);
                    next_claimed = true;
                }
                s_desc_super[st] = p_super;
                s_desc_j[st] = p_j;
                s_desc_nsub[st] = p_nsub;
                s_desc_copied[st] = (int)copied;
                mbar_expect_tx(&s_full[st], copied * (unsigned)sizeof(V2));
                if (copied > 0)
                    tma_load_1d(stage + (size_t)st * K2_SUB, xy + 2 * base, copied * (unsigned)sizeof(V2), &s_full[st]);
                if (++p_j == p_nsub) {
                    p_super = p_next >= nsuper ? TILE_DONE : p_next;
                    next_claimed = false;
                    p_j = 0;
                    p_nsub = 0;
                    if (p_super < nsuper)
                        p_nsub = (int)min((long long)subs,
                                          (n - (long long)p_super * super_pts + K2_SUB - 1) / K2_SUB);
                }
            }
        }
        __syncwarp();
    } else if (warp < K2_CWARPS) {
        // ------------------------------------------------ consumer warps --
        // Survivors of the super-tile held in buffer bb, written by every
        // consumer warp for its own 32-point groups, once the publisher has
        // resolved the super-tile's global offset.
        // Group e of a super-tile holds its points [32 e, 32 e + 32) (e =
        // (j * K2_NP + u) * K2_CWARPS + warp); its ballot word and offset sit
        // at [warp][j * K2_NP + u], so warp w writes the groups it tested,
        // four per step (one 16-byte load of ballots, one of offsets).
        auto write_survivors = [&](int bb) {
            bar_sync(K2_BAR_BASE + 2 + bb, K2_CTHREADS + 32); // offset of buffer bb is known
            if (s_total[bb] > 0) {
                // this warp's own slots (the groups it tested): slot t is
                // group e = 8 t + warp, points [32 e, 32 e + 32) of the
                // super-tile; its ballot and offset words are contiguous
                const int per = s_nsub[bb] * K2_NP;
                long long *ob = out + s_excl[bb];
                asm("" : "+l"(ob)); // one base register: offsets below are 32-bit
                long long v = (long long)s_tile[bb] * super_pts + index_base + 32LL * warp + lane;
                const uint4 *bw = (const uint4 *)(bits + bb * K2_ENTRIES + warp * K2_SLOTS);
                const int4 *sc = (const int4 *)(gscan + bb * K2_ENTRIES + warp * K2_SLOTS);
                const unsigned lb = 1u << lane;
                const long long vend = v - lane + 256LL * (per - 1) + 32; // this warp's index range: [v - lane, vend)
                if ((v >> 32) == ((vend - 1) >> 32)) {
                    // no 2^32 crossing: the high word is constant, the low word a 32-bit add
                    const unsigned hi = (unsigned)(v >> 32);
                    unsigned lo = (unsigned)v;
                    for (int q = 0; q < per / 4; q++, lo += 1024) {
                        const uint4 m = bw[q];
                        if ((m.x | m.y | m.z | m.w) == 0u)
                            continue;
                        const int4 c = sc[q];
                        store_group32(ob, m.x, c.x, lo, hi, lb, lt);
                        store_group32(ob, m.y, c.y, lo + 256, hi, lb, lt);
                        store_group32(ob, m.z, c.z, lo + 512, hi, lb, lt);
                        store_group32(ob, m.w, c.w, lo + 768, hi, lb, lt);
                    }
                    __syncwarp();
                    return;
                }
                for (int q = 0; q < per / 4; q++, v += 1024) {
                    const uint4 m = bw[q];
                    if ((m.x | m.y | m.z | m.w) == 0u)
                        continue;
                    const int4 c = sc[q];
                    store_group(ob, m.x, c.x, v, lb, lt);
                    store_group(ob, m.y, c.y, v + 256, lb, lt);
                    store_group(ob, m.z, c.z, v + 512, lb, lt);
                    store_group(ob, m.w, c.w, v + 768, lb, lt);
                }
            }
            __syncwarp(); // every lane's reads of its ballot words before lane 0 refills them
        };
        int b = 0, uses0 = 0, uses1 = 0;
        int guess_mode = 0; // adaptive: see classify()
        int box_mode = 0;   // adaptive: see consume_cert()
        for (unsigned seq = 0;; seq++) {
            const int st = (int)(seq % K2_STAGES);
            mbar_wait(&s_full[st], (seq / K2_STAGES) & 1u);
            const unsigned sup = s_desc_super[st];
            if (sup == TILE_DONE)
                break;
            const int j = s_desc_j[st], nsub = s_desc_nsub[st];
            if (j == 0 && (b ? uses1 : uses0) > 0) {
                // super-tile handed off two rounds ago.  Each warp reads only
                // the ballot words it wrote itself (its own slots) and the
                // offsets the block scan wrote before the hand-off, so no
                // barrier is needed before the warp refills buffer b; the
                // next scan's barrier orders every warp's reads before the
                // scan overwrites the offsets
                write_survivors(b);
            }
            const long long base = (long long)sup * super_pts + (long long)j * K2_SUB;
            const V2 *sp = stage + (size_t)st * K2_SUB;
            const int copied = s_desc_copied[st];
            unsigned *bw = bits + b * K2_ENTRIES + warp * K2_SLOTS + j * K2_NP; // this warp's slots (j, u)
            if (so.has_f32 && copied == (int)K2_SUB) {
                // adaptive (warp-uniform): a pass where the accept box left
                // >= 8 lanes with points outside it (ring-like data) makes
                // the next 64 sub-tiles skip the box test
                if (CH_K2_BOX && box_mode == 0) {
                    consume_cert<T, K2_NP, true>(so, sp, bw, box_mode);
                } else {
                    box_mode -= box_mode > 0;
                    consume_cert<T, K2_NP, false>(so, sp, bw, box_mode);
                }
                __syncwarp();
                if (lane == 0)
                    mbar_arrive(&s_empty[st]); // this warp is done with stage st
            } else {
            // (the per-lane-mask path, in chunks of <= 8 points per thread so
            // that its registers stay below consume_cert's; rare on the bench
            // workloads, so the stage is held until the last chunk is read)
            constexpr int CHK = K2_NP < 8 ? K2_NP : 8;
#pragma unroll 1
            for (int h0 = 0; h0 < K2_NP; h0 += CHK) {
                T px[CHK], py[CHK]; // storage precision; widened exactly where fp64 is needed
                unsigned valid = (1u << CHK) - 1u;
#pragma unroll
                for (int u = 0; u < CHK; u++) {
                    const V2 v = sp[(h0 + u) * K2_CTHREADS + tid];
                    px[u] = v.x;
                    py[u] = v.y;
                }
                if (copied < (int)K2_SUB) { // the partial last sub-tile (uniform branch)
                    valid = 0;
#pragma unroll
                    for (int u = 0; u < CHK; u++) {
                        const int q = (h0 + u) * K2_CTHREADS + tid;
                        if (q >= copied && base + q < n)
                            ld1raw(xy, base + q, px[u], py[u]); // odd float tail point
                        valid |= (base + q < n ? 1u : 0u) << u;
                    }
                }
                const unsigned keep = so.degenerate ? valid : classify<T, CHK>(so, px, py, valid, guess_mode);
#pragma unroll
                for (int u = 0; u < CHK; u++) {
                    const unsigned m = __ballot_sync(FULL, keep & (1u << u));
                    if (lane == 0)
                        bw[h0 + u] = m;
                }
            }
            __syncwarp();
            if (lane == 0)
                mbar_arrive(&s_empty[st]); // this warp is done with stage st
            }
            if (j == nsub - 1) {
                // ---- end of super-tile: group prefix (block scan) + aggregate ----
                bar_sync(K2_BAR_BASE + 4, K2_CTHREADS);
                const int E = nsub * K2_GROUPS;
                const unsigned *bb = bits + b * K2_ENTRIES;
                // group e (index order) = slot e / 8 of warp e % 8, stored at
                // [warp][slot]
                int c[4], sum = 0;
#pragma unroll
                for (int q = 0; q < 4; q++) {
                    const int e = 4 * tid + q;
                    c[q] = e < E ? __popc(bb[(e % K2_CWARPS) * K2_SLOTS + e / K2_CWARPS]) : 0;
                    sum += c[q];
                }
                int inc = sum;
#pragma unroll
                for (int off = 1; off < 32; off <<= 1) {
                    int t = __shfl_up_sync(FULL, inc, off);
                    if (lane >= off)
                        inc += t;
                }
                if (lane == 31)
                    s_wsum[warp] = inc;
                bar_sync(K2_BAR_BASE + 4, K2_CTHREADS);
                int ex = inc - sum, total = 0;
#pragma unroll
                for (int w = 0; w < K2_CWARPS; w++) {
                    const int v = s_wsum[w];
                    ex += w < warp ? v : 0;
                    total += v;
                }
                int *sc = gscan + b * K2_ENTRIES;
#pragma unroll
                for (int q = 0; q < 4; q++) {
                    const int e = 4 * tid + q;
                    sc[(e % K2_CWARPS) * K2_SLOTS + e / K2_CWARPS] = ex;
                    ex += c[q];
                }
                if (tid == 0) {
                    // Publish the aggregate right away (flag A; P for super-tile 0)
                    // so successors' look-backs never wait on this CTA's publisher.
                    st_release(&status[sup], ((sup == 0 ? ST_P : ST_A) << 62) | ((unsigned long long)epoch << 40) |
                                                 ((unsigned long long)total & ST_VALUE_MASK));
                    s_total[b] = total;
                    s_tile[b] = sup;
                    s_nsub[b] = nsub;
                }
                bar_arrive(K2_BAR_BASE + b, K2_CTHREADS + 32); // hand buffer b to the publisher
                if (b) uses1++; else uses0++;
                b ^= 1;
            }
        }
        // flush: the older pending buffer first
        if ((b ? uses1 : uses0) > 0)
            write_survivors(b);
        if ((b ? uses0 : uses1) > 0)
            write_survivors(b ^ 1);
        bar_sync(K2_BAR_BASE + 4, K2_CTHREADS);
        if (tid == 0)
            s_tile[b] = TILE_DONE;
        bar_arrive(K2_BAR_BASE + b, K2_CTHREADS + 32);
    } else {
        // ------------------------------------------------ publisher warp --
        // Decoupled look-back (Merrill & Garland) for each handed-off
        // super-tile: its global offset, then the inclusive prefix (flag P).
        int b = 0;
        while (true) {
            bar_sync(K2_BAR_BASE + b, K2_CTHREADS + 32);
            const unsigned tile = s_tile[b];
            if (tile == TILE_DONE)
                break;
            const int total = s_total[b];
            long long excl = 0;
            if (tile != 0) {
                long long pos = (long long)tile - 1;
                while (true) {
                    long long j = pos - lane;
                    unsigned long long flag = ST_P, val = 0;
                    unsigned pm, xm, need;
                    while (true) {
                        if (j >= 0) {
                            unsigned long long stw = ld_acquire(&status[j]);
                            bool ok = (unsigned)((stw >> 40) & ST_EPOCH_MASK) == epoch && (stw >> 62) != 0;
                            flag = ok ? (stw >> 62) : 0;
                            val = stw & ST_VALUE_MASK;
                        }
                        pm = __ballot_sync(FULL, flag == ST_P);
                        xm = __ballot_sync(FULL, flag == 0);
                        need = pm ? (((pm & (0u - pm)) << 1) - 1u) : FULL; // lanes up to the first P
                        if ((xm & need) == 0)
                            break;
                        __nanosleep(64);
                    }
                    unsigned long long c = ((need >> lane) & 1u) ? val : 0ull;
#pragma unroll
                    for (int off = 16; off > 0; off >>= 1)
                        c += __shfl_xor_sync(FULL, c, off);
                    excl += (long long)c;
                    if (pm)
                        break;
                    pos -= 32;
                }
                if (lane == 0)
                    st_release(&status[tile], (ST_P << 62) | ((unsigned long long)epoch << 40) |
                                                  ((unsigned long long)(excl + total) & ST_VALUE_MASK));
            }
            if (lane == 0) {
                s_excl[b] = excl;
                if (tile == nsuper - 1) {
                    hdr->result.count = excl + total;
                    if (d_count)
                        *d_count = excl + total;
                }
            }
            bar_arrive(K2_BAR_BASE + 2 + b, K2_CTHREADS + 32);
            b ^= 1;
        }
    }
    __syncthreads();
    // exit protocol: the last CTA to leave resets the counters, bumps the epoch
    __shared__ int s_exit_last;
    if (tid == 0) {
        __threadfence();
        s_exit_last = atomicAdd(&hdr->k2_exit, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    const unsigned next_epoch = (s_epoch + 1) & ST_EPOCH_MASK;
    if (s_exit_last && next_epoch == 0) {
        // the epoch wraps (every 2^22 launches): clear every status word of
        // the workspace, so that none written 2^22 launches ago can pass for
        // one of the coming launches
        for (long long q = tid; q < nstatus; q += K2_THREADS)
            status[q] = 0ull;
        __threadfence();
        __syncthreads();
    }
    if (tid == 0) {
        if (s_exit_last) {
            hdr->k2_claim = 0;
            hdr->k2_exit = 0;
            hdr->epoch = next_epoch;
            if (nsuper == 0) {
                hdr->result.count = 0;
                if (d_count)
                    *d_count = 0;
            }
            if (pp.world > 0) { // a7 fused: this rank's count into every peer's buffer
                __threadfence();
                peer_push_count(pp, *(volatile long long *)&hdr->result.count);
            }
        }
    }
}

// ===================================================================== K5 ==
// Small inputs (n <= KS_MAX_N, the latency-bound C1 case): the whole step in
// ONE CTA and one launch -- extremes (per-thread runs, block reduction),
// octagon (build_octagon_cta), octagon test and a block-wide stable
// compaction -- so no grid combine, no look-back, no second launch.  Same
// results as K1 + K2 (same functions, same order of decisions).
constexpr int KS_THREADS = 512;
constexpr int KS_BATCH = 4;
#ifndef CH_KS_MAX_N
#define CH_KS_MAX_N 2048
#endif
constexpr long long KS_MAX_N = CH_KS_MAX_N; // K5 / K6 crossover (profiles/r01_small_n.txt)

template <typename T>
__global__ void __launch_bounds__(KS_THREADS, 1)
k5_small_filter(const T *__restrict__ xy, long long n, int flags, WsHeader *hdr, long long *__restrict__ out,
                long long *d_count)
{
    constexpr int B = KS_BATCH;                 // point slots per thread
    static_assert(KS_MAX_N <= (long long)B * KS_THREADS, "K5 holds every point in registers");
    constexpr int NW = KS_THREADS / 32;
    __shared__ double s_v[NW][8];
    __shared__ long long s_i[NW][8];
    constexpr int GPL = B * NW / 32;            // scan groups per lane
    static_assert(B * NW % 32 == 0, "K5 group count");
    __shared__ int s_cnt[B * NW], s_pre[B * NW], s_tot;
    __shared__ ch_extremes s_e;
    __shared__ ch_octagon s_o;
    __shared__ SOct so;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int P = (int)((n + KS_THREADS - 1) / KS_THREADS); // slots in use (block-uniform)
    CH_TR(0);
    // ---- the points, once, into registers (point j * KS_THREADS + tid);
    //      extremes walking upward (equal keys keep the lower index) ----
    double px[B], py[B];
#pragma unroll
    for (int j = 0; j < B; j++) {
        const long long i = (long long)j * KS_THREADS + tid;
        px[j] = py[j] = 0.0;
        if (j < P && i < n)
            ld1pt(xy, i, px[j], py[j]);
    }
    Best bst;
    best_init(bst);
    double acc = 0.0;
    unsigned valid = 0;
#pragma unroll
    for (int j = 0; j < B; j++) {
        if (j >= P)
            break;
        const long long i = (long long)j * KS_THREADS + tid;
        if (i < n) {
            best_point(bst, px[j], py[j], i);
            acc = __fma_rn(px[j], 0.0, acc);
            acc = __fma_rn(py[j], 0.0, acc);
            valid |= 1u << j;
        }
    }
    CH_TR(1);
    {
        double wv;
        long long wi;
        best_warp_rs(bst, wv, wi);
        if ((lane & 3) == 0) {
            s_v[warp][rs_key(lane)] = wv;
            s_i[warp][rs_key(lane)] = wi;
        }
    }
    const int nf = __syncthreads_or(acc != acc);
    CH_TR(2);
    if (warp == 0) { // the NW warp results; lane k < 8 ends with key k
        double cv;
        long long ci;
        rows_combine<NW>(s_v, s_i, cv, ci);
        if (lane < 8) {
            s_e.idx[lane] = ci;
            s_e.x[lane] = (double)xy[2 * ci];
            s_e.y[lane] = (double)xy[2 * ci + 1];
        }
    }
    __syncthreads();
    CH_TR(3);
    build_octagon_cta(s_e, flags, s_o);
    CH_TR(4);
    load_soct(so, &s_o);
    __syncthreads();
    CH_TR(5);
    // ---- octagon test + stable compaction: groups (j, warp) of 32
    //      consecutive points, block scan of their popcounts ----
    int guess_mode = 0; // adaptive: see classify()
    const unsigned keep = so.degenerate ? valid
                          : so.has_f32  ? cert_classify<B>(so, px, py, valid, P)
                                        : classify<double, B>(so, px, py, valid, guess_mode, P);
    CH_TR(6);
    unsigned m[B];
#pragma unroll
    for (int j = 0; j < B; j++) {
        m[j] = __ballot_sync(FULL, (keep >> j) & 1u);
        if (lane == 0)
            s_cnt[j * NW + warp] = __popc(m[j]);
    }
    __syncthreads();
    // exclusive prefix of the B * NW group counts (index order: j, warp),
    // one warp scan: lane l owns groups [GPL*l, GPL*l + GPL)
    if (warp == 0) {
        int c[GPL], run = 0;
#pragma unroll
        for (int t = 0; t < GPL; t++) {
            c[t] = s_cnt[lane * GPL + t];
            run += c[t];
        }
        int inc = run;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const int v = __shfl_up_sync(FULL, inc, off);
            if (lane >= off)
                inc += v;
        }
        int ex = inc - run;
#pragma unroll
        for (int t = 0; t < GPL; t++) {
            s_pre[lane * GPL + t] = ex;
            ex += c[t];
        }
        if (lane == 31)
            s_tot = inc;
    }
    __syncthreads();
    CH_TR(7);
    const long long base_out = s_tot;
    const unsigned lt = lanemask_lt();
#pragma unroll
    for (int j = 0; j < B; j++) {
        if (j >= P)
            break;
        const int pre = s_pre[j * NW + warp];
        if ((m[j] >> lane) & 1u)
            out[pre + __popc(m[j] & lt)] = (long long)j * KS_THREADS + tid;
    }
    CH_TR(8);
    // ---- publish (the same workspace fields K1/K2 write) ----
    const unsigned *src = (const unsigned *)&s_o;
    unsigned *dst = (unsigned *)&hdr->oct;
    for (int q = tid; q < (int)(sizeof(ch_octagon) / 4); q += KS_THREADS)
        dst[q] = src[q];
    const unsigned *se = (const unsigned *)&s_e;
    unsigned *de = (unsigned *)&hdr->ext;
    for (int q = tid; q < (int)(sizeof(ch_extremes) / 4); q += KS_THREADS)
        de[q] = se[q];
    if (tid == 0) {
        hdr->result.count = base_out;
        hdr->result.nonfinite = nf;
        hdr->result.degenerate = s_o.degenerate;
        hdr->peer_timeout = 0;
        set_tag(hdr, xy, n, 0);
        if (d_count)
            *d_count = base_out;
    }
}

// ===================================================================== K6 ==
// Mid-small inputs (KS_MAX_N < n <= KC_MAX_N, e.g. the C1 config): the whole
// step in ONE launch of one 8-CTA thread-block cluster, each point read once
// into registers.  CTA r holds points [r P T, (r + 1) P T) (T threads, P =
// ceil(n / 8T) slots per thread, so every CTA has work).  Extremes per CTA
// (selects, butterflies), pushed into EVERY CTA's shared memory; every CTA
// combines them and builds the octagon itself (build_octagon_cta; the same
// values everywhere); the octagon test, and a stable compaction whose
// per-CTA totals are pushed to every CTA.  Only remote STORES cross the
// cluster, each followed by one cluster barrier (release / acquire): two in
// all.  Same decisions as K1 + K2.
constexpr int KC_CTAS = 8, KC_THREADS = 512, KC_P = 8;
constexpr long long KC_MAX_N = (long long)KC_CTAS * KC_THREADS * KC_P;

template <typename T>
__global__ void __cluster_dims__(KC_CTAS, 1, 1) __launch_bounds__(KC_THREADS, 1)
k6_cluster_filter(const T *__restrict__ xy, long long n, int flags, WsHeader *hdr, long long *__restrict__ out,
                  long long *d_count)
{
    namespace cg = cooperative_groups;
    cg::cluster_group cluster = cg::this_cluster();
    constexpr int NW = KC_THREADS / 32;
    __shared__ double s_v[NW][8];
    __shared__ long long s_i[NW][8];
    __shared__ double s_cv[KC_CTAS][8];     // every CTA's extremes (pushed to every CTA)
    __shared__ long long s_ci[KC_CTAS][8];
    __shared__ int s_cnf[KC_CTAS];          // every CTA's non-finite flag (pushed)
    __shared__ int s_nfall;                 // the cluster's
    __shared__ ch_extremes s_e;             // built by every CTA (the same values)
    __shared__ ch_octagon s_o;
    __shared__ SOct so;
    __shared__ int s_cnt[KC_P * NW], s_pre[KC_P * NW];
    __shared__ int s_tots[KC_CTAS];         // every CTA's survivor total (pushed)
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int r = (int)cluster.block_rank();
    const int P = (int)((n + KC_CTAS * KC_THREADS - 1) / (KC_CTAS * KC_THREADS)); // 1..KC_P
    const long long base = (long long)r * P * KC_THREADS;
    // shared memory of another CTA may be written only once that CTA runs:
    // arrive now, wait before the first remote store
    asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
    CH_TR(10);
    // ---- the points, once, into registers; extremes walking upward ----
    double px[KC_P], py[KC_P];
#pragma unroll
    for (int j = 0; j < KC_P; j++) {
        const long long i = base + (long long)j * KC_THREADS + tid;
        px[j] = py[j] = 0.0;
        if (j < P && i < n)
            ld1pt(xy, i, px[j], py[j]);
    }
    Best bst;
    best_init(bst);
    double acc = 0.0;
    unsigned valid = 0;
    CH_TR(11);
#pragma unroll
    for (int j = 0; j < KC_P; j++) {
        if (j >= P)
            break;
        const long long i = base + (long long)j * KC_THREADS + tid;
        if (i < n) {
            best_point(bst, px[j], py[j], i);
            acc = __fma_rn(px[j], 0.0, acc);
            acc = __fma_rn(py[j], 0.0, acc);
            valid |= 1u << j;
        }
    }
    {
        double wv;
        long long wi;
        best_warp_rs(bst, wv, wi);
        if ((lane & 3) == 0) {
            s_v[warp][rs_key(lane)] = wv;
            s_i[warp][rs_key(lane)] = wi;
        }
    }
    const int nf = __syncthreads_or(acc != acc);
    asm volatile("barrier.cluster.wait.aligned;" ::: "memory"); // every CTA of the cluster runs
    CH_TR(12);
    if (warp == 0) { // this CTA's extremes (lane k < 8: key k) -> every CTA's shared memory
        double cv;
        long long ci;
        rows_combine<NW>(s_v, s_i, cv, ci);
        // lane L pushes key L & 7 to CTAs (L >> 3) and (L >> 3) + 4
        const int k = lane & 7, d0 = lane >> 3;
        cv = __shfl_sync(FULL, cv, k);
        ci = __shfl_sync(FULL, ci, k);
#pragma unroll
        for (int h = 0; h < 2; h++) {
            const int d = d0 + 4 * h;
            *cluster.map_shared_rank(&s_cv[r][k], d) = cv;
            *cluster.map_shared_rank(&s_ci[r][k], d) = ci;
            if (k == 0)
                *cluster.map_shared_rank(&s_cnf[r], d) = nf;
        }
    }
    cluster.sync(); // every CTA holds every CTA's partial
    CH_TR(13);
    // Every CTA combines the partials and builds the octagon itself (the
    // same operations on the same values, so the same octagon): no second
    // push and no cluster barrier for it.
    if (warp == 0) {
        double cv;
        long long ci;
        rows_combine<KC_CTAS>(s_cv, s_ci, cv, ci);
        const int anynf = __any_sync(FULL, lane < KC_CTAS && s_cnf[lane]);
        if (lane < 8) {
            s_e.idx[lane] = ci;
            s_e.x[lane] = (double)xy[2 * ci];
            s_e.y[lane] = (double)xy[2 * ci + 1];
        }
        if (lane == 0)
            s_nfall = anynf;
    }
    __syncthreads();
    CH_TR(14);
    build_octagon_cta(s_e, flags, s_o);
    load_soct(so, &s_o);
    __syncthreads();
    CH_TR(16);
    // ---- octagon test + stable compaction (groups (j, warp) of 32 points) ----
    int guess_mode = 0;
    const unsigned keep = so.degenerate ? valid
                          : so.has_f32  ? cert_classify<KC_P>(so, px, py, valid, P)
                                        : classify<double, KC_P>(so, px, py, valid, guess_mode, P);
    CH_TR(17);
    unsigned m[KC_P];
#pragma unroll
    for (int j = 0; j < KC_P; j++) {
        m[j] = j < P ? __ballot_sync(FULL, (keep >> j) & 1u) : 0u; // (P is CTA-uniform)
        if (lane == 0)
            s_cnt[j * NW + warp] = __popc(m[j]);
    }
    __syncthreads();
    constexpr int GPL = KC_P * NW / 32; // scan groups per lane
    if (warp == 0) {
        int c[GPL], run = 0;
#pragma unroll
        for (int t = 0; t < GPL; t++) {
            c[t] = s_cnt[lane * GPL + t];
            run += c[t];
        }
        int inc = run;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const int v = __shfl_up_sync(FULL, inc, off);
            if (lane >= off)
                inc += v;
        }
        int ex = inc - run;
#pragma unroll
        for (int t = 0; t < GPL; t++) {
            s_pre[lane * GPL + t] = ex;
            ex += c[t];
        }
        const int tot = __shfl_sync(FULL, inc, 31);
        if (lane < KC_CTAS) // this CTA's total -> every CTA
            *cluster.map_shared_rank(&s_tots[r], lane) = tot;
    }
    cluster.sync(); // every CTA's survivor total is known everywhere (last remote access)
    CH_TR(18);
    long long off = 0, total = 0;
#pragma unroll
    for (int q = 0; q < KC_CTAS; q++) {
        const int t = s_tots[q];
        off += q < r ? t : 0;
        total += t;
    }
    const unsigned lt = lanemask_lt();
    CH_TR(19);
#pragma unroll
    for (int j = 0; j < KC_P; j++) {
        if (j >= P)
            break;
        const int pre = s_pre[j * NW + warp];
        if ((m[j] >> lane) & 1u)
            out[off + pre + __popc(m[j] & lt)] = base + (long long)j * KC_THREADS + tid;
    }
    if (r == 0) {   // publish (the same workspace fields K1 / K2 write)
        const unsigned *src = (const unsigned *)&s_o;
        unsigned *dst = (unsigned *)&hdr->oct;
        for (int q = tid; q < (int)(sizeof(ch_octagon) / 4); q += KC_THREADS)
            dst[q] = src[q];
        const unsigned *se = (const unsigned *)&s_e;
        unsigned *de = (unsigned *)&hdr->ext;
        for (int q = tid; q < (int)(sizeof(ch_extremes) / 4); q += KC_THREADS)
            de[q] = se[q];
        if (tid == 0) {
            hdr->result.count = total;
            hdr->result.nonfinite = s_nfall;
            hdr->result.degenerate = s_o.degenerate;
            hdr->peer_timeout = 0;
            set_tag(hdr, xy, n, 0);
            if (d_count)
                *d_count = total;
        }
    }
    CH_TR(20);
}

// ===================================================================== K4 ==
__global__ void __launch_bounds__(K4_THREADS)
k4_octagon_bits(const double *__restrict__ xy, long long n, const ch_octagon *__restrict__ oct,
                unsigned *__restrict__ bits)
{
    __shared__ SOct so;
    load_soct(so, oct);
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const long long nwords = (n + 31) / 32;
    const long long wstride = (long long)gridDim.x * (K4_THREADS / 32);
    for (long long w = (long long)blockIdx.x * (K4_THREADS / 32) + (threadIdx.x >> 5); w < nwords; w += wstride) {
        long long p = w * 32 + lane;
        bool k = false;
        if (p < n) {
            double x, y;
            ld128(xy + 2 * p, x, y);
            k = so.degenerate ? true : keep_point(so, x, y);
        }
        unsigned b = __ballot_sync(FULL, k);
        if (lane == 0)
            bits[w] = b;
    }
}

__global__ void k_gather(const double *__restrict__ xy, long long index_base, const long long *__restrict__ idx,
                         long long m, double *__restrict__ outp)
{
    for (long long j = (long long)blockIdx.x * blockDim.x + threadIdx.x; j < m; j += (long long)gridDim.x * blockDim.x) {
        long long i = idx[j] - index_base;
        double x, y;
        ld128(xy + 2 * i, x, y);
        outp[2 * j] = x;
        outp[2 * j + 1] = y;
    }
}

// ================================================================ host side ==
using chi::fail;

ch_status cuda_check(const char *what)
{
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess)
        return fail(CH_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
    return CH_OK;
}

struct DevInfo {
    int sms = 0;
    int k1_per_sm = 0;   // float64 storage
    int k1_per_sm_f = 0; // float32 storage
    int k2_per_sm_d = 0; // double points
    int k2_per_sm_f = 0; // float points
};

DevInfo dev_info()
{
    static thread_local int cached_dev = -1;
    static thread_local DevInfo info;
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev != cached_dev) {
        cudaDeviceGetAttribute(&info.sms, cudaDevAttrMultiProcessorCount, dev);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&info.k1_per_sm, k1_extremes8<double, true>, K1_THREADS, 0);
        info.k1_per_sm = std::max(1, info.k1_per_sm);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&info.k1_per_sm_f, k1_extremes8<float, true>, K1_THREADS, 0);
        info.k1_per_sm_f = std::max(1, info.k1_per_sm_f);
        cudaFuncSetAttribute(k2_filter_compact<double>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)k2_dsmem<double>());
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&info.k2_per_sm_d, k2_filter_compact<double>, K2_THREADS,
                                                      k2_dsmem<double>());
        info.k2_per_sm_d = std::max(1, info.k2_per_sm_d);
        cudaFuncSetAttribute(k2_filter_compact<float>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)k2_dsmem<float>());
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&info.k2_per_sm_f, k2_filter_compact<float>, K2_THREADS,
                                                      k2_dsmem<float>());
        info.k2_per_sm_f = std::max(1, info.k2_per_sm_f);
        cached_dev = dev;
    }
    return info;
}

ch_status check_ws(const void *d_ws, size_t ws_bytes, long long n)
{
    if (!d_ws)
        return fail(CH_ERR_WORKSPACE, "workspace is NULL");
    if (((uintptr_t)d_ws & 255u) != 0)
        return fail(CH_ERR_WORKSPACE, "workspace must be 256-byte aligned");
    if (ws_bytes < ch_workspace_bytes(n))
        return fail(CH_ERR_WORKSPACE, "workspace too small for n");
    return CH_OK;
}

template <typename T>
ch_status check_points(const T *d_xy, long long n)
{
    if (n < 0)
        return fail(CH_ERR_INVALID_ARG, "n < 0");
    if (n == 0)
        return fail(CH_ERR_EMPTY, "n == 0 (EmptySet)");
    if (!d_xy)
        return fail(CH_ERR_INVALID_ARG, "d_xy is NULL");
    if (((uintptr_t)d_xy & 15u) != 0)
        return fail(CH_ERR_MISALIGNED, "d_xy must be 16-byte aligned");
    if (n > (1ll << 39))
        return fail(CH_ERR_INVALID_ARG, "n > 2^39 unsupported");
    return CH_OK;
}

inline WsHeader *hdr_of(void *d_ws) { return (WsHeader *)d_ws; }
inline Partial *parts_of(void *d_ws) { return (Partial *)((char *)d_ws + WS_HEADER); }
inline unsigned long long *status_of(void *d_ws)
{
    return (unsigned long long *)((char *)d_ws + WS_HEADER + WS_PARTIALS);
}

template <typename T>
ch_status launch_k1(const T *d_xy, long long n, long long index_base, int flags, void *d_ext_out,
                    void *d_ws, cudaStream_t st, const PeerPush &pp = PeerPush{})
{
    DevInfo di = dev_info();
    constexpr long long K1_CHUNK = k1_chunk<T>();
    long long nchunks = (n + K1_CHUNK - 1) / K1_CHUNK;
    long long g = std::min<long long>((long long)di.sms * (sizeof(T) == 8 ? di.k1_per_sm : di.k1_per_sm_f), nchunks);
    g = std::min<long long>(g, K1_MAX_CTAS);
    if (g < 1)
        g = 1;
    // wide loads need their points aligned to the load size (32 B / 16 B)
    if (((uintptr_t)d_xy & (2 * PtTraits<T>::K1_PPL * sizeof(T) - 1)) == 0)
        k1_extremes8<T, true><<<(unsigned)g, K1_THREADS, 0, st>>>(d_xy, n, index_base, flags, hdr_of(d_ws),
                                                                   parts_of(d_ws), d_ext_out, pp);
    else
        k1_extremes8<T, false><<<(unsigned)g, K1_THREADS, 0, st>>>(d_xy, n, index_base, flags, hdr_of(d_ws),
                                                                    parts_of(d_ws), d_ext_out, pp);
    return cuda_check("k1_extremes8");
}

// A caller-supplied octagon (ch_filter_compact / ch_octagon_filter with
// h_oct != NULL) defines the predicate by its vertices, edges and thresholds
// (D_k > thr[k] on every edge, R4).  The shortcuts the kernels take are
// re-derived here, never trusted: nv must lie in [0, 8] and agree with
// `degenerate` (else CH_ERR_INVALID_ARG); the accept box is kept only if
// every corner passes every edge (chf::box_corner_ok, the proof at
// octagon.cuh), else it is replaced by the empty box; guessed edges outside
// [0, nv) become 0; the fp32 certificates are off (their bound needs the
// points inside the octagon's bbox).
ch_status sanitize_octagon(const ch_octagon &in, ch_octagon &o)
{
    o = in;
    if (o.nv < 0 || o.nv > 8)
        return fail(CH_ERR_INVALID_ARG, "octagon: nv outside [0, 8]");
    if ((o.degenerate != 0) != (o.nv < 3))
        return fail(CH_ERR_INVALID_ARG, "octagon: degenerate must be (nv < 3)");
    o.degenerate = o.nv < 3;
    o.plain = o.plain ? 1 : 0;
    o.exact = (!o.plain && o.exact) ? 1 : 0;
    o.has_f32 = 0;
    for (int k = 0; k < 8; k++)
        if (o.guess_edge[k] < 0 || o.guess_edge[k] >= (o.nv > 0 ? o.nv : 1))
            o.guess_edge[k] = 0;
    bool box_ok = o.has_box && !o.degenerate && o.box[0] <= o.box[1] && o.box[2] <= o.box[3];
    for (int k = 0; k < o.nv && box_ok; k++)
        for (int c = 0; c < 4 && box_ok; c++)
            box_ok = chf::box_corner_ok(o, k, o.box, c);
    if (!box_ok) {
        o.has_box = 0;
        o.box[0] = o.box[2] = CH_INF;
        o.box[1] = o.box[3] = -CH_INF;
    }
    return CH_OK;
}

ch_status stage_octagon(const ch_octagon *h_oct, void *d_ws, cudaStream_t st, const ch_octagon **d_oct)
{
    WsHeader *h = hdr_of(d_ws);
    if (h_oct) {
        ch_octagon o;
        ch_status s = sanitize_octagon(*h_oct, o);
        if (s != CH_OK)
            return s;
        // (pageable source: the copy is staged before cudaMemcpyAsync returns)
        cudaMemcpyAsync(&h->oct, &o, sizeof(ch_octagon), cudaMemcpyHostToDevice, st);
        cudaMemsetAsync(&h->result.nonfinite, 0, sizeof(int32_t), st); // no K1 pass: nothing checked
        cudaMemsetAsync(&h->tag_valid, 0, sizeof(unsigned), st);      // not built from the data
        s = cuda_check("octagon upload");
        if (s != CH_OK)
            return s;
    }
    *d_oct = &h->oct;
    return CH_OK;
}

template <typename T>
// pdl: launch with programmatic stream serialization.  Only when the kernel
// just before K2 on the stream is our K1 or K3 (they trigger early and never
// touch K2's claim counter, epoch or status words); a K2 right after another
// K2 on the same workspace must see that K2's exit protocol, so by default
// K2 is serialized normally.
ch_status launch_k2(const T *d_xy, long long n, long long index_base, const ch_octagon *d_oct,
                    long long *d_surv, long long *d_count, void *d_ws, size_t ws_bytes, cudaStream_t st,
                    const PeerPush &pp = PeerPush{}, bool pdl = false)
{
    const long long nstatus = (long long)((ws_bytes - WS_HEADER - WS_PARTIALS) / sizeof(unsigned long long));
    DevInfo di = dev_info();
    long long resident = (long long)di.sms * (sizeof(T) == 8 ? di.k2_per_sm_d : di.k2_per_sm_f);
    constexpr long long K2_SUB = k2_sub<T>();
    long long nsub_total = (n + K2_SUB - 1) / K2_SUB;
    // aim for >= CH_K2_SUPERS super-tiles per CTA (load balance: the last
    // super-tiles' look-backs wait on their predecessors), <= k2_maxsub
    // sub-tiles each
    long long subs = (nsub_total + resident * CH_K2_SUPERS - 1) / (resident * CH_K2_SUPERS);
    subs = std::max<long long>(1, std::min<long long>(subs, (long long)k2_maxsub<T>()));
    long long nsuper = (nsub_total + subs - 1) / subs;
    long long grid = std::max<long long>(1, std::min<long long>(resident, nsuper));
    // programmatic dependent launch: K2's producer overlaps the tail of K1
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3(K2_THREADS);
    cfg.dynamicSmemBytes = k2_dsmem<T>();
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
    const cudaError_t e = cudaLaunchKernelEx(&cfg, k2_filter_compact<T>, d_xy, (long long)n, (long long)index_base, d_oct,
                                             hdr_of(d_ws), status_of(d_ws), (long long *)d_surv, (long long *)d_count,
                                             (unsigned)nsuper, (int)subs, nstatus, pp);
    if (e != cudaSuccess)
        return fail(CH_ERR_CUDA, std::string("k2_filter_compact: ") + cudaGetErrorString(e));
    return cuda_check("k2_filter_compact");
}

template <typename T>
ch_status extremes8_impl(const T *d_xy, int64_t n, int64_t index_base, int flags, void *d_ext_out,
                         ch_extremes *h_ext, ch_octagon *h_oct, void *d_ws, size_t ws_bytes, void *stream);
template <typename T>
ch_status filter_compact_impl(const T *d_xy, int64_t n, int64_t index_base, const ch_octagon *h_oct,
                              int64_t *d_survivors, int64_t *d_count, void *d_ws, size_t ws_bytes, void *stream,
                              bool after_k1 = false);
template <typename T>
ch_status filter_impl(const T *d_xy, int64_t n, int flags, int64_t *d_survivors, int64_t *h_count, void *d_ws,
                      size_t ws_bytes, void *stream);
template <typename T>
ch_status filter_async_impl(const T *d_xy, int64_t n, int flags, int64_t *d_survivors, int64_t *d_count, void *d_ws,
                            size_t ws_bytes, void *stream);

} // namespace

// ================================================================== C ABI ==
extern "C" {

int ch_abi_version(void) { return CH_ABI_VERSION; }

#ifdef CH_TRACE
int ch_debug_trace(long long *h, int n)
{
    if (n > 32)
        n = 32;
    return cudaMemcpyFromSymbol(h, g_trace, n * sizeof(long long)) == cudaSuccess ? n : -1;
}
#endif

int ch_occupancy(int kernel)
{
    const DevInfo d = dev_info();
    if (cudaGetLastError() != cudaSuccess)
        return -1;
    switch (kernel) {
    case 0: return d.k1_per_sm;
    case 1: return d.k2_per_sm_d;
    case 2: return d.k2_per_sm_f;
    default: return -1;
    }
}

const char *ch_status_str(ch_status s)
{
    switch (s) {
    case CH_OK: return "CH_OK";
    case CH_ERR_INVALID_ARG: return "CH_ERR_INVALID_ARG";
    case CH_ERR_EMPTY: return "CH_ERR_EMPTY";
    case CH_ERR_NONFINITE: return "CH_ERR_NONFINITE";
    case CH_ERR_MISALIGNED: return "CH_ERR_MISALIGNED";
    case CH_ERR_WORKSPACE: return "CH_ERR_WORKSPACE";
    case CH_ERR_CUDA: return "CH_ERR_CUDA";
    case CH_ERR_PEER: return "CH_ERR_PEER";
    case CH_ERR_NCCL: return "CH_ERR_NCCL";
    }
    return "CH_ERR_UNKNOWN";
}

const char *ch_last_error(void) { return chi::last_error(); }

size_t ch_workspace_bytes(int64_t n)
{
    if (n < 0)
        n = 0;
    size_t tiles = (size_t)ntiles_of(n) + 1;
    size_t b = WS_HEADER + WS_PARTIALS + tiles * sizeof(unsigned long long);
    return (b + 4095) & ~(size_t)4095;
}

ch_status ch_workspace_init(void *d_ws, size_t ws_bytes, void *stream)
{
    if (!d_ws || ws_bytes < WS_HEADER + WS_PARTIALS)
        return fail(CH_ERR_WORKSPACE, "workspace missing or too small");
    cudaMemsetAsync(d_ws, 0, ws_bytes, (cudaStream_t)stream);
    return cuda_check("workspace init");
}

ch_status ch_octagon_build(const ch_extremes *ext, int flags, ch_octagon *out)
{
    if (!ext || !out)
        return fail(CH_ERR_INVALID_ARG, "NULL argument");
    chf::build_octagon(*ext, flags, *out);
    return CH_OK;
}

ch_status ch_read_octagon(const void *d_ws, ch_extremes *h_ext, ch_octagon *h_oct, void *stream)
{
    if (!d_ws)
        return fail(CH_ERR_INVALID_ARG, "NULL workspace");
    cudaStream_t st = (cudaStream_t)stream;
    if (h_ext)
        cudaMemcpyAsync(h_ext, &((const WsHeader *)d_ws)->ext, sizeof(ch_extremes), cudaMemcpyDeviceToHost, st);
    if (h_oct)
        cudaMemcpyAsync(h_oct, &((const WsHeader *)d_ws)->oct, sizeof(ch_octagon), cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    return cuda_check("read octagon");
}

ch_status ch_read_result(const void *d_ws, ch_result *h_res, void *stream)
{
    if (!d_ws || !h_res)
        return fail(CH_ERR_INVALID_ARG, "NULL argument");
    cudaStream_t st = (cudaStream_t)stream;
    unsigned late = 0;
    cudaMemcpyAsync(h_res, &((const WsHeader *)d_ws)->result, sizeof(ch_result), cudaMemcpyDeviceToHost, st);
    cudaMemcpyAsync(&late, &((const WsHeader *)d_ws)->peer_timeout, sizeof(unsigned), cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    ch_status s = cuda_check("read result");
    if (s != CH_OK)
        return s;
    if (h_res->nonfinite)
        return fail(CH_ERR_NONFINITE, "non-finite coordinate in input");
    if (late)
        return fail(CH_ERR_PEER, "peer exchange timed out (a rank's record did not arrive)");
    return CH_OK;
}

} // extern "C"

namespace {
template <typename T>
ch_status extremes8_impl(const T *d_xy, int64_t n, int64_t index_base, int flags, void *d_ext_out,
                         ch_extremes *h_ext, ch_octagon *h_oct, void *d_ws, size_t ws_bytes, void *stream)
{
    ch_status s = check_points(d_xy, n);
    if (s != CH_OK)
        return s;
    if ((s = check_ws(d_ws, ws_bytes, n)) != CH_OK)
        return s;
    cudaStream_t st = (cudaStream_t)stream;
    if ((s = launch_k1(d_xy, n, index_base, flags, d_ext_out, d_ws, st)) != CH_OK)
        return s;
    if (h_ext || h_oct) {
        WsHeader *h = hdr_of(d_ws);
        if (h_ext)
            cudaMemcpyAsync(h_ext, &h->ext, sizeof(ch_extremes), cudaMemcpyDeviceToHost, st);
        if (h_oct)
            cudaMemcpyAsync(h_oct, &h->oct, sizeof(ch_octagon), cudaMemcpyDeviceToHost, st);
        ch_result r;
        return ch_read_result(d_ws, &r, stream);
    }
    return CH_OK;
}

template <typename T>
ch_status filter_compact_impl(const T *d_xy, int64_t n, int64_t index_base, const ch_octagon *h_oct,
                              int64_t *d_survivors, int64_t *d_count, void *d_ws, size_t ws_bytes, void *stream,
                              bool after_k1)
{
    ch_status s = check_points(d_xy, n);
    if (s != CH_OK)
        return s;
    if (!d_survivors)
        return fail(CH_ERR_INVALID_ARG, "d_survivors is NULL");
    if ((s = check_ws(d_ws, ws_bytes, n)) != CH_OK)
        return s;
    cudaStream_t st = (cudaStream_t)stream;
    const ch_octagon *d_oct;
    if ((s = stage_octagon(h_oct, d_ws, st, &d_oct)) != CH_OK)
        return s;
    return launch_k2(d_xy, n, index_base, d_oct, (long long *)d_survivors, (long long *)d_count, d_ws, ws_bytes,
                     st, PeerPush{}, after_k1 && !h_oct);
}

// One step, asynchronous: K5 (one CTA, one launch) for small n, else K1 + K2.
template <typename T>
ch_status filter_async_impl(const T *d_xy, int64_t n, int flags, int64_t *d_survivors, int64_t *d_count, void *d_ws,
                            size_t ws_bytes, void *stream)
{
    if (n <= KS_MAX_N) {
        ch_status s = check_points(d_xy, n);
        if (s != CH_OK)
            return s;
        if (!d_survivors)
            return fail(CH_ERR_INVALID_ARG, "d_survivors is NULL");
        if ((s = check_ws(d_ws, ws_bytes, n)) != CH_OK)
            return s;
        k5_small_filter<T><<<1, KS_THREADS, 0, (cudaStream_t)stream>>>(d_xy, n, flags, hdr_of(d_ws),
                                                                       (long long *)d_survivors, (long long *)d_count);
        return cuda_check("k5_small_filter");
    }
    if (n <= KC_MAX_N && !(flags & CH_NO_CLUSTER)) {
        ch_status s = check_points(d_xy, n);
        if (s != CH_OK)
            return s;
        if (!d_survivors)
            return fail(CH_ERR_INVALID_ARG, "d_survivors is NULL");
        if ((s = check_ws(d_ws, ws_bytes, n)) != CH_OK)
            return s;
        k6_cluster_filter<T><<<KC_CTAS, KC_THREADS, 0, (cudaStream_t)stream>>>(
            d_xy, n, flags, hdr_of(d_ws), (long long *)d_survivors, (long long *)d_count);
        return cuda_check("k6_cluster_filter");
    }
    ch_status s = extremes8_impl(d_xy, n, 0, flags, nullptr, nullptr, nullptr, d_ws, ws_bytes, stream);
    if (s != CH_OK)
        return s;
    return filter_compact_impl(d_xy, n, 0, nullptr, d_survivors, d_count, d_ws, ws_bytes, stream, true);
}

template <typename T>
ch_status filter_impl(const T *d_xy, int64_t n, int flags, int64_t *d_survivors, int64_t *h_count, void *d_ws,
                      size_t ws_bytes, void *stream)
{
    ch_status s = filter_async_impl(d_xy, n, flags, d_survivors, (int64_t *)nullptr, d_ws, ws_bytes, stream);
    if (s != CH_OK)
        return s;
    ch_result r;
    s = ch_read_result(d_ws, &r, stream);
    if (h_count)
        *h_count = r.count;
    return s;
}
} // namespace

extern "C" {

ch_status ch_extremes8(const double *d_xy, int64_t n, int64_t index_base, int flags, void *d_ext_out,
                       ch_extremes *h_ext, ch_octagon *h_oct, void *d_ws, size_t ws_bytes, void *stream)
{
    return extremes8_impl(d_xy, n, index_base, flags, d_ext_out, h_ext, h_oct, d_ws, ws_bytes, stream);
}

ch_status ch_extremes8_f32(const float *d_xy, int64_t n, int64_t index_base, int flags, void *d_ext_out,
                           ch_extremes *h_ext, ch_octagon *h_oct, void *d_ws, size_t ws_bytes, void *stream)
{
    return extremes8_impl(d_xy, n, index_base, flags, d_ext_out, h_ext, h_oct, d_ws, ws_bytes, stream);
}

ch_status ch_combine8(const void *d_ext_all, int world, int flags, void *d_ws, size_t ws_bytes, void *stream)
{
    if (!d_ext_all || world < 1)
        return fail(CH_ERR_INVALID_ARG, "bad extremes array / world");
    ch_status s = check_ws(d_ws, ws_bytes, 0);
    if (s != CH_OK)
        return s;
    k3_combine8<<<1, 256, 0, (cudaStream_t)stream>>>((const ch_extremes *)d_ext_all, world, flags, hdr_of(d_ws));
    return cuda_check("k3_combine8");
}

ch_status ch_octagon_filter(const double *d_xy, int64_t n, const ch_octagon *h_oct, uint32_t *d_keep_bits,
                            void *d_ws, size_t ws_bytes, void *stream)
{
    ch_status s = check_points(d_xy, n);
    if (s != CH_OK)
        return s;
    if (!d_keep_bits)
        return fail(CH_ERR_INVALID_ARG, "d_keep_bits is NULL");
    if ((s = check_ws(d_ws, ws_bytes, 0)) != CH_OK)
        return s;
    cudaStream_t st = (cudaStream_t)stream;
    const ch_octagon *d_oct;
    if ((s = stage_octagon(h_oct, d_ws, st, &d_oct)) != CH_OK)
        return s;
    DevInfo di = dev_info();
    long long nwords = (n + 31) / 32;
    long long g = std::min<long long>((nwords + 7) / 8, (long long)di.sms * 8);
    k4_octagon_bits<<<(unsigned)std::max<long long>(g, 1), K4_THREADS, 0, st>>>(d_xy, n, d_oct, d_keep_bits);
    return cuda_check("k4_octagon_bits");
}

ch_status ch_filter_compact(const double *d_xy, int64_t n, int64_t index_base, const ch_octagon *h_oct,
                            int64_t *d_survivors, int64_t *d_count, void *d_ws, size_t ws_bytes, void *stream)
{
    return filter_compact_impl(d_xy, n, index_base, h_oct, d_survivors, d_count, d_ws, ws_bytes, stream);
}

ch_status ch_filter_compact_f32(const float *d_xy, int64_t n, int64_t index_base, const ch_octagon *h_oct,
                                int64_t *d_survivors, int64_t *d_count, void *d_ws, size_t ws_bytes, void *stream)
{
    return filter_compact_impl(d_xy, n, index_base, h_oct, d_survivors, d_count, d_ws, ws_bytes, stream);
}

ch_status ch_filter(const double *d_xy, int64_t n, int flags, int64_t *d_survivors, int64_t *h_count,
                    void *d_ws, size_t ws_bytes, void *stream)
{
    return filter_impl(d_xy, n, flags, d_survivors, h_count, d_ws, ws_bytes, stream);
}

ch_status ch_filter_async(const double *d_xy, int64_t n, int flags, int64_t *d_survivors, int64_t *d_count,
                          void *d_ws, size_t ws_bytes, void *stream)
{
    return filter_async_impl(d_xy, n, flags, d_survivors, d_count, d_ws, ws_bytes, stream);
}

ch_status ch_filter_async_f32(const float *d_xy, int64_t n, int flags, int64_t *d_survivors, int64_t *d_count,
                              void *d_ws, size_t ws_bytes, void *stream)
{
    return filter_async_impl(d_xy, n, flags, d_survivors, d_count, d_ws, ws_bytes, stream);
}

ch_status ch_filter_f32(const float *d_xy, int64_t n, int flags, int64_t *d_survivors, int64_t *h_count,
                        void *d_ws, size_t ws_bytes, void *stream)
{
    return filter_impl(d_xy, n, flags, d_survivors, h_count, d_ws, ws_bytes, stream);
}

} // extern "C"

struct ch_graph {
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
};

namespace {
template <typename T>
ch_status graph_create(const T *d_xy, int64_t n, int flags, int64_t *d_survivors, int64_t *d_count, void *d_ws,
                       size_t ws_bytes, ch_graph **out)
{
    if (!out)
        return fail(CH_ERR_INVALID_ARG, "out is NULL");
    *out = nullptr;
    dev_info(); // function attributes / occupancy queried before capture
    cudaStream_t cs;
    if (cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking) != cudaSuccess)
        return fail(CH_ERR_CUDA, "graph: stream create failed");
    ch_graph *g = new ch_graph();
    ch_status s = CH_OK;
    if (cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal) != cudaSuccess) {
        s = fail(CH_ERR_CUDA, "graph: begin capture failed");
    } else {
        s = filter_async_impl(d_xy, n, flags, d_survivors, d_count, d_ws, ws_bytes, (void *)cs);
        const cudaError_t e = cudaStreamEndCapture(cs, &g->graph);
        if (s == CH_OK && e != cudaSuccess)
            s = fail(CH_ERR_CUDA, std::string("graph: capture failed: ") + cudaGetErrorString(e));
        if (s == CH_OK && cudaGraphInstantiate(&g->exec, g->graph, 0) != cudaSuccess)
            s = fail(CH_ERR_CUDA, "graph: instantiate failed");
    }
    cudaGetLastError();
    cudaStreamDestroy(cs);
    if (s != CH_OK) {
        if (g->exec)
            cudaGraphExecDestroy(g->exec);
        if (g->graph)
            cudaGraphDestroy(g->graph);
        delete g;
        return s;
    }
    *out = g;
    return CH_OK;
}
} // namespace

extern "C" {

ch_status ch_filter_graph_create(const double *d_xy, int64_t n, int flags, int64_t *d_survivors, int64_t *d_count,
                                 void *d_ws, size_t ws_bytes, ch_graph **out)
{
    return graph_create(d_xy, n, flags, d_survivors, d_count, d_ws, ws_bytes, out);
}

ch_status ch_filter_graph_create_f32(const float *d_xy, int64_t n, int flags, int64_t *d_survivors,
                                     int64_t *d_count, void *d_ws, size_t ws_bytes, ch_graph **out)
{
    return graph_create(d_xy, n, flags, d_survivors, d_count, d_ws, ws_bytes, out);
}

ch_status ch_graph_launch(ch_graph *g, void *stream)
{
    if (!g || !g->exec)
        return fail(CH_ERR_INVALID_ARG, "graph is NULL");
    const cudaError_t e = cudaGraphLaunch(g->exec, (cudaStream_t)stream);
    if (e != cudaSuccess)
        return fail(CH_ERR_CUDA, std::string("graph launch: ") + cudaGetErrorString(e));
    return CH_OK;
}

ch_status ch_graph_destroy(ch_graph *g)
{
    if (!g)
        return CH_OK;
    if (g->exec)
        cudaGraphExecDestroy(g->exec);
    if (g->graph)
        cudaGraphDestroy(g->graph);
    delete g;
    return CH_OK;
}

} // extern "C"

struct ch_peer {
    int rank = 0, world = 0;
    unsigned long long *d_buf = nullptr;           // this rank's exchange buffer
    unsigned long long *base[CH_MAX_PEERS] = {};   // every rank's, mapped here
    bool opened[CH_MAX_PEERS] = {};
    unsigned long long epoch = 0;                  // steps issued
    unsigned long long timeout_ms = 60000;         // waits for a peer's record / count
};

namespace {
template <typename T>
ch_status step_peer(ch_peer *p, const T *d_xy, int64_t n_local, int64_t index_base, int flags, int64_t *d_survivors,
                    void *d_ws, size_t ws_bytes, void *stream)
{
    if (!p || !p->base[0])
        return fail(CH_ERR_INVALID_ARG, "peer exchange not opened");
    if (n_local < 0 || (n_local > 0 && !d_survivors))
        return fail(CH_ERR_INVALID_ARG, "bad shard arguments");
    ch_status s;
    if (n_local > 0 && (s = check_points(d_xy, n_local)) != CH_OK)
        return s;
    if ((s = check_ws(d_ws, ws_bytes, n_local)) != CH_OK)
        return s;
    cudaStream_t st = (cudaStream_t)stream;
    PeerPush pp{};
    for (int r = 0; r < p->world; r++)
        pp.base[r] = p->base[r];
    pp.world = p->world;
    pp.rank = p->rank;
    pp.epoch = ++p->epoch;
    pp.timeout_ns = p->timeout_ms * 1000000ull;
    if (n_local > 0) {
        if ((s = launch_k1(d_xy, n_local, index_base, flags, nullptr, d_ws, st, pp)) != CH_OK)
            return s;
    } else {
        k_peer_push<<<1, 256, 0, st>>>(pp, 0);
    }
    k3_combine8_peer<<<1, 256, 0, st>>>(pp, flags, hdr_of(d_ws));
    if ((s = cuda_check("k3_combine8_peer")) != CH_OK)
        return s;
    if (n_local > 0)
        return launch_k2(d_xy, n_local, index_base, &hdr_of(d_ws)->oct, (long long *)d_survivors, nullptr, d_ws,
                         ws_bytes, st, pp, true); // K3 (peer) just before
    k_peer_push<<<1, 32, 0, st>>>(pp, 1);
    return cuda_check("k_peer_push");
}
} // namespace

extern "C" {

size_t ch_peer_handle_bytes(void) { return sizeof(cudaIpcMemHandle_t); }

ch_status ch_peer_create(int rank, int world, ch_peer **out, void *h_handle)
{
    if (!out || !h_handle || world < 1 || world > CH_MAX_PEERS || rank < 0 || rank >= world)
        return fail(CH_ERR_INVALID_ARG, "bad rank / world (1 <= world <= CH_MAX_PEERS)");
    ch_peer *p = new ch_peer();
    p->rank = rank;
    p->world = world;
    if (const char *t = getenv("CH_PEER_TIMEOUT_MS")) // tests: a short timeout
        p->timeout_ms = std::max(1ull, strtoull(t, nullptr, 10));
    if (cudaMalloc((void **)&p->d_buf, PEER_BUF_BYTES) != cudaSuccess ||
        cudaMemset(p->d_buf, 0, PEER_BUF_BYTES) != cudaSuccess) {
        delete p;
        return cuda_check("peer buffer");
    }
    cudaIpcMemHandle_t h;
    if (cudaIpcGetMemHandle(&h, p->d_buf) != cudaSuccess) {
        cudaFree(p->d_buf);
        delete p;
        return fail(CH_ERR_CUDA, "cudaIpcGetMemHandle failed");
    }
    memcpy(h_handle, &h, sizeof(h));
    p->base[rank] = p->d_buf;
    *out = p;
    return CH_OK;
}

ch_status ch_peer_open(ch_peer *p, const void *h_handles)
{
    if (!p || !h_handles)
        return fail(CH_ERR_INVALID_ARG, "NULL argument");
    for (int r = 0; r < p->world; r++) {
        if (r == p->rank || p->opened[r])
            continue;
        cudaIpcMemHandle_t h;
        memcpy(&h, (const char *)h_handles + r * sizeof(h), sizeof(h));
        void *ptr = nullptr;
        const cudaError_t e = cudaIpcOpenMemHandle(&ptr, h, cudaIpcMemLazyEnablePeerAccess);
        if (e != cudaSuccess) {
            cudaGetLastError();
            return fail(CH_ERR_CUDA, std::string("cudaIpcOpenMemHandle failed: ") + cudaGetErrorString(e));
        }
        p->base[r] = (unsigned long long *)ptr;
        p->opened[r] = true;
    }
    cudaDeviceSynchronize();
    return cuda_check("peer open");
}

ch_status ch_peer_destroy(ch_peer *p)
{
    if (!p)
        return CH_OK;
    cudaDeviceSynchronize();
    for (int r = 0; r < p->world; r++)
        if (p->opened[r])
            cudaIpcCloseMemHandle(p->base[r]);
    cudaFree(p->d_buf);
    delete p;
    cudaGetLastError();
    return CH_OK;
}

ch_status ch_filter_step_peer(ch_peer *p, const double *d_xy, int64_t n_local, int64_t index_base, int flags,
                              int64_t *d_survivors, void *d_ws, size_t ws_bytes, void *stream)
{
    return step_peer(p, d_xy, n_local, index_base, flags, d_survivors, d_ws, ws_bytes, stream);
}

ch_status ch_filter_step_peer_f32(ch_peer *p, const float *d_xy, int64_t n_local, int64_t index_base, int flags,
                                  int64_t *d_survivors, void *d_ws, size_t ws_bytes, void *stream)
{
    return step_peer(p, d_xy, n_local, index_base, flags, d_survivors, d_ws, ws_bytes, stream);
}

ch_status ch_peer_counts(ch_peer *p, int64_t *h_counts, int64_t *h_offset, int64_t *h_total, void *stream)
{
    if (!p)
        return fail(CH_ERR_INVALID_ARG, "NULL argument");
    cudaStreamSynchronize((cudaStream_t)stream);
    ch_status s = cuda_check("peer counts");
    if (s != CH_OK)
        return s;
    const size_t bank = (size_t)(p->epoch & 1) * CH_MAX_PEERS * PEER_SLOT;
    std::vector<unsigned long long> buf((size_t)p->world * PEER_SLOT);
    const auto t0 = std::chrono::steady_clock::now();
    while (true) {
        cudaMemcpyAsync(buf.data(), p->d_buf + bank, buf.size() * 8, cudaMemcpyDeviceToHost, (cudaStream_t)stream);
        cudaStreamSynchronize((cudaStream_t)stream);
        bool all = true;
        for (int r = 0; r < p->world; r++)
            all = all && buf[(size_t)r * PEER_SLOT + PEER_CNT_FLAG] == p->epoch;
        if (all)
            break;
        if (std::chrono::steady_clock::now() - t0 > std::chrono::milliseconds(p->timeout_ms))
            return fail(CH_ERR_PEER, "peer exchange timed out (a rank's count did not arrive)");
        std::this_thread::sleep_for(std::chrono::microseconds(50));
    }
    // a7: this rank's exclusive offset in the global order, and the total
    int64_t off = 0, total = 0;
    for (int r = 0; r < p->world; r++) {
        const int64_t c = (int64_t)buf[(size_t)r * PEER_SLOT + PEER_CNT];
        if (h_counts)
            h_counts[r] = c;
        off += r < p->rank ? c : 0;
        total += c;
    }
    if (h_offset)
        *h_offset = off;
    if (h_total)
        *h_total = total;
    return cuda_check("peer counts");
}

ch_status ch_exclusive_offset(const int64_t *h_counts, int world, int rank, int64_t *h_offset, int64_t *h_total)
{
    if (!h_counts || world < 1 || rank < 0 || rank >= world)
        return fail(CH_ERR_INVALID_ARG, "bad counts / world / rank");
    int64_t off = 0, total = 0;
    for (int r = 0; r < world; r++) {
        if (h_counts[r] < 0)
            return fail(CH_ERR_INVALID_ARG, "negative count");
        off += r < rank ? h_counts[r] : 0;
        total += h_counts[r];
    }
    if (h_offset)
        *h_offset = off;
    if (h_total)
        *h_total = total;
    return CH_OK;
}

ch_status ch_filter_host(const double *h_xy, int64_t n, int flags, double *d_xy_staging, int64_t *d_survivors,
                         int64_t *h_survivors, int64_t *h_count, void *d_ws, size_t ws_bytes, void *stream)
{
    if (!h_xy || !h_survivors || !d_xy_staging)
        return fail(CH_ERR_INVALID_ARG, "NULL argument");
    cudaStream_t st = (cudaStream_t)stream;
    if (n > 0) {
        cudaMemcpyAsync(d_xy_staging, h_xy, (size_t)n * 16, cudaMemcpyHostToDevice, st);
        ch_status s0 = cuda_check("h2d copy");
        if (s0 != CH_OK)
            return s0;
    }
    int64_t cnt = 0;
    ch_status s = ch_filter(d_xy_staging, n, flags, d_survivors, &cnt, d_ws, ws_bytes, stream);
    if (s != CH_OK)
        return s;
    if (cnt > 0)
        cudaMemcpyAsync(h_survivors, d_survivors, (size_t)cnt * 8, cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    if ((s = cuda_check("d2h copy")) != CH_OK)
        return s;
    if (h_count)
        *h_count = cnt;
    return CH_OK;
}

ch_status ch_gather_points(const double *d_xy, int64_t index_base, const int64_t *d_idx, int64_t m, double *d_out,
                           void *stream)
{
    if (m < 0 || (m > 0 && (!d_xy || !d_idx || !d_out)))
        return fail(CH_ERR_INVALID_ARG, "bad gather arguments");
    if (m == 0)
        return CH_OK;
    DevInfo di = dev_info();
    long long g = std::min<long long>((m + 255) / 256, (long long)di.sms * 8);
    k_gather<<<(unsigned)g, 256, 0, (cudaStream_t)stream>>>(d_xy, index_base, (const long long *)d_idx, m, d_out);
    return cuda_check("gather");
}

ch_status ch_hull_points(const double *h_pts, const int64_t *h_ids, int64_t m, int64_t *h_hull, int64_t *h_n_hull)
{
    if (m < 0 || !h_n_hull || (m > 0 && (!h_pts || !h_ids || !h_hull)))
        return fail(CH_ERR_INVALID_ARG, "bad hull arguments");
    *h_n_hull = ch_internal_hull(h_pts, h_ids, m, h_hull);
    return CH_OK;
}

static size_t ws_tail_offset(int64_t n) { return (ch_workspace_bytes(n) + 255) & ~(size_t)255; }

size_t ch_hull_workspace_bytes(int64_t n)
{
    return ws_tail_offset(n) + ch_hull_gpu_temp_bytes(n < 1 ? 1 : n);
}

ch_status ch_hull_end_to_end(const double *d_xy, int64_t n, int flags, int64_t *d_survivors, int64_t *h_n_survivors,
                             int64_t *h_hull, int64_t *h_n_hull, ch_stats *h_stats, void *d_ws, size_t ws_bytes,
                             void *stream)
{
    if (!h_hull || !h_n_hull || !d_survivors)
        return fail(CH_ERR_INVALID_ARG, "NULL argument");
    cudaStream_t st = (cudaStream_t)stream;
    // pass 1 and pass 2 timed apart (events between K1 and K2); for n <=
    // 32768 the one-launch step (K5 / K6) counts as pass 1
    cudaEvent_t e0, e1, e2;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventCreate(&e2);
    cudaEventRecord(e0, st);
    int64_t cnt = 0;
    ch_status s;
    const bool one_launch = n <= KC_MAX_N;
    if (one_launch) {
        s = filter_async_impl(d_xy, n, flags & 3, d_survivors, (int64_t *)nullptr, d_ws, ws_bytes, stream);
        cudaEventRecord(e1, st);
    } else {
        s = extremes8_impl(d_xy, n, 0, flags & 3, nullptr, nullptr, nullptr, d_ws, ws_bytes, stream);
        cudaEventRecord(e1, st);
        if (s == CH_OK)
            s = filter_compact_impl(d_xy, n, 0, nullptr, d_survivors, (int64_t *)nullptr, d_ws, ws_bytes, stream);
    }
    cudaEventRecord(e2, st);
    if (s == CH_OK) {
        ch_result res;
        s = ch_read_result(d_ws, &res, stream);
        cnt = res.count;
    }
    float ms_p1 = 0.f, ms_p2 = 0.f;
    if (s == CH_OK) {
        cudaEventSynchronize(e2);
        cudaEventElapsedTime(&ms_p1, e0, e1);
        cudaEventElapsedTime(&ms_p2, e1, e2);
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaEventDestroy(e2);
    if (s != CH_OK)
        return s;
    const float ms_filter = ms_p1 + ms_p2;

    auto t0 = std::chrono::steady_clock::now();
    auto t1 = t0;
    int64_t h = 0;
    if (!(flags & CH_HULL_HOST)) {
        // f1: the hull on the device; only the hull ids come back
        // scratch: the workspace tail when the caller sized it for the hull
        const size_t off = ws_tail_offset(n), tb = ch_hull_gpu_temp_bytes(cnt);
        const bool tail = ws_bytes >= off + tb;
        void *d_tmp = tail ? (void *)((char *)d_ws + off) : nullptr;
        if (!tail && cudaMallocAsync(&d_tmp, tb, st) != cudaSuccess)
            return fail(CH_ERR_CUDA, "cudaMallocAsync for the device hull failed");
        s = ch_hull_gpu(d_xy, n, d_survivors, cnt, h_hull, &h, d_tmp, tb, stream);
        if (!tail)
            cudaFreeAsync(d_tmp, st);
        cudaStreamSynchronize(st);
        if (s != CH_OK)
            return fail(s, "ch_hull_gpu failed");
        t1 = std::chrono::steady_clock::now();
    } else {
    std::vector<double> pts((size_t)cnt * 2);
    std::vector<int64_t> ids((size_t)cnt);
    if (cnt > 0) {
        double *d_pts = nullptr;
        if (cudaMallocAsync((void **)&d_pts, (size_t)cnt * 16, st) != cudaSuccess)
            return fail(CH_ERR_CUDA, "cudaMallocAsync for the hull gather failed");
        if ((s = ch_gather_points(d_xy, 0, d_survivors, cnt, d_pts, stream)) != CH_OK)
            return s;
        cudaMemcpyAsync(pts.data(), d_pts, (size_t)cnt * 16, cudaMemcpyDeviceToHost, st);
        cudaMemcpyAsync(ids.data(), d_survivors, (size_t)cnt * 8, cudaMemcpyDeviceToHost, st);
        cudaFreeAsync(d_pts, st);
        cudaStreamSynchronize(st);
        if ((s = cuda_check("hull gather")) != CH_OK)
            return s;
    }
    t1 = std::chrono::steady_clock::now();
    h = ch_internal_hull(pts.data(), ids.data(), cnt, h_hull);
    }
    auto t2 = std::chrono::steady_clock::now();
    *h_n_hull = h;
    if (h_n_survivors)
        *h_n_survivors = cnt;
    if (h_stats) {
        h_stats->n = n;
        h_stats->n_survivors = cnt;
        h_stats->n_hull = h;
        h_stats->ms_filter = ms_filter;
        h_stats->ms_gather = std::chrono::duration<double, std::milli>(t1 - t0).count();
        h_stats->ms_hull = std::chrono::duration<double, std::milli>(t2 - t1).count();
        h_stats->ms_pass1 = ms_p1;
        h_stats->ms_pass2 = ms_p2;
        h_stats->ms_exchange = 0.0;
    }
    return CH_OK;
}

// Test hook (not part of the documented ABI): the hull's exact orientation.
int ch_orient_sign(double ax, double ay, double bx, double by, double cx, double cy)
{
    extern int ch_internal_orient_sign(double, double, double, double, double, double);
    return ch_internal_orient_sign(ax, ay, bx, by, cx, cy);
}

} // extern "C"

// ================================================ internal API (internal.h) ==
// Host entry points the multi-GPU translation unit (comm.cu) builds its
// steps from.  Not part of the C ABI.
namespace {
__global__ void k_pack_status(const WsHeader *__restrict__ hdr, int empty, long long *__restrict__ w)
{
    if (threadIdx.x == 0) {
        w[0] = empty ? 0 : hdr->result.count;
        w[1] = (empty ? 0 : (hdr->result.nonfinite ? 1 : 0)) | (hdr->peer_timeout ? 2 : 0);
    }
}
__global__ void k_empty_record(unsigned long long *__restrict__ rec)
{
    if (threadIdx.x < 24)
        rec[threadIdx.x] = threadIdx.x < 8 ? ~0ull : 0ull; // idx = -1, x = y = 0
}
} // namespace

namespace chi {

thread_local std::string g_err;

ch_status fail(ch_status s, const std::string &msg)
{
    g_err = msg;
    return s;
}

const char *last_error() { return g_err.c_str(); }

ch_status k1(const void *d_xy, bool f32, int64_t n, int64_t index_base, int flags, void *d_ext_out, void *d_ws,
             size_t ws_bytes, cudaStream_t st)
{
    return f32 ? extremes8_impl((const float *)d_xy, n, index_base, flags, d_ext_out, nullptr, nullptr, d_ws,
                                ws_bytes, (void *)st)
               : extremes8_impl((const double *)d_xy, n, index_base, flags, d_ext_out, nullptr, nullptr, d_ws,
                                ws_bytes, (void *)st);
}

ch_status k3(const void *d_ext_all, int world, int flags, void *d_ws, size_t ws_bytes, cudaStream_t st)
{
    return ch_combine8(d_ext_all, world, flags, d_ws, ws_bytes, (void *)st);
}

ch_status k2(const void *d_xy, bool f32, int64_t n, int64_t index_base, int64_t *d_surv, int64_t *d_count,
             void *d_ws, size_t ws_bytes, cudaStream_t st, bool pdl)
{
    return f32 ? filter_compact_impl((const float *)d_xy, n, index_base, nullptr, d_surv, d_count, d_ws, ws_bytes,
                                     (void *)st, pdl)
               : filter_compact_impl((const double *)d_xy, n, index_base, nullptr, d_surv, d_count, d_ws, ws_bytes,
                                     (void *)st, pdl);
}

ch_status pack_status(const void *d_ws, bool empty, int64_t *d_words, cudaStream_t st)
{
    k_pack_status<<<1, 32, 0, st>>>((const WsHeader *)d_ws, empty ? 1 : 0, (long long *)d_words);
    return cuda_check("pack status");
}

ch_status empty_record(void *d_ext, cudaStream_t st)
{
    k_empty_record<<<1, 32, 0, st>>>((unsigned long long *)d_ext);
    return cuda_check("empty record");
}

const void *ws_extremes(const void *d_ws) { return &((const WsHeader *)d_ws)->ext; }

} // namespace chi
