// radix_sort.cuh -- hand-written LSD radix sort for sm_100a, used by the
// device hull (f1: "a complete parallel convex hull ... on the GPU") to
// put the survivors in x order for the monotone chain (§3.3).
//
// Onesweep-style (one read and one write of keys and values per 8-bit digit
// pass, no separate upsweep):
//   * one kernel quantises the keys and builds the 256-bin histogram of every
//     pass at once (hull_gpu.cu, k_keys_hist);
//   * per pass, each CTA claims the next RS_TILE-item tile with an atomic
//     ticket (so every tile it waits on is already resident) and ranks the
//     tile's items by digit: warp w owns items [RS_WARP_ITEMS w, ...) in
//     RS_ITEMS rounds of 32, and the lanes of a round that share a digit find
//     each other through a shared atomicOr of lane bits, so the rank is stable
//     (tile order).  It publishes the tile's per-digit counts; a decoupled
//     look-back (one thread per digit) over earlier tiles' counts gives the
//     tile's global offset per digit; the tile is reordered by digit in
//     shared memory and written out, so lanes with the same digit write
//     consecutive addresses.
//   * status words are {flag:2, pass tag:2, count:60}: one memset per sort
//     clears them, the tag keeps a pass from reading the previous pass's
//     words.
// cta_sort_pass: the same ranking inside ONE CTA over a segment of global
// memory, tiles in order (no look-back) -- the device hull's fallback for runs
// of equal quantised keys longer than a thread sorts by itself.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace chrs {

#ifdef CH_RS_STATS
// debug build only: look-back windows read, windows re-read (unpublished), tiles
__device__ unsigned long long g_rs_stats[4];
#endif

constexpr int RS_BINS = 256;
constexpr int RS_THREADS = 256; // one thread per digit in the per-digit steps
constexpr int RS_WARPS = RS_THREADS / 32;
#ifndef RS_ITEMS_N
#define RS_ITEMS_N 24 // keys per thread per tile (A/B: 8 -> 4.79, 12 -> 3.61, 16 -> 3.12, 24 -> 2.97 ms for 4 passes at 1e8)
#endif
constexpr int RS_ITEMS = RS_ITEMS_N;
constexpr int RS_TILE = RS_THREADS * RS_ITEMS;
constexpr int RS_WARP_ITEMS = 32 * RS_ITEMS;
constexpr int RS_LOOKBACK = 4; // earlier tiles read per look-back round trip
#ifndef RS_PACK
#define RS_PACK 1 // 32-bit keys with 32-bit values: one 64-bit shared word per item in the reorder
#endif
#ifndef RS_MINB
#define RS_MINB 2 // resident CTAs per SM the pass kernel's registers are bounded for
#endif
static_assert(RS_THREADS == RS_BINS, "one thread per digit");

constexpr unsigned long long RS_FLAG_AGG = 1ull << 62;  // this tile's count only
constexpr unsigned long long RS_FLAG_INC = 2ull << 62;  // count of this and every earlier tile
constexpr unsigned long long RS_COUNT = (1ull << 60) - 1;

template <typename K, typename V> struct TileSmem {
    K key[RS_TILE];
    V val[RS_TILE];
    unsigned whist[RS_WARPS][RS_BINS]; // per-warp digit counts, then per-warp exclusive offsets
    unsigned match[2][RS_WARPS][RS_BINS]; // per-warp lane masks by digit (two rounds in flight), zero between uses
    unsigned cnt[RS_BINS];             // the tile's count per digit
    unsigned excl[RS_BINS];            // tile-local exclusive offset per digit
    long long gofs[RS_BINS];           // output position of the digit's item j is gofs[d] + j
    unsigned wsum[RS_WARPS];
    unsigned long long wsum64[RS_WARPS];
    unsigned long long lo, hi, tile;
};

__device__ __forceinline__ unsigned lanemask_lt()
{
    unsigned m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

template <typename K> __device__ __forceinline__ unsigned digit_of(K k, int shift)
{
    return (unsigned)(k >> shift) & (RS_BINS - 1);
}

// The lanes of the (full) warp whose 8-bit digit d equals this lane's, among
// the lanes with the same `ok`: one ballot per bit (__match_any_sync measured
// several times slower here).
__device__ __forceinline__ unsigned match_digit(unsigned d, bool ok)
{
    const unsigned okm = __ballot_sync(0xffffffffu, ok);
    unsigned peers = ok ? okm : ~okm;
#pragma unroll
    for (int b = 0; b < 8; b++) {
        const bool bit = (d >> b) & 1u;
        const unsigned bal = __ballot_sync(0xffffffffu, bit);
        peers &= bit ? bal : ~bal;
    }
    return peers;
}

__device__ __forceinline__ void st_volatile(unsigned long long *p, unsigned long long v)
{
    *(volatile unsigned long long *)p = v;
}
__device__ __forceinline__ unsigned long long ld_volatile(const unsigned long long *p)
{
    return *(const volatile unsigned long long *)p;
}

// Block-wide exclusive scan of one value per thread (RS_THREADS threads).
template <typename T> __device__ __forceinline__ T block_excl_scan(T v, T *wsum)
{
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    T incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const T t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o)
            incl += t;
    }
    if (lane == 31)
        wsum[w] = incl;
    __syncthreads();
    T base = 0;
#pragma unroll
    for (int i = 0; i < RS_WARPS; i++)
        if (i < w)
            base += wsum[i];
    __syncthreads(); // wsum is reused by the next scan
    return base + incl - v;
}

// Ranks a tile of items held in registers (item i of lane l of warp w sits at
// tile position RS_WARP_ITEMS w + 32 i + l; items at 32 i + l >= nv, the
// warp's valid count, are past the end).  Per round the lanes sharing a digit
// find each other through a shared-memory atomicOr of their lane bits (the
// first lane of the group then clears the word; rounds alternate between two
// mask arrays, so two warp barriers per round suffice).  On return (after a
// block barrier): rank[i] = the item's place among its warp's items with the
// same digit, s.whist[w][d] = the tile position of warp w's first digit-d item
// (the tile's exclusive digit offset s.excl[d] plus the warp's offset among
// the tile's digit-d items), s.cnt[d], s.excl[d].
template <typename K, typename V>
__device__ __forceinline__ void rank_tile(TileSmem<K, V> &s, const K (&k)[RS_ITEMS], int nv,
                                          unsigned (&rank)[RS_ITEMS], int shift)
{
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int b = threadIdx.x; b < RS_WARPS * RS_BINS; b += RS_THREADS)
        (&s.whist[0][0])[b] = 0;
    __syncthreads();
    const unsigned lt = lanemask_lt();
#pragma unroll
    for (int i = 0; i < RS_ITEMS; i++) {
        const bool ok = 32 * i + lane < nv;
        const unsigned d = digit_of(k[i], shift);
        unsigned *mw = &s.match[i & 1][w][d];
        if (ok)
            atomicOr(mw, 1u << lane);
        __syncwarp();
        unsigned peers = 0, old = 0;
        if (ok) {
            peers = *mw;
            old = s.whist[w][d];
        }
        __syncwarp();
        if (ok && (peers & lt) == 0) {
            s.whist[w][d] = old + __popc(peers);
            *mw = 0;
        }
        rank[i] = old + __popc(peers & lt);
    }
    __syncthreads();
    const int d = threadIdx.x;
    unsigned run = 0;
#pragma unroll
    for (int ww = 0; ww < RS_WARPS; ww++) {
        const unsigned c = s.whist[ww][d];
        s.whist[ww][d] = run;
        run += c;
    }
    s.cnt[d] = run;
    const unsigned ex = block_excl_scan<unsigned>(run, s.wsum);
    s.excl[d] = ex;
#pragma unroll
    for (int ww = 0; ww < RS_WARPS; ww++)
        s.whist[ww][d] += ex; // now the tile position of warp ww's first digit-d item
    __syncthreads();
}

// The ranked tile reordered by digit in shared memory; each value is read
// from vsrc at its item's position here (not held through the ranking).
template <typename K, typename V>
__device__ __forceinline__ void local_scatter(TileSmem<K, V> &s, const K (&k)[RS_ITEMS], const V *__restrict__ vsrc,
                                              long long wb, int nv, const unsigned (&rank)[RS_ITEMS], int shift)
{
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
    for (int i = 0; i < RS_ITEMS; i++)
        if (32 * i + lane < nv) {
            const unsigned d = digit_of(k[i], shift);
            const unsigned pos = s.whist[w][d] + rank[i];
            if constexpr (RS_PACK && sizeof(K) == 4 && sizeof(V) == 4) {
                // key and value as one 64-bit word (the key and value arrays
                // are contiguous: 2 RS_TILE words)
                reinterpret_cast<unsigned long long *>(s.key)[pos] =
                    ((unsigned long long)vsrc[wb + 32 * i] << 32) | (unsigned)k[i];
            } else {
                s.key[pos] = k[i];
                s.val[pos] = vsrc[wb + 32 * i];
            }
        }
}

// One digit pass over m items: kin/vin -> kout/vout, stable.  hist: the
// pass's global digit counts; status: ceil(m / RS_TILE) * RS_BINS words,
// cleared before the first pass of the sort; ticket: zero before this pass.
// One tile per CTA (grid ceil(m / RS_TILE)); O: output offset type (unsigned
// when m < 2^32).  Dynamic smem sizeof(TileSmem).
template <typename K, typename V, typename O>
__global__ void __launch_bounds__(RS_THREADS, RS_MINB) k_rs_pass(const K *__restrict__ kin, K *__restrict__ kout,
                                                              const V *__restrict__ vin, V *__restrict__ vout,
                                                              long long m, int shift, int tag,
                                                              const unsigned long long *__restrict__ hist,
                                                              unsigned long long *status, unsigned long long *ticket,
                                                              const long long *__restrict__ dm = nullptr)
{
    // dm (nullable): the key count is on the device (<= m; the grid is sized for m)
    if (dm)
        m = *dm < m ? *dm : m;
    extern __shared__ __align__(16) unsigned char rs_smem[];
    TileSmem<K, V> &s = *reinterpret_cast<TileSmem<K, V> *>(rs_smem);
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31, d = threadIdx.x;
    if (threadIdx.x == 0)
        s.tile = atomicAdd(ticket, 1ull);
    for (int b = threadIdx.x; b < 2 * RS_WARPS * RS_BINS; b += RS_THREADS)
        (&s.match[0][0][0])[b] = 0;
    __syncthreads();
    const long long tile = (long long)s.tile;
    const long long base = tile * RS_TILE;
    if (base >= m)
        return;
    K k[RS_ITEMS];
    unsigned rank[RS_ITEMS];
    const long long wb = base + (long long)w * RS_WARP_ITEMS + lane;
    const long long wrem = m - (base + (long long)w * RS_WARP_ITEMS);
    const int nv = wrem >= RS_WARP_ITEMS ? RS_WARP_ITEMS : (wrem > 0 ? (int)wrem : 0);
#pragma unroll
    for (int i = 0; i < RS_ITEMS; i++)
        k[i] = 32 * i + lane < nv ? kin[wb + 32 * i] : (K)0;
    rank_tile(s, k, nv, rank, shift);

    // publish this tile's counts, then look back for the earlier tiles':
    // windows of up to RS_LOOKBACK earlier tiles (independent loads), summed
    // down to the window's latest inclusive word; a window with an
    // unpublished word is re-read
    const unsigned long long c = s.cnt[d];
    const unsigned long long tg = (unsigned long long)(tag & 3) << 60;
    unsigned long long *my = status + tile * RS_BINS + d;
    st_volatile(my, (tile == 0 ? RS_FLAG_INC : RS_FLAG_AGG) | tg | c);
    const unsigned long long hb = block_excl_scan<unsigned long long>(hist[d], s.wsum64);
    unsigned long long pre = 0;
    if (tile > 0) {
        long long p = tile - 1;
        while (true) {
            const int nw = p >= RS_LOOKBACK - 1 ? RS_LOOKBACK : (int)p + 1;
            unsigned long long wv[RS_LOOKBACK];
#pragma unroll
            for (int u = 0; u < RS_LOOKBACK; u++)
                wv[u] = u < nw ? ld_volatile(status + (p - u) * RS_BINS + d) : 0;
            unsigned long long sum = 0;
            bool ready = true, inc = false;
#pragma unroll
            for (int u = 0; u < RS_LOOKBACK; u++) {
                if (u >= nw || inc || !ready)
                    continue;
                const unsigned long long f = wv[u] & (3ull << 62);
                if (f == 0 || (wv[u] & (3ull << 60)) != tg) {
                    ready = false; // not published for this pass yet
                    continue;
                }
                sum += wv[u] & RS_COUNT;
                inc = f == RS_FLAG_INC;
            }
#ifdef CH_RS_STATS
            atomicAdd(&g_rs_stats[ready ? 0 : 1], 1ull);
#endif
            if (!ready)
                continue;
            pre += sum;
            if (inc)
                break;
            p -= nw;
        }
        st_volatile(my, RS_FLAG_INC | tg | (pre + c));
#ifdef CH_RS_STATS
        const long long ntiles = (m + RS_TILE - 1) / RS_TILE;
        if (d == 0 && atomicAdd(&g_rs_stats[2], 1ull) + 2 == (unsigned long long)ntiles)
            printf("rs_stats pass tag %d: tiles %lld windows %llu (per digit-tile %.2f) unpublished re-reads %llu\n",
                   tag, ntiles, g_rs_stats[0], (double)g_rs_stats[0] / RS_BINS / ntiles, g_rs_stats[1]);
#endif
    }
    O *gofs = reinterpret_cast<O *>(s.gofs);
    gofs[d] = (O)(hb + pre) - (O)s.excl[d];
    local_scatter(s, k, vin, wb, nv, rank, shift);
    __syncthreads();
    const int nvalid = (int)(m - base < RS_TILE ? m - base : RS_TILE);
    for (int j = threadIdx.x; j < nvalid; j += RS_THREADS) {
        K kk;
        V vv;
        if constexpr (RS_PACK && sizeof(K) == 4 && sizeof(V) == 4) {
            const unsigned long long kv = reinterpret_cast<const unsigned long long *>(s.key)[j];
            kk = (K)(unsigned)kv;
            vv = (V)(kv >> 32);
        } else {
            kk = s.key[j];
            vv = s.val[j];
        }
        const O g = gofs[digit_of(kk, shift)] + (O)j;
        kout[g] = kk;
        vout[g] = vv;
    }
}

// One digit pass of a single CTA over the segment [a, a + L) of kin/vin into
// the same segment of kout/vout, stable.  Returns false (and writes nothing)
// when every key has the same digit (the pass is the identity).
template <typename K, typename V>
__device__ bool cta_sort_pass(TileSmem<K, V> &s, const K *kin, K *kout, const V *vin, V *vout, long long a, long long L,
                              int shift)
{
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31, d = threadIdx.x;
    // histogram of the segment (cnt as scratch)
    s.cnt[d] = 0;
    for (int b = threadIdx.x; b < 2 * RS_WARPS * RS_BINS; b += RS_THREADS)
        (&s.match[0][0][0])[b] = 0;
    __syncthreads();
    const unsigned lt = lanemask_lt();
    for (long long t0 = 0; t0 < L; t0 += RS_THREADS) {
        const long long t = t0 + threadIdx.x;
        const bool okk = t < L;
        const unsigned dd = okk ? digit_of(kin[a + t], shift) : 0u;
        const unsigned peers = match_digit(dd, okk);
        if (okk && (peers & lt) == 0)
            atomicAdd(&s.cnt[dd], (unsigned)__popc(peers));
    }
    __syncthreads();
    const unsigned long long hc = s.cnt[d];
    if (__syncthreads_or(hc == (unsigned long long)L))
        return false;
    // running output offset per digit, advanced tile by tile
    s.gofs[d] = (long long)block_excl_scan<unsigned long long>(hc, s.wsum64);
    __syncthreads();
    for (long long c0 = 0; c0 < L; c0 += RS_TILE) {
        K k[RS_ITEMS];
        unsigned rank[RS_ITEMS];
        const long long wb = a + c0 + (long long)w * RS_WARP_ITEMS + lane;
        const long long wrem = L - (c0 + (long long)w * RS_WARP_ITEMS);
        const int nv = wrem >= RS_WARP_ITEMS ? RS_WARP_ITEMS : (wrem > 0 ? (int)wrem : 0);
#pragma unroll
        for (int i = 0; i < RS_ITEMS; i++)
            k[i] = 32 * i + lane < nv ? kin[wb + 32 * i] : (K)0;
        rank_tile(s, k, nv, rank, shift);
        local_scatter(s, k, vin, wb, nv, rank, shift);
        __syncthreads();
        const int nvalid = (int)(L - c0 < RS_TILE ? L - c0 : RS_TILE);
        for (int j = threadIdx.x; j < nvalid; j += RS_THREADS) {
            const K kk = s.key[j];
            const unsigned dd = digit_of(kk, shift);
            const long long g = a + s.gofs[dd] + (j - (long long)s.excl[dd]);
            kout[g] = kk;
            vout[g] = s.val[j];
        }
        __syncthreads();
        s.gofs[d] += s.cnt[d];
        __syncthreads();
    }
    return true;
}

} // namespace chrs
