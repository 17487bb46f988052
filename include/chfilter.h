/*
 * chfilter.h -- C ABI of the B200-native convex-hull pre-filter
 * (Carrasco, Ferrada, Navarro, Hitschfeld, arXiv 2303.10581).
 *
 * Citations: "P:<line>" = PAPER.md line, "S:<line>" = SPEC.md line (both in
 * the paper's source bundle), "DESIGN Rk" = reading k in DESIGN.md.
 *
 * The library computes Algorithm 1:
 *   line 1  findingPolygon          -> ch_extremes8  (+ ch_octagon_build)
 *   line 2  buildingFilter          -> ch_octagon_filter (bit vector)
 *   line 3  compactingFilteredPoints-> ch_filter_compact (fused with line 2)
 *   line 4  convexHull_algorithm    -> ch_hull_end_to_end
 *
 * Conventions (all entry points):
 *  - Points are float64 AoS: point i is (xy[2i], xy[2i+1]); the array must be
 *    16-byte aligned (CH_ERR_MISALIGNED otherwise).  n and every index are
 *    int64 (n > 2^31 is supported).
 *  - "d_" pointers are device memory of the current CUDA device, "h_" host.
 *    The caller owns every buffer; the library never allocates device memory
 *    on hot calls and never frees caller memory.
 *  - Scratch lives in a caller-provided workspace of ch_workspace_bytes(n)
 *    bytes, zero-filled once before first use (ch_workspace_init).  A
 *    workspace must not be used by two calls concurrently; calls on distinct
 *    workspaces are reentrant.
 *  - `stream` is a cudaStream_t passed as void* (NULL = legacy default).
 *    Calls enqueue asynchronously unless they fill a host output ("h_"),
 *    in which case they synchronize that stream before returning.
 *  - Errors are returned as ch_status; nothing is thrown.  On error the
 *    outputs are unspecified; ch_last_error() gives a thread-local detail.
 *    Non-finite coordinates are detected inside the first pass and reported
 *    (CH_ERR_NONFINITE) by the next call that synchronizes.
 *  - Degenerate input (fewer than 3 distinct octagon vertices) is not an
 *    error: every point survives (DESIGN R6).
 *  - Arithmetic: binary64, round-to-nearest-even, no FMA contraction, in the
 *    order stated for each step.  Results are bit-identical to the sequential
 *    definition (DESIGN.md section "Readings") for every grid shape and
 *    world size.
 */
#ifndef CHFILTER_H
#define CHFILTER_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CH_ABI_VERSION 3 /* 2: ch_comm_* (NCCL), ch_gather_survivors, ch_peer_counts with offsets, ch_stats pass times;
                            3: ch_octagon's fp32 certificate as scaled edges with one keep bound */

typedef enum {
    CH_OK = 0,
    CH_ERR_INVALID_ARG = 1,
    CH_ERR_EMPTY = 2,      /* n == 0 (S:75 EmptySet)                    */
    CH_ERR_NONFINITE = 3,  /* a NaN / infinite coordinate        */
    CH_ERR_MISALIGNED = 4, /* d_xy not 16-byte aligned                  */
    CH_ERR_WORKSPACE = 5,  /* workspace missing or too small            */
    CH_ERR_CUDA = 6,       /* a CUDA runtime error (see ch_last_error)  */
    CH_ERR_PEER = 7,       /* peer exchange: a rank's record did not arrive (timeout) */
    CH_ERR_NCCL = 8        /* NCCL missing, or an NCCL call failed (see ch_last_error) */
} ch_status;

/* Predicate switch (DESIGN R4).  Default: certified thresholds T_k. */
#define CH_CERTIFIED 0
#define CH_PLAIN 1 /* T_k = 0: the plain fp64 test (not hull-safe adversarially) */
#define CH_EXACT 2 /* f3: discard iff the EXACT orientation is > 0 on
                      every edge -- the maximal hull-safe discard.  Certified T_k and
                      Shewchuk's per-point bound decide all but a thin band, which is
                      evaluated with exact expansion arithmetic on the device. */

/* The eight extremes, slot order R, TR, T, TL, L, BL, B, BR:
 *   R = argmax x, TR = argmax fl(x+y), T = argmax y, TL = argmin fl(x-y),
 *   L = argmin x, BL = argmin fl(x+y), B = argmin y, BR = argmax fl(x-y);
 * ties go to the lowest global index, -0.0 == +0.0 (DESIGN R1, R2). */
typedef struct {
    int64_t idx[8]; /* global point index                                  */
    double x[8];    /* coordinates of that point                           */
    double y[8];
} ch_extremes;      /* 192 bytes */

/* The discard polygon ("counterclockwise"; DESIGN R5).  Vertices are
 * the cycle [R,TR,T,TL,L,BL,B,BR] with consecutive duplicates (and trailing
 * copies of the first) removed.  Edge k runs from v[k] to v[(k+1) % nv]:
 *   ex = fl(vx[k+1] - vx[k]),  ey = fl(vy[k+1] - vy[k]),
 *   thr = T_k = 2^-50 * fl(fl(|ex| Y) + fl(|ey| X)) (certified) or 0 (plain),
 *   X = max(fl(xmax - vx[k]), fl(vx[k] - xmin)), Y likewise in y.
 * A point is discarded iff for every k
 *   D_k = fl(fl(ex * fl(y - vy[k])) - fl(ey * fl(x - vx[k]))) > thr[k].
 * box/has_box: a closed axis box on which every D_k > thr[k] was verified at
 * the four corners (D_k is monotone in x and in y under round-to-nearest, so
 * the corners bound it); points inside it are discarded without edge tests.
 * It never changes a result.  guess_edge/cx/cy: the octant of (x-cx, y-cy)
 * picks the edge tested first (a pure speed hint).
 * f32_*: an fp32 pre-filter with static error bounds (DESIGN.md "fp32
 * certification"), edge k scaled by an exact power of two 2^s_k so that
 * max(|a|, |b|) is in [1, 2): v_k = fma(a, fl32(x), fma(b, fl32(y), c)) >= 0
 * proves D_k > thr[k], v_k < -f32_dk[k] proves D_k < thr[k] (CH_EXACT:
 * < -thr[k]); with G = min_k v_k, G >= 0 proves the point is discarded and
 * G + f32_delta < 0 that it is kept; otherwise D_k is evaluated in fp64.  Valid only for
 * points inside bbox, so the kernels use it only with octagons they built
 * themselves from the same points (has_f32 is cleared on a caller-supplied
 * octagon; a workspace octagon is tagged with the (pointer, n, index_base) it
 * was built from, and K2 uses its fp32 stage only on those points).  It never
 * changes a result.
 * A caller-supplied octagon (h_oct != NULL below) is validated on the host:
 * nv outside [0, 8] or degenerate != (nv < 3) is CH_ERR_INVALID_ARG; its box
 * is kept only if every corner passes every edge test (else no box is used);
 * guess_edge entries outside [0, nv) become 0. */
typedef struct {
    int32_t nv;
    int32_t degenerate;
    int64_t vidx[8];
    double vx[8], vy[8];
    double ex[8], ey[8], thr[8];
    double bbox[4];    /* xmin, xmax, ymin, ymax                         */
    double box[4];     /* x0, x1, y0, y1 (closed)                        */
    int32_t has_box;
    int32_t plain;     /* 1 if built with CH_PLAIN                       */
    int32_t guess_edge[8];
    double cx, cy;
    float f32_a[8], f32_b[8], f32_c[8]; /* fp32 certificate of edge k scaled by 2^s_k */
    float f32_dk[8];   /* edge k's keep bound (scaled)                   */
    float f32_delta;   /* max over the edges of f32_dk                   */
    int32_t has_f32;
    int32_t exact;     /* 1 if built with CH_EXACT                       */
} ch_octagon;

/* Result of the last filter call on a workspace (device-resident copy in the
 * workspace; read with ch_read_result). */
typedef struct {
    int64_t count;      /* number of survivors                            */
    int32_t nonfinite;  /* 1 if a non-finite coordinate was seen          */
    int32_t degenerate; /* 1 if the octagon had < 3 distinct vertices     */
} ch_result;

typedef struct {
    int64_t n, n_survivors, n_hull;
    double ms_filter;   /* extremes + octagon + filter + compaction (device)       */
    double ms_gather;   /* survivor coordinates to the hull stage (host or root)    */
    double ms_hull;     /* the exact hull (device or host)                          */
    double ms_pass1;    /* pass 1: K1 extremes + octagon (device events)            */
    double ms_pass2;    /* pass 2: K2 octagon test + compaction (device events)     */
    double ms_exchange; /* multi-GPU: extremes all-gather + K3 + count all-gather   */
} ch_stats;

int ch_abi_version(void);
const char *ch_status_str(ch_status s);
const char *ch_last_error(void); /* thread-local, valid until the next call */

/* Diagnostics: resident CTAs per SM the streaming kernels launch with, from
 * the CUDA occupancy API on the current device (kernel 0 = K1, 1 = K2 on
 * float64 points, 2 = K2 on float32 points).  K1 runs 3 and K2 2 per SM by
 * design; a smaller number means a resource regression.
 * Returns < 0 for an unknown kernel or a CUDA error. */
int ch_occupancy(int kernel);

/* Bytes of workspace needed for inputs of up to n points. */
size_t ch_workspace_bytes(int64_t n);
/* Zero-fill a workspace (once, before first use).  Async on `stream`. */
ch_status ch_workspace_init(void *d_ws, size_t ws_bytes, void *stream);

/* Algorithm 1 line 1: the eight extremes of d_xy[0..n) in one
 * pass, indices offset by index_base (a shard's global offset), then the
 * octagon (flags: CH_CERTIFIED or CH_PLAIN) built on the device into the
 * workspace.  If d_ext_out != NULL the extremes are also written there as a
 * device ch_extremes (for the multi-GPU exchange).  If h_ext != NULL and/or
 * h_oct != NULL the call synchronizes and copies them out (and reports
 * CH_ERR_NONFINITE). */
ch_status ch_extremes8(const double *d_xy, int64_t n, int64_t index_base, int flags,
                       void *d_ext_out, ch_extremes *h_ext, ch_octagon *h_oct,
                       void *d_ws, size_t ws_bytes, void *stream);

/* Multi-GPU exchange step (north_star): combine W device ch_extremes records
 * (d_ext_all, contiguous, one per rank -- e.g. the output of an all-gather)
 * with the same ordering (best key, then lowest global index), and build the
 * octagon into the workspace.  Bit-identical to a single-GPU ch_extremes8
 * over the concatenated shards.  d_xy is not needed (coordinates travel in
 * the records). */
ch_status ch_combine8(const void *d_ext_all, int world, int flags,
                      void *d_ws, size_t ws_bytes, void *stream);

/* Host-side octagon assembly (DESIGN R5): pure, no CUDA. */
ch_status ch_octagon_build(const ch_extremes *ext, int flags, ch_octagon *out);

/* Algorithm 1 line 2: the paper's n-bit flag vector.
 * Bit (i % 32) of d_keep_bits[i / 32] is 1 iff point i survives; the padding
 * bits of the last word are 0.  h_oct == NULL uses the workspace octagon
 * from the last ch_extremes8 / ch_combine8 on d_ws. */
ch_status ch_octagon_filter(const double *d_xy, int64_t n, const ch_octagon *h_oct,
                            uint32_t *d_keep_bits, void *d_ws, size_t ws_bytes, void *stream);

/* Algorithm 1 lines 2-3 fused: the octagon test and a
 * single-pass stable stream compaction.  Writes the survivors as int64
 * global indices (index_base + i) in increasing order to d_survivors
 * (capacity n) and their count to *d_count (device, nullable) and to the
 * workspace result.  h_oct == NULL uses the workspace octagon. */
ch_status ch_filter_compact(const double *d_xy, int64_t n, int64_t index_base,
                            const ch_octagon *h_oct, int64_t *d_survivors, int64_t *d_count,
                            void *d_ws, size_t ws_bytes, void *stream);

/* float32 storage (the paper's precision): the same
 * three calls on AoS float32 points (8 B/pt, 16-byte aligned base).  Each
 * coordinate is widened to double exactly, so every result equals the
 * float64 call on the widened array (and the oracle on it). */
ch_status ch_extremes8_f32(const float *d_xy, int64_t n, int64_t index_base, int flags,
                           void *d_ext_out, ch_extremes *h_ext, ch_octagon *h_oct,
                           void *d_ws, size_t ws_bytes, void *stream);
ch_status ch_filter_compact_f32(const float *d_xy, int64_t n, int64_t index_base,
                                const ch_octagon *h_oct, int64_t *d_survivors, int64_t *d_count,
                                void *d_ws, size_t ws_bytes, void *stream);
ch_status ch_filter_f32(const float *d_xy, int64_t n, int flags, int64_t *d_survivors,
                        int64_t *h_count, void *d_ws, size_t ws_bytes, void *stream);

/* Synchronize `stream` and copy the workspace result to the host.  Returns
 * CH_ERR_NONFINITE if the last pass saw a non-finite coordinate. */
ch_status ch_read_result(const void *d_ws, ch_result *h_res, void *stream);

/* Synchronize `stream` and copy the eight extremes and the octagon (Algorithm
 * 1 line 1) that the last step on this workspace built on the
 * device (K1's last CTA, K3, K5 or K6) to the host.  Either pointer may be
 * NULL.  Unspecified before the first step. */
ch_status ch_read_octagon(const void *d_ws, ch_extremes *h_ext, ch_octagon *h_oct, void *stream);

/* One filter step on device-resident input: ch_extremes8 + ch_filter_compact
 * (two kernels, no host round trip in between; one launch -- K5, or K6 -- for
 * n <= 32768, see ch_filter_async)
 * + ch_read_result. */
ch_status ch_filter(const double *d_xy, int64_t n, int flags, int64_t *d_survivors,
                    int64_t *h_count, void *d_ws, size_t ws_bytes, void *stream);

/* The same step without synchronizing: the count goes to *d_count (device,
 * nullable) and to the workspace result.  For n <= 2048 the whole step runs
 * as ONE single-CTA kernel (K5); for n <= 32768 (the latency-bound C1 case)
 * as ONE launch of an 8-CTA thread-block cluster (K6: extremes combined and
 * the octagon shared through distributed shared memory); above, K1 + K2.
 * _f32: float32 storage. */
ch_status ch_filter_async(const double *d_xy, int64_t n, int flags, int64_t *d_survivors,
                          int64_t *d_count, void *d_ws, size_t ws_bytes, void *stream);
ch_status ch_filter_async_f32(const float *d_xy, int64_t n, int flags, int64_t *d_survivors,
                              int64_t *d_count, void *d_ws, size_t ws_bytes, void *stream);

/* The step of ch_filter_async captured once into a CUDA graph, then replayed
 * with one launch per step (Blackwell: a graph launch costs one host call
 * for the whole K1 + K2, K5 or K6 sequence, the point of the latency-bound C1
 * config).  Capture happens on a private stream; the arguments (pointers,
 * n, flags) are baked into the graph, so the caller keeps the buffers alive
 * and unchanged in place until ch_graph_destroy.  *out receives an opaque
 * handle owned by the caller.  Errors: the ch_filter_async ones, or
 * CH_ERR_CUDA if capture / instantiation fails.  ch_graph_launch enqueues one
 * step on `stream` (asynchronous, like ch_filter_async). */
typedef struct ch_graph ch_graph;
ch_status ch_filter_graph_create(const double *d_xy, int64_t n, int flags, int64_t *d_survivors,
                                 int64_t *d_count, void *d_ws, size_t ws_bytes, ch_graph **out);
ch_status ch_filter_graph_create_f32(const float *d_xy, int64_t n, int flags, int64_t *d_survivors,
                                     int64_t *d_count, void *d_ws, size_t ws_bytes, ch_graph **out);
ch_status ch_graph_launch(ch_graph *g, void *stream);
ch_status ch_graph_destroy(ch_graph *g);

/* ---- Multi-GPU with the exchanges fused into the kernels (north_star a4, a7;
 * SURVEY 8(e) "v2") ------------------------------------------------------------
 * One process per GPU, points sharded by contiguous index ranges.  Every rank
 * owns a small exchange buffer (2 banks x CH_MAX_PEERS slots x 256 B), exported
 * with cudaIpcGetMemHandle and opened by every peer (NVLink / NVSwitch peer
 * memory; on one GPU shared by several processes, plain device memory).
 *   K1's last CTA stores its eight extremes (one ch_extremes record) straight
 *   into slot[rank] of every peer's buffer, then a release flag (the step
 *   epoch) -- the all-gather of a4 without a collective launch;
 *   K3 (one CTA) acquires the W flags of its own buffer and combines the W
 *   records into the global octagon, identically on every rank;
 *   K2's last CTA stores the survivor count into every peer's slot[rank]
 *   (a7), read back on the host by ch_peer_counts.
 * Banks alternate with the step epoch (a rank can run at most one step ahead
 * of a peer's reads).  Waits time out after 60 s (or $CH_PEER_TIMEOUT_MS at
 * ch_peer_create) with CH_ERR_PEER from the next
 * ch_read_result / ch_peer_counts) instead of hanging.
 *   ch_peer_create: allocates the buffer, writes its IPC handle (64 bytes,
 *     ch_peer_handle_bytes()) to h_handle.  ch_peer_open: takes the world
 *     handles in rank order (the caller all-gathers them, e.g. with
 *     torch.distributed) and opens the peers'.  Both synchronize.
 *   ch_filter_step_peer: one sharded step on `stream` (asynchronous); n_local
 *     may be 0 (an empty shard still takes part).  index_base = the shard's
 *     first global index.  d_survivors: global indices, increasing.
 *   ch_peer_counts: synchronizes `stream`, then waits for every rank's count of
 *     the last step; h_counts[world] in rank order (exclusive scan = offsets). */
#define CH_MAX_PEERS 16
typedef struct ch_peer ch_peer;
size_t ch_peer_handle_bytes(void);
ch_status ch_peer_create(int rank, int world, ch_peer **out, void *h_handle);
ch_status ch_peer_open(ch_peer *p, const void *h_handles);
ch_status ch_peer_destroy(ch_peer *p);
ch_status ch_filter_step_peer(ch_peer *p, const double *d_xy, int64_t n_local, int64_t index_base, int flags,
                              int64_t *d_survivors, void *d_ws, size_t ws_bytes, void *stream);
ch_status ch_filter_step_peer_f32(ch_peer *p, const float *d_xy, int64_t n_local, int64_t index_base, int flags,
                                  int64_t *d_survivors, void *d_ws, size_t ws_bytes, void *stream);
/* h_counts[world] (nullable): every rank's count; h_offset / h_total
 * (nullable): this rank's exclusive offset in the global survivor order and
 * the total (a7's scan, done here). */
ch_status ch_peer_counts(ch_peer *p, int64_t *h_counts, int64_t *h_offset, int64_t *h_total, void *stream);

/* a7's scan for callers that exchange the counts themselves (host, pure):
 * *h_offset = sum of h_counts[0..rank), *h_total = sum of h_counts[0..world). */
ch_status ch_exclusive_offset(const int64_t *h_counts, int world, int rank, int64_t *h_offset, int64_t *h_total);

/* ---- Multi-GPU over a library-owned NCCL communicator (north_star: "a tiny
 * NCCL allgather ... survivor counts are exclusive-scanned to gather
 * survivors") ------------------------------------------------
 * One process per GPU.  NCCL is loaded at run time (the libnccl.so.2 the
 * process already has, e.g. PyTorch's, else the system one); without it these
 * calls return CH_ERR_NCCL and everything else still works.
 *   ch_comm_unique_id: rank 0 creates the 128-byte ncclUniqueId; the caller
 *     broadcasts it (e.g. torch.distributed) -- the only bytes that cross the
 *     caller's transport.  ch_comm_init: collective over the `world` ranks;
 *     binds `device` (cudaSetDevice) and allocates the communicator's own
 *     ~1 KB of device buffers.  ch_comm_nccl_version: NCCL_VERSION_CODE of the
 *     loaded library, or -1.
 *   ch_filter_compact_dist: one sharded step (rows a1-a7): K1 on the shard
 *     (global indices, shard = DESIGN R14: rank r owns [floor(r n/W),
 *     floor((r+1) n/W)), n_local must be that size, may be 0), ncclAllGather
 *     of the 192-byte extremes records, K3 (combine + octagon, identical on
 *     every rank, bit-identical to 1 GPU), K2 on the shard, ncclAllGather of
 *     {count, flags}, and the exclusive scan on the device.
 *     d_survivors_local: this shard's survivors as increasing GLOBAL indices.
 *     h_count_local / h_offset / h_total / h_ext (global extremes), all
 *     nullable: if any is given the call synchronizes `stream` and returns
 *     CH_ERR_NONFINITE on EVERY rank if any shard held a non-finite
 *     coordinate; if none is given the call is asynchronous and
 *     ch_comm_result reads the outcome later.
 *   ch_comm_result: synchronizes `stream`; h_counts[world] (every rank's
 *     count), this rank's offset, the total; the same status rule.
 *   ch_comm_step_times: device-event times of the last step's phases.
 *   ch_gather_survivors (the hull stage's gather, a8): the survivors of the
 *     last step to `root`, in global order, by grouped ncclSend / ncclRecv:
 *     d_all_ids (root, capacity total) gets the ids; with_points (same value
 *     on every rank) also sends the coordinates, d_all_pts (root, capacity
 *     2 * total doubles), staged on non-root ranks in d_tmp (>= 16 bytes per
 *     local survivor).  d_local / d_xy_shard: this rank's survivors and shard.
 *   ch_hull_end_to_end_dist: Algorithm 1 on W GPUs: the step, the gather
 *     to `root`, the exact device hull of the gathered survivors there (f1).
 *     h_hull (root, capacity >= total) and *h_n_hull at the root; *h_n_hull
 *     = 0 elsewhere.  Stage times to h_stats (nullable).  Synchronizes. */
#define CH_NCCL_ID_BYTES 128
typedef struct ch_comm ch_comm;
ch_status ch_comm_unique_id(void *h_id);
int ch_comm_nccl_version(void);
ch_status ch_comm_init(ch_comm **out, const void *h_id, int rank, int world, int device);
ch_status ch_comm_destroy(ch_comm *c);
ch_status ch_filter_compact_dist(ch_comm *c, const double *d_xy_shard, int64_t n_local, int64_t n_global, int flags,
                                 int64_t *d_survivors_local, int64_t *h_count_local, int64_t *h_offset,
                                 int64_t *h_total, ch_extremes *h_ext, void *d_ws, size_t ws_bytes, void *stream);
ch_status ch_filter_compact_dist_f32(ch_comm *c, const float *d_xy_shard, int64_t n_local, int64_t n_global,
                                     int flags, int64_t *d_survivors_local, int64_t *h_count_local,
                                     int64_t *h_offset, int64_t *h_total, ch_extremes *h_ext, void *d_ws,
                                     size_t ws_bytes, void *stream);
ch_status ch_comm_result(ch_comm *c, int64_t *h_counts, int64_t *h_offset, int64_t *h_total, void *stream);
ch_status ch_comm_step_times(ch_comm *c, double *h_ms_pass1, double *h_ms_exchange, double *h_ms_pass2);
ch_status ch_gather_survivors(ch_comm *c, const double *d_xy_shard, const int64_t *d_local, int root, int with_points,
                              int64_t *d_all_ids, double *d_all_pts, void *d_tmp, size_t tmp_bytes, void *stream);
ch_status ch_hull_end_to_end_dist(ch_comm *c, const double *d_xy_shard, int64_t n_local, int64_t n_global, int flags,
                                  int64_t *d_survivors_local, int root, int64_t *h_hull, int64_t *h_n_hull,
                                  int64_t *h_n_survivors, ch_stats *h_stats, void *d_ws, size_t ws_bytes,
                                  void *stream);

/* The same step end to end from HOST memory: copies h_xy (pinned for full
 * speed) into d_xy_staging (capacity n points), filters, and copies the
 * survivor indices back to h_survivors (capacity n).  Synchronizes. */
ch_status ch_filter_host(const double *h_xy, int64_t n, int flags, double *d_xy_staging,
                         int64_t *d_survivors, int64_t *h_survivors, int64_t *h_count,
                         void *d_ws, size_t ws_bytes, void *stream);

/* Gather d_xy[d_idx[j] - index_base] into d_out[2j..2j+1] for j < m. */
ch_status ch_gather_points(const double *d_xy, int64_t index_base, const int64_t *d_idx,
                           int64_t m, double *d_out, void *stream);

/* Exact strict convex hull on the host (Algorithm 1 line 4, P:149-151;
 * DESIGN R8): h_pts[2j..2j+1] are the coordinates of point h_ids[j].
 * Output: hull vertex ids, counter-clockwise from the lexicographic minimum
 * (x, then y), duplicates resolved to the lowest id, collinear points
 * excluded.  h_hull capacity >= m.  Exact orientation (adaptive filter with
 * an exact expansion fallback); valid for |coordinates| in [2^-450, 2^450]
 * or zero. */
ch_status ch_hull_points(const double *h_pts, const int64_t *h_ids, int64_t m,
                         int64_t *h_hull, int64_t *h_n_hull);

/* f1: Algorithm 1 line 4 on the device (future work P:432):
 * the exact strict hull of the m survivors d_surv (indices into d_xy, which
 * holds n_points points), same canonical form as ch_hull_points (DESIGN R8).
 * n_points < 2^32 lets the sort carry 32-bit ids.  m <= 1024: one CTA
 * (sort and chains in shared memory).  For m >= 2^16 a second
 * filtering round first drops survivors strictly inside a triangle of input
 * points (exact orientation; 64-direction extremes of a sample), then one
 * hand-written radix sort by x (32-bit monotone keys, equal-key runs sorted
 * exactly), each run of equal x reduced in place to its lowest and highest
 * point (the only possible strict hull vertices among them), per-chunk
 * exact monotone chains, a tree of exact bridge merges.
 * Scratch: ch_hull_gpu_temp_bytes(m) bytes at d_tmp.  Hull ids go to h_hull
 * (host, capacity m); synchronizes `stream`. */
size_t ch_hull_gpu_temp_bytes(int64_t m);
ch_status ch_hull_gpu(const double *d_xy, int64_t n_points, const int64_t *d_surv, int64_t m, int64_t *h_hull,
                      int64_t *h_n_hull, void *d_tmp, size_t tmp_bytes, void *stream);
/* The same hull kept on the device ("avoiding unnecessary data copying
 * between the device and host"): ids to d_hull (device, capacity m), the
 * count to *d_n_hull (device int64).  Fully asynchronous on `stream`; d_tmp
 * (ch_hull_gpu_temp_bytes(m)) must stay untouched until the stream reaches
 * this point.  m == 0 writes a zero count.  The second filtering round runs
 * here too, decided on the device (its count never reaches the host). */
ch_status ch_hull_gpu_async(const double *d_xy, int64_t n_points, const int64_t *d_surv, int64_t m,
                            int64_t *d_hull, int64_t *d_n_hull, void *d_tmp, size_t tmp_bytes, void *stream);

/* f1 on given coordinates: the hull of the m points d_pts[2j..2j+1] with ids
 * d_ids[j] (e.g. survivors gathered to a root, in increasing id order: then
 * duplicates resolve to the lowest id, as in ch_hull_gpu).  Asynchronous;
 * scratch ch_hull_gpu_temp_bytes(m). */
ch_status ch_hull_gpu_pts_async(const double *d_pts, const int64_t *d_ids, int64_t m, int64_t *d_hull,
                                int64_t *d_n_hull, void *d_tmp, size_t tmp_bytes, void *stream);

#define CH_HULL_HOST 4 /* flag for ch_hull_end_to_end: gather + host monotone chain */
#define CH_NO_CLUSTER 8 /* flag for ch_filter / ch_filter_async: no single-cluster step (K6)
                           for mid-small n; K1 + K2 instead (tests, A/B) */

/* Algorithm 1 complete: ch_filter on device-resident d_xy, then
 * the exact hull of the survivors -- on the device (ch_hull_gpu, default)
 * or, with flags & CH_HULL_HOST, gathered to the host and computed there
 * (ch_hull_points).  Stage times go to h_stats (nullable).  h_hull capacity
 * >= number of survivors (<= n).  Device-hull scratch: when ws_bytes >=
 * ch_hull_workspace_bytes(n) it is the tail of d_ws (no allocation);
 * otherwise it is taken with cudaMallocAsync for the call. */
size_t ch_hull_workspace_bytes(int64_t n); /* filter workspace + device-hull scratch */
ch_status ch_hull_end_to_end(const double *d_xy, int64_t n, int flags, int64_t *d_survivors,
                             int64_t *h_n_survivors, int64_t *h_hull, int64_t *h_n_hull,
                             ch_stats *h_stats, void *d_ws, size_t ws_bytes, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* CHFILTER_H */
