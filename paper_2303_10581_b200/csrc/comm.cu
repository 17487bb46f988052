// comm.cu -- the multi-GPU step over a library-owned NCCL communicator
// (north_star: "Per-rank extremes are combined with a tiny NCCL allgather ...
// survivor counts are exclusive-scanned to gather survivors"; SURVEY 8(b),
// 8(e); the paper itself is single-GPU).
//
// One process per GPU, points sharded by contiguous index ranges (DESIGN
// R14: rank r owns [floor(r n / W), floor((r + 1) n / W))).  One step:
//   K1 on the shard (global indices)           -> 192-byte extremes record
//   ncclAllGather of the W records             (a4)
//   K3: combine8 + octagon, identical on every rank
//   K2 on the shard (programmatic launch after K3)
//   ncclAllGather of {count, flags} per rank   (a7)
//   k_scan: the exclusive scan -> {count, offset, total, flags} on the device
// plus, for the hull stage (a8, timed separately), a grouped ncclSend /
// ncclRecv gather of survivor ids and coordinates to a root, and the device
// hull of the gathered points there (f1).
//
// NCCL is loaded at run time (dlopen "libnccl.so.2": the copy the process
// already has -- e.g. PyTorch's -- else the system one), so the library loads
// and every single-GPU entry point works without NCCL; ch_comm_* report
// CH_ERR_NCCL if it is missing.  Only the 128-byte ncclUniqueId crosses the
// caller's own transport (torch.distributed broadcasts it).
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/chfilter.h"
#include "internal.h"

static_assert(sizeof(ncclUniqueId) == CH_NCCL_ID_BYTES, "ncclUniqueId size");

namespace {

using chi::fail;

// ------------------------------------------------------------ NCCL loader --
struct Nccl {
    bool ok = false;
    std::string err;
    int version = 0;
    ncclResult_t (*GetVersion)(int *);
    ncclResult_t (*GetUniqueId)(ncclUniqueId *);
    ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int);
    ncclResult_t (*CommDestroy)(ncclComm_t);
    ncclResult_t (*CommAbort)(ncclComm_t);
    ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t *);
    const char *(*GetErrorString)(ncclResult_t);
    ncclResult_t (*AllGather)(const void *, void *, size_t, ncclDataType_t, ncclComm_t, cudaStream_t);
    ncclResult_t (*Send)(const void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
    ncclResult_t (*Recv)(void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
    ncclResult_t (*GroupStart)();
    ncclResult_t (*GroupEnd)();
};

const Nccl &nccl()
{
    static Nccl api;
    static std::once_flag once;
    std::call_once(once, [] {
        void *h = nullptr;
        for (const char *name : {"libnccl.so.2", "libnccl.so"})
            if ((h = dlopen(name, RTLD_NOW | RTLD_GLOBAL)))
                break;
        if (!h) {
            api.err = std::string("cannot load libnccl.so.2: ") + (dlerror() ? dlerror() : "?");
            return;
        }
        bool all = true;
        auto sym = [&](auto &fp, const char *name) {
            fp = reinterpret_cast<std::remove_reference_t<decltype(fp)>>(dlsym(h, name));
            if (!fp) {
                all = false;
                api.err += std::string(api.err.empty() ? "" : ", ") + "missing " + name;
            }
        };
        sym(api.GetVersion, "ncclGetVersion");
        sym(api.GetUniqueId, "ncclGetUniqueId");
        sym(api.CommInitRank, "ncclCommInitRank");
        sym(api.CommDestroy, "ncclCommDestroy");
        sym(api.CommAbort, "ncclCommAbort");
        sym(api.CommGetAsyncError, "ncclCommGetAsyncError");
        sym(api.GetErrorString, "ncclGetErrorString");
        sym(api.AllGather, "ncclAllGather");
        sym(api.Send, "ncclSend");
        sym(api.Recv, "ncclRecv");
        sym(api.GroupStart, "ncclGroupStart");
        sym(api.GroupEnd, "ncclGroupEnd");
        api.ok = all;
        if (all)
            api.GetVersion(&api.version);
    });
    return api;
}

ch_status nccl_check(ncclResult_t r, const char *what)
{
    if (r == ncclSuccess)
        return CH_OK;
    return fail(CH_ERR_NCCL, std::string(what) + ": " + nccl().GetErrorString(r));
}

ch_status cuda_ok(cudaError_t e, const char *what)
{
    if (e == cudaSuccess)
        return CH_OK;
    cudaGetLastError();
    return fail(CH_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

// a7: every rank's {count, flags} pair (gathered, rank order) -> this rank's
// {count, exclusive offset, total, OR of all flags}.
__global__ void k_scan_counts(const long long *__restrict__ all, int world, int rank, long long *__restrict__ out)
{
    if (threadIdx.x == 0) {
        long long off = 0, total = 0, flags = 0;
        for (int r = 0; r < world; r++) {
            const long long c = all[2 * r];
            off += r < rank ? c : 0;
            total += c;
            flags |= all[2 * r + 1];
        }
        out[0] = all[2 * rank];
        out[1] = off;
        out[2] = total;
        out[3] = flags;
    }
}

enum { EV_START, EV_K1, EV_EXCH1, EV_K2, EV_END, EV_N };

} // namespace

// Device layout of the communicator's buffers (one allocation):
//   ext_send[24]  this rank's extremes record (K1's d_ext_out)
//   ext_all[24 W] the gathered records (K3's input)
//   st_send[2]    {count, flags} of this rank
//   st_all[2 W]   the gathered pairs
//   scan[4]       {count, offset, total, flags} (k_scan_counts)
struct ch_comm {
    ncclComm_t comm = nullptr;
    int rank = 0, world = 0, device = 0;
    long long *d_buf = nullptr;
    long long *ext_send = nullptr, *ext_all = nullptr, *st_send = nullptr, *st_all = nullptr, *scan = nullptr;
    long long *h_pinned = nullptr; // scan[4] + st_all[2 W], copied back when a call synchronizes
    cudaEvent_t ev[EV_N] = {};
    // the last step
    long long index_base = 0, n_local = 0;
    bool stepped = false, host_valid = false;
    cudaStream_t last_stream = nullptr;
    std::vector<long long> counts; // valid when host_valid
};

namespace {

// Copy {scan, st_all} of the last step to the host (synchronizes the stream).
ch_status comm_sync_host(ch_comm *c, cudaStream_t st)
{
    if (!c->stepped)
        return fail(CH_ERR_INVALID_ARG, "no ch_filter_compact_dist step on this communicator yet");
    if (c->host_valid)
        return CH_OK;
    cudaMemcpyAsync(c->h_pinned, c->scan, 4 * sizeof(long long), cudaMemcpyDeviceToHost, st);
    cudaMemcpyAsync(c->h_pinned + 4, c->st_all, 2 * c->world * sizeof(long long), cudaMemcpyDeviceToHost, st);
    ch_status s = cuda_ok(cudaStreamSynchronize(st), "comm sync");
    if (s != CH_OK)
        return s;
    ncclResult_t ae = ncclSuccess;
    nccl().CommGetAsyncError(c->comm, &ae);
    if (ae != ncclSuccess)
        return nccl_check(ae, "NCCL async error");
    c->counts.assign((size_t)c->world, 0);
    for (int r = 0; r < c->world; r++)
        c->counts[(size_t)r] = c->h_pinned[4 + 2 * r];
    c->host_valid = true;
    return CH_OK;
}

ch_status comm_flags_status(const ch_comm *c)
{
    const long long flags = c->h_pinned[3];
    if (flags & 1)
        return fail(CH_ERR_NONFINITE, "non-finite coordinate in some rank's shard");
    if (flags & 2)
        return fail(CH_ERR_PEER, "a rank's exchange timed out");
    return CH_OK;
}

ch_status dist_step(ch_comm *c, const void *d_xy, bool f32, int64_t n_local, int64_t n_global, int flags,
                    int64_t *d_survivors, int64_t *h_count_local, int64_t *h_offset, int64_t *h_total,
                    ch_extremes *h_ext, void *d_ws, size_t ws_bytes, void *stream)
{
    if (!c || !c->comm)
        return fail(CH_ERR_INVALID_ARG, "communicator is NULL");
    if (n_global < 0 || n_local < 0)
        return fail(CH_ERR_INVALID_ARG, "negative size");
    const long long W = c->world, r = c->rank;
    // R14 shard bounds, computed without overflow for n_global < 2^39
    const long long lo = (long long)(((__int128)r * n_global) / W);
    const long long hi = (long long)(((__int128)(r + 1) * n_global) / W);
    if (n_local != hi - lo)
        return fail(CH_ERR_INVALID_ARG, "n_local must be the R14 shard size floor((r+1)n/W) - floor(rn/W)");
    if (n_global == 0)
        return fail(CH_ERR_EMPTY, "n_global == 0 (EmptySet)");
    if (n_local > 0 && !d_survivors)
        return fail(CH_ERR_INVALID_ARG, "d_survivors is NULL");
    cudaStream_t st = (cudaStream_t)stream;
    const Nccl &N = nccl();
    c->host_valid = false;
    c->stepped = false;
    ch_status s;
    cudaEventRecord(c->ev[EV_START], st);
    // a2/a3 on the shard; an empty shard sends the empty record
    if (n_local > 0)
        s = chi::k1(d_xy, f32, n_local, lo, flags, c->ext_send, d_ws, ws_bytes, st);
    else
        s = chi::empty_record(c->ext_send, st);
    if (s != CH_OK)
        return s;
    cudaEventRecord(c->ev[EV_K1], st);
    // a4: all-gather of the records, K3 on every rank
    if ((s = nccl_check(N.AllGather(c->ext_send, c->ext_all, 24, ncclInt64, c->comm, st), "ncclAllGather(extremes)")) !=
        CH_OK)
        return s;
    if ((s = chi::k3(c->ext_all, (int)W, flags, d_ws, ws_bytes, st)) != CH_OK)
        return s;
    cudaEventRecord(c->ev[EV_EXCH1], st);
    // a5/a6 on the shard (programmatic launch after K3)
    if (n_local > 0 && (s = chi::k2(d_xy, f32, n_local, lo, d_survivors, nullptr, d_ws, ws_bytes, st, true)) != CH_OK)
        return s;
    cudaEventRecord(c->ev[EV_K2], st);
    // a7: {count, flags} all-gather and the exclusive scan, on the device
    if ((s = chi::pack_status(d_ws, n_local == 0, (int64_t *)c->st_send, st)) != CH_OK)
        return s;
    if ((s = nccl_check(N.AllGather(c->st_send, c->st_all, 2, ncclInt64, c->comm, st), "ncclAllGather(counts)")) !=
        CH_OK)
        return s;
    k_scan_counts<<<1, 32, 0, st>>>(c->st_all, (int)W, (int)r, c->scan);
    if ((s = cuda_ok(cudaGetLastError(), "k_scan_counts")) != CH_OK)
        return s;
    cudaEventRecord(c->ev[EV_END], st);
    c->index_base = lo;
    c->n_local = n_local;
    c->stepped = true;
    c->last_stream = st;
    if (!h_count_local && !h_offset && !h_total && !h_ext)
        return CH_OK; // asynchronous: results in ch_comm_result / the next synchronizing call
    if (h_ext)
        cudaMemcpyAsync(h_ext, chi::ws_extremes(d_ws), sizeof(ch_extremes), cudaMemcpyDeviceToHost, st);
    if ((s = comm_sync_host(c, st)) != CH_OK)
        return s;
    if (h_count_local)
        *h_count_local = c->h_pinned[0];
    if (h_offset)
        *h_offset = c->h_pinned[1];
    if (h_total)
        *h_total = c->h_pinned[2];
    return comm_flags_status(c);
}

} // namespace

extern "C" {

ch_status ch_comm_unique_id(void *h_id)
{
    if (!h_id)
        return fail(CH_ERR_INVALID_ARG, "h_id is NULL");
    const Nccl &N = nccl();
    if (!N.ok)
        return fail(CH_ERR_NCCL, "NCCL unavailable: " + N.err);
    ncclUniqueId id;
    ch_status s = nccl_check(N.GetUniqueId(&id), "ncclGetUniqueId");
    if (s == CH_OK)
        memcpy(h_id, &id, sizeof(id));
    return s;
}

int ch_comm_nccl_version(void)
{
    const Nccl &N = nccl();
    return N.ok ? N.version : -1;
}

ch_status ch_comm_init(ch_comm **out, const void *h_id, int rank, int world, int device)
{
    if (!out || !h_id || world < 1 || rank < 0 || rank >= world || device < 0)
        return fail(CH_ERR_INVALID_ARG, "bad communicator arguments");
    *out = nullptr;
    const Nccl &N = nccl();
    if (!N.ok)
        return fail(CH_ERR_NCCL, "NCCL unavailable: " + N.err);
    ch_status s = cuda_ok(cudaSetDevice(device), "cudaSetDevice");
    if (s != CH_OK)
        return s;
    ch_comm *c = new ch_comm();
    c->rank = rank;
    c->world = world;
    c->device = device;
    const size_t words = 24 + 24 * (size_t)world + 2 + 2 * (size_t)world + 4;
    if ((s = cuda_ok(cudaMalloc((void **)&c->d_buf, words * sizeof(long long)), "comm buffers")) != CH_OK ||
        (s = cuda_ok(cudaMemset(c->d_buf, 0, words * sizeof(long long)), "comm buffers")) != CH_OK ||
        (s = cuda_ok(cudaMallocHost((void **)&c->h_pinned, (4 + 2 * (size_t)world) * sizeof(long long)),
                     "comm host buffer")) != CH_OK) {
        ch_comm_destroy(c);
        return s;
    }
    c->ext_send = c->d_buf;
    c->ext_all = c->ext_send + 24;
    c->st_send = c->ext_all + 24 * (size_t)world;
    c->st_all = c->st_send + 2;
    c->scan = c->st_all + 2 * (size_t)world;
    for (auto &e : c->ev)
        cudaEventCreate(&e);
    ncclUniqueId id;
    memcpy(&id, h_id, sizeof(id));
    if ((s = nccl_check(N.CommInitRank(&c->comm, world, id, rank), "ncclCommInitRank")) != CH_OK) {
        c->comm = nullptr;
        ch_comm_destroy(c);
        return s;
    }
    *out = c;
    return CH_OK;
}

ch_status ch_comm_destroy(ch_comm *c)
{
    if (!c)
        return CH_OK;
    if (c->last_stream)
        cudaStreamSynchronize(c->last_stream);
    if (c->comm)
        nccl().CommDestroy(c->comm);
    for (auto &e : c->ev)
        if (e)
            cudaEventDestroy(e);
    if (c->d_buf)
        cudaFree(c->d_buf);
    if (c->h_pinned)
        cudaFreeHost(c->h_pinned);
    delete c;
    cudaGetLastError();
    return CH_OK;
}

ch_status ch_filter_compact_dist(ch_comm *c, const double *d_xy_shard, int64_t n_local, int64_t n_global, int flags,
                                 int64_t *d_survivors_local, int64_t *h_count_local, int64_t *h_offset,
                                 int64_t *h_total, ch_extremes *h_ext, void *d_ws, size_t ws_bytes, void *stream)
{
    return dist_step(c, d_xy_shard, false, n_local, n_global, flags, d_survivors_local, h_count_local, h_offset,
                     h_total, h_ext, d_ws, ws_bytes, stream);
}

ch_status ch_filter_compact_dist_f32(ch_comm *c, const float *d_xy_shard, int64_t n_local, int64_t n_global,
                                     int flags, int64_t *d_survivors_local, int64_t *h_count_local,
                                     int64_t *h_offset, int64_t *h_total, ch_extremes *h_ext, void *d_ws,
                                     size_t ws_bytes, void *stream)
{
    return dist_step(c, d_xy_shard, true, n_local, n_global, flags, d_survivors_local, h_count_local, h_offset,
                     h_total, h_ext, d_ws, ws_bytes, stream);
}

ch_status ch_comm_result(ch_comm *c, int64_t *h_counts, int64_t *h_offset, int64_t *h_total, void *stream)
{
    if (!c)
        return fail(CH_ERR_INVALID_ARG, "communicator is NULL");
    ch_status s = comm_sync_host(c, (cudaStream_t)stream);
    if (s != CH_OK)
        return s;
    if (h_counts)
        for (int r = 0; r < c->world; r++)
            h_counts[r] = c->counts[(size_t)r];
    if (h_offset)
        *h_offset = c->h_pinned[1];
    if (h_total)
        *h_total = c->h_pinned[2];
    return comm_flags_status(c);
}

ch_status ch_comm_step_times(ch_comm *c, double *h_ms_pass1, double *h_ms_exchange, double *h_ms_pass2)
{
    if (!c || !c->stepped)
        return fail(CH_ERR_INVALID_ARG, "no step on this communicator yet");
    if (cudaEventSynchronize(c->ev[EV_END]) != cudaSuccess)
        return cuda_ok(cudaGetLastError(), "step events");
    float a = 0, b = 0, d = 0, e = 0;
    cudaEventElapsedTime(&a, c->ev[EV_START], c->ev[EV_K1]);
    cudaEventElapsedTime(&b, c->ev[EV_K1], c->ev[EV_EXCH1]);
    cudaEventElapsedTime(&d, c->ev[EV_EXCH1], c->ev[EV_K2]);
    cudaEventElapsedTime(&e, c->ev[EV_K2], c->ev[EV_END]);
    if (h_ms_pass1)
        *h_ms_pass1 = a;
    if (h_ms_exchange)
        *h_ms_exchange = (double)b + e;
    if (h_ms_pass2)
        *h_ms_pass2 = d;
    return CH_OK;
}

ch_status ch_gather_survivors(ch_comm *c, const double *d_xy_shard, const int64_t *d_local, int root, int with_points,
                              int64_t *d_all_ids, double *d_all_pts, void *d_tmp, size_t tmp_bytes, void *stream)
{
    if (!c || root < 0 || root >= c->world)
        return fail(CH_ERR_INVALID_ARG, "bad communicator / root");
    cudaStream_t st = (cudaStream_t)stream;
    ch_status s = comm_sync_host(c, st);
    if (s != CH_OK)
        return s;
    const long long mine = c->counts[(size_t)c->rank];
    const bool is_root = c->rank == root;
    if (mine > 0 && (!d_local || !d_xy_shard))
        return fail(CH_ERR_INVALID_ARG, "d_local / d_xy_shard is NULL");
    if (is_root && c->h_pinned[2] > 0 && (!d_all_ids || (with_points && !d_all_pts)))
        return fail(CH_ERR_INVALID_ARG, "d_all_ids / d_all_pts is NULL at the root");
    const Nccl &N = nccl();
    if (is_root) {
        long long off = 0;
        for (int r = 0; r < c->rank; r++)
            off += c->counts[(size_t)r];
        if (mine > 0) { // the root's own part: copies, no NCCL
            cudaMemcpyAsync(d_all_ids + off, d_local, (size_t)mine * 8, cudaMemcpyDeviceToDevice, st);
            if (with_points &&
                (s = ch_gather_points(d_xy_shard, c->index_base, d_local, mine, d_all_pts + 2 * off, st)) != CH_OK)
                return s;
        }
    } else if (mine > 0 && with_points) {
        // stage this rank's survivor coordinates for the send
        if (!d_tmp || tmp_bytes < (size_t)mine * 16)
            return fail(CH_ERR_WORKSPACE, "d_tmp must hold 16 bytes per local survivor");
        if ((s = ch_gather_points(d_xy_shard, c->index_base, d_local, mine, (double *)d_tmp, st)) != CH_OK)
            return s;
    }
    if ((s = nccl_check(N.GroupStart(), "ncclGroupStart")) != CH_OK)
        return s;
    if (is_root) {
        long long off = 0;
        for (int r = 0; r < c->world; r++) {
            const long long cnt = c->counts[(size_t)r];
            if (r != root && cnt > 0) {
                N.Recv(d_all_ids + off, (size_t)cnt, ncclInt64, r, c->comm, st);
                if (with_points)
                    N.Recv(d_all_pts + 2 * off, 2 * (size_t)cnt, ncclFloat64, r, c->comm, st);
            }
            off += cnt;
        }
    } else if (mine > 0) {
        N.Send(d_local, (size_t)mine, ncclInt64, root, c->comm, st);
        if (with_points)
            N.Send(d_tmp, 2 * (size_t)mine, ncclFloat64, root, c->comm, st);
    }
    return nccl_check(N.GroupEnd(), "ncclGroupEnd");
}

ch_status ch_hull_end_to_end_dist(ch_comm *c, const double *d_xy_shard, int64_t n_local, int64_t n_global, int flags,
                                  int64_t *d_survivors_local, int root, int64_t *h_hull, int64_t *h_n_hull,
                                  int64_t *h_n_survivors, ch_stats *h_stats, void *d_ws, size_t ws_bytes,
                                  void *stream)
{
    if (!c || !h_n_hull || root < 0 || root >= (c ? c->world : 1))
        return fail(CH_ERR_INVALID_ARG, "bad arguments");
    cudaStream_t st = (cudaStream_t)stream;
    int64_t cnt = 0, off = 0, total = 0;
    ch_status s = dist_step(c, d_xy_shard, false, n_local, n_global, flags & 3, d_survivors_local, &cnt, &off, &total,
                            nullptr, d_ws, ws_bytes, stream);
    if (s != CH_OK)
        return s;
    double p1 = 0, ex = 0, p2 = 0;
    ch_comm_step_times(c, &p1, &ex, &p2);
    const bool is_root = c->rank == root;
    if (is_root && total > 0 && !h_hull)
        return fail(CH_ERR_INVALID_ARG, "h_hull is NULL at the root");
    const auto t0 = std::chrono::steady_clock::now();
    // scratch for this call only (the hull stage, not the filter's hot path)
    void *ids = nullptr, *pts = nullptr, *tmp = nullptr, *htmp = nullptr, *hout = nullptr;
    size_t hb = 0;
    auto cleanup = [&] {
        for (void *p : {ids, pts, tmp, htmp, hout})
            if (p)
                cudaFreeAsync(p, st);
    };
    if (is_root) {
        hb = ch_hull_gpu_temp_bytes(total);
        if (cudaMallocAsync(&ids, (size_t)std::max<int64_t>(total, 1) * 8, st) != cudaSuccess ||
            cudaMallocAsync(&pts, (size_t)std::max<int64_t>(total, 1) * 16, st) != cudaSuccess ||
            cudaMallocAsync(&htmp, hb, st) != cudaSuccess ||
            cudaMallocAsync(&hout, (size_t)(std::max<int64_t>(total, 1) + 1) * 8, st) != cudaSuccess) {
            cleanup();
            return cuda_ok(cudaGetLastError(), "hull-stage allocation at the root");
        }
    } else if (cnt > 0 && cudaMallocAsync(&tmp, (size_t)cnt * 16, st) != cudaSuccess) {
        return cuda_ok(cudaGetLastError(), "gather staging");
    }
    s = ch_gather_survivors(c, d_xy_shard, d_survivors_local, root, 1, (int64_t *)ids, (double *)pts, tmp,
                            (size_t)cnt * 16, stream);
    if (s != CH_OK) {
        cleanup();
        return s;
    }
    const auto t1 = std::chrono::steady_clock::now();
    int64_t nh = 0;
    if (is_root) {
        int64_t *d_nh = (int64_t *)hout + std::max<int64_t>(total, 1);
        s = chi::hull_pts_refined((const double *)pts, (const int64_t *)ids, total, (int64_t *)hout, d_nh, htmp, hb,
                                  st);
        if (s == CH_OK) {
            cudaMemcpyAsync(&nh, d_nh, 8, cudaMemcpyDeviceToHost, st);
            cudaStreamSynchronize(st);
            if (nh > 0)
                cudaMemcpyAsync(h_hull, hout, (size_t)nh * 8, cudaMemcpyDeviceToHost, st);
        }
    }
    cleanup();
    ch_status s2 = cuda_ok(cudaStreamSynchronize(st), "hull stage");
    if (s != CH_OK)
        return fail(s, "device hull of the gathered survivors failed");
    if (s2 != CH_OK)
        return s2;
    const auto t2 = std::chrono::steady_clock::now();
    *h_n_hull = is_root ? nh : 0;
    if (h_n_survivors)
        *h_n_survivors = total;
    if (h_stats) {
        h_stats->n = n_global;
        h_stats->n_survivors = total;
        h_stats->n_hull = *h_n_hull;
        h_stats->ms_filter = p1 + ex + p2;
        h_stats->ms_gather = std::chrono::duration<double, std::milli>(t1 - t0).count();
        h_stats->ms_hull = std::chrono::duration<double, std::milli>(t2 - t1).count();
        h_stats->ms_pass1 = p1;
        h_stats->ms_pass2 = p2;
        h_stats->ms_exchange = ex;
    }
    return CH_OK;
}

} // extern "C"
