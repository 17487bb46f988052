// internal.h -- host-side entry points shared by the library's translation
// units (chfilter.cu defines them; comm.cu builds the NCCL steps from them).
// Not part of the C ABI of include/chfilter.h.
#pragma once

#include <cuda_runtime.h>

#include <string>

#include "../../include/chfilter.h"

namespace chi {

// Records the thread-local detail string ch_last_error() returns.
ch_status fail(ch_status s, const std::string &msg);
const char *last_error();

// K1 on n points (float32 storage if f32) with global indices index_base + i;
// the eight extremes also to d_ext_out (device ch_extremes, nullable).
ch_status k1(const void *d_xy, bool f32, int64_t n, int64_t index_base, int flags, void *d_ext_out, void *d_ws,
             size_t ws_bytes, cudaStream_t st);
// K3: combine `world` device ch_extremes records into the workspace octagon.
ch_status k3(const void *d_ext_all, int world, int flags, void *d_ws, size_t ws_bytes, cudaStream_t st);
// K2 with the workspace octagon; pdl: programmatic launch after our K1 / K3.
ch_status k2(const void *d_xy, bool f32, int64_t n, int64_t index_base, int64_t *d_surv, int64_t *d_count,
             void *d_ws, size_t ws_bytes, cudaStream_t st, bool pdl);
// d_words[0] = the survivor count of the last step on d_ws (0 for an empty
// shard), d_words[1] = flags: bit 0 non-finite input, bit 1 late peer.
ch_status pack_status(const void *d_ws, bool empty, int64_t *d_words, cudaStream_t st);
// An empty shard's extremes record (idx -1) at d_ext.
ch_status empty_record(void *d_ext, cudaStream_t st);
// Device address of the workspace's (global) extremes record.
const void *ws_extremes(const void *d_ws);
// The device hull of m gathered points d_pts with ids d_ids (increasing),
// after the second filtering round (hull_gpu.cu); synchronizes `st`.
// Scratch ch_hull_gpu_temp_bytes(m).
ch_status hull_pts_refined(const double *d_pts, const int64_t *d_ids, int64_t m, int64_t *d_hull, int64_t *d_n_hull,
                           void *d_tmp, size_t tmp_bytes, cudaStream_t st);

} // namespace chi
