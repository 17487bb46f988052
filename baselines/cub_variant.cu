// baselines/cub_variant.cu -- SURVEY 8(f) f4: the paper's library variant
// rebuilt on this B200 as an in-box prior-art bar (NOT the product path).
//
// Variant #4 "cub-flagged" (§4.3):
//   * CUB ArgMin / ArgMax for each of the eight keys ("ArgMax and ArgMin
//     ... key-value"): one device-wide reduction -- one read of the input --
//     per key;
//   * the octagon from those extremes (the product's ch_octagon_build, so the
//     survivor set is the same);
//   * a per-point kernel writing one flag byte per point;
//   * cub::DeviceSelect::Flagged over the point indices ("d_flags ...
//     d_num_selected_out").
// It reads the input 9 times plus the flags, against the product's two
// fused passes; bench.py --impl cub times it next to K1 + K2.
//
// Variants #2 "thrust-scan" and #3 "thrust-copy" (§4.2), with
// Thrust as the paper used it:
//   * thrust::min_element / max_element for each key (eight more
//     reads of the input);
//   * #2: a transform to int flags, thrust::exclusive_scan of the flags, and
//     a scatter kernel;
//   * #3: thrust::copy_if of the point indices with the inside test as the
//     predicate.
// bench.py --impl thrust-scan / thrust-copy.
#include <cuda_runtime.h>

#include <cub/cub.cuh>
#include <cuda/std/cstdint>
#include <thrust/copy.h>
#include <thrust/execution_policy.h>
#include <thrust/extrema.h>
#include <thrust/iterator/counting_iterator.h>
#include <thrust/iterator/transform_iterator.h>
#include <thrust/scan.h>
#include <thrust/transform.h>

#include <cstdint>
#include <cstring>

#include "../include/chfilter.h"

namespace {

struct KeyOf {
    const double *xy;
    int kind; // 0 x, 1 x+y, 2 y, 3 x-y
    __host__ __device__ double operator()(int64_t i) const
    {
#ifdef __CUDA_ARCH__
        const double x = xy[2 * i], y = xy[2 * i + 1];
        switch (kind) {
        case 0: return x;
        case 1: return __dadd_rn(x, y);
        case 2: return y;
        default: return __dsub_rn(x, y);
        }
#else
        return 0.0; // never dereferenced on the host
#endif
    }
};

// The paper's buildingFilter kernel: one thread per point, all edges, a flag
// byte out (1 = hull candidate).  Same predicate as the oracle (R4).
__global__ void flags_kernel(const double *__restrict__ xy, int64_t n, ch_octagon o, uint8_t *__restrict__ flags)
{
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const double x = xy[2 * i], y = xy[2 * i + 1];
        bool inside = !o.degenerate;
        for (int k = 0; k < o.nv && inside; k++) {
            const double D = __dsub_rn(__dmul_rn(o.ex[k], __dsub_rn(y, o.vy[k])),
                                       __dmul_rn(o.ey[k], __dsub_rn(x, o.vx[k])));
            inside = D > o.thr[k];
        }
        flags[i] = inside ? 0 : 1;
    }
}

size_t g_temp_reduce = 0, g_temp_select = 0;

// The inside test of the paper's filter kernel as a functor (for copy_if /
// transform): true if point i is a hull candidate.
struct Candidate {
    const double *xy;
    ch_octagon o;
    __host__ __device__ bool operator()(int64_t i) const
    {
#ifdef __CUDA_ARCH__
        const double x = xy[2 * i], y = xy[2 * i + 1];
        bool inside = !o.degenerate;
        for (int k = 0; k < o.nv && inside; k++) {
            const double D = __dsub_rn(__dmul_rn(o.ex[k], __dsub_rn(y, o.vy[k])),
                                       __dmul_rn(o.ey[k], __dsub_rn(x, o.vx[k])));
            inside = D > o.thr[k];
        }
        return !inside;
#else
        return false;
#endif
    }
};
struct FlagOf {
    Candidate c;
    __host__ __device__ int operator()(int64_t i) const { return c(i) ? 1 : 0; }
};

__global__ void scatter_kernel(const int *__restrict__ flags, const int64_t *__restrict__ pos, int64_t n,
                               int64_t *__restrict__ out)
{
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        if (flags[i])
            out[pos[i]] = i;
}

// The eight extremes with thrust::min_element / max_element over the keys,
// then the octagon on the host (as the paper's host code would).
ch_octagon thrust_octagon(const double *d_xy, int64_t n, cudaStream_t st)
{
    thrust::counting_iterator<int64_t> cnt(0);
    const int kind[8] = {0, 1, 2, 3, 0, 1, 2, 3};
    const bool is_max[8] = {true, true, true, false, false, false, false, true};
    ch_extremes ext;
    for (int k = 0; k < 8; k++) {
        auto it = thrust::make_transform_iterator(cnt, KeyOf{d_xy, kind[k]});
        // first occurrence of the extreme value: the lowest index (R2)
        auto r = is_max[k] ? thrust::max_element(thrust::cuda::par.on(st), it, it + n)
                           : thrust::min_element(thrust::cuda::par.on(st), it, it + n);
        const int64_t i = (int64_t)(r - it);
        double p[2];
        cudaMemcpyAsync(p, d_xy + 2 * i, sizeof(p), cudaMemcpyDeviceToHost, st);
        cudaStreamSynchronize(st);
        ext.idx[k] = i;
        ext.x[k] = p[0];
        ext.y[k] = p[1];
    }
    ch_octagon o;
    ch_octagon_build(&ext, CH_CERTIFIED, &o);
    return o;
}

} // namespace

extern "C" {

// Scratch bytes for n points: CUB temp storage + 8 (value, index) outputs +
// n flag bytes + the selected count.
size_t chb_cub_temp_bytes(int64_t n)
{
    size_t r = 0, s = 0;
    thrust::counting_iterator<int64_t> cnt(0);
    auto it = thrust::make_transform_iterator(cnt, KeyOf{nullptr, 0});
    cub::DeviceReduce::ArgMax(nullptr, r, it, (double *)nullptr, (int64_t *)nullptr, n);
    cub::DeviceSelect::Flagged(nullptr, s, cnt, (const uint8_t *)nullptr, (int64_t *)nullptr, (int64_t *)nullptr, n);
    g_temp_reduce = r;
    g_temp_select = s;
    size_t t = (r > s ? r : s);
    t = (t + 255) & ~(size_t)255;
    return t + 256 * 2 + ((size_t)n + 255) / 256 * 256 + 256;
}

// One filter step the library way.  Returns 0 on success.
int chb_cub_filter(const double *d_xy, int64_t n, int64_t *d_survivors, int64_t *h_count, void *d_temp,
                   size_t temp_bytes, void *stream)
{
    cudaStream_t st = (cudaStream_t)stream;
    const size_t need = chb_cub_temp_bytes(n);
    if (temp_bytes < need || n < 1)
        return 1;
    size_t tb = (g_temp_reduce > g_temp_select ? g_temp_reduce : g_temp_select);
    tb = (tb + 255) & ~(size_t)255;
    char *base = (char *)d_temp;
    double *d_val = (double *)(base + tb);           // 8 values
    int64_t *d_idx = (int64_t *)(base + tb + 256);   // 8 indices
    uint8_t *d_flags = (uint8_t *)(base + tb + 512);
    int64_t *d_nsel = (int64_t *)(base + tb + 512 + ((size_t)n + 255) / 256 * 256);
    thrust::counting_iterator<int64_t> cnt(0);
    // slots R, TR, T, TL, L, BL, B, BR (R1): key kind and direction
    const int kind[8] = {0, 1, 2, 3, 0, 1, 2, 3};
    const bool is_max[8] = {true, true, true, false, false, false, false, true};
    for (int k = 0; k < 8; k++) {
        auto it = thrust::make_transform_iterator(cnt, KeyOf{d_xy, kind[k]});
        size_t b = tb;
        cudaError_t e = is_max[k] ? cub::DeviceReduce::ArgMax(d_temp, b, it, d_val + k, d_idx + k, n, st)
                                  : cub::DeviceReduce::ArgMin(d_temp, b, it, d_val + k, d_idx + k, n, st);
        if (e != cudaSuccess)
            return 2;
    }
    // extremes -> octagon on the host (as the paper's host code would)
    int64_t idx[8];
    cudaMemcpyAsync(idx, d_idx, sizeof(idx), cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    ch_extremes ext;
    for (int k = 0; k < 8; k++) {
        double p[2];
        cudaMemcpy(p, d_xy + 2 * idx[k], sizeof(p), cudaMemcpyDeviceToHost);
        ext.idx[k] = idx[k];
        ext.x[k] = p[0];
        ext.y[k] = p[1];
    }
    ch_octagon o;
    ch_octagon_build(&ext, CH_CERTIFIED, &o);
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    flags_kernel<<<sms * 8, 256, 0, st>>>(d_xy, n, o, d_flags);
    size_t b = tb;
    if (cub::DeviceSelect::Flagged(d_temp, b, cnt, d_flags, d_survivors, d_nsel, n, st) != cudaSuccess)
        return 3;
    cudaMemcpyAsync(h_count, d_nsel, sizeof(int64_t), cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    return cudaGetLastError() == cudaSuccess ? 0 : 4;
}

// Scratch for the Thrust variants: int flags + int64 scan positions.
size_t chb_thrust_temp_bytes(int64_t n) { return ((size_t)n * 4 + 255) / 256 * 256 + (size_t)n * 8 + 256; }

// Variant #2 (variant == 2, "thrust-scan") or #3 (variant == 3,
// "thrust-copy").  Returns 0 on success.
int chb_thrust_filter(int variant, const double *d_xy, int64_t n, int64_t *d_survivors, int64_t *h_count,
                      void *d_temp, size_t temp_bytes, void *stream)
{
    cudaStream_t st = (cudaStream_t)stream;
    if (n < 1 || temp_bytes < chb_thrust_temp_bytes(n))
        return 1;
    const ch_octagon o = thrust_octagon(d_xy, n, st);
    thrust::counting_iterator<int64_t> cnt(0);
    const Candidate cand{d_xy, o};
    if (variant == 3) {
        int64_t *end = thrust::copy_if(thrust::cuda::par.on(st), cnt, cnt + n, d_survivors, cand);
        *h_count = (int64_t)(end - d_survivors);
    } else if (variant == 2) {
        int *flags = (int *)d_temp;
        int64_t *pos = (int64_t *)((char *)d_temp + ((size_t)n * 4 + 255) / 256 * 256);
        thrust::transform(thrust::cuda::par.on(st), cnt, cnt + n, flags, FlagOf{cand});
        thrust::exclusive_scan(thrust::cuda::par.on(st), flags, flags + n, pos, (int64_t)0);
        int dev = 0, sms = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        scatter_kernel<<<sms * 8, 256, 0, st>>>(flags, pos, n, d_survivors);
        int64_t last_pos = 0;
        int last_flag = 0;
        cudaMemcpyAsync(&last_pos, pos + n - 1, 8, cudaMemcpyDeviceToHost, st);
        cudaMemcpyAsync(&last_flag, flags + n - 1, 4, cudaMemcpyDeviceToHost, st);
        cudaStreamSynchronize(st);
        *h_count = last_pos + last_flag;
    } else {
        return 5;
    }
    cudaStreamSynchronize(st);
    return cudaGetLastError() == cudaSuccess ? 0 : 4;
}

} // extern "C"
