// mxfft_metrics.cu -- image-quality metrics over magnitude (RSS) images on the
// device (metrics.py:38-93).  FP64 throughout.  The
// reductions run in a different order than numpy's pairwise sums, so results
// agree to ~1e-15 relative, not bit for bit (the north star's PSNR/NRMSE bar
// is 0.01 dB / 1e-4).
#include <cfloat>

#include "mxfft_common.cuh"
#include "mxfft_internal.h"

namespace mxfft {

__device__ __forceinline__ void atomic_max_d(double* a, double v) {
    unsigned long long* p = reinterpret_cast<unsigned long long*>(a);
    unsigned long long old = *p;
    while (__longlong_as_double((long long)old) < v) {
        const unsigned long long prev = atomicCAS(p, old, (unsigned long long)__double_as_longlong(v));
        if (prev == old) break;
        old = prev;
    }
}
__device__ __forceinline__ void atomic_min_d(double* a, double v) {
    unsigned long long* p = reinterpret_cast<unsigned long long*>(a);
    unsigned long long old = *p;
    while (__longlong_as_double((long long)old) > v) {
        const unsigned long long prev = atomicCAS(p, old, (unsigned long long)__double_as_longlong(v));
        if (prev == old) break;
        old = prev;
    }
}

template <int NT>
__device__ __forceinline__ double block_sum(double v, double* sh) {
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0) sh[w] = v;
    __syncthreads();
    double s = 0.0;
    if (threadIdx.x == 0)
        for (int i = 0; i < NT / 32; ++i) s += sh[i];
    __syncthreads();
    return s;
}

// out[0] += sum (r - t)^2, out[1] += sum r^2, out[2] = max r, out[3] = min r
__global__ void __launch_bounds__(256) k_metric_sums(const double* __restrict__ r, const double* __restrict__ t,
                                                     int64_t n, double* out) {
    __shared__ double sh[8];
    double d2 = 0.0, r2 = 0.0, mx = -DBL_MAX, mn = DBL_MAX;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const double a = r[i], b = t[i], d = a - b;
        d2 = __fma_rn(d, d, d2);
        r2 = __fma_rn(a, a, r2);
        mx = fmax(mx, a);
        mn = fmin(mn, a);
    }
    for (int o = 16; o; o >>= 1) {
        mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    }
    if ((threadIdx.x & 31) == 0) {
        atomic_max_d(out + 2, mx);
        atomic_min_d(out + 3, mn);
    }
    const double s0 = block_sum<256>(d2, sh), s1 = block_sum<256>(r2, sh);
    if (threadIdx.x == 0) {
        atomicAdd(out, s0);
        atomicAdd(out + 1, s1);
    }
}

// Mean local SSIM over the valid (h-10) x (w-10) positions of an 11 x 11
// window `win` (row-major, symmetric Gaussian, so convolution == correlation).
// out[0] += sum of num/den.
__global__ void __launch_bounds__(256) k_ssim(const double* __restrict__ r, const double* __restrict__ t, int h,
                                              int w, const double* __restrict__ win, double c1, double c2,
                                              double* out) {
    __shared__ double wk[121];
    __shared__ double sh[8];
    for (int i = threadIdx.x; i < 121; i += blockDim.x) wk[i] = win[i];
    __syncthreads();
    const int oh = h - 10, ow = w - 10;
    const int64_t total = (int64_t)oh * ow;
    double acc = 0.0;
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < total;
         p += (int64_t)gridDim.x * blockDim.x) {
        const int y = (int)(p / ow), x = (int)(p - (int64_t)y * ow);
        double m1 = 0, m2 = 0, e11 = 0, e22 = 0, e12 = 0;
        for (int dy = 0; dy < 11; ++dy) {
            const double* rr = r + (int64_t)(y + dy) * w + x;
            const double* tt = t + (int64_t)(y + dy) * w + x;
#pragma unroll
            for (int dx = 0; dx < 11; ++dx) {
                const double k = wk[dy * 11 + dx], a = rr[dx], b = tt[dx];
                m1 = __fma_rn(k, a, m1);
                m2 = __fma_rn(k, b, m2);
                e11 = __fma_rn(k, a * a, e11);
                e22 = __fma_rn(k, b * b, e22);
                e12 = __fma_rn(k, a * b, e12);
            }
        }
        const double s1 = e11 - m1 * m1, s2 = e22 - m2 * m2, s12 = e12 - m1 * m2;
        const double num = (2 * m1 * m2 + c1) * (2 * s12 + c2);
        const double den = (m1 * m1 + m2 * m2 + c1) * (s1 + s2 + c2);
        acc += num / den;
    }
    const double s = block_sum<256>(acc, sh);
    if (threadIdx.x == 0) atomicAdd(out, s);
}

__global__ void k_metric_init(double* out) {
    out[0] = out[1] = 0.0;
    out[2] = -DBL_MAX;
    out[3] = DBL_MAX;
    out[4] = 0.0;
}

cudaError_t launch_metrics(const double* r, const double* t, int64_t h, int64_t w, int do_ssim, const double* win,
                           double c1, double c2, double* out, cudaStream_t st) {
    k_metric_init<<<1, 1, 0, st>>>(out);
    note_launch();
    const int64_t n = h * w;
    const unsigned g1 = (unsigned)((n + 255) / 256 < 148 * 8 ? (n + 255) / 256 : 148 * 8);
    if (n > 0) {
        k_metric_sums<<<g1 < 1 ? 1 : g1, 256, 0, st>>>(r, t, n, out);
        note_launch();
    }
    if (do_ssim && h >= 11 && w >= 11) {
        const int64_t m = (h - 10) * (w - 10);
        const unsigned g2 = (unsigned)((m + 255) / 256 < 148 * 16 ? (m + 255) / 256 : 148 * 16);
        k_ssim<<<g2, 256, 0, st>>>(r, t, (int)h, (int)w, win, c1, c2, out + 4);
        note_launch();
    }
    return cudaGetLastError();
}

}  // namespace mxfft
