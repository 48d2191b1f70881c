// mxfft_modes.cu -- the non-MX transform modes of ModeSpec on the GPU
// (SURVEY.md §8(f) ranks 1-2).
//
//  * FP16 positive control (_fft_batch_fp16, fftcore.py:285-311): inputs
//    quantized to FP16 (from FP64 for complex128 input), every intermediate
//    of the complex multiply rounded to FP16 the way numpy's half ufuncs do
//    it (FP32 compute, one rounding back to FP16; overflow -> inf), add/sub in
//    FP32, outputs quantized to the FP16 grid with saturation
//    (quantize_array, minifloat.py:105-120).  One CTA per line, the line in
//    shared memory.
//  * FP64 reference (_fft_batch_reference, fftcore.py:243-256): radix-2 DIT
//    in complex128 with numpy 2.3's complex product rounding
//    (re = fma(ar, br, -(ai*bi)), im = fma(ar, bi, ai*br); verified against
//    numpy on this host), add/sub in FP64.  A bit-reversal kernel, then one
//    kernel per stage over a work buffer (lines of any length up to 2^14).
#include <cuda_fp16.h>

#include "mxfft_common.cuh"
#include "mxfft_internal.h"

namespace mxfft {

static int grid_for(int64_t n, int threads) {
    int64_t g = (n + threads - 1) / threads;
    if (g > 148 * 32) g = 148 * 32;
    return (int)(g < 1 ? 1 : g);
}

__device__ __forceinline__ float h16(float v) { return __half2float(__float2half_rn(v)); }
__device__ __forceinline__ float in16(float v) { return h16(v); }
__device__ __forceinline__ float in16(double v) { return __half2float(__double2half(v)); }

template <typename T>
__global__ void __launch_bounds__(512) k_fp16_lines(const T* __restrict__ x, float2* __restrict__ y, int n,
                                                    int log2n, const __half2* __restrict__ tw, int inverse,
                                                    FmtDesc f16fmt, int* __restrict__ nonfinite) {
    extern __shared__ float2 L16[];
    const int64_t line = blockIdx.x;
    const T* xl = x + line * (int64_t)n;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const int r = log2n ? (int)(__brev((unsigned)i) >> (32 - log2n)) : 0;
        const T v = xl[r];
        L16[i] = make_float2(in16(v.x), in16(v.y));
    }
    __syncthreads();
    const int m = n / 2;
    for (int s = 0; s < log2n; ++s) {
        const int half = 1 << s;
        for (int t = threadIdx.x; t < m; t += blockDim.x) {
            const int g = t >> s, j = t & (half - 1);
            const int pu = g * 2 * half + j, pv = pu + half;
            const float2 v = L16[pv], u = L16[pu];
            const float vr = h16(v.x), vi = h16(v.y);
            const __half2 w = tw[half + j];
            const float wr = __low2float(w), wi = inverse ? -__high2float(w) : __high2float(w);
            const float pr = h16(__fsub_rn(h16(__fmul_rn(wr, vr)), h16(__fmul_rn(wi, vi))));
            const float pi = h16(__fadd_rn(h16(__fmul_rn(wr, vi)), h16(__fmul_rn(wi, vr))));
            L16[pu] = make_float2(__fadd_rn(u.x, pr), __fadd_rn(u.y, pi));
            L16[pv] = make_float2(__fsub_rn(u.x, pr), __fsub_rn(u.y, pi));
        }
        __syncthreads();
    }
    float2* yl = y + line * (int64_t)n;
    int bad = 0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const float2 v = L16[i];
        if (!isfinite(v.x) || !isfinite(v.y)) bad = 1;
        yl[i] = make_float2((float)quantize_ref((double)v.x, f16fmt), (float)quantize_ref((double)v.y, f16fmt));
    }
    if (bad) atomicOr(nonfinite, 1);
}

__global__ void k_ref_bitrev(const double2* __restrict__ x, double2* __restrict__ w, int64_t rows, int n,
                             int log2n) {
    const int64_t total = rows * n;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = e / n;
        const int i = (int)(e - r * n);
        const int src = log2n ? (int)(__brev((unsigned)i) >> (32 - log2n)) : 0;
        w[e] = x[r * n + src];
    }
}

__global__ void k_ref_stage(double2* __restrict__ w, int64_t rows, int n, int s,
                            const double2* __restrict__ tw, int inverse) {
    const int half = 1 << s, m = n / 2;
    const int64_t total = rows * m;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = e / m;
        const int t = (int)(e - r * m);
        const int g = t >> s, j = t & (half - 1);
        double2* l = w + r * n;
        const int pu = g * 2 * half + j, pv = pu + half;
        const double2 u = l[pu], v = l[pv];
        const double2 c = tw[half + j];
        const double br = c.x, bi = inverse ? -c.y : c.y;
        const double tr = __fma_rn(v.x, br, -__dmul_rn(v.y, bi));
        const double ti = __fma_rn(v.x, bi, __dmul_rn(v.y, br));
        l[pu] = make_double2(__dadd_rn(u.x, tr), __dadd_rn(u.y, ti));
        l[pv] = make_double2(__dsub_rn(u.x, tr), __dsub_rn(u.y, ti));
    }
}

cudaError_t launch_fp16_rows(const void* x, int x_is_c128, void* y, int64_t batch, int n, const void* tw,
                             int inverse, int* nonfinite, cudaStream_t st) {
    if (batch <= 0) return cudaSuccess;
    int log2n = 0;
    while ((1 << log2n) < n) ++log2n;
    const size_t smem = (size_t)n * sizeof(float2);
    {
        cudaError_t e = x_is_c128 ? ensure_smem_attr((const void*)k_fp16_lines<double2>, 227 * 1024)
                                  : ensure_smem_attr((const void*)k_fp16_lines<float2>, 227 * 1024);
        if (e != cudaSuccess) return e;
    }
    const FmtDesc f16 = make_fmt(5, 10, POL_IEEE, 15);
    const int nt = n / 2 < 512 ? (n / 2 < 32 ? 32 : n / 2) : 512;
    if (x_is_c128)
        k_fp16_lines<double2><<<(unsigned)batch, nt, smem, st>>>(reinterpret_cast<const double2*>(x),
                                                                 reinterpret_cast<float2*>(y), n, log2n,
                                                                 reinterpret_cast<const __half2*>(tw), inverse,
                                                                 f16, nonfinite);
    else
        k_fp16_lines<float2><<<(unsigned)batch, nt, smem, st>>>(reinterpret_cast<const float2*>(x),
                                                                reinterpret_cast<float2*>(y), n, log2n,
                                                                reinterpret_cast<const __half2*>(tw), inverse,
                                                                f16, nonfinite);
    note_launch();
    return cudaGetLastError();
}

cudaError_t launch_f64_rows(const void* x, void* y, int64_t batch, int n, const void* tw, int inverse,
                            cudaStream_t st) {
    if (batch <= 0) return cudaSuccess;
    int log2n = 0;
    while ((1 << log2n) < n) ++log2n;
    double2* w = reinterpret_cast<double2*>(y);
    k_ref_bitrev<<<grid_for(batch * n, 256), 256, 0, st>>>(reinterpret_cast<const double2*>(x), w, batch, n, log2n);
    note_launch();
    for (int s = 0; s < log2n; ++s) {
        k_ref_stage<<<grid_for(batch * (n / 2), 256), 256, 0, st>>>(w, batch, n, s,
                                                                   reinterpret_cast<const double2*>(tw), inverse);
        note_launch();
    }
    return cudaGetLastError();
}

}  // namespace mxfft
