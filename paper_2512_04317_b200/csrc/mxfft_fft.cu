// mxfft_fft.cu -- generic reference-literal MX transform + pass dispatch.
//
// The hot path is the line kernel in mxfft_lines.cu.  This file holds the
// generic kernel used for everything the line kernel does not cover (element
// formats without a hardware quantizer -- FP16, the test-only WIDE E8M23, any
// custom MinifloatFormat --, block sizes with cpb > 32, n < 32): a direct
// restatement of _fft_batch_mx (fftcore.py:259-282) with the FP64 quantizer and
// products in FP32 or FP64 per fftcore.py:163.  One CTA per line.
#include "mxfft_common.cuh"
#include "mxfft_generic.cuh"
#include "mxfft_internal.h"

namespace mxfft {

// ---------------------------------------------------------------------------
// generic kernel: any format / block size / n >= 2 (reference-literal, FP64
// quantizer, products in FP32 or FP64 per fftcore.py:163).  One CTA per line.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_lines_generic(GenericArgs a) {
    extern __shared__ float4 smem4[];
    float2* L = reinterpret_cast<float2*>(smem4);
    const FmtDesc f = a.fmt;
    const int n = a.n, m = n / 2, cpb = a.cpb;
    const int64_t line = blockIdx.x;
    int64_t base;
    int64_t img;
    if (a.col_mode) {
        img = line / n;
        base = img * a.img_elems + (line % n);
    } else {
        img = line / a.lines_per_image;
        base = line * n;
    }
    const int64_t es = a.col_mode ? n : 1;
    const int kin = a.kin_sign * (a.kvec ? a.kvec[img / a.k_group] : 0) + a.kin_const;
    const int kout = a.kout_sign * (a.kvec ? a.kvec[img / a.k_group] : 0) + a.kout_const;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        int r = (int)(__brev((unsigned)i) >> (32 - a.log2n));
        if (a.log2n == 0) r = 0;
        L[i] = gscale(a.in[base + (int64_t)r * es], kin);
    }
    __syncthreads();
    auto acc = [L](int i) { return L + i; };
    for (int s = 0; s < a.log2n; ++s) {
        generic_stage(acc, s, m, cpb, f, a.wcr, a.wci, a.wsexp, a.inverse, threadIdx.x, blockDim.x);
        __syncthreads();
    }
    for (int i = threadIdx.x; i < n; i += blockDim.x) a.out[base + (int64_t)i * es] = gscale(L[i], kout);
}


cudaError_t run_lines(const Plan& p, const LinePass& lp, cudaStream_t st) {
    if (mx_lines_ok(p)) return run_mx_lines(p, lp, st);
    if (lp.d_vexp) return cudaErrorNotSupported;  // stage capture is a line-kernel feature
    GenericArgs g{};
    g.in = reinterpret_cast<const float2*>(lp.in);
    g.out = reinterpret_cast<float2*>(lp.out);
    g.n = p.n;
    g.log2n = p.log2n;
    g.cpb = p.cpb;
    g.fmt = p.fmt;
    g.wcr = p.d_wcr;
    g.wci = p.d_wci;
    g.wsexp = p.d_wsexp;
    g.inverse = lp.inverse;
    g.col_mode = lp.col_mode;
    g.img_elems = lp.img_elems;
    g.lines_per_image = lp.lines_per_image;
    g.kvec = lp.kvec;
    g.k_group = lp.k_group > 0 ? lp.k_group : 1;
    g.kin_sign = lp.kin_sign;
    g.kout_sign = lp.kout_sign;
    g.kout_const = lp.kout_const;
    g.kin_const = lp.kin_const;
    const size_t smem = (size_t)p.n * sizeof(float2);
    if (smem > 227 * 1024) return cudaErrorInvalidValue;
    {
        cudaError_t e = ensure_smem_attr((const void*)k_lines_generic, 227 * 1024);
        if (e != cudaSuccess) return e;
    }
    const int64_t lines = lp.col_mode ? lp.batch * p.n : lp.total_lines;
    k_lines_generic<<<(unsigned)lines, 256, smem, st>>>(g);
    note_launch();
    return cudaGetLastError();
}

}  // namespace mxfft
