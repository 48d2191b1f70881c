// mxfft_fft.cu -- generic reference-literal MX transform + pass dispatch.
//
// The hot path is the line kernel in mxfft_lines.cu.  This file holds the
// generic kernel used for everything the line kernel does not cover (element
// formats without a hardware quantizer -- FP16, the test-only WIDE E8M23, any
// custom MinifloatFormat --, block sizes with cpb > 32, n < 32): a direct
// restatement of _fft_batch_mx (fftcore.py:259-282) with the FP64 quantizer and
// products in FP32 or FP64 per fftcore.py:163.  One CTA per line.
#include "mxfft_common.cuh"
#include "mxfft_internal.h"

namespace mxfft {

__device__ __forceinline__ float2 gscale(float2 a, int e) {
    if (e == 0) return a;
    const double f = ldexp(1.0, e);
    return make_float2((float)((double)a.x * f), (float)((double)a.y * f));
}

// ---------------------------------------------------------------------------
// generic kernel: any format / block size / n >= 2 (reference-literal, FP64
// quantizer, products in FP32 or FP64 per fftcore.py:163).  One CTA per line.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_lines_generic(GenericArgs a) {
    extern __shared__ float4 smem4[];
    float2* L = reinterpret_cast<float2*>(smem4);
    const FmtDesc f = a.fmt;
    const int n = a.n, m = n / 2, cpb = a.cpb, nb = m / cpb;
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
    const int kin = a.kin_sign * (a.kvec ? a.kvec[img / a.k_group] : 0);
    const int kout = a.kout_sign * (a.kvec ? a.kvec[img / a.k_group] : 0) + a.kout_const;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        int r = (int)(__brev((unsigned)i) >> (32 - a.log2n));
        if (a.log2n == 0) r = 0;
        L[i] = gscale(a.in[base + (int64_t)r * es], kin);
    }
    __syncthreads();
    for (int s = 0; s < a.log2n; ++s) {
        const int half = 1 << s;
        const double* wcr = a.wcr + (int64_t)s * m;
        const double* wci = a.wci + (int64_t)s * m;
        const int* wse = a.wsexp + (int64_t)s * nb;
        for (int blk = threadIdx.x; blk < nb; blk += blockDim.x) {
            double amax = 0.0;
            for (int i = 0; i < cpb; ++i) {
                const int t = blk * cpb + i, g = t >> s, j = t & (half - 1);
                const float2 v = L[g * 2 * half + half + j];
                amax = fmax(amax, fmax(fabs((double)v.x), fabs((double)v.y)));
            }
            const int ev = block_scale_exp(amax, f);
            const double inv = ldexp(1.0, -ev);
            const double wsign = a.inverse ? -1.0 : 1.0;
            // pass A: product block amax
            double ap = 0.0;
            for (int i = 0; i < cpb; ++i) {
                const int t = blk * cpb + i, g = t >> s, j = t & (half - 1);
                const float2 v = L[g * 2 * half + half + j];
                const double cvr = quantize_ref((double)v.x * inv, f);
                const double cvi = quantize_ref((double)v.y * inv, f);
                const double xr = wcr[t], xi = wsign * wci[t];
                if (f.prod_f32) {
                    const float pr = __fsub_rn(__fmul_rn((float)xr, (float)cvr), __fmul_rn((float)xi, (float)cvi));
                    const float pi = __fadd_rn(__fmul_rn((float)xr, (float)cvi), __fmul_rn((float)xi, (float)cvr));
                    ap = fmax(ap, (double)fmaxf(fabsf(pr), fabsf(pi)));
                } else {
                    const double pr = __dsub_rn(__dmul_rn(xr, cvr), __dmul_rn(xi, cvi));
                    const double pi = __dadd_rn(__dmul_rn(xr, cvi), __dmul_rn(xi, cvr));
                    ap = fmax(ap, fmax(fabs(pr), fabs(pi)));
                }
            }
            int sh = 0;
            if (ap > f.max_finite) {
                int ea, em;
                const double ma = frexp(ap, &ea), mm = frexp(f.max_finite, &em);
                sh = ea - em + (ma > mm ? 1 : 0);
            }
            const int E = wse[blk] + ev + sh;
            const double sc = ldexp(1.0, E);
            // pass B: requantize, decode, butterfly
            for (int i = 0; i < cpb; ++i) {
                const int t = blk * cpb + i, g = t >> s, j = t & (half - 1);
                const int pu = g * 2 * half + j, pv = pu + half;
                const float2 v = L[pv];
                const double cvr = quantize_ref((double)v.x * inv, f);
                const double cvi = quantize_ref((double)v.y * inv, f);
                const double xr = wcr[t], xi = wsign * wci[t];
                double pr, pi;
                if (f.prod_f32) {
                    float r = __fsub_rn(__fmul_rn((float)xr, (float)cvr), __fmul_rn((float)xi, (float)cvi));
                    float im = __fadd_rn(__fmul_rn((float)xr, (float)cvi), __fmul_rn((float)xi, (float)cvr));
                    if (sh) {
                        const float fac = (float)ldexp(1.0, -sh);
                        r = __fmul_rn(r, fac);
                        im = __fmul_rn(im, fac);
                    }
                    pr = r;
                    pi = im;
                } else {
                    pr = __dsub_rn(__dmul_rn(xr, cvr), __dmul_rn(xi, cvi));
                    pi = __dadd_rn(__dmul_rn(xr, cvi), __dmul_rn(xi, cvr));
                    if (sh) {
                        pr = __dmul_rn(pr, ldexp(1.0, -sh));
                        pi = __dmul_rn(pi, ldexp(1.0, -sh));
                    }
                }
                const float tr = (float)(quantize_ref(pr, f) * sc);
                const float ti = (float)(quantize_ref(pi, f) * sc);
                const float2 u = L[pu];
                L[pu] = make_float2(__fadd_rn(u.x, tr), __fadd_rn(u.y, ti));
                L[pv] = make_float2(__fsub_rn(u.x, tr), __fsub_rn(u.y, ti));
            }
        }
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
    const size_t smem = (size_t)p.n * sizeof(float2);
    if (smem > 227 * 1024) return cudaErrorInvalidValue;
    static bool attr_done = false;
    if (!attr_done) {
        cudaError_t e = cudaFuncSetAttribute(k_lines_generic, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             227 * 1024);
        if (e != cudaSuccess) return e;
        attr_done = true;
    }
    const int64_t lines = lp.col_mode ? lp.batch * p.n : lp.total_lines;
    k_lines_generic<<<(unsigned)lines, 256, smem, st>>>(g);
    note_launch();
    return cudaGetLastError();
}

}  // namespace mxfft
