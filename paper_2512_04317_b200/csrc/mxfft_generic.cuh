// mxfft_generic.cuh -- reference-literal MX butterfly stages over a line held
// in shared memory (FP64 quantizer, products in FP32 or FP64 per
// fftcore.py:163).  Used by the generic kernel (formats without a hardware
// quantizer) and by the line kernel's exact replay of a group whose block
// exponents left the fast range.
#pragma once
#include "mxfft_common.cuh"

namespace mxfft {

__device__ __forceinline__ float2 gscale(float2 a, int e) {
    if (e == 0) return a;
    const double f = ldexp(1.0, e);
    return make_float2((float)((double)a.x * f), (float)((double)a.y * f));
}

// Stage s of _fft_batch_mx (fftcore.py:269-281) on the line L (accessor:
// L(i) -> float2* of position i).  Blocks of cpb butterflies are spread over
// threads tid, tid + nthr, ...; the caller synchronises between stages.
template <class Acc>
__device__ __forceinline__ void generic_stage(Acc L, int s, int m, int cpb, const FmtDesc& f,
                                              const double* wcr_all, const double* wci_all,
                                              const int* wse_all, bool inverse, int tid, int nthr) {
    const int half = 1 << s, nb = m / cpb;
    const double* wcr = wcr_all + (int64_t)s * m;
    const double* wci = wci_all + (int64_t)s * m;
    const int* wse = wse_all + (int64_t)s * nb;
    const double wsign = inverse ? -1.0 : 1.0;
    for (int blk = tid; blk < nb; blk += nthr) {
        double amax = 0.0;
        for (int i = 0; i < cpb; ++i) {
            const int t = blk * cpb + i, g = t >> s, j = t & (half - 1);
            const float2 v = *L(g * 2 * half + half + j);
            amax = fmax(amax, fmax(fabs((double)v.x), fabs((double)v.y)));
        }
        const int ev = block_scale_exp(amax, f);
        const double inv = ldexp(1.0, -ev);
        // pass A: product block amax
        double ap = 0.0;
        for (int i = 0; i < cpb; ++i) {
            const int t = blk * cpb + i, g = t >> s, j = t & (half - 1);
            const float2 v = *L(g * 2 * half + half + j);
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
            const float2 v = *L(pv);
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
            const float2 u = *L(pu);
            *L(pu) = make_float2(__fadd_rn(u.x, tr), __fadd_rn(u.y, ti));
            *L(pv) = make_float2(__fsub_rn(u.x, tr), __fsub_rn(u.y, ti));
        }
    }
}

}  // namespace mxfft
