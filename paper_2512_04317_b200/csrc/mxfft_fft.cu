// mxfft_fft.cu -- MX-scaled radix-2 DIT transforms for sm_100a.
//
// Reproduces _fft_batch_mx (fftcore.py:259-282) with _mx_multiply_batch
// (fftcore.py:150-183) inside every stage, bit-exactly:
//   * bit-reversed input order (fftcore.py:262);
//   * per stage, blocks of cpb consecutive butterflies in (group, j) order
//     (fftcore.py:269-272); v-block shared power-of-two scale (mxblock.py:27-38)
//     and element codes (RNE, saturating: hardware cvt.rn.satfinite);
//   * FP32 mantissa-space complex product of prequantized twiddle codes and v
//     codes (exact), per-block renormalization shift, requantization;
//   * FP32 butterfly u +- c*2^E (decode folded into an exact FMA).
//
// Layout: a "line" is one 1-D transform (a row, or a column of an n x n image).
// A CTA stages a tile of LT lines in shared memory; each thread owns CH
// consecutive (bit-reversed) positions of one line, so the first log2(CH)
// stages run entirely in registers with in-thread block maxima; the remaining
// stages exchange through shared memory, each thread taking CH/2 consecutive
// butterflies (= CH/(2 cpb) whole MX blocks) per stage.
#include <cstdio>

#include "mxfft_common.cuh"
#include "mxfft_internal.h"

namespace mxfft {

// ---------------------------------------------------------------------------
// per-block MX multiply + butterfly, hardware quantizer
// ---------------------------------------------------------------------------
struct DbgCtx {
    int32_t* vexp;
    float* vcodes;
    int32_t* pexp;
    int32_t* pshift;
    float* pcodes;
    int64_t row;   // global row index
    int nb;        // blocks per row per stage
    int m;         // n/2
    int64_t rows;  // rows in the batch
    int stage;
};

template <int ID, int CPB, bool DBG>
__device__ __noinline__ void mx_block_slow(float2* u, float2* v, const float2* w, int ew,
                                           const DbgCtx* dc, int blk) {
    using F = HwFmt<ID>;
    float am = 0.f;
    for (int i = 0; i < CPB; ++i) am = fmax3(am, fabsf(v[i].x), fabsf(v[i].y));
    const int ev = am > 0.f ? floor_log2f(am) - F::EMAX : 0;
    const double inv = ldexp(1.0, -ev);
    float cr[CPB], ci[CPB], pr[CPB], pi[CPB];
    float ap = 0.f;
    for (int i = 0; i < CPB; ++i) {
        F::q2((float)((double)v[i].x * inv), (float)((double)v[i].y * inv), cr[i], ci[i]);
        pr[i] = __fsub_rn(__fmul_rn(w[i].x, cr[i]), __fmul_rn(w[i].y, ci[i]));
        pi[i] = __fadd_rn(__fmul_rn(w[i].x, ci[i]), __fmul_rn(w[i].y, cr[i]));
        ap = fmax3(ap, fabsf(pr[i]), fabsf(pi[i]));
    }
    const int sh = ap > F::MAXF ? shift_for<F>(ap) : 0;
    const float fac = exp2i(-sh);
    const int E = ew + ev + sh;
    const double sc = ldexp(1.0, E);
    for (int i = 0; i < CPB; ++i) {
        float qr, qi;
        F::q2(__fmul_rn(pr[i], fac), __fmul_rn(pi[i], fac), qr, qi);
        const float tr = (float)((double)qr * sc), ti = (float)((double)qi * sc);
        const float2 uu = u[i];
        u[i] = make_float2(__fadd_rn(uu.x, tr), __fadd_rn(uu.y, ti));
        v[i] = make_float2(__fsub_rn(uu.x, tr), __fsub_rn(uu.y, ti));
        if (DBG) {
            int64_t o = ((int64_t)dc->stage * dc->rows + dc->row) * dc->m + (int64_t)blk * CPB + i;
            dc->vcodes[2 * o] = cr[i];
            dc->vcodes[2 * o + 1] = ci[i];
            dc->pcodes[2 * o] = qr;
            dc->pcodes[2 * o + 1] = qi;
        }
    }
    if (DBG) {
        int64_t o = ((int64_t)dc->stage * dc->rows + dc->row) * dc->nb + blk;
        dc->vexp[o] = ev;
        dc->pexp[o] = E;
        dc->pshift[o] = sh;
    }
}

// u, v: the block's cpb butterfly operands; w: twiddle codes (conjugated for the
// inverse); ew: log2 of the twiddle block scale.  On return u = u + wv,
// v = u - wv (fftcore.py:280-281).
template <int ID, int CPB, bool DBG>
__device__ __forceinline__ void mx_block(float2 (&u)[CPB], float2 (&v)[CPB],
                                         const float2 (&w)[CPB], int ew, const DbgCtx* dc,
                                         int blk) {
    using F = HwFmt<ID>;
    using R = DecodeRange<F>;
    // (1) v-block amax -> shared scale exponent (mxblock.py:27-38)
    float am = 0.f;
#pragma unroll
    for (int i = 0; i < CPB; ++i) am = fmax3(am, fabsf(v[i].x), fabsf(v[i].y));
    const int ev = am > 0.f ? floor_log2f(am) - F::EMAX : 0;
    // (2) v codes (fftcore.py:144-146)
    const float inv = exp2i(-ev);
    float cr[CPB], ci[CPB];
#pragma unroll
    for (int i = 0; i < CPB; ++i) F::q2(v[i].x * inv, v[i].y * inv, cr[i], ci[i]);
    // (3) exact mantissa-space products, one FP32 rounding each (fftcore.py:168-169)
    float pr[CPB], pi[CPB];
    float ap = 0.f;
#pragma unroll
    for (int i = 0; i < CPB; ++i) {
        pr[i] = __fmaf_rn(w[i].x, cr[i], -(w[i].y * ci[i]));
        pi[i] = __fmaf_rn(w[i].x, ci[i], w[i].y * cr[i]);
        ap = fmax3(ap, fabsf(pr[i]), fabsf(pi[i]));
    }
    // (4) renormalization (fftcore.py:171-179)
    const int sh = ap > F::MAXF ? shift_for<F>(ap) : 0;
    const int E = ew + ev + sh;
    const bool fast = (ev >= -127) & (ev <= 126) & (E >= R::ELO) & (E <= R::EHI);
    if (__builtin_expect(!fast, 0)) {
        // rare (extreme magnitudes): exact FP64-assisted path on a local copy so
        // that the register arrays never have their address taken
        float2 tmp[3 * CPB];
#pragma unroll
        for (int i = 0; i < CPB; ++i) {
            tmp[i] = u[i];
            tmp[CPB + i] = v[i];
            tmp[2 * CPB + i] = w[i];
        }
        mx_block_slow<ID, CPB, DBG>(tmp, tmp + CPB, tmp + 2 * CPB, ew, dc, blk);
#pragma unroll
        for (int i = 0; i < CPB; ++i) {
            u[i] = tmp[i];
            v[i] = tmp[CPB + i];
        }
        return;
    }
    const float fac = exp2i(-sh);
    const float sc = exp2i(E);
    // (5) requantize, (6) decode folded into the FP32 butterfly: c*2^E is an
    // exact FP32 value here, so fma(c, 2^E, u) == u + fl(c*2^E).
#pragma unroll
    for (int i = 0; i < CPB; ++i) {
        float qr, qi;
        F::q2(pr[i] * fac, pi[i] * fac, qr, qi);
        const float2 uu = u[i];
        u[i] = make_float2(__fmaf_rn(qr, sc, uu.x), __fmaf_rn(qi, sc, uu.y));
        v[i] = make_float2(__fmaf_rn(-qr, sc, uu.x), __fmaf_rn(-qi, sc, uu.y));
        if (DBG) {
            int64_t o = ((int64_t)dc->stage * dc->rows + dc->row) * dc->m + (int64_t)blk * CPB + i;
            dc->vcodes[2 * o] = cr[i];
            dc->vcodes[2 * o + 1] = ci[i];
            dc->pcodes[2 * o] = qr;
            dc->pcodes[2 * o + 1] = qi;
        }
    }
    if (DBG) {
        int64_t o = ((int64_t)dc->stage * dc->rows + dc->row) * dc->nb + blk;
        dc->vexp[o] = ev;
        dc->pexp[o] = E;
        dc->pshift[o] = sh;
    }
}

// ---------------------------------------------------------------------------
// line kernel
// ---------------------------------------------------------------------------
template <int BITS>
__host__ __device__ constexpr int brev_c(int i) {
    int r = 0;
    for (int b = 0; b < BITS; ++b) r |= ((i >> b) & 1) << (BITS - 1 - b);
    return r;
}

__device__ __forceinline__ float2 scale2(float2 a, float f) { return make_float2(a.x * f, a.y * f); }

// exact power-of-two scaling of an FP32 value (one rounding of the exact
// product, like the reference's FP64 scale followed by a complex64 cast)
__device__ __forceinline__ float2 pow2_scale(float2 a, int e) {
    if (e == 0) return a;
    if (e >= -126 && e <= 127) return scale2(a, exp2i(e));
    const double f = ldexp(1.0, e);
    return make_float2((float)((double)a.x * f), (float)((double)a.y * f));
}

__device__ __forceinline__ int line_k(const LinesArgs& a, int64_t img) {
    return a.kvec ? a.kvec[img / a.k_group] : 0;
}

template <int ID, int CPB, int LOGCH, bool DBG>
__global__ void __launch_bounds__(LOGCH == 6 ? 256 : 512) k_lines(LinesArgs a) {
    constexpr int CH = 1 << LOGCH;
    constexpr int HB = CH / 2;  // butterflies per thread per stage
    extern __shared__ float4 smem4[];
    float2* sm = reinterpret_cast<float2*>(smem4);
    const int tid = threadIdx.x;
    const int NT = blockDim.x;
    const int n = a.n;

    // ---- tile -> shared memory (apply_prescale fused: x * 2^k) ----
    int64_t img0 = 0, l0 = 0;
    if (a.col_mode) {
        img0 = blockIdx.x / a.tiles_per_image;
        l0 = (int64_t)(blockIdx.x % a.tiles_per_image) * a.LT;
        const float2* src = a.in + img0 * a.img_elems + l0;
        const int kin = a.kin_sign * line_k(a, img0);
        const int half_lt = a.LT >> 1;
        for (int idx = tid; idx < a.LT * n / 2; idx += NT) {
            const int p = idx / half_lt, lp = idx - p * half_lt;
            float4 q = __ldg(reinterpret_cast<const float4*>(src + (int64_t)p * n + 2 * lp));
            float2 e0 = pow2_scale(make_float2(q.x, q.y), kin);
            float2 e1 = pow2_scale(make_float2(q.z, q.w), kin);
            sm[(2 * lp) * a.LS + p] = e0;
            sm[(2 * lp + 1) * a.LS + p] = e1;
        }
    } else {
        l0 = (int64_t)blockIdx.x * a.LT;
        const int lt = (int)min((int64_t)a.LT, a.total_lines - l0);
        const float2* src = a.in + l0 * n;
        for (int idx = tid; idx < lt * n / 2; idx += NT) {
            const int l = (2 * idx) / n, p = 2 * idx - l * n;
            const int kin = a.kin_sign * line_k(a, (l0 + l) / a.lines_per_image);
            float4 q = __ldg(reinterpret_cast<const float4*>(src + (int64_t)l * n + p));
            float2 e0 = pow2_scale(make_float2(q.x, q.y), kin);
            float2 e1 = pow2_scale(make_float2(q.z, q.w), kin);
            *reinterpret_cast<float4*>(sm + l * a.LS + p) = make_float4(e0.x, e0.y, e1.x, e1.y);
        }
    }
    __syncthreads();

    const int line = tid >> a.log2T;
    const int tl = tid & (a.T - 1);
    const bool active = line < a.LT && (a.col_mode || l0 + line < a.total_lines);
    float2* L = sm + line * a.LS;
    DbgCtx dc;
    if (DBG) {
        dc.vexp = a.d_vexp;
        dc.vcodes = a.d_vcodes;
        dc.pexp = a.d_pexp;
        dc.pshift = a.d_pshift;
        dc.pcodes = a.d_pcodes;
        dc.row = l0 + line;
        dc.m = n / 2;
        dc.nb = (n / 2) / CPB;
        dc.rows = a.total_lines;
    }

    float2 x[CH];
    if (active) {
        // ---- bit-reversed gather (fftcore.py:262) ----
        const int rt = a.log2T ? (int)(__brev((unsigned)tl) >> (32 - a.log2T)) : 0;
#pragma unroll
        for (int i = 0; i < CH; ++i) x[i] = L[(brev_c<LOGCH>(i) << a.log2T) + rt];

        // ---- register-resident stages s < log2(CH) ----
#pragma unroll
        for (int s = 0; s < LOGCH; ++s) {
            if (s < a.stage_limit) {
                const int half = 1 << s;
                const float2* tw = a.tw + (half - 1);
                const int* twe = a.tw_exp + (half - 1);
                if (DBG) dc.stage = s;
#pragma unroll
                for (int k = 0; k < HB / CPB; ++k) {
                    float2 ub[CPB], vb[CPB], wb[CPB];
#pragma unroll
                    for (int i = 0; i < CPB; ++i) {
                        const int b = k * CPB + i;  // thread-local butterfly index
                        const int g = b >> s, j = b & (half - 1);
                        ub[i] = x[g * 2 * half + j];
                        vb[i] = x[g * 2 * half + half + j];
                        wb[i] = __ldg(tw + j);
                    }
                    const int j0 = (k * CPB) & (half - 1);
                    mx_block<ID, CPB, DBG>(ub, vb, wb, __ldg(twe + j0), &dc, tl * (HB / CPB) + k);
#pragma unroll
                    for (int i = 0; i < CPB; ++i) {
                        const int b = k * CPB + i;
                        const int g = b >> s, j = b & (half - 1);
                        x[g * 2 * half + j] = ub[i];
                        x[g * 2 * half + half + j] = vb[i];
                    }
                }
            }
        }
#pragma unroll
        for (int i = 0; i < CH; i += 2)
            *reinterpret_cast<float4*>(L + tl * CH + i) =
                make_float4(x[i].x, x[i].y, x[i + 1].x, x[i + 1].y);
    }

    // ---- shared-memory stages s >= log2(CH) ----
    for (int s = LOGCH; s < a.stage_limit; ++s) {
        __syncthreads();
        if (active) {
            const int half = 1 << s;
            const int b0 = tl * HB;
            const int g = b0 >> s, j0 = b0 & (half - 1);
            float2* U = L + g * 2 * half + j0;
            float2* V = U + half;
            float2 ub[HB], vb[HB];
#pragma unroll
            for (int i = 0; i < HB; i += 2) {
                float4 qu = *reinterpret_cast<const float4*>(U + i);
                float4 qv = *reinterpret_cast<const float4*>(V + i);
                ub[i] = make_float2(qu.x, qu.y);
                ub[i + 1] = make_float2(qu.z, qu.w);
                vb[i] = make_float2(qv.x, qv.y);
                vb[i + 1] = make_float2(qv.z, qv.w);
            }
            const float2* tw = a.tw + (half - 1) + j0;
            const int* twe = a.tw_exp + (half - 1) + j0;
            if (DBG) dc.stage = s;
#pragma unroll
            for (int k = 0; k < HB / CPB; ++k) {
                float2 ubk[CPB], vbk[CPB], wb[CPB];
#pragma unroll
                for (int i = 0; i < CPB; ++i) {
                    ubk[i] = ub[k * CPB + i];
                    vbk[i] = vb[k * CPB + i];
                    wb[i] = __ldg(tw + k * CPB + i);
                }
                mx_block<ID, CPB, DBG>(ubk, vbk, wb, __ldg(twe + k * CPB), &dc,
                                       b0 / CPB + k);
#pragma unroll
                for (int i = 0; i < CPB; ++i) {
                    ub[k * CPB + i] = ubk[i];
                    vb[k * CPB + i] = vbk[i];
                }
            }
#pragma unroll
            for (int i = 0; i < HB; i += 2) {
                *reinterpret_cast<float4*>(U + i) = make_float4(ub[i].x, ub[i].y, ub[i + 1].x, ub[i + 1].y);
                *reinterpret_cast<float4*>(V + i) = make_float4(vb[i].x, vb[i].y, vb[i + 1].x, vb[i + 1].y);
            }
        }
    }
    __syncthreads();

    // ---- shared memory -> global (undo_prescale / 1/n^2 fused: x * 2^(kout)) ----
    if (a.col_mode) {
        float2* dst = a.out + img0 * a.img_elems + l0;
        const int kout = a.kout_sign * line_k(a, img0) + a.kout_const;
        const int half_lt = a.LT >> 1;
        for (int idx = tid; idx < a.LT * n / 2; idx += NT) {
            const int p = idx / half_lt, lp = idx - p * half_lt;
            float2 e0 = pow2_scale(sm[(2 * lp) * a.LS + p], kout);
            float2 e1 = pow2_scale(sm[(2 * lp + 1) * a.LS + p], kout);
            *reinterpret_cast<float4*>(dst + (int64_t)p * n + 2 * lp) = make_float4(e0.x, e0.y, e1.x, e1.y);
        }
    } else {
        const int lt = (int)min((int64_t)a.LT, a.total_lines - l0);
        float2* dst = a.out + l0 * n;
        for (int idx = tid; idx < lt * n / 2; idx += NT) {
            const int l = (2 * idx) / n, p = 2 * idx - l * n;
            const int kout = a.kout_sign * line_k(a, (l0 + l) / a.lines_per_image) + a.kout_const;
            float4 q = *reinterpret_cast<const float4*>(sm + l * a.LS + p);
            float2 e0 = pow2_scale(make_float2(q.x, q.y), kout);
            float2 e1 = pow2_scale(make_float2(q.z, q.w), kout);
            *reinterpret_cast<float4*>(dst + (int64_t)l * n + p) = make_float4(e0.x, e0.y, e1.x, e1.y);
        }
    }
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
        L[i] = pow2_scale(a.in[base + (int64_t)r * es], kin);
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
    for (int i = threadIdx.x; i < n; i += blockDim.x) a.out[base + (int64_t)i * es] = pow2_scale(L[i], kout);
}

// ---------------------------------------------------------------------------
// launchers
// ---------------------------------------------------------------------------
template <int ID, int CPB, int LOGCH, bool DBG>
static cudaError_t launch_lines_t(const LinesArgs& a, int nt, size_t smem, cudaStream_t st) {
    auto k = k_lines<ID, CPB, LOGCH, DBG>;
    static bool attr_done = false;  // per instantiation
    if (!attr_done) {
        cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
        if (e != cudaSuccess) return e;
        attr_done = true;
    }
    int grid = a.col_mode ? (int)(a.batch * a.tiles_per_image) : (int)((a.total_lines + a.LT - 1) / a.LT);
    k<<<grid, nt, smem, st>>>(a);
    note_launch();
    return cudaGetLastError();
}

template <int ID, int CPB, bool DBG>
static cudaError_t dispatch_ch(const LinesArgs& a, int nt, size_t smem, cudaStream_t st) {
    constexpr int LOGCH = (2 * CPB > 32) ? 6 : 5;
    return launch_lines_t<ID, CPB, LOGCH, DBG>(a, nt, smem, st);
}

template <int ID, bool DBG>
static cudaError_t dispatch_cpb(const LinesArgs& a, int cpb, int nt, size_t smem, cudaStream_t st) {
    switch (cpb) {
        case 1: return dispatch_ch<ID, 1, DBG>(a, nt, smem, st);
        case 2: return dispatch_ch<ID, 2, DBG>(a, nt, smem, st);
        case 4: return dispatch_ch<ID, 4, DBG>(a, nt, smem, st);
        case 8: return dispatch_ch<ID, 8, DBG>(a, nt, smem, st);
        case 16: return dispatch_ch<ID, 16, DBG>(a, nt, smem, st);
        case 32: return dispatch_ch<ID, 32, DBG>(a, nt, smem, st);
    }
    return cudaErrorInvalidValue;
}

template <bool DBG>
static cudaError_t dispatch_fmt(const LinesArgs& a, int id, int cpb, int nt, size_t smem, cudaStream_t st) {
    switch (id) {
        case F_E4M3: return dispatch_cpb<F_E4M3, DBG>(a, cpb, nt, smem, st);
        case F_E5M2: return dispatch_cpb<F_E5M2, DBG>(a, cpb, nt, smem, st);
        case F_E2M3: return dispatch_cpb<F_E2M3, DBG>(a, cpb, nt, smem, st);
        case F_E3M2: return dispatch_cpb<F_E3M2, DBG>(a, cpb, nt, smem, st);
        case F_E2M1: return dispatch_cpb<F_E2M1, DBG>(a, cpb, nt, smem, st);
    }
    return cudaErrorInvalidValue;
}

bool fast_path_ok(const Plan& p) {
    if (p.fmt.id == F_GENERIC) return false;
    if (p.cpb > 32 || (p.cpb & (p.cpb - 1))) return false;
    const int logch = (2 * p.cpb > 32) ? 6 : 5;
    if (p.log2n < logch) return false;
    const int T = p.n >> logch;
    if (T > (logch == 6 ? 256 : 512)) return false;
    return true;
}

// Launch one pass of 1-D transforms over lines.
cudaError_t run_lines(const Plan& p, const LinePass& lp, cudaStream_t st) {
    if (fast_path_ok(p)) {
        LinesArgs a{};
        const int logch = (2 * p.cpb > 32) ? 6 : 5;
        a.in = reinterpret_cast<const float2*>(lp.in);
        a.out = reinterpret_cast<float2*>(lp.out);
        a.n = p.n;
        a.log2n = p.log2n;
        a.T = p.n >> logch;
        a.log2T = p.log2n - logch;
        int nt = a.T >= 128 ? a.T : 128;
        if (lp.col_mode && a.T < 16) nt = 16 * a.T;  // >= 16 columns per tile
        if (nt < 32) nt = 32;
        a.LT = nt / a.T;
        a.LS = a.LT > 1 ? p.n + 2 : p.n;
        a.col_mode = lp.col_mode;
        a.img_elems = lp.img_elems;
        a.lines_per_image = lp.lines_per_image;
        a.tiles_per_image = lp.col_mode ? (int)(p.n / a.LT) : 0;
        a.total_lines = lp.total_lines;
        a.batch = lp.batch;
        a.tw = lp.inverse ? p.d_tw_inv : p.d_tw_fwd;
        a.tw_exp = p.d_tw_exp;
        a.kvec = lp.kvec;
        a.k_group = lp.k_group > 0 ? lp.k_group : 1;
        a.kin_sign = lp.kin_sign;
        a.kout_sign = lp.kout_sign;
        a.kout_const = lp.kout_const;
        a.stage_limit = lp.stage_limit >= 0 ? lp.stage_limit : p.log2n;
        a.d_vexp = lp.d_vexp;
        a.d_vcodes = lp.d_vcodes;
        a.d_pexp = lp.d_pexp;
        a.d_pshift = lp.d_pshift;
        a.d_pcodes = lp.d_pcodes;
        if (lp.col_mode && (a.LT & 1)) return cudaErrorInvalidValue;
        size_t smem = (size_t)a.LT * a.LS * sizeof(float2);
        const bool dbg = lp.d_vexp != nullptr;
        return dbg ? dispatch_fmt<true>(a, p.fmt.id, p.cpb, nt, smem, st)
                   : dispatch_fmt<false>(a, p.fmt.id, p.cpb, nt, smem, st);
    }
    // generic path
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
    size_t smem = (size_t)p.n * sizeof(float2);
    if (smem > 227 * 1024) return cudaErrorInvalidValue;
    static bool attr_done = false;
    if (!attr_done) {
        cudaError_t e = cudaFuncSetAttribute(k_lines_generic, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
        if (e != cudaSuccess) return e;
        attr_done = true;
    }
    const int64_t lines = lp.col_mode ? lp.batch * p.n : lp.total_lines;
    k_lines_generic<<<(unsigned)lines, 256, smem, st>>>(g);
    note_launch();
    return cudaGetLastError();
}

}  // namespace mxfft
