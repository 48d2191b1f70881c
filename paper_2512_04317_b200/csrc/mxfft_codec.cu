// mxfft_codec.cu -- element/MX block codec kernels, plan-table construction, RSS.
//
// These serve the public codec API (quantize_array, encode_block_mx,
// decode_block_mx) and plan creation.  They use the reference-literal FP64
// quantizer (quantize_ref == minifloat.py:114-120) because the API takes FP64
// inputs: rounding FP64 -> FP32 before a hardware cvt would double-round.
#include "mxfft_common.cuh"
#include "mxfft_internal.h"

namespace mxfft {

__global__ void k_quantize_f64(const double* __restrict__ x, double* __restrict__ out, int64_t n,
                               FmtDesc f, int32_t* nonfinite) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const double v = x[i];
        if (!isfinite(v)) {
            if (nonfinite) *nonfinite = 1;
            out[i] = 0.0;
            continue;
        }
        out[i] = quantize_ref(v, f);
    }
}

static int grid_for(int64_t n, int threads) {
    int64_t g = (n + threads - 1) / threads;
    if (g > 148 * 32) g = 148 * 32;
    return (int)(g < 1 ? 1 : g);
}

cudaError_t launch_quantize_f64(const double* x, double* out, int64_t n, const FmtDesc& f,
                                int32_t* d_nonfinite, cudaStream_t st) {
    if (n <= 0) return cudaSuccess;
    k_quantize_f64<<<grid_for(n, 256), 256, 0, st>>>(x, out, n, f, d_nonfinite);
    note_launch();
    return cudaGetLastError();
}

// encode_block_mx (mxblock.py:41-51), one warp per block.
__global__ void k_encode_f64(const double* __restrict__ v, int64_t nblocks, int len, FmtDesc f,
                             double* __restrict__ codes, double* __restrict__ scales,
                             int* __restrict__ scale_exp, int32_t* nonfinite) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t b = warp; b < nblocks; b += nwarps) {
        const double* x = v + b * len;
        double amax = 0.0;
        int bad = 0;
        for (int i = lane; i < len; i += 32) {
            const double a = x[i];
            bad |= !isfinite(a);
            amax = fmax(amax, fabs(a));
        }
        for (int o = 16; o; o >>= 1) {
            amax = fmax(amax, __shfl_xor_sync(0xffffffffu, amax, o));
            bad |= __shfl_xor_sync(0xffffffffu, bad, o);
        }
        if (bad) {
            if (lane == 0 && nonfinite) *nonfinite = 1;
            continue;
        }
        const int se = block_scale_exp(amax, f);
        const double inv = ldexp(1.0, -se);
        for (int i = lane; i < len; i += 32) codes[b * len + i] = quantize_ref(x[i] * inv, f);
        if (lane == 0) {
            if (scales) scales[b] = ldexp(1.0, se);
            if (scale_exp) scale_exp[b] = se;
        }
    }
}

cudaError_t launch_encode_f64(const double* v, int64_t nblocks, int block_len, const FmtDesc& f,
                              double* codes, double* scales, int* scale_exp, int32_t* d_nonfinite,
                              cudaStream_t st) {
    if (nblocks <= 0) return cudaSuccess;
    k_encode_f64<<<grid_for(nblocks * 32, 256), 256, 0, st>>>(v, nblocks, block_len, f, codes,
                                                               scales, scale_exp, d_nonfinite);
    note_launch();
    return cudaGetLastError();
}

// decode_block_mx (mxblock.py:86-90): (codes[0::2] + i codes[1::2]) * scale
__global__ void k_decode_f64(const double* __restrict__ codes, const double* __restrict__ scales,
                             int64_t nblocks, int len, double* __restrict__ out) {
    const int64_t half = len / 2;
    const int64_t total = nblocks * half;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t b = i / half, j = i - b * half;
        const double s = scales[b];
        out[2 * i] = codes[b * len + 2 * j] * s;
        out[2 * i + 1] = codes[b * len + 2 * j + 1] * s;
    }
}

cudaError_t launch_decode_f64(const double* codes, const double* scales, int64_t nblocks,
                              int block_len, double* out, cudaStream_t st) {
    if (nblocks <= 0) return cudaSuccess;
    k_decode_f64<<<grid_for(nblocks * (block_len / 2), 256), 256, 0, st>>>(codes, scales, nblocks,
                                                                          block_len, out);
    note_launch();
    return cudaGetLastError();
}

// Twiddle encoding (fftcore.py:108-113 -> _encode_blocks_batch): one thread per
// (stage, block); tw: complex128 (stages, m) in butterfly order.
__global__ void k_plan_encode(const double* __restrict__ tw, int stages, int m, int cpb, FmtDesc f,
                              double* wcr, double* wci, int* wsexp) {
    const int nb = m / cpb;
    const int64_t total = (int64_t)stages * nb;
    for (int64_t id = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; id < total;
         id += (int64_t)gridDim.x * blockDim.x) {
        const int s = (int)(id / nb), k = (int)(id % nb);
        const double* w = tw + 2 * ((int64_t)s * m + (int64_t)k * cpb);
        double amax = 0.0;
        for (int j = 0; j < cpb; ++j) amax = fmax(amax, fmax(fabs(w[2 * j]), fabs(w[2 * j + 1])));
        const int se = block_scale_exp(amax, f);
        const double inv = ldexp(1.0, -se);
        for (int j = 0; j < cpb; ++j) {
            const int64_t o = (int64_t)s * m + (int64_t)k * cpb + j;
            wcr[o] = quantize_ref(w[2 * j] * inv, f);
            wci[o] = quantize_ref(w[2 * j + 1] * inv, f);
        }
        wsexp[id] = se;
    }
}

// Kernel tables: stage s, j < 2^s at entry 2^s + j (entry 0 unused).
// Butterfly t = j of group 0 carries twiddle j, and its block is j / cpb
// (fftcore.py:101-113), so one entry per (s, j) describes every block.
// Codes are packed f16x2 (exact for every MX element format).
__global__ void k_plan_tables(const double* wcr, const double* wci, const int* wsexp, int stages,
                              int m, int cpb, unsigned* tw_fwd, unsigned* tw_inv,
                              signed char* tw_exp) {
    const int nb = m / cpb;
    const int total = 1 << stages;
    for (int id = blockIdx.x * blockDim.x + threadIdx.x; id < total; id += gridDim.x * blockDim.x) {
        if (id == 0) {
            tw_fwd[0] = tw_inv[0] = 0u;
            tw_exp[0] = 0;
            continue;
        }
        const int s = 31 - __clz(id);
        const int j = id - (1 << s);
        const double r = wcr[(int64_t)s * m + j], im = wci[(int64_t)s * m + j];
        const __half2 f = __halves2half2(__double2half(r), __double2half(im));
        const __half2 c = __halves2half2(__double2half(r), __double2half(-im));
        tw_fwd[id] = *reinterpret_cast<const unsigned*>(&f);
        tw_inv[id] = *reinterpret_cast<const unsigned*>(&c);
        const int e = wsexp[(int64_t)s * nb + j / cpb];
        tw_exp[id] = (signed char)(e < -128 ? -128 : (e > 127 ? 127 : e));
    }
}

cudaError_t plan_encode(Plan& p, const double* d_tw, cudaStream_t st) {
    const int m = p.n / 2;
    const int nb = m / p.cpb;
    const int64_t total = (int64_t)p.log2n * nb;
    k_plan_encode<<<grid_for(total, 128), 128, 0, st>>>(d_tw, p.log2n, m, p.cpb, p.fmt, p.d_wcr,
                                                        p.d_wci, p.d_wsexp);
    note_launch();
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    k_plan_tables<<<grid_for(p.n, 256), 256, 0, st>>>(p.d_wcr, p.d_wci, p.d_wsexp, p.log2n, m,
                                                       p.cpb, p.d_tw16_fwd, p.d_tw16_inv, p.d_twe8);
    note_launch();
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    // stage 0/1 shortcut is valid only if the encoded twiddles are exactly
    // w = 1 (j = 0) and w = -i (stage 1, j = 1) at block scale 2^-emax
    p.trivial01 = 0;
    if (p.log2n >= 2 && p.fmt.id != F_GENERIC) {
        double cr[3], ci[3];
        int ex0 = 0, ex1 = 0, ex1b = 0;
        const int nb = m / p.cpb;
        if ((e = cudaStreamSynchronize(st)) != cudaSuccess) return e;
        cudaMemcpy(&cr[0], p.d_wcr, sizeof(double), cudaMemcpyDeviceToHost);
        cudaMemcpy(&ci[0], p.d_wci, sizeof(double), cudaMemcpyDeviceToHost);
        cudaMemcpy(&cr[1], p.d_wcr + m, 2 * sizeof(double), cudaMemcpyDeviceToHost);
        cudaMemcpy(&ci[1], p.d_wci + m, 2 * sizeof(double), cudaMemcpyDeviceToHost);
        cudaMemcpy(&ex0, p.d_wsexp, sizeof(int), cudaMemcpyDeviceToHost);
        cudaMemcpy(&ex1, p.d_wsexp + nb, sizeof(int), cudaMemcpyDeviceToHost);
        cudaMemcpy(&ex1b, p.d_wsexp + nb + (1 / p.cpb), sizeof(int), cudaMemcpyDeviceToHost);
        const double one = ldexp(1.0, p.fmt.emax);
        p.trivial01 = cr[0] == one && ci[0] == 0.0 && cr[1] == one && ci[1] == 0.0 &&
                      cr[2] == 0.0 && ci[2] == -one && ex0 == -p.fmt.emax && ex1 == -p.fmt.emax &&
                      ex1b == -p.fmt.emax;
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
    }
    return cudaSuccess;
}

// _mx_multiply_batch (fftcore.py:150-183) and butterfly_mx (fftcore.py:186-235)
// on FP64 operands, one thread per MX block of cpb complex values: the v block
// is encoded (fftcore.py:131-147: amax of |re|, |im|, shared power-of-two
// scale, quantize_array of v * 2^-e), the mantissa-space products are taken in
// the reference's product dtype (FP32 unless the format is too wide,
// fftcore.py:163), renormalized by 2^-shift when the block maximum exceeds
// max_finite (exact integer shift, fftcore.py:172-177), requantized and
// decoded with the scale ws * sv * 2^shift.  wv (complex128) receives the
// decoded products; with u, y0 = u32 + wv32 and y1 = u32 - wv32 (complex64).
// Twiddle tables (wcr, wci: nb x cpb, ws: nb) are shared by every row.
__global__ void k_mx_multiply(const double2* __restrict__ v, const double* __restrict__ wcr,
                              const double* __restrict__ wci, const double* __restrict__ ws, int64_t rows, int m,
                              int cpb, FmtDesc f, double2* __restrict__ wv, const double2* __restrict__ u,
                              float2* __restrict__ y0, float2* __restrict__ y1, int32_t* nonfinite) {
    const int nb = m / cpb;
    for (int64_t gb = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; gb < rows * nb;
         gb += (int64_t)gridDim.x * blockDim.x) {
        const int64_t row = gb / nb;
        const int blk = (int)(gb - row * nb);
        const double2* vb = v + row * m + (int64_t)blk * cpb;
        double amax = 0.0;
        bool bad = false;
        for (int i = 0; i < cpb; ++i) {
            const double2 t = vb[i];
            bad |= !isfinite(t.x) || !isfinite(t.y);
            amax = fmax(amax, fmax(fabs(t.x), fabs(t.y)));
        }
        if (bad) {
            if (nonfinite) *nonfinite = 1;
            continue;
        }
        const int se = block_scale_exp(amax, f);
        const double inv = ldexp(1.0, -se);
        const double* xr = wcr + (int64_t)blk * cpb;
        const double* xi = wci + (int64_t)blk * cpb;
        // products and their block maximum
        double ap = 0.0;
        for (int i = 0; i < cpb; ++i) {
            const double2 t = vb[i];
            const double yr = quantize_ref(__dmul_rn(t.x, inv), f), yi = quantize_ref(__dmul_rn(t.y, inv), f);
            if (f.prod_f32) {
                const float pr = __fsub_rn(__fmul_rn((float)xr[i], (float)yr), __fmul_rn((float)xi[i], (float)yi));
                const float pi = __fadd_rn(__fmul_rn((float)xr[i], (float)yi), __fmul_rn((float)xi[i], (float)yr));
                ap = fmax(ap, (double)fmaxf(fabsf(pr), fabsf(pi)));
            } else {
                const double pr = __dsub_rn(__dmul_rn(xr[i], yr), __dmul_rn(xi[i], yi));
                const double pi = __dadd_rn(__dmul_rn(xr[i], yi), __dmul_rn(xi[i], yr));
                ap = fmax(ap, fmax(fabs(pr), fabs(pi)));
            }
        }
        int sh = 0;
        if (ap > f.max_finite) {
            int ea, em;
            const double ma = frexp(ap, &ea), mm = frexp(f.max_finite, &em);
            sh = ea - em + (ma > mm ? 1 : 0);  // = ceil(log2(ap / max_finite)), exactly
        }
        const double s_out = __dmul_rn(__dmul_rn(ws[blk], ldexp(1.0, se)), ldexp(1.0, sh));
        for (int i = 0; i < cpb; ++i) {
            const double2 t = vb[i];
            const double yr = quantize_ref(__dmul_rn(t.x, inv), f), yi = quantize_ref(__dmul_rn(t.y, inv), f);
            double pr, pi;
            if (f.prod_f32) {
                float r = __fsub_rn(__fmul_rn((float)xr[i], (float)yr), __fmul_rn((float)xi[i], (float)yi));
                float im = __fadd_rn(__fmul_rn((float)xr[i], (float)yi), __fmul_rn((float)xi[i], (float)yr));
                if (sh) {
                    const float fac = (float)ldexp(1.0, -sh);
                    r = __fmul_rn(r, fac);
                    im = __fmul_rn(im, fac);
                }
                pr = r;
                pi = im;
            } else {
                pr = __dsub_rn(__dmul_rn(xr[i], yr), __dmul_rn(xi[i], yi));
                pi = __dadd_rn(__dmul_rn(xr[i], yi), __dmul_rn(xi[i], yr));
                if (sh) {
                    pr = __dmul_rn(pr, ldexp(1.0, -sh));
                    pi = __dmul_rn(pi, ldexp(1.0, -sh));
                }
            }
            const double2 w = make_double2(__dmul_rn(quantize_ref(pr, f), s_out), __dmul_rn(quantize_ref(pi, f), s_out));
            const int64_t o = row * m + (int64_t)blk * cpb + i;
            if (wv) wv[o] = w;
            if (u) {
                const double2 uu = u[o];
                const float ur = (float)uu.x, ui = (float)uu.y, wr = (float)w.x, wi = (float)w.y;
                y0[o] = make_float2(__fadd_rn(ur, wr), __fadd_rn(ui, wi));
                y1[o] = make_float2(__fsub_rn(ur, wr), __fsub_rn(ui, wi));
            }
        }
    }
}

cudaError_t launch_mx_multiply(const void* v, const double* wcr, const double* wci, const double* ws, int64_t rows,
                               int m, int cpb, const FmtDesc& f, void* wv, const void* u, void* y0, void* y1,
                               int32_t* nonfinite, cudaStream_t st) {
    const int64_t nblk = rows * (m / cpb);
    if (nblk <= 0) return cudaSuccess;
    k_mx_multiply<<<grid_for(nblk, 128), 128, 0, st>>>(
        reinterpret_cast<const double2*>(v), wcr, wci, ws, rows, m, cpb, f, reinterpret_cast<double2*>(wv),
        reinterpret_cast<const double2*>(u), reinterpret_cast<float2*>(y0), reinterpret_cast<float2*>(y1), nonfinite);
    note_launch();
    return cudaGetLastError();
}

// |z| exactly as numpy 2.3.5 computes np.abs(complex128) on FMA hosts:
// larger * sqrt(fma(r, r, 1)), r = smaller / larger (IEEE-rounded ops only).
__device__ __forceinline__ double np_cabs(double re, double im) {
    const double a = fabs(re), b = fabs(im);
    const double larger = fmax(a, b), smaller = fmin(a, b);
    if (larger == 0.0) return 0.0;
    const double r = __ddiv_rn(smaller, larger);
    return __dmul_rn(__dsqrt_rn(__fma_rn(r, r, 1.0)), larger);
}

// rss (mri.py:70-81): sqrt(sum_c |T_c|^2), coils accumulated in order.
// With kvec / econst, every coil value of group g is first multiplied by
// 2^(ksign * kvec[g] + econst) in FP64 (exact): the pipelines' x 1/N^2 and
// undo_prescale (mri.py:101-107, prescale.py:89-91) applied in FP64, as the
// reference does, before |.|.
template <typename T>
__global__ void k_rss(const T* __restrict__ x, int64_t groups, int coils, int64_t npix,
                      const int32_t* __restrict__ kvec, int ksign, int econst, double* __restrict__ out) {
    const int64_t total = groups * npix;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t g = i / npix, p = i - g * npix;
        const int e = (kvec ? ksign * kvec[g] : 0) + econst;
        const double f = ldexp(1.0, e);
        double acc = 0.0;
        for (int c = 0; c < coils; ++c) {
            const T v = x[(g * coils + c) * npix + p];
            const double m = e ? np_cabs(__dmul_rn((double)v.x, f), __dmul_rn((double)v.y, f))
                               : np_cabs((double)v.x, (double)v.y);
            const double sq = __dmul_rn(m, m);
            acc = c == 0 ? sq : __dadd_rn(acc, sq);
        }
        out[i] = __dsqrt_rn(acc);
    }
}

// apply_prescale (prescale.py:76-86) followed by the complex64 cast of the
// transform's first gather (fftcore.py:262): y = complex64(x * 2^k[seg]),
// the product taken in FP64 (exact) and rounded to FP32 once.
__global__ void k_prescale_apply_c128(const double2* __restrict__ x, float2* __restrict__ y, int64_t seg_points,
                                      int64_t total, const int32_t* __restrict__ kvec) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        const double f = ldexp(1.0, kvec[i / seg_points]);
        const double2 v = x[i];
        y[i] = make_float2(__double2float_rn(__dmul_rn(v.x, f)), __double2float_rn(__dmul_rn(v.y, f)));
    }
}

// data * math.ldexp(1.0, k) of apply_prescale for float32 / float64 arrays
// (flat real scalars; complex arrays as interleaved pairs): the factor comes
// in already rounded to the array's precision, as numpy rounds the weak
// Python-float scalar, and each product is rounded once.
// Complex arrays are multiplied as numpy multiplies complex by the scalar
// cast to complex, (re f - im 0, re 0 + im f): identical to (re f, im f)
// except for infinities and NaNs (inf * 0 = NaN), which it reproduces.
template <typename T, bool CPLX>
__global__ void k_scale(const T* __restrict__ x, T* __restrict__ y, int64_t n, T f) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        if (CPLX) {
            const T re = x[2 * i], im = x[2 * i + 1];
            y[2 * i] = re * f - im * T(0);
            y[2 * i + 1] = re * T(0) + im * f;
        } else {
            y[i] = x[i] * f;
        }
    }
}

// Batched square transpose of complex64 images, y[b][j][i] = x[b][i][j]
// (np.ascontiguousarray(rows.T), fftcore.py:352): 64 x 64 tiles through
// shared memory; every global access is a 512-byte warp-contiguous run.
constexpr int TT = 64;
#ifndef MXFFT_TRANSPOSE_V2
#define MXFFT_TRANSPOSE_V2 1  // 16-byte global accesses, XOR-swizzled tile (when everything is 16-byte aligned)
#endif
template <bool V2>
__global__ void __launch_bounds__(256) k_transpose_c64(const float2* __restrict__ x, float2* __restrict__ y,
                                                       int n, int tiles_per_dim, int64_t ntiles, int64_t ldx,
                                                       int64_t bsx) {
if constexpr (V2) {
    // Each warp moves whole 512-byte rows as float4 (two complex per thread).
    // Tile element (r, c) lives at column c ^ ((r >> 1) & 15): a half-warp of
    // the store pass reads column k of rows 2l (or 2l + 1), l < 16, which then
    // hit 16 different 8-byte bank slots.
    __shared__ float2 tile[TT][TT];
    const int l = threadIdx.x & 31, w = threadIdx.x >> 5;  // 32 lanes x 8 warps
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const int64_t per = (int64_t)tiles_per_dim * tiles_per_dim;
        const int64_t b = t / per;
        const int r = (int)(t - b * per);
        const int i0 = (r / tiles_per_dim) * TT, j0 = (r % tiles_per_dim) * TT;
        const float2* xb = x + b * bsx;
        float2* yb = y + b * (int64_t)n * n;
        float4 v[8];
#pragma unroll
        for (int q = 0; q < 8; ++q)  // rows w + 8q, columns 2l, 2l + 1
            v[q] = __ldg(reinterpret_cast<const float4*>(xb + (int64_t)(i0 + w + 8 * q) * ldx + j0) + l);
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const int rr = w + 8 * q, f = (rr >> 1) & 15;
            tile[rr][(2 * l) ^ f] = make_float2(v[q].x, v[q].y);
            tile[rr][(2 * l + 1) ^ f] = make_float2(v[q].z, v[q].w);
        }
        __syncthreads();
#pragma unroll
        for (int q = 0; q < 8; ++q) {  // output row j0 + k, k = w + 8q: input rows 2l, 2l + 1 at column k
            const int k = w + 8 * q;
            const float2 a = tile[2 * l][k ^ (l & 15)], c = tile[2 * l + 1][k ^ (l & 15)];
            reinterpret_cast<float4*>(yb + (int64_t)(j0 + k) * n + i0)[l] = make_float4(a.x, a.y, c.x, c.y);
        }
        __syncthreads();
    }
    } else {
    __shared__ float2 tile[TT][TT + 1];
    const int tx = threadIdx.x & 63, ty = threadIdx.x >> 6;  // 64 x 4 threads
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const int64_t per = (int64_t)tiles_per_dim * tiles_per_dim;
        const int64_t b = t / per;
        const int r = (int)(t - b * per);
        const int i0 = (r / tiles_per_dim) * TT, j0 = (r % tiles_per_dim) * TT;
        const float2* xb = x + b * bsx;
        float2* yb = y + b * (int64_t)n * n;
#pragma unroll 4
        for (int k = ty; k < TT; k += 4) tile[k][tx] = xb[(int64_t)(i0 + k) * ldx + j0 + tx];
        __syncthreads();
#pragma unroll 4
        for (int k = ty; k < TT; k += 4) yb[(int64_t)(j0 + k) * n + i0 + tx] = tile[tx][k];
        __syncthreads();
    }
    }
}

cudaError_t launch_transpose_c64(const void* x, void* y, int64_t batch, int n, cudaStream_t st,
                                 int64_t ldx, int64_t bsx) {
    if (batch <= 0) return cudaSuccess;
    if (n % TT) return cudaErrorInvalidValue;
    if (ldx <= 0) ldx = n;
    if (bsx <= 0) bsx = (int64_t)n * n;
    const int tpd = n / TT;
    const int64_t ntiles = batch * (int64_t)tpd * tpd;
    const unsigned grid = (unsigned)(ntiles < 148 * 8 ? ntiles : 148 * 8);
    const bool v2 = MXFFT_TRANSPOSE_V2 && ((ldx | bsx) & 1) == 0 &&
                    ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(y)) & 15) == 0;
    if (v2)
        k_transpose_c64<true><<<grid, 256, 0, st>>>(reinterpret_cast<const float2*>(x), reinterpret_cast<float2*>(y),
                                                    n, tpd, ntiles, ldx, bsx);
    else
        k_transpose_c64<false><<<grid, 256, 0, st>>>(reinterpret_cast<const float2*>(x), reinterpret_cast<float2*>(y),
                                                     n, tpd, ntiles, ldx, bsx);
    note_launch();
    return cudaGetLastError();
}

// |z| exactly as numpy's np.abs(complex128) (the prescale magnitude,
// prescale.py:66), FP64 out.
template <typename T>
__global__ void k_cabs(const T* __restrict__ x, int64_t n, double* __restrict__ out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const T v = x[i];
        out[i] = np_cabs((double)v.x, (double)v.y);
    }
}

cudaError_t launch_cabs(const void* x, int is_c128, int64_t n, double* out, cudaStream_t st) {
    if (n <= 0) return cudaSuccess;
    if (is_c128)
        k_cabs<double2><<<grid_for(n, 256), 256, 0, st>>>(reinterpret_cast<const double2*>(x), n, out);
    else
        k_cabs<float2><<<grid_for(n, 256), 256, 0, st>>>(reinterpret_cast<const float2*>(x), n, out);
    note_launch();
    return cudaGetLastError();
}

cudaError_t launch_rss(const void* x, int is_c128, int64_t groups, int coils, int64_t npix,
                       double* out, cudaStream_t st, const int32_t* kvec, int ksign, int econst) {
    if (groups * npix <= 0) return cudaSuccess;
    if (is_c128)
        k_rss<double2><<<grid_for(groups * npix, 256), 256, 0, st>>>(
            reinterpret_cast<const double2*>(x), groups, coils, npix, kvec, ksign, econst, out);
    else
        k_rss<float2><<<grid_for(groups * npix, 256), 256, 0, st>>>(
            reinterpret_cast<const float2*>(x), groups, coils, npix, kvec, ksign, econst, out);
    note_launch();
    return cudaGetLastError();
}

cudaError_t launch_prescale_apply_c128(const void* x, void* y, int64_t seg_points, int64_t nseg,
                                       const int32_t* kvec, cudaStream_t st) {
    const int64_t total = seg_points * nseg;
    if (total <= 0) return cudaSuccess;
    k_prescale_apply_c128<<<grid_for(total, 256), 256, 0, st>>>(reinterpret_cast<const double2*>(x),
                                                               reinterpret_cast<float2*>(y), seg_points, total,
                                                               kvec);
    note_launch();
    return cudaGetLastError();
}

cudaError_t launch_scale(const void* x, void* y, int64_t n, int dtype, double f, cudaStream_t st) {
    if (n <= 0) return cudaSuccess;
    const int g = grid_for(n, 256);
    switch (dtype) {
        case 0: k_scale<float, false><<<g, 256, 0, st>>>((const float*)x, (float*)y, n, (float)f); break;
        case 1: k_scale<double, false><<<g, 256, 0, st>>>((const double*)x, (double*)y, n, f); break;
        case 2: k_scale<float, true><<<g, 256, 0, st>>>((const float*)x, (float*)y, n, (float)f); break;
        case 3: k_scale<double, true><<<g, 256, 0, st>>>((const double*)x, (double*)y, n, f); break;
        default: return cudaErrorInvalidValue;
    }
    note_launch();
    return cudaGetLastError();
}

}  // namespace mxfft

namespace mxfft {

// Self-test (test instrumentation): for every finite FP32 bit pattern x, compare
// the hardware quantizer used inside the transform (HwFmt<ID>::q2) with the
// reference-literal FP64 quantizer (quantize_ref); count mismatches.
template <int ID>
__global__ void k_selftest_hwq(FmtDesc f, unsigned long long* mismatches, unsigned* first_bad) {
    const uint64_t total = 1ull << 32;
    unsigned long long bad = 0;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < total / 2;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const unsigned b0 = (unsigned)(2 * i), b1 = b0 + 1;
        float a = __uint_as_float(b0), b = __uint_as_float(b1);
        const bool fa = isfinite(a), fb = isfinite(b);
        if (!fa) a = 0.f;
        if (!fb) b = 0.f;
        float qa, qb;
        HwFmt<ID>::q2(a, b, qa, qb);
        if (fa && (double)qa != quantize_ref((double)a, f)) {
            ++bad;
            atomicMin(first_bad, b0);
        }
        if (fb && (double)qb != quantize_ref((double)b, f)) {
            ++bad;
            atomicMin(first_bad, b1);
        }
    }
    if (bad) atomicAdd(mismatches, bad);
}

cudaError_t launch_selftest_hwq(const FmtDesc& f, unsigned long long* mism, unsigned* first_bad,
                                cudaStream_t st) {
    const int grid = 148 * 16, thr = 256;
    switch (f.id) {
        case F_E4M3: k_selftest_hwq<F_E4M3><<<grid, thr, 0, st>>>(f, mism, first_bad); break;
        case F_E5M2: k_selftest_hwq<F_E5M2><<<grid, thr, 0, st>>>(f, mism, first_bad); break;
        case F_E2M3: k_selftest_hwq<F_E2M3><<<grid, thr, 0, st>>>(f, mism, first_bad); break;
        case F_E3M2: k_selftest_hwq<F_E3M2><<<grid, thr, 0, st>>>(f, mism, first_bad); break;
        case F_E2M1: k_selftest_hwq<F_E2M1><<<grid, thr, 0, st>>>(f, mism, first_bad); break;
        default: return cudaErrorInvalidValue;
    }
    note_launch();
    return cudaGetLastError();
}

}  // namespace mxfft
