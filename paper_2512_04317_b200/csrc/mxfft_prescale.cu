// mxfft_prescale.cu -- compute_prescale (prescale.py:61-73) on the device.
//
// Per segment (one coil stack / one image):
//   m     = |x| exactly as numpy's np.abs(complex128) (see np_cabs below)
//   a_max = max m ;  p_tau = np.percentile(m[m > 0], tau), method "linear"
//   k1 = round_half_away(log2(target / max(a_max, 1e-30)))
//   k2 = ceil(log2(tau_min / max(p_tau, 1e-30)))
//   k  = clip(max(k1, k2), k_min, k_max)
//
// The percentile needs two order statistics of the nonzero magnitudes.  They
// are found with a histogram radix-select that never sorts the segment:
//   pass 1: bin every nonzero point by a cheap monotone key of |z|^2 (1/8
//           binade of |z|^2 = 1/16 binade of |z|); count nnz; track the top key;
//   scan  : locate the bins holding ranks r_lo, r_hi;
//   pass 2: compute the exact numpy magnitude only for points in those bins
//           (+-1 bin, which absorbs any key rounding) and sort that handful in
//           shared memory (bitonic); a radix-select over the exact FP64 bits is
//           the fallback when the window overflows the candidate buffer.
// One CTA per segment; pass 2 re-reads the segment from L2.
#include <cfloat>

#include "mxfft_common.cuh"
#include "mxfft_internal.h"
#include "../../include/mxfft_b200.h"

namespace mxfft {

constexpr int PS_THREADS = 1024;
constexpr int NBINS = 8192;
constexpr int CAND_CAP = 4096;

__device__ __forceinline__ double np_cabs_d(double re, double im) {
    const double a = fabs(re), b = fabs(im);
    const double larger = fmax(a, b), smaller = fmin(a, b);
    if (larger == 0.0) return 0.0;
    const double r = __ddiv_rn(smaller, larger);
    return __dmul_rn(__dsqrt_rn(__fma_rn(r, r, 1.0)), larger);
}

// Monotone bin key (non-decreasing in |z| up to key rounding) for complex64.
// key = 8 * (unbiased exponent of |z|^2 + 171) + top 3 mantissa bits; |z|^2 of
// complex64 spans [2^-298, 2^257] -> keys [0, 4447].
__device__ __forceinline__ int key_c64(float re, float im) {
    const float a = fmaxf(fabsf(re), fabsf(im));
    if (a >= 0x1p-60f && a <= 0x1p60f) {
        const float s = __fmaf_rn(re, re, __fmul_rn(im, im));
        return (int)(__float_as_uint(s) >> 20) + 352;  // (be-127+171)*8 + mant3
    }
    // rescale so that max(|re|,|im|) is in [1,2): |z|^2 = s' * 2^(-2 sc)
    const int sc = -floor_log2f(a);
    double f = ldexp(1.0, sc);
    const float r2 = (float)((double)re * f), i2 = (float)((double)im * f);
    const float s = __fmaf_rn(r2, r2, __fmul_rn(i2, i2));
    const unsigned b = __float_as_uint(s);
    const int be = (int)(b >> 23) - 127 - 2 * sc;
    int key = (be + 171) * 8 + (int)((b >> 20) & 7);
    return key < 0 ? 0 : (key > NBINS - 1 ? NBINS - 1 : key);
}

// complex128 inputs (public API): key straight from the exact magnitude bits
// (11-bit exponent + 2 mantissa bits); exactly monotone.
__device__ __forceinline__ int key_of_m(double m) {
    return (int)(__double_as_longlong(m) >> 50);
}

template <typename T>
struct Elem;
template <>
struct Elem<float2> {
    static __device__ __forceinline__ bool finite(float2 v) { return isfinite(v.x) && isfinite(v.y); }
    static __device__ __forceinline__ bool nonzero(float2 v) { return v.x != 0.f || v.y != 0.f; }
    static __device__ __forceinline__ int key(float2 v) { return key_c64(v.x, v.y); }
    static __device__ __forceinline__ double mag(float2 v) { return np_cabs_d((double)v.x, (double)v.y); }
};
template <>
struct Elem<double2> {
    static __device__ __forceinline__ bool finite(double2 v) { return isfinite(v.x) && isfinite(v.y); }
    static __device__ __forceinline__ bool nonzero(double2 v) { return v.x != 0.0 || v.y != 0.0; }
    static __device__ __forceinline__ int key(double2 v) { return key_of_m(np_cabs_d(v.x, v.y)); }
    static __device__ __forceinline__ double mag(double2 v) { return np_cabs_d(v.x, v.y); }
};

struct PsCfg {
    double target, q, tau_min;  // q = tau / 100 (np.percentile's true_divide)
    int k_min, k_max;
};

__device__ __forceinline__ int round_half_away(double v) {
    return v >= 0 ? (int)floor(__dadd_rn(v, 0.5)) : (int)ceil(__dsub_rn(v, 0.5));
}

// block-wide exclusive prefix sum over NBINS bins held in smem (in place),
// returns nothing; every thread owns NBINS / PS_THREADS consecutive bins.
__device__ void block_scan_bins(unsigned* hist, unsigned* warp_sums) {
    constexpr int PER = NBINS / PS_THREADS;
    const int t = threadIdx.x;
    unsigned loc[PER];
    unsigned s = 0;
#pragma unroll
    for (int i = 0; i < PER; ++i) {
        loc[i] = hist[t * PER + i];
        s += loc[i];
    }
    // inclusive warp scan of s
    const int lane = t & 31, w = t >> 5;
    unsigned x = s;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        unsigned y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) warp_sums[w] = x;
    __syncthreads();
    if (w == 0) {
        unsigned v = warp_sums[lane];
        unsigned z = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            unsigned y = __shfl_up_sync(0xffffffffu, z, o);
            if (lane >= o) z += y;
        }
        warp_sums[lane] = z - v;  // exclusive
    }
    __syncthreads();
    unsigned run = warp_sums[w] + x - s;
#pragma unroll
    for (int i = 0; i < PER; ++i) {
        hist[t * PER + i] = run;  // exclusive prefix
        run += loc[i];
    }
    __syncthreads();
}

struct PsShared {
    unsigned hist[NBINS];
    unsigned warp_sums[32];
    double cand[CAND_CAP];
    unsigned long long amax_bits;
    unsigned long long nnz;
    int maxkey;
    int nonfinite;
    unsigned ncand;
    int jlo, jhi;          // bins holding ranks r_lo, r_hi
    unsigned off;          // number of points in bins < jlo - 1
    unsigned wcount;       // points in window bins [jlo-1, jhi+1]
    unsigned rh[256];      // radix-select digit histogram
    unsigned long long prefix;
};

// k-th smallest (0-based) exact magnitude among window points, by MSB-first
// radix select over the FP64 bit pattern (nonnegative doubles order as ints).
template <typename T>
__device__ double radix_select(const T* x, int64_t npts, int wlo, int whi, unsigned k, PsShared& S) {
    unsigned long long prefix = 0;
    for (int shift = 56; shift >= 0; shift -= 8) {
        for (int i = threadIdx.x; i < 256; i += blockDim.x) S.rh[i] = 0;
        __syncthreads();
        const unsigned long long hi_mask = shift == 56 ? 0ull : (~0ull << (shift + 8));
        for (int64_t i = threadIdx.x; i < npts; i += blockDim.x) {
            const T v = x[i];
            if (!Elem<T>::nonzero(v)) continue;
            const int key = Elem<T>::key(v);
            if (key < wlo || key > whi) continue;
            const unsigned long long b = (unsigned long long)__double_as_longlong(Elem<T>::mag(v));
            if ((b & hi_mask) != (prefix & hi_mask)) continue;
            atomicAdd(&S.rh[(b >> shift) & 255], 1u);
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            unsigned c = 0;
            int d = 0;
            for (; d < 256; ++d) {
                if (c + S.rh[d] > k) break;
                c += S.rh[d];
            }
            S.prefix = prefix | ((unsigned long long)d << shift);
            S.rh[0] = c;  // reuse slot to broadcast the count below
        }
        __syncthreads();
        prefix = S.prefix;
        k -= S.rh[0];
        __syncthreads();
    }
    return __longlong_as_double((long long)prefix);
}

template <typename T>
__device__ void ps_segment(const T* __restrict__ xall, int64_t npts, const PsCfg& cfg,
                           mxfft_prescale_result* out, int32_t* kvec, const int seg, PsShared& S) {
    const T* x = xall + (int64_t)seg * npts;
    const int tid = threadIdx.x;
    for (int i = tid; i < NBINS; i += blockDim.x) S.hist[i] = 0;
    if (tid == 0) {
        S.amax_bits = 0;
        S.nnz = 0;
        S.maxkey = -1;
        S.nonfinite = 0;
        S.ncand = 0;
    }
    __syncthreads();

    // ---- pass 1: finiteness, nnz, key histogram, top key ----
    unsigned long long my_nnz = 0;
    int my_max = -1, bad = 0;
    for (int64_t i = tid; i < npts; i += blockDim.x) {
        const T v = x[i];
        if (!Elem<T>::finite(v)) {
            bad = 1;
            continue;
        }
        if (!Elem<T>::nonzero(v)) continue;
        const int key = Elem<T>::key(v);
        ++my_nnz;
        my_max = max(my_max, key);
        atomicAdd(&S.hist[key], 1u);
    }
    for (int o = 16; o; o >>= 1) {
        my_nnz += __shfl_xor_sync(0xffffffffu, my_nnz, o);
        my_max = max(my_max, __shfl_xor_sync(0xffffffffu, my_max, o));
        bad |= __shfl_xor_sync(0xffffffffu, bad, o);
    }
    if ((tid & 31) == 0) {
        atomicAdd(&S.nnz, my_nnz);
        atomicMax(&S.maxkey, my_max);
        if (bad) S.nonfinite = 1;
    }
    __syncthreads();
    if (S.nonfinite) {
        if (tid == 0) {
            mxfft_prescale_result r{};
            r.flags = 1;
            out[seg] = r;
            if (kvec) kvec[seg] = 0;
        }
        return;
    }
    const unsigned long long nnz = S.nnz;
    double a_max = 0.0, p_tau = 0.0;
    if (nnz > 0) {
        // ranks of the two neighbouring order statistics (numpy _get_indexes)
        const double virt = __dmul_rn((double)(nnz - 1), cfg.q);
        unsigned r_lo, r_hi;
        double gamma;
        if (virt >= (double)(nnz - 1)) {
            r_lo = r_hi = (unsigned)(nnz - 1);
            gamma = __dadd_rn(virt, 1.0);
        } else {
            r_lo = (unsigned)floor(virt);
            r_hi = r_lo + 1;
            gamma = __dsub_rn(virt, (double)r_lo);
        }
        // counts -> exclusive prefix; locate the bins of r_lo / r_hi
        block_scan_bins(S.hist, S.warp_sums);
        for (int b = tid; b < NBINS; b += blockDim.x) {
            const unsigned lo = S.hist[b];
            const unsigned hi = b + 1 < NBINS ? S.hist[b + 1] : (unsigned)nnz;
            if (lo <= r_lo && r_lo < hi) S.jlo = b;
            if (lo <= r_hi && r_hi < hi) S.jhi = b;
        }
        __syncthreads();
        const int wlo = max(S.jlo - 1, 0), whi = min(S.jhi + 1, NBINS - 1);
        const unsigned off = S.hist[wlo];
        const unsigned wend = whi + 1 < NBINS ? S.hist[whi + 1] : (unsigned)nnz;
        const unsigned wcount = wend - off;
        const int mk = S.maxkey;
        __syncthreads();

        // ---- pass 2: exact magnitudes for the window and for the top bins ----
        for (int64_t i = tid; i < npts; i += blockDim.x) {
            const T v = x[i];
            if (!Elem<T>::nonzero(v)) continue;
            const int key = Elem<T>::key(v);
            const bool in_w = key >= wlo && key <= whi;
            const bool in_top = key >= mk - 1;
            if (!in_w && !in_top) continue;
            const double m = Elem<T>::mag(v);
            if (in_top) atomicMax(&S.amax_bits, (unsigned long long)__double_as_longlong(m));
            if (in_w && wcount <= CAND_CAP) {
                const unsigned slot = atomicAdd(&S.ncand, 1u);
                S.cand[slot] = m;
            }
        }
        __syncthreads();
        a_max = __longlong_as_double((long long)S.amax_bits);
        double vlo, vhi;
        if (wcount <= CAND_CAP) {
            // bitonic sort of the candidates (padded with +inf)
            int P = 1;
            while (P < (int)wcount) P <<= 1;
            for (int i = wcount + tid; i < P; i += blockDim.x) S.cand[i] = DBL_MAX;
            __syncthreads();
            for (int k = 2; k <= P; k <<= 1)
                for (int j = k >> 1; j > 0; j >>= 1) {
                    for (int i = tid; i < P; i += blockDim.x) {
                        const int l = i ^ j;
                        if (l > i) {
                            const double a = S.cand[i], b = S.cand[l];
                            const bool up = (i & k) == 0;
                            if ((a > b) == up) {
                                S.cand[i] = b;
                                S.cand[l] = a;
                            }
                        }
                    }
                    __syncthreads();
                }
            vlo = S.cand[r_lo - off];
            vhi = S.cand[r_hi - off];
        } else {
            vlo = radix_select<T>(x, npts, wlo, whi, r_lo - off, S);
            vhi = r_hi == r_lo ? vlo : radix_select<T>(x, npts, wlo, whi, r_hi - off, S);
        }
        // numpy _lerp: a + (b-a)*t, or b - (b-a)*(1-t) where t >= 0.5
        const double diff = __dsub_rn(vhi, vlo);
        p_tau = gamma >= 0.5 ? __dsub_rn(vhi, __dmul_rn(diff, __dsub_rn(1.0, gamma)))
                             : __dadd_rn(vlo, __dmul_rn(diff, gamma));
    }
    if (tid == 0) {
        const double EPS = 1e-30;
        const double L1 = log2(__ddiv_rn(cfg.target, a_max > EPS ? a_max : EPS));
        const double L2 = log2(__ddiv_rn(cfg.tau_min, p_tau > EPS ? p_tau : EPS));
        const int k1 = round_half_away(L1);
        const int k2 = (int)ceil(L2);
        int k = max(k1, k2);
        k = min(max(k, cfg.k_min), cfg.k_max);
        // near a rounding boundary the host re-derives k with its own log2
        const double d1 = fabs(fabs(L1 - trunc(L1)) - 0.5);
        const double d2 = fabs(L2 - rint(L2));
        const double tol1 = 1e-12 * fmax(1.0, fabs(L1)), tol2 = 1e-12 * fmax(1.0, fabs(L2));
        const double ratio2 = __ddiv_rn(cfg.tau_min, p_tau > EPS ? p_tau : EPS);
        const bool pow2 = (__double_as_longlong(ratio2) & 0xFFFFFFFFFFFFFll) == 0;
        const int amb = (d1 < tol1 || (d2 < tol2 && !pow2)) ? 2 : 0;
        mxfft_prescale_result r;
        r.a_max = a_max;
        r.p_tau = p_tau;
        r.k1 = k1;
        r.k2 = k2;
        r.k = k;
        r.flags = amb;
        r.nnz = (int64_t)nnz;
        out[seg] = r;
        if (kvec) kvec[seg] = k;
    }
}

// Exact kernel: one CTA per segment, or -- after the sampled fast path -- a
// small grid working through the list of segments the fast path flagged.
template <typename T>
__global__ void __launch_bounds__(PS_THREADS) k_prescale(const T* __restrict__ xall, int64_t npts,
                                                         PsCfg cfg, mxfft_prescale_result* out,
                                                         int32_t* kvec, const int* list, const int* list_n) {
    extern __shared__ unsigned long long ps_smem[];
    PsShared& S = *reinterpret_cast<PsShared*>(ps_smem);
    if (!list) {
        ps_segment(xall, npts, cfg, out, kvec, (int)blockIdx.x, S);
        return;
    }
    // launched with programmatic stream serialization behind the sampled kernels (its launch
    // overlaps their tail; the list is almost always empty): wait for them before the list
    pdl_launch_dependents();
    pdl_wait();
    const int cnt = *list_n;
    for (int i = blockIdx.x; i < cnt; i += gridDim.x) {
        ps_segment(xall, npts, cfg, out, kvec, list[i], S);
        __syncthreads();
    }
}

cudaError_t launch_prescale_fast(const float2* x, int64_t nseg, int64_t npts, double q,
                                 const mxfft_prescale_cfg& c, mxfft_prescale_result* out,
                                 int32_t* kvec, void* ws, int** list, int** list_n, cudaStream_t st);
int64_t prescale_fast_ws_bytes(int64_t nseg, int64_t npts);
bool prescale_fast_ok(int64_t npts);

cudaError_t launch_prescale(const void* x, int is_c128, int64_t nseg, int64_t npts,
                            const mxfft_prescale_cfg& c, mxfft_prescale_result* out, int32_t* kvec,
                            void* ws, int64_t ws_bytes, cudaStream_t st) {
    PsCfg cfg;
    cfg.target = c.target;
    cfg.q = c.tau / 100.0;
    cfg.tau_min = c.tau_min;
    cfg.k_min = c.k_min;
    cfg.k_max = c.k_max;
    const size_t smem = sizeof(PsShared);
    if (is_c128) {
        {
            cudaError_t e = ensure_smem_attr((const void*)k_prescale<double2>, (int)smem);
            if (e != cudaSuccess) return e;
        }
        k_prescale<double2><<<(unsigned)nseg, PS_THREADS, smem, st>>>(
            reinterpret_cast<const double2*>(x), npts, cfg, out, kvec, nullptr, nullptr);
        note_launch();
        return cudaGetLastError();
    }
    {
        cudaError_t e = ensure_smem_attr((const void*)k_prescale<float2>, (int)smem);
        if (e != cudaSuccess) return e;
    }
    if (ws && prescale_fast_ok(npts) && ws_bytes >= prescale_fast_ws_bytes(nseg, npts)) {
        // sampled fast path; segments it cannot settle are listed for the exact kernel
        int* list = nullptr;
        int* list_n = nullptr;
        cudaError_t e = launch_prescale_fast(reinterpret_cast<const float2*>(x), nseg, npts, cfg.q, c,
                                             out, kvec, ws, &list, &list_n, st);
        if (e != cudaSuccess) return e;
        const unsigned grid = (unsigned)(nseg < 64 ? nseg : 64);
        e = launch_pdl(k_prescale<float2>, grid, PS_THREADS, smem, st, reinterpret_cast<const float2*>(x), npts, cfg,
                       out, kvec, (const int*)list, (const int*)list_n);
        note_launch();
        return e != cudaSuccess ? e : cudaGetLastError();
    }
    k_prescale<float2><<<(unsigned)nseg, PS_THREADS, smem, st>>>(reinterpret_cast<const float2*>(x),
                                                                  npts, cfg, out, kvec, nullptr, nullptr);
    note_launch();
    return cudaGetLastError();
}

}  // namespace mxfft
