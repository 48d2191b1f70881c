// mxfft_prescale_fast.cu -- sampled selection for compute_prescale on complex64
// segments (the pipeline hot path).  Exact; segments it cannot settle are
// flagged and recomputed by the histogram kernel in mxfft_prescale.cu.
//
//   sample : one CTA per segment reads pseudo-random whole 32-byte sectors
//            (S = 256 points for segments <= 2^16, 1024 <= 2^18, else 4096),
//            bitonic-sorts their squared magnitudes and brackets the rank of
//            the tau-percentile by +-(8 + 4 sigma) sample ranks (Floyd-Rivest);
//            the sample maximum is the threshold for peak candidates.
//   count  : one streaming pass, 16-byte loads, no per-point atomics: nnz, the
//            points strictly below the bracket, and bitmasks of the points in
//            the bracket / above the sample max, appended with one warp scan +
//            one atomic per warp.
//   select : a 512-bin histogram of the candidates' keys locates the bins of
//            the two order statistics; only the candidates of those bins (+-1)
//            get the exact numpy magnitude (np.abs, FP64) and a small bitonic
//            sort.  Guards: the selected magnitudes must sit clear of the
//            window edges by more than the FP32 key rounding, else fall back.
#include <cfloat>

#include "../../include/mxfft_b200.h"
#include "mxfft_common.cuh"
#include "mxfft_internal.h"

namespace mxfft {

constexpr int SAMPLE_MAX = 4096;
constexpr int SEL_THREADS = 256;
constexpr int TOPCAP = 2048;
constexpr int NBIN = 512;
constexpr int WCAP = 2048;  // exact-sort window capacity
constexpr int CNT_THREADS = 256;
constexpr int CNT_PER_THREAD = 16;  // complex values per thread per chunk
constexpr int CHUNK = CNT_THREADS * CNT_PER_THREAD;

struct SegState {
    float lo, hi, top;
    int pad0;
    unsigned long long nnz;
    unsigned below, ncand, ntop, flags;  // flags: 1 non-finite, 2 extreme range
};

// the bracket keeps ~(16 + 8 sqrt(q S)) / S of the points: 256 -> ~7%,
// 1024 -> ~3%, 4096 -> ~1.5%
static inline int sample_size(int64_t npts) {
    return npts < 32768 ? 256 : (npts <= 262144 ? 1024 : SAMPLE_MAX);
}

static inline int64_t cand_cap(int64_t npts) {
    int64_t c = npts / 4;
    return c < 1024 ? 1024 : (c > 16384 ? 16384 : c);
}

bool prescale_fast_ok(int64_t npts) { return npts >= 1024 && npts <= (int64_t(1) << 24); }

int64_t prescale_fast_ws_bytes(int64_t nseg, int64_t npts) {
    const int64_t st = ((int64_t)sizeof(SegState) * nseg + 255) / 256 * 256;
    const int64_t fb = ((int64_t)sizeof(int) * nseg + 255) / 256 * 256;
    return st + fb + nseg * (cand_cap(npts) + TOPCAP) * (int64_t)sizeof(float2);
}

__device__ __forceinline__ double np_cabs_f(double re, double im) {
    const double a = fabs(re), b = fabs(im);
    const double larger = fmax(a, b), smaller = fmin(a, b);
    if (larger == 0.0) return 0.0;
    const double r = __ddiv_rn(smaller, larger);
    return __dmul_rn(__dsqrt_rn(__fma_rn(r, r, 1.0)), larger);
}

// squared-magnitude key (FP32); points with |re|,|im| outside [2^-60, 2^60]
// are flagged and the segment goes to the exact kernel
__device__ __forceinline__ float skey(float re, float im) { return __fmaf_rn(re, re, __fmul_rn(im, im)); }

template <typename T>
__device__ void bitonic_sort(T* a, int P) {  // ascending, P a power of two, whole block
    for (int k = 2; k <= P; k <<= 1)
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int i = threadIdx.x; i < P; i += blockDim.x) {
                const int l = i ^ j;
                if (l > i) {
                    const T x = a[i], y = a[l];
                    if ((x > y) == ((i & k) == 0)) {
                        a[i] = y;
                        a[l] = x;
                    }
                }
            }
            __syncthreads();
        }
}

// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(SEL_THREADS) k_ps_sample(const float2* __restrict__ xall, int64_t npts,
                                                           int S, double q, SegState* st, int* fb) {
    __shared__ unsigned keys[SAMPLE_MAX];
    __shared__ int snz;
    const int seg = blockIdx.x, tid = threadIdx.x;
    const float2* x = xall + (int64_t)seg * npts;
    if (tid == 0) snz = 0;
    __syncthreads();
    // sector h(j) = j * odd mod nsec is a permutation when nsec is a power of two
    const int64_t nsec = npts / 4;
    int cnt = 0;
    for (int j = tid; j < S / 4; j += SEL_THREADS) {
        const uint64_t h = (uint64_t)j * 2654435761ull;
        const uint64_t sec = (nsec & (nsec - 1)) == 0 ? (h & (uint64_t)(nsec - 1)) : h % (uint64_t)nsec;
        const float4* p = reinterpret_cast<const float4*>(x + sec * 4);
        const float4 a = __ldg(p), b = __ldg(p + 1);
        const float v[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
#pragma unroll
        for (int h = 0; h < 4; ++h) {
            const float re = v[2 * h], im = v[2 * h + 1];
            const float m = fmaxf(fabsf(re), fabsf(im));
            unsigned k = 0xffffffffu;  // zeros / NaN sort last, excluded by count
            if (m > 0.f) {
                const float sk = (m >= 0x1p-60f && m <= 0x1p60f) ? skey(re, im) : (m < 1.f ? 0.f : 0x1p125f);
                k = __float_as_uint(sk);
                ++cnt;
            }
            keys[j * 4 + h] = k;
        }
    }
    for (int o = 16; o; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
    if ((tid & 31) == 0) atomicAdd(&snz, cnt);
    __syncthreads();
    bitonic_sort<unsigned>(keys, S);
    if (tid == 0) {
        SegState g;
        const int n = snz;
        if (n == 0) {
            g.lo = 0.f;
            g.hi = __int_as_float(0x7f800000);
            g.top = 0.f;
        } else {
            const double rs = (double)(n - 1) * q;
            const int d = 8 + (int)(4.0 * sqrt(rs + 1.0));
            const int ilo = (int)floor(rs) - d, ihi = (int)ceil(rs) + 1 + d;
            g.lo = ilo <= 0 ? 0.f : __uint_as_float(keys[ilo]) * (1.f - 0x1p-20f);
            g.hi = ihi >= n ? __int_as_float(0x7f800000) : __uint_as_float(keys[ihi]) * (1.f + 0x1p-20f);
            g.top = __uint_as_float(keys[n - 1]) * (1.f - 0x1p-20f);
        }
        g.pad0 = 0;
        g.nnz = 0;
        g.below = g.ncand = g.ntop = g.flags = 0;
        st[seg] = g;
        fb[seg] = 0;
    }
}

// ---------------------------------------------------------------------------
// warp-aggregated reservation of this thread's `cnt` slots: one atomic per warp
__device__ __forceinline__ unsigned warp_reserve(unsigned cnt, unsigned* counter) {
    const unsigned lane = threadIdx.x & 31;
    unsigned incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= (unsigned)o) incl += y;
    }
    unsigned base = 0;
    if (lane == 31 && incl) base = atomicAdd(counter, incl);
    base = __shfl_sync(0xffffffffu, base, 31);
    return base + incl - cnt;
}

__global__ void __launch_bounds__(CNT_THREADS, 4) k_ps_count(const float2* __restrict__ xall, int64_t npts,
                                                          int chunks_per_seg, SegState* st,
                                                          float2* cand, int64_t cap, float2* top) {
    const int64_t chunk = blockIdx.x;
    const int seg = (int)(chunk / chunks_per_seg);
    const int64_t start = (chunk - (int64_t)seg * chunks_per_seg) * CHUNK;
    const float2* x = xall + (int64_t)seg * npts;
    const SegState g = st[seg];
    unsigned nnz = 0, below = 0, cbits = 0, tbits = 0;
    float ksum = 0.f;  // NaN / Inf / key overflow propagate into the sum
    const int64_t p0 = start / 2;  // pairs of complex values per 16-byte load
    const int64_t pend = (npts / 2 < (start + CHUNK) / 2) ? npts / 2 : (start + CHUNK) / 2;
    const float4* x4 = reinterpret_cast<const float4*>(x);
    float4 v[CNT_PER_THREAD / 2];
#pragma unroll
    for (int it = 0; it < CNT_PER_THREAD / 2; ++it) {
        const int64_t pi = p0 + it * CNT_THREADS + threadIdx.x;
        v[it] = pi < pend ? __ldg(x4 + pi) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int it = 0; it < CNT_PER_THREAD / 2; ++it) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const float re = h ? v[it].z : v[it].x, im = h ? v[it].w : v[it].y;
            const bool nz = (re != 0.f) | (im != 0.f);
            const float sk = skey(re, im);
            ksum += sk;
            nnz += nz;
            below += nz & (sk < g.lo);
            cbits |= (unsigned)(nz & (sk >= g.lo) & (sk <= g.hi)) << (2 * it + h);
            tbits |= (unsigned)(nz & (sk >= g.top)) << (2 * it + h);
        }
    }
    unsigned slot = warp_reserve(__popc(cbits), &st[seg].ncand);
    if (cbits) {
        float2* cb = cand + (int64_t)seg * cap;
#pragma unroll
        for (int it = 0; it < CNT_PER_THREAD / 2; ++it)
#pragma unroll
            for (int h = 0; h < 2; ++h)
                if ((cbits >> (2 * it + h)) & 1) {
                    if (slot < cap) cb[slot] = h ? make_float2(v[it].z, v[it].w) : make_float2(v[it].x, v[it].y);
                    ++slot;
                }
    }
    slot = warp_reserve(__popc(tbits), &st[seg].ntop);
    if (tbits) {
        float2* tb = top + (int64_t)seg * TOPCAP;
#pragma unroll
        for (int it = 0; it < CNT_PER_THREAD / 2; ++it)
#pragma unroll
            for (int h = 0; h < 2; ++h)
                if ((tbits >> (2 * it + h)) & 1) {
                    if (slot < TOPCAP) tb[slot] = h ? make_float2(v[it].z, v[it].w) : make_float2(v[it].x, v[it].y);
                    ++slot;
                }
    }
    // non-finite input, or keys beyond FP32 range: let the exact kernel decide
    unsigned flags = (ksum <= 0x1p126f) ? 0u : 1u;
    for (int o = 16; o; o >>= 1) {
        nnz += __shfl_xor_sync(0xffffffffu, nnz, o);
        below += __shfl_xor_sync(0xffffffffu, below, o);
        flags |= __shfl_xor_sync(0xffffffffu, flags, o);
    }
    if ((threadIdx.x & 31) == 0) {
        atomicAdd(&st[seg].nnz, (unsigned long long)nnz);
        atomicAdd(&st[seg].below, below);
        if (flags) atomicOr(&st[seg].flags, flags);
    }
}

// ---------------------------------------------------------------------------
__device__ __forceinline__ int round_half_away_d(double v) {
    return v >= 0 ? (int)floor(__dadd_rn(v, 0.5)) : (int)ceil(__dsub_rn(v, 0.5));
}

struct SelShared {
    unsigned hist[NBIN];
    double w[WCAP];
    unsigned warp_sums[SEL_THREADS / 32];
    unsigned long long amax_b;
    unsigned wn;
    int bt, bt1, fail;
    unsigned woff, wend;
};

// bin of a key bit pattern inside [klo, khi] (monotone non-decreasing in k)
__device__ __forceinline__ int kbin(unsigned k, unsigned klo, float inv) {
    k = k < klo ? klo : k;
    const int b = (int)((float)(k - klo) * inv);
    return b >= NBIN ? NBIN - 1 : b;
}
// (approximately) the smallest key bit pattern of bin b; only used by the
// rounding guard, which has a 2^-18 relative margin
__device__ __forceinline__ unsigned bin_lo(int b, unsigned klo, float inv) {
    return klo + (unsigned)ceilf((float)b / inv);
}

__global__ void __launch_bounds__(SEL_THREADS) k_ps_select(SegState* st, int* fb, const float2* cand,
                                                           int64_t cap, const float2* top, double q,
                                                           mxfft_prescale_cfg c,
                                                           mxfft_prescale_result* out, int32_t* kvec) {
    __shared__ SelShared S;
    const int seg = blockIdx.x, tid = threadIdx.x;
    const SegState g = st[seg];
    const unsigned long long nnz = g.nnz;
    if (g.flags) {
        if (tid == 0) fb[seg] = 1;
        return;
    }
    double a_max = 0.0, p_tau = 0.0;
    if (nnz > 0) {
        const double virt = __dmul_rn((double)(nnz - 1), q);
        unsigned long long r_lo, r_hi;
        double gamma;
        if (virt >= (double)(nnz - 1)) {
            r_lo = r_hi = nnz - 1;
            gamma = __dadd_rn(virt, 1.0);
        } else {
            r_lo = (unsigned long long)floor(virt);
            r_hi = r_lo + 1;
            gamma = __dsub_rn(virt, (double)r_lo);
        }
        const unsigned nc = g.ncand, nt = g.ntop;
        if (!(nc <= cap && nt <= TOPCAP && nt >= 1 && g.below <= r_lo && r_hi < g.below + nc)) {
            if (tid == 0) fb[seg] = 1;
            return;
        }
        const unsigned t = (unsigned)(r_lo - g.below), t1 = (unsigned)(r_hi - g.below);
        const unsigned klo = __float_as_uint(g.lo), khi = __float_as_uint(g.hi);
        const float inv = (float)NBIN / ((float)(khi - klo) + 1.f);
        const float2* cb = cand + (int64_t)seg * cap;
        for (int i = tid; i < NBIN; i += SEL_THREADS) S.hist[i] = 0;
        if (tid == 0) {
            S.amax_b = 0;
            S.wn = 0;
            S.fail = 0;
        }
        __syncthreads();
        for (unsigned i = tid; i < nc; i += SEL_THREADS) {
            const float2 v = cb[i];
            atomicAdd(&S.hist[kbin(__float_as_uint(skey(v.x, v.y)), klo, inv)], 1u);
        }
        // peak: exact magnitudes of the few points above the sample maximum
        unsigned long long am = 0;
        for (unsigned i = tid; i < nt; i += SEL_THREADS) {
            const float2 v = top[(int64_t)seg * TOPCAP + i];
            am = max(am, (unsigned long long)__double_as_longlong(np_cabs_f((double)v.x, (double)v.y)));
        }
        for (int o = 16; o; o >>= 1) am = max(am, __shfl_xor_sync(0xffffffffu, am, o));
        if ((tid & 31) == 0) atomicMax(&S.amax_b, am);
        __syncthreads();
        // exclusive scan of the histogram (2 bins per thread)
        {
            const unsigned h0 = S.hist[2 * tid], h1 = S.hist[2 * tid + 1];
            unsigned incl = h0 + h1;
            const int lane = tid & 31, wp = tid >> 5;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const unsigned y = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += y;
            }
            if (lane == 31) S.warp_sums[wp] = incl;
            __syncthreads();
            unsigned wbase = 0;
            for (int w2 = 0; w2 < wp; ++w2) wbase += S.warp_sums[w2];
            const unsigned e0 = wbase + incl - h0 - h1, e1 = e0 + h0;
            if (e0 <= t && t < e1) S.bt = 2 * tid;
            if (e1 <= t && t < e1 + h1) S.bt = 2 * tid + 1;
            if (e0 <= t1 && t1 < e1) S.bt1 = 2 * tid;
            if (e1 <= t1 && t1 < e1 + h1) S.bt1 = 2 * tid + 1;
            __syncthreads();
            const int wlo = S.bt > 0 ? S.bt - 1 : 0, whi = S.bt1 < NBIN - 1 ? S.bt1 + 1 : NBIN - 1;
            if (2 * tid == wlo) S.woff = e0;
            if (2 * tid + 1 == wlo) S.woff = e1;
            if (2 * tid == whi) S.wend = e1;
            if (2 * tid + 1 == whi) S.wend = e1 + h1;
        }
        __syncthreads();
        const int wlo = S.bt > 0 ? S.bt - 1 : 0, whi = S.bt1 < NBIN - 1 ? S.bt1 + 1 : NBIN - 1;
        const unsigned woff = S.woff, wcount = S.wend - S.woff;
        if (wcount > WCAP) {
            if (tid == 0) fb[seg] = 1;
            return;
        }
        for (unsigned i = tid; i < nc; i += SEL_THREADS) {
            const float2 v = cb[i];
            const int b = kbin(__float_as_uint(skey(v.x, v.y)), klo, inv);
            if (b >= wlo && b <= whi) S.w[atomicAdd(&S.wn, 1u)] = np_cabs_f((double)v.x, (double)v.y);
        }
        __syncthreads();
        int P = 1;
        while (P < (int)wcount) P <<= 1;
        for (int i = (int)wcount + tid; i < P; i += SEL_THREADS) S.w[i] = DBL_MAX;
        __syncthreads();
        bitonic_sort<double>(S.w, P);
        const double vlo = S.w[t - woff], vhi = S.w[t1 - woff];
        // every point outside the window must order strictly on its side:
        // the picks must clear the window's key edges by more than the key rounding
        const float elo = wlo > 0 ? __uint_as_float(bin_lo(wlo, klo, inv)) : g.lo;
        const float ehi = whi < NBIN - 1 ? __uint_as_float(bin_lo(whi + 1, klo, inv)) : g.hi;
        bool good = true;
        if (elo > 0.f && !(elo >= 0x1p-100f && vlo * vlo > (double)elo * (1.0 + 0x1p-18))) good = false;
        if (ehi <= FLT_MAX && !(vhi * vhi < (double)ehi * (1.0 - 0x1p-18))) good = false;
        if (!good) {
            if (tid == 0) fb[seg] = 1;
            return;
        }
        a_max = __longlong_as_double((long long)S.amax_b);
        const double diff = __dsub_rn(vhi, vlo);
        p_tau = gamma >= 0.5 ? __dsub_rn(vhi, __dmul_rn(diff, __dsub_rn(1.0, gamma)))
                             : __dadd_rn(vlo, __dmul_rn(diff, gamma));
    }
    if (tid == 0) {
        const double EPS = 1e-30;
        const double r1 = __ddiv_rn(c.target, a_max > EPS ? a_max : EPS);
        const double r2 = __ddiv_rn(c.tau_min, p_tau > EPS ? p_tau : EPS);
        const double L1 = log2(r1), L2 = log2(r2);
        const int k1 = round_half_away_d(L1);
        const int k2 = (int)ceil(L2);
        int k = max(k1, k2);
        k = min(max(k, c.k_min), c.k_max);
        const double d1 = fabs(fabs(L1 - trunc(L1)) - 0.5);
        const double d2 = fabs(L2 - rint(L2));
        const bool pow2 = (__double_as_longlong(r2) & 0xFFFFFFFFFFFFFll) == 0;
        const int amb = (d1 < 1e-12 * fmax(1.0, fabs(L1)) || (d2 < 1e-12 * fmax(1.0, fabs(L2)) && !pow2)) ? 2 : 0;
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

cudaError_t launch_prescale_fast(const float2* x, int64_t nseg, int64_t npts, double q,
                                 const mxfft_prescale_cfg& c, mxfft_prescale_result* out,
                                 int32_t* kvec, void* ws, int** fallback, cudaStream_t st) {
    char* w = reinterpret_cast<char*>(ws);
    SegState* sst = reinterpret_cast<SegState*>(w);
    w += ((int64_t)sizeof(SegState) * nseg + 255) / 256 * 256;
    int* fb = reinterpret_cast<int*>(w);
    w += ((int64_t)sizeof(int) * nseg + 255) / 256 * 256;
    const int64_t cap = cand_cap(npts);
    float2* cand = reinterpret_cast<float2*>(w);
    float2* top = cand + nseg * cap;
    *fallback = fb;
    k_ps_sample<<<(unsigned)nseg, SEL_THREADS, 0, st>>>(x, npts, sample_size(npts), q, sst, fb);
    note_launch();
    const int cps = (int)((npts + CHUNK - 1) / CHUNK);
    k_ps_count<<<(unsigned)(nseg * cps), CNT_THREADS, 0, st>>>(x, npts, cps, sst, cand, cap, top);
    note_launch();
    k_ps_select<<<(unsigned)nseg, SEL_THREADS, 0, st>>>(sst, fb, cand, cap, top, q, c, out, kvec);
    note_launch();
    return cudaGetLastError();
}

}  // namespace mxfft
