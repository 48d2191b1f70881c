// mxfft_prescale_fast.cu -- sampled selection for compute_prescale on complex64
// segments (the pipeline hot path).  Exact; segments it cannot settle are
// listed and recomputed by the histogram kernel in mxfft_prescale.cu.
//
// Segments of up to 2^18 points (one image / coil stack of the pipelines) run
// ONE fused kernel, one CTA per segment: the three steps below back to back,
// with the bracket candidates kept in shared memory (no global atomics, one
// read of the segment).  Larger segments use the three kernels:
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
#include <cstdlib>
#include <climits>
#include <cstdio>

#include <cooperative_groups.h>

#include "../../include/mxfft_b200.h"
#include "mxfft_common.cuh"
#include "mxfft_internal.h"
#include "mxfft_stats.cuh"

namespace mxfft {

constexpr int SAMPLE_MAX = 4096;
constexpr int SEL_THREADS = 256;
constexpr int TOPCAP = 2048;
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

constexpr int64_t FUSED_MAX = int64_t(1) << 18;
#ifndef MXFFT_C3_CLUSTER
#define MXFFT_C3_CLUSTER 2  // CTAs per cluster (2 or 4; 0: off) when few large segments leave SMs idle (4 measured slower: 109 vs 80 us on C3)
#endif
#ifndef MXFFT_PS_SAMPLE_FIRST
#define MXFFT_PS_SAMPLE_FIRST 1  // lean statistics: issue the sample loads before the L2 prefetch
#endif
#ifndef MXFFT_PS_FPREFETCH
#define MXFFT_PS_FPREFETCH 4  // fused statistics (segments > 2^17 points): rounds prefetched into L2
#endif
#ifndef MXFFT_PS_HISTSEL
#define MXFFT_PS_HISTSEL 1  // fused statistics: sample order statistics by histogram + exact in-bin rank (no sort)
#endif
#ifndef MXFFT_PS_LEAN_S512
#define MXFFT_PS_LEAN_S512 4096  // lean statistics, 512-thread variant: sample size
#endif
#ifndef MXFFT_PS_LEAN_SMALL_NT
#define MXFFT_PS_LEAN_SMALL_NT 128  // lean statistics: threads per CTA for segments <= 2^15 points (128: C4 162.4 -> 158.9 us vs 256)
#endif
#ifndef MXFFT_CR_MINB
#define MXFFT_CR_MINB 4  // count_range kernel: min CTAs per SM for the register budget (4: 63 registers, no spills)
#endif
#ifndef MXFFT_PS_PREFETCH
#define MXFFT_PS_PREFETCH 4  // lean statistics: stream rounds prefetched into L2 ahead of the loads
#endif
#ifndef MXFFT_PS_LEAN
#define MXFFT_PS_LEAN 1  // k_ps_lean for segments of 2^13 .. 2^17 points
#endif
#ifndef MXFFT_FUSED_MIN_SEG
#define MXFFT_FUSED_MIN_SEG 1  // fewer segments: the grid-wide path (1: per-segment kernels always; 256^2 x1 stats 34.6 -> 22.8 us)
#endif
// fused kernel: 256 threads for segments <= 2^15 points
// (several CTAs per SM hide each other's select phase), else 512; 4096 candidates
constexpr int F_TOPCAP = 1024;  // points above the sample maximum
constexpr int F_UNR = 4;        // float4 loads per thread per round (double-buffered)

static inline int fused_sample_size(int64_t npts) { return npts < 32768 ? 256 : (npts <= 65536 ? 1024 : 4096); }

static inline int64_t cand_cap(int64_t npts) {
    int64_t c = npts / 4;
    return c < 1024 ? 1024 : (c > 16384 ? 16384 : c);
}

bool prescale_fast_ok(int64_t npts) { return npts >= 1024 && npts <= (int64_t(1) << 24); }

// workspace: SegState[nseg] | fallback list int[nseg] + count | candidates
int64_t prescale_fast_ws_bytes(int64_t nseg, int64_t npts) {
    const int64_t st = ((int64_t)sizeof(SegState) * nseg + 255) / 256 * 256;
    const int64_t fb = ((int64_t)sizeof(int) * (nseg + 1) + 255) / 256 * 256;
    if (npts <= FUSED_MAX && nseg >= MXFFT_FUSED_MIN_SEG) return st + fb;
    return st + fb + nseg * (cand_cap(npts) + TOPCAP) * (int64_t)sizeof(float2);
}



// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(SEL_THREADS) k_ps_sample(const float2* __restrict__ xall, int64_t npts,
                                                           int S, double q, SegState* st, int* list_n) {
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
    sort_block<unsigned, SEL_THREADS, SAMPLE_MAX / SEL_THREADS>(keys, S);
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
        if (seg == 0) *list_n = 0;
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
                                                          float2* cand, int64_t cap, float2* top,
                                                          int64_t topcap) {
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
        float2* tb = top + (int64_t)seg * topcap;
#pragma unroll
        for (int it = 0; it < CNT_PER_THREAD / 2; ++it)
#pragma unroll
            for (int h = 0; h < 2; ++h)
                if ((tbits >> (2 * it + h)) & 1) {
                    if (slot < topcap) tb[slot] = h ? make_float2(v[it].z, v[it].w) : make_float2(v[it].x, v[it].y);
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

struct SelShared {
    unsigned hist[NBIN];
    double w[WCAP];
    double wsel[3];
    unsigned warp_sums[SEL_THREADS / 32];
    unsigned long long amax_b;
    unsigned wn;
    int bt, bt1, fail;
    unsigned woff, wend;
};


__device__ __forceinline__ void fail_seg(int* list, int* list_n, int seg) { list[atomicAdd(list_n, 1)] = seg; }

__global__ void __launch_bounds__(SEL_THREADS) k_ps_select(SegState* st, int* list, int* list_n, const float2* cand,
                                                           int64_t cap, const float2* top, double q,
                                                           mxfft_prescale_cfg c,
                                                           mxfft_prescale_result* out, int32_t* kvec) {
    __shared__ SelShared S;
    const int seg = blockIdx.x, tid = threadIdx.x;
    const SegState g = st[seg];
    const unsigned long long nnz = g.nnz;
    if (g.flags) {
        if (tid == 0) fail_seg(list, list_n, seg);
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
            if (tid == 0) fail_seg(list, list_n, seg);
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
            if (tid == 0) fail_seg(list, list_n, seg);
            return;
        }
        for (unsigned i = tid; i < nc; i += SEL_THREADS) {
            const float2 v = cb[i];
            const int b = kbin(__float_as_uint(skey(v.x, v.y)), klo, inv);
            if (b >= wlo && b <= whi) S.w[atomicAdd(&S.wn, 1u)] = np_cabs_f((double)v.x, (double)v.y);
        }
        __syncthreads();
        pick_two<double, SEL_THREADS, WCAP / SEL_THREADS>(S.w, (int)wcount, (int)(t - woff), (int)(t1 - woff), S.wsel);
        const double vlo = S.wsel[0], vhi = S.wsel[1];
        // every point outside the window must order strictly on its side:
        // the picks must clear the window's key edges by more than the key rounding
        const float elo = wlo > 0 ? __uint_as_float(bin_lo(wlo, klo, inv)) : g.lo;
        const float ehi = whi < NBIN - 1 ? __uint_as_float(bin_lo(whi + 1, klo, inv)) : g.hi;
        bool good = true;
        if (elo > 0.f && !(elo >= 0x1p-100f && vlo * vlo > (double)elo * (1.0 + 0x1p-18))) good = false;
        if (ehi <= FLT_MAX && !(vhi * vhi < (double)ehi * (1.0 - 0x1p-18))) good = false;
        if (!good) {
            if (tid == 0) fail_seg(list, list_n, seg);
            return;
        }
        a_max = __longlong_as_double((long long)S.amax_b);
        const double diff = __dsub_rn(vhi, vlo);
        p_tau = gamma >= 0.5 ? __dsub_rn(vhi, __dmul_rn(diff, __dsub_rn(1.0, gamma)))
                             : __dadd_rn(vlo, __dmul_rn(diff, gamma));
    }
    if (tid == 0) finish_result(c, a_max, p_tau, nnz, out, kvec, seg);
}


// ---------------------------------------------------------------------------
// fused sample -> count -> select, one CTA per segment (segments <= 2^18 points)
// ---------------------------------------------------------------------------
template <int NT, int CCAP, int SMAX, int WC, int TC>
struct FusedShared {
    union {
        unsigned keys[SMAX];  // sample phase
        double w[WC];         // exact-sort window (select phase)
    } u;
    float2 cand[CCAP];
    float2 topb[TC];
    unsigned hist[NBIN];
    unsigned warp_sums[NT / 32];
    unsigned long long amax_b;
    unsigned snz, nnz, below, ncand, ntop, flags, wn;
    unsigned sel[3];  // selected sample keys
    double wsel[3];   // selected window magnitudes
    float lo, hi, top;
    int bt, bt1;
    unsigned woff, wend;
};

// CL = 2 (not dispatched): a 2-CTA cluster per segment -- both CTAs draw the
// same sample (so the same bracket), each streams half of the segment, and
// CTA 0 merges CTA 1's counts and candidates through distributed shared
// memory and selects.  Measured slower on C2 (78 vs 57 us, 256-thread CTAs).
template <int NT, int CCAP, int CL, int SMAX, int WC, int TC>
__global__ void __launch_bounds__(NT, 1024 / NT) k_ps_fused(const float2* __restrict__ xall, int64_t npts, int S,
                                                           double q, mxfft_prescale_cfg c,
                                                           mxfft_prescale_result* out, int32_t* kvec, int* list,
                                                           int* list_n) {
    constexpr int F_THREADS = NT, F_CCAP = CCAP, F_TOPCAP = TC, SAMPLE_MAX = SMAX, WCAP = WC;
    using Shared = FusedShared<NT, CCAP, SMAX, WC, TC>;
    extern __shared__ unsigned long long fused_smem[];
    Shared& F = *reinterpret_cast<Shared*>(fused_smem);
    const int seg = blockIdx.x / CL, crank = CL > 1 ? (int)(blockIdx.x % CL) : 0;
    const int tid = threadIdx.x, lane = tid & 31;
#ifdef PS_TIMING
    long long T0 = clock64(), TS[8];
#define PS_T(i) if (tid == 0) TS[i] = clock64() - T0;
#else
#define PS_T(i)
#endif
    const float2* x = xall + (int64_t)seg * npts;
    if (tid == 0) {
        F.snz = F.nnz = F.below = F.ncand = F.ntop = F.flags = F.wn = 0;
        F.amax_b = 0;
    }
    for (int i = tid; i < NBIN; i += F_THREADS) F.hist[i] = 0;
    __syncthreads();

    // ---- sample: pseudo-random whole sectors, sorted squared magnitudes ----
    {
        const int64_t nsec = npts / 4;
        int cnt = 0;
        for (int j = tid; j < S / 4; j += F_THREADS) {
            const uint64_t h = (uint64_t)j * 2654435761ull;
            const uint64_t sec = (nsec & (nsec - 1)) == 0 ? (h & (uint64_t)(nsec - 1)) : h % (uint64_t)nsec;
            const float4* p = reinterpret_cast<const float4*>(x + sec * 4);
            const float4 a = __ldg(p), b = __ldg(p + 1);
            const float v[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
#pragma unroll
            for (int hh = 0; hh < 4; ++hh) {
                const float re = v[2 * hh], im = v[2 * hh + 1];
                const float m = fmaxf(fabsf(re), fabsf(im));
                unsigned k = 0xffffffffu;
                if (m > 0.f) {
                    const float sk = (m >= 0x1p-60f && m <= 0x1p60f) ? skey(re, im) : (m < 1.f ? 0.f : 0x1p125f);
                    k = __float_as_uint(sk);
                    ++cnt;
                }
                F.u.keys[j * 4 + hh] = k;
            }
        }
        for (int o = 16; o; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
        if (lane == 0) atomicAdd(&F.snz, (unsigned)cnt);
        __syncthreads();
        PS_T(0)
        // the bracket needs three order statistics of the sample
        const int n = (int)F.snz;
        const double rs = (double)(n - 1) * q;
        const int d = 8 + (int)(4.0 * sqrt(rs + 1.0));
        const int ilo = (int)floor(rs) - d, ihi = (int)ceil(rs) + 1 + d;
        if (S <= F_THREADS) {
            rank_select<unsigned, F_THREADS>(F.u.keys, S, ilo > 0 ? ilo : -1, ihi < n ? ihi : -1, n - 1, F.sel);
        } else if (MXFFT_PS_HISTSEL) {
            // the same three order statistics without sorting: a 512-bin
            // histogram of key >> 22 finds the bins holding ranks ilo and ihi,
            // then ranks are counted exactly among those bins' keys (the sort of
            // 4096 keys took ~47k cycles on C3)
            unsigned* l0 = reinterpret_cast<unsigned*>(F.cand);  // free until the stream
            unsigned* l1 = l0 + SAMPLE_MAX;
            unsigned kmax = 0;
            for (int i = tid; i < S; i += F_THREADS) {
                const unsigned k = F.u.keys[i];
                if (k != 0xffffffffu) {
                    atomicAdd(&F.hist[k >> 22], 1u);
                    kmax = max(kmax, k);
                }
            }
            for (int o = 16; o; o >>= 1) kmax = max(kmax, __shfl_xor_sync(0xffffffffu, kmax, o));
            if (tid == 0) {
                F.sel[2] = 0;
                F.bt = F.bt1 = -1;
                F.woff = F.wend = 0;  // (reused here: list lengths)
            }
            __syncthreads();
            if (lane == 0) atomicMax(&F.sel[2], kmax);
            {  // exclusive scan, one bin per thread (NBIN == 512 <= F_THREADS)
                const unsigned h = tid < NBIN ? F.hist[tid] : 0u;
                unsigned incl = h;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const unsigned y = __shfl_up_sync(0xffffffffu, incl, o);
                    if (lane >= o) incl += y;
                }
                if (lane == 31) F.warp_sums[tid >> 5] = incl;
                __syncthreads();
                unsigned base = incl - h;
                for (int w = 0; w < (tid >> 5); ++w) base += F.warp_sums[w];
                if (h && ilo > 0 && (unsigned)ilo >= base && (unsigned)ilo < base + h) {
                    F.bt = tid;
                    F.wn = (unsigned)ilo - base;  // rank within the bin
                }
                if (h && ihi < n && (unsigned)ihi >= base && (unsigned)ihi < base + h) {
                    F.bt1 = tid;
                    F.nnz = (unsigned)ihi - base;  // (reused: rank within the bin)
                }
            }
            __syncthreads();
            const int b0 = F.bt, b1 = F.bt1;
            for (int i = tid; i < S; i += F_THREADS) {
                const unsigned k = F.u.keys[i];
                if (k == 0xffffffffu) continue;
                if ((int)(k >> 22) == b0) l0[atomicAdd(&F.woff, 1u)] = k;
                if ((int)(k >> 22) == b1) l1[atomicAdd(&F.wend, 1u)] = k;
            }
            __syncthreads();
            const unsigned c0 = F.woff, c1 = F.wend, r0 = F.wn, r1 = F.nnz;
            for (unsigned i = tid; i < c0; i += F_THREADS) {  // exact rank among the bin's keys
                const unsigned e = l0[i];
                unsigned lt = 0, eq = 0;
                for (unsigned j = 0; j < c0; ++j) {
                    lt += l0[j] < e;
                    eq += l0[j] == e;
                }
                if (lt <= r0 && r0 < lt + eq) F.sel[0] = e;
            }
            for (unsigned i = tid; i < c1; i += F_THREADS) {
                const unsigned e = l1[i];
                unsigned lt = 0, eq = 0;
                for (unsigned j = 0; j < c1; ++j) {
                    lt += l1[j] < e;
                    eq += l1[j] == e;
                }
                if (lt <= r1 && r1 < lt + eq) F.sel[1] = e;
            }
            for (int i = tid; i < NBIN; i += F_THREADS) F.hist[i] = 0;  // the select phase reuses it
            if (tid == 0) F.wn = F.nnz = F.woff = F.wend = 0;
            __syncthreads();
        } else {
            sort_block<unsigned, F_THREADS, SAMPLE_MAX / F_THREADS>(F.u.keys, S);
            if (tid == 0) {
                if (ilo > 0) F.sel[0] = F.u.keys[ilo];
                if (ihi < n) F.sel[1] = F.u.keys[ihi];
                if (n > 0) F.sel[2] = F.u.keys[n - 1];
            }
            __syncthreads();
        }
        PS_T(1)
        if (tid == 0) {
            if (n == 0) {
                F.lo = 0.f;
                F.hi = __int_as_float(0x7f800000);
                F.top = 0.f;
            } else {
                F.lo = ilo <= 0 ? 0.f : __uint_as_float(F.sel[0]) * (1.f - 0x1p-20f);
                F.hi = ihi >= n ? __int_as_float(0x7f800000) : __uint_as_float(F.sel[1]) * (1.f + 0x1p-20f);
                F.top = __uint_as_float(F.sel[2]) * (1.f - 0x1p-20f);
            }
        }
        __syncthreads();
    }
    const float glo = F.lo, ghi = F.hi, gtop = F.top;
    PS_T(2)

    // ---- count: one streaming pass, candidates appended to shared memory ----
    {
        unsigned nnz = 0, below = 0;
        float ksum = 0.f;
        const int64_t part = (npts / 2 + CL - 1) / CL;  // this CTA's pairs of the segment
        const int64_t p_begin = crank * part;
        const int64_t npairs = (npts / 2 - p_begin) < part ? (npts / 2 - p_begin) : part;
        const float4* x4 = reinterpret_cast<const float4*>(x) + p_begin;
        constexpr int64_t STEP = (int64_t)F_THREADS * F_UNR;
        // bulk L2 prefetch MXFFT_PS_FPREFETCH rounds ahead (one thread): a lone CTA
        // per SM (C3's few large segments) is otherwise bound by its loads in flight
        constexpr int FPF = MXFFT_PS_FPREFETCH;
        auto fprefetch = [&](int64_t b) {
            if (FPF > 0 && tid == 0 && b < npairs) {
                const int64_t cnt = npairs - b < STEP ? npairs - b : STEP;
                asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(x4 + b), "r"((unsigned)(cnt * 16))
                             : "memory");
            }
        };
        for (int r = 0; r < FPF; ++r) fprefetch((int64_t)r * STEP);
        float4 vn[F_UNR];  // next round's loads are in flight while this one is classified
#pragma unroll
        for (int it = 0; it < F_UNR; ++it) {
            const int64_t pi = it * F_THREADS + tid;
            vn[it] = pi < npairs ? __ldg(x4 + pi) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
        for (int64_t base = 0; base < npairs; base += STEP) {
            fprefetch(base + (int64_t)FPF * STEP);
            float4 v[F_UNR];
#pragma unroll
            for (int it = 0; it < F_UNR; ++it) {
                v[it] = vn[it];
                const int64_t pi = base + STEP + it * F_THREADS + tid;
                vn[it] = pi < npairs ? __ldg(x4 + pi) : make_float4(0.f, 0.f, 0.f, 0.f);
            }
            unsigned cbits = 0, tbits = 0;
#pragma unroll
            for (int it = 0; it < F_UNR; ++it) {
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const float re = h ? v[it].z : v[it].x, im = h ? v[it].w : v[it].y;
                    const bool nz = (re != 0.f) | (im != 0.f);
                    const float sk = skey(re, im);
                    ksum += sk;
                    nnz += nz;
                    below += nz & (sk < glo);
                    cbits |= (unsigned)(nz & (sk >= glo) & (sk <= ghi)) << (2 * it + h);
                    tbits |= (unsigned)(nz & (sk >= gtop)) << (2 * it + h);
                }
            }
            // candidates are a few percent of the points: one shared atomic per
            // lane that has any is cheaper than a warp scan every round
            if (cbits) {
                unsigned slot = atomicAdd(&F.ncand, (unsigned)__popc(cbits));
#pragma unroll
                for (int it = 0; it < F_UNR; ++it)
#pragma unroll
                    for (int h = 0; h < 2; ++h)
                        if ((cbits >> (2 * it + h)) & 1) {
                            if (slot < F_CCAP) F.cand[slot] = h ? make_float2(v[it].z, v[it].w) : make_float2(v[it].x, v[it].y);
                            ++slot;
                        }
            }
            if (tbits) {
                unsigned slot = atomicAdd(&F.ntop, (unsigned)__popc(tbits));
#pragma unroll
                for (int it = 0; it < F_UNR; ++it)
#pragma unroll
                    for (int h = 0; h < 2; ++h)
                        if ((tbits >> (2 * it + h)) & 1) {
                            if (slot < F_TOPCAP) F.topb[slot] = h ? make_float2(v[it].z, v[it].w) : make_float2(v[it].x, v[it].y);
                            ++slot;
                        }
            }
        }
        unsigned flags = (ksum <= 0x1p126f) ? 0u : 1u;  // non-finite / keys beyond FP32 range
        for (int o = 16; o; o >>= 1) {
            nnz += __shfl_xor_sync(0xffffffffu, nnz, o);
            below += __shfl_xor_sync(0xffffffffu, below, o);
            flags |= __shfl_xor_sync(0xffffffffu, flags, o);
        }
        if (lane == 0) {
            atomicAdd(&F.nnz, nnz);
            atomicAdd(&F.below, below);
            if (flags) atomicOr(&F.flags, flags);
        }
        __syncthreads();
    }
    if constexpr (CL > 1) {  // merge the other CTA's half into CTA 0
        namespace cg = cooperative_groups;
        cg::cluster_group cluster = cg::this_cluster();
        cluster.sync();
        if (crank == 0) {
            // append ranks 1 .. CL-1 in order (counts may exceed the capacity:
            // the select phase then fails the segment over to the exact kernel)
            unsigned nc = F.ncand, nt = F.ntop, flags = F.flags;
            unsigned nnz = F.nnz, below = F.below;
            for (int r = 1; r < CL; ++r) {
                const Shared& R = *cluster.map_shared_rank(&F, r);
                const unsigned nc1 = R.ncand, nt1 = R.ntop;
                for (unsigned i = tid; i < nc1; i += F_THREADS)
                    if (nc + i < F_CCAP && i < F_CCAP) F.cand[nc + i] = R.cand[i];
                for (unsigned i = tid; i < nt1; i += F_THREADS)
                    if (nt + i < F_TOPCAP && i < F_TOPCAP) F.topb[nt + i] = R.topb[i];
                nc += nc1;
                nt += nt1;
                nnz += R.nnz;
                below += R.below;
                flags |= R.flags;
            }
            __syncthreads();
            if (tid == 0) {
                F.ncand = nc;
                F.ntop = nt;
                F.nnz = nnz;
                F.below = below;
                F.flags = flags;
            }
        }
        cluster.sync();  // CTA 1's shared memory stays alive until CTA 0 has read it
        if (crank != 0) return;
    }

    // ---- select: histogram of the candidates, exact sort of a small window ----
    PS_T(3)
    const unsigned long long nnz = F.nnz;
    if (F.flags) {
        if (tid == 0) fail_seg(list, list_n, seg);
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
        const unsigned nc = F.ncand, nt = F.ntop, below = F.below;
        if (!(nc <= F_CCAP && nt <= F_TOPCAP && nt >= 1 && below <= r_lo && r_hi < below + nc)) {
            if (tid == 0) fail_seg(list, list_n, seg);
            return;
        }
        const unsigned t = (unsigned)(r_lo - below), t1 = (unsigned)(r_hi - below);
        const unsigned klo = __float_as_uint(glo), khi = __float_as_uint(ghi);
        const float inv = (float)NBIN / ((float)(khi - klo) + 1.f);
        for (unsigned i = tid; i < nc; i += F_THREADS) {
            const float2 v = F.cand[i];
            atomicAdd(&F.hist[kbin(__float_as_uint(skey(v.x, v.y)), klo, inv)], 1u);
        }
        unsigned long long am = 0;
        for (unsigned i = tid; i < nt; i += F_THREADS) {
            const float2 v = F.topb[i];
            am = max(am, (unsigned long long)__double_as_longlong(np_cabs_f((double)v.x, (double)v.y)));
        }
        for (int o = 16; o; o >>= 1) am = max(am, __shfl_xor_sync(0xffffffffu, am, o));
        if (lane == 0) atomicMax(&F.amax_b, am);
        __syncthreads();
        {  // exclusive scan of the histogram (2 bins per thread; threads >= NBIN/2 hold none)
            const bool has = tid < NBIN / 2;
            const unsigned h0 = has ? F.hist[2 * tid] : 0u, h1 = has ? F.hist[2 * tid + 1] : 0u;
            unsigned incl = h0 + h1;
            const int wp = tid >> 5;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const unsigned y = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += y;
            }
            if (lane == 31) F.warp_sums[wp] = incl;
            __syncthreads();
            unsigned wbase = 0;
            for (int w2 = 0; w2 < wp; ++w2) wbase += F.warp_sums[w2];
            const unsigned e0 = wbase + incl - h0 - h1, e1 = e0 + h0;
            if (has) {
                if (e0 <= t && t < e1) F.bt = 2 * tid;
                if (e1 <= t && t < e1 + h1) F.bt = 2 * tid + 1;
                if (e0 <= t1 && t1 < e1) F.bt1 = 2 * tid;
                if (e1 <= t1 && t1 < e1 + h1) F.bt1 = 2 * tid + 1;
            }
            __syncthreads();
            const int wlo = F.bt > 0 ? F.bt - 1 : 0, whi = F.bt1 < NBIN - 1 ? F.bt1 + 1 : NBIN - 1;
            if (has) {
                if (2 * tid == wlo) F.woff = e0;
                if (2 * tid + 1 == wlo) F.woff = e1;
                if (2 * tid == whi) F.wend = e1;
                if (2 * tid + 1 == whi) F.wend = e1 + h1;
            }
        }
        __syncthreads();
        const int wlo = F.bt > 0 ? F.bt - 1 : 0, whi = F.bt1 < NBIN - 1 ? F.bt1 + 1 : NBIN - 1;
        const unsigned woff = F.woff, wcount = F.wend - F.woff;
        if (wcount > WCAP) {
            if (tid == 0) fail_seg(list, list_n, seg);
            return;
        }
        PS_T(4)
        for (unsigned i = tid; i < nc; i += F_THREADS) {
            const float2 v = F.cand[i];
            const int b = kbin(__float_as_uint(skey(v.x, v.y)), klo, inv);
            if (b >= wlo && b <= whi) F.u.w[atomicAdd(&F.wn, 1u)] = np_cabs_f((double)v.x, (double)v.y);
        }
        __syncthreads();
        PS_T(5)
        const int P = (int)wcount;
        pick_two<double, F_THREADS, WCAP / F_THREADS>(F.u.w, P, (int)(t - woff), (int)(t1 - woff), F.wsel);
        PS_T(6)
#ifdef PS_TIMING
        if (tid == 0 && (seg == 0 || seg == 100))
            printf("seg %d S=%d nc=%u wcount=%u P=%d | sampled %lld sorted %lld stream0 %lld streamed %lld hist+scan %lld window %lld wsorted %lld\n",
                   seg, S, nc, wcount, P, TS[0], TS[1], TS[2], TS[3], TS[4], TS[5], TS[6]);
#endif
        const double vlo = F.wsel[0], vhi = F.wsel[1];
        const float elo = wlo > 0 ? __uint_as_float(bin_lo(wlo, klo, inv)) : glo;
        const float ehi = whi < NBIN - 1 ? __uint_as_float(bin_lo(whi + 1, klo, inv)) : ghi;
        bool good = true;
        if (elo > 0.f && !(elo >= 0x1p-100f && vlo * vlo > (double)elo * (1.0 + 0x1p-18))) good = false;
        if (ehi <= FLT_MAX && !(vhi * vhi < (double)ehi * (1.0 - 0x1p-18))) good = false;
        if (!good) {
            if (tid == 0) fail_seg(list, list_n, seg);
            return;
        }
        a_max = __longlong_as_double((long long)F.amax_b);
        const double diff = __dsub_rn(vhi, vlo);
        p_tau = gamma >= 0.5 ? __dsub_rn(vhi, __dmul_rn(diff, __dsub_rn(1.0, gamma)))
                             : __dadd_rn(vlo, __dmul_rn(diff, gamma));
    }
    if (tid == 0) finish_result(c, a_max, p_tau, nnz, out, kvec, seg);
}

// ---------------------------------------------------------------------------
// Lean fused statistics, one CTA per segment (C2 / C4 image sizes).  Same
// result contract and exactness argument as k_ps_fused; three changes make it
// issue-light:
//  * bracket: a 2048-bin histogram of the sample keys (bin = key bits >> 20,
//    1/8 binade of the key) instead of sorting the sample: lo / hi are the
//    edges of the bins holding sample ranks ilo / ihi (so the bracket only
//    widens), lo never drops below the sample minimum's bin edge / 2^8;
//  * stream: per point a squared-magnitude key, an exact zero test, an
//    integer "below lo" count and one "rare" test (bracket or peak); rare
//    points go to a per-thread shared-memory list with a predicated store --
//    no branch, no atomic on the hot loop;
//  * select: candidate bins span [min candidate key, hi], so the exact
//    window (np.abs in FP64) is a few dozen points and counted ranks pick
//    the order statistics.
// Anything that does not settle (list overflow, ranks outside the bracket,
// selected values within key rounding of a window edge, extreme / non-finite
// keys) sends the segment to the exact fallback list, as before.
// ---------------------------------------------------------------------------
constexpr int LB_BINS = 2048;  // sample histogram: key >> 20

template <int NT, int K, int WC, int OV>
struct LeanShared {
    union {
        struct {
            unsigned hist[LB_BINS];
        } s;  // sample phase
        struct {
            unsigned hist[NBIN];
            double w[WC];
        } q;  // select phase
    } u;
    float2 buf[(K + 8) * NT];  // per-thread rare lists, entry k of thread t at k * NT + t; rows >= K: sink
    float2 ovf[OV];      // shared spill for threads whose list is full
    unsigned warp_a[NT / 32], warp_b[NT / 32], warp_c[NT / 32];
    unsigned long long amax_b;
    unsigned snz, smax, wn, flags, kmin, novf;
    int bsel[3];
    double wsel[3];
    float lo, hi, top;
    int bt, bt1;
    unsigned woff, wend;
};


template <int NT, int K, int WC, int OV>
__global__ void __launch_bounds__(NT, 1024 / NT)
    k_ps_lean(const float2* __restrict__ xall, int64_t npts, int S, double q, mxfft_prescale_cfg c,
              mxfft_prescale_result* out, int32_t* kvec, int* list, int* list_n) {
#ifdef PS_TIMING
    long long T0 = clock64(), TL[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#define PL_T(i) if (threadIdx.x == 0) TL[i] = clock64() - T0;
#else
#define PL_T(i)
#endif
    using Shared = LeanShared<NT, K, WC, OV>;
    extern __shared__ unsigned long long lean_smem[];
    Shared& F = *reinterpret_cast<Shared*>(lean_smem);
    const int seg = blockIdx.x, tid = threadIdx.x, lane = tid & 31;
    const float2* x = xall + (int64_t)seg * npts;
    constexpr unsigned HUGEB = 0x7e800000u;  // key 2^126: beyond it the segment goes to the exact kernel

    // the stream's first rounds head for L2 while the sample is drawn
    constexpr int PF = MXFFT_PS_PREFETCH;  // rounds of look-ahead (bulk L2 prefetch, one thread)
    constexpr unsigned RB = NT * 4 * 16;   // bytes per stream round
    const int nrounds_pf = (int)(npts * 8 / RB);
    auto prefetch_head = [&]() {
        if (tid == 0)
            for (int r = 0; r < PF && r < nrounds_pf; ++r)
                asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(
                                 reinterpret_cast<const char*>(x) + (size_t)r * RB),
                             "n"(RB)
                             : "memory");
    };
#if !MXFFT_PS_SAMPLE_FIRST
    prefetch_head();
#endif
    // ---- sample -> histogram bracket ----
    for (int i = tid; i < LB_BINS; i += NT) F.u.s.hist[i] = 0;
    if (tid == 0) {
        F.snz = 0;
        F.smax = 0;
        F.wn = 0;
        F.flags = 0;
        F.kmin = 0xffffffffu;
        F.novf = 0;
        F.amax_b = 0;
        F.bsel[0] = F.bsel[1] = F.bsel[2] = -1;
    }
    __syncthreads();
    {
        const int64_t nsec = npts / 4;
        unsigned cnt = 0, mx = 0, mn = 0xffffffffu;
        // all of this thread's sample sectors are requested before any is used
        constexpr int SPT = 4;  // sectors per thread per batch (S <= 4 * 4 * NT)
        for (int j0 = tid; j0 < S / 4; j0 += SPT * NT) {
            float4 sa[SPT], sb[SPT];
#pragma unroll
            for (int u = 0; u < SPT; ++u) {
                const int j = j0 + u * NT;
                const uint64_t h = (uint64_t)j * 2654435761ull;
                const uint64_t sec = (nsec & (nsec - 1)) == 0 ? (h & (uint64_t)(nsec - 1)) : h % (uint64_t)nsec;
                const float4* p = reinterpret_cast<const float4*>(x + sec * 4);
                if (j < S / 4) {
                    sa[u] = __ldg(p);
                    sb[u] = __ldg(p + 1);
                } else {
                    sa[u] = sb[u] = make_float4(0.f, 0.f, 0.f, 0.f);
                }
            }
#if MXFFT_PS_SAMPLE_FIRST
            // the sample's sector loads go out ahead of the stream's bulk L2
            // prefetch, so they do not queue behind it
            if (j0 == tid) prefetch_head();
#endif
#pragma unroll
          for (int u = 0; u < SPT; ++u) {
            const float4 a = sa[u], b = sb[u];
            const float v[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
#pragma unroll
            for (int hh = 0; hh < 4; ++hh) {
                const float re = v[2 * hh], im = v[2 * hh + 1];
                const float m = fmaxf(fabsf(re), fabsf(im));
                if (m > 0.f) {
                    const float sk = (m >= 0x1p-60f && m <= 0x1p60f) ? skey(re, im) : (m < 1.f ? 0.f : 0x1p125f);
                    const unsigned k = __float_as_uint(sk);
                    atomicAdd(&F.u.s.hist[k >> 20], 1u);
                    mx = max(mx, k);
                    mn = min(mn, k);
                    ++cnt;
                }
            }
          }
        }
        for (int o = 16; o; o >>= 1) {
            cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
            mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
            mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, o));
        }
        if (lane == 0) {
            atomicAdd(&F.snz, cnt);
            atomicMax(&F.smax, mx);
            atomicMin(&F.kmin, mn);  // (reused: sample minimum here)
        }
    }
    __syncthreads();
    PL_T(0)
    {
        const int n = (int)F.snz;
        const double rs = (double)(n - 1) * q;
        const int d = 8 + (int)(4.0 * sqrt(rs + 1.0));
        const int ilo = (int)floor(rs) - d, ihi = (int)ceil(rs) + 1 + d;
        // exclusive scan of the 2048 bins, B consecutive bins per thread
        constexpr int B = LB_BINS / NT;
        unsigned hv[B], tot = 0;
#pragma unroll
        for (int i = 0; i < B; ++i) {
            hv[i] = F.u.s.hist[tid * B + i];
            tot += hv[i];
        }
        unsigned incl = tot;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        if (lane == 31) F.warp_a[tid >> 5] = incl;
        __syncthreads();
        unsigned base = incl - tot;
        for (int w = 0; w < (tid >> 5); ++w) base += F.warp_a[w];
        const int want[2] = {ilo, ihi};
#pragma unroll
        for (int r = 0; r < 2; ++r) {
            const int rk = want[r];
            if (rk >= 0 && rk < n && (unsigned)rk >= base && (unsigned)rk < base + tot) {
                unsigned e = base;
#pragma unroll
                for (int i = 0; i < B; ++i) {
                    if ((unsigned)rk >= e && (unsigned)rk < e + hv[i]) F.bsel[r] = tid * B + i;
                    e += hv[i];
                }
            }
        }
        __syncthreads();
        if (tid == 0) {
            if (n == 0) {
                F.lo = 0x1p-126f;  // no nonzero sample: everything nonzero is a candidate (-> fallback)
                F.hi = __int_as_float(0x7f800000);
                F.top = __int_as_float(0x7f800000);
            } else {
                // lo > 0 always (zeros, key 0, are then never rare)
                unsigned lob;
                if (ilo > 0) {
                    lob = (unsigned)F.bsel[0] << 20;
                } else {
                    const unsigned e = (F.kmin >> 20) << 20;
                    lob = e > (8u << 23) ? e - (8u << 23) : 0u;
                }
                F.lo = __uint_as_float(lob > 1u ? lob : 1u);
                F.hi = ihi < n ? __uint_as_float((((unsigned)F.bsel[1] + 1u) << 20) - 1u) : __int_as_float(0x7f800000);
                F.top = __uint_as_float(F.smax) * (1.f - 0x1p-20f);
            }
            F.kmin = 0xffffffffu;
        }
        __syncthreads();
    }
    const unsigned lob = __float_as_uint(F.lo), hib = __float_as_uint(F.hi), topb = __float_as_uint(F.top);
    const unsigned rng = hib - lob;
    PL_T(1)

    // ---- stream: counts + per-thread rare lists ----
    // npts is a multiple of 2 * NT * U (dispatch), so rounds need no bounds checks.
    // A thread's list has K rows plus 2U sink rows: a round appends at most 2U
    // entries, and a round that crosses row K spills its late entries.
    unsigned nzero = 0, below_all = 0;
    constexpr int U = 4;
    const unsigned row0 = (unsigned)__cvta_generic_to_shared(&F.buf[tid]);
    unsigned wa = row0;  // next free row of this thread's list
    {
        const int nrounds = (int)(npts / (2 * NT * U));
        const float4* x4 = reinterpret_cast<const float4*>(x) + tid;
        float4 vn[U];
#pragma unroll
        for (int it = 0; it < U; ++it) vn[it] = __ldg(x4 + it * NT);
        for (int r = 0; r < nrounds; ++r) {
            if (tid == 0 && r + PF < nrounds)
                asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(
                                 reinterpret_cast<const char*>(x) + (size_t)(r + PF) * RB),
                             "n"(RB)
                             : "memory");
            float4 v[U];
#pragma unroll
            for (int it = 0; it < U; ++it) v[it] = vn[it];
            if (r + 1 < nrounds) {
#pragma unroll
                for (int it = 0; it < U; ++it) vn[it] = __ldg(x4 + (r + 1) * (NT * U) + it * NT);
            }
            const unsigned wa0 = wa;
#pragma unroll
            for (int it = 0; it < U; ++it) {
#pragma unroll
                for (int hh = 0; hh < 2; ++hh) {
                    const float re = hh ? v[it].z : v[it].x, im = hh ? v[it].w : v[it].y;
                    const unsigned kb = __float_as_uint(skey(re, im));
                    const unsigned z = (__float_as_uint(re) | __float_as_uint(im)) & 0x7fffffffu;
                    const unsigned d = kb - lob;
                    nzero += (z - 1u) >> 31;   // z == 0
                    below_all += d >> 31;      // kb < lob (keys and lob are < 2^31; NaN keys are flagged)
                    asm volatile(
                        "{\n\t.reg .pred p, q;\n\t"
                        "setp.le.u32 p, %1, %2;\n\t"
                        "setp.ge.u32 q, %3, %4;\n\t"
                        "or.pred p, p, q;\n\t"
                        "@p st.shared.v2.f32 [%0], {%5, %6};\n\t"
                        "@p add.u32 %0, %0, %7;\n\t}"
                        : "+r"(wa)
                        : "r"(d), "r"(rng), "r"(kb), "r"(topb), "f"(re), "f"(im), "n"(NT * 8)
                        : "memory");
                }
            }
            if (wa >= row0 + (unsigned)(K * NT * 8)) {  // list full: spill this round's entries past row K
                unsigned w2 = wa0;
#pragma unroll
                for (int it = 0; it < U; ++it) {
#pragma unroll
                    for (int hh = 0; hh < 2; ++hh) {
                        const float re = hh ? v[it].z : v[it].x, im = hh ? v[it].w : v[it].y;
                        const unsigned kb = __float_as_uint(skey(re, im));
                        if ((kb - lob <= rng) | (kb >= topb)) {
                            if (w2 >= row0 + (unsigned)(K * NT * 8)) {
                                const unsigned o = atomicAdd(&F.novf, 1u);
                                if (o < (unsigned)OV) F.ovf[o] = make_float2(re, im);
                            }
                            w2 += NT * 8;
                        }
                    }
                }
                wa = row0 + (unsigned)(K * NT * 8);  // later rounds spill everything
            }
        }
    }
    const unsigned nr = (wa - row0) / (unsigned)(NT * 8);

    // ---- select ----
    __syncthreads();
    PL_T(2)
    const unsigned nsp = F.novf < (unsigned)OV ? F.novf : (unsigned)OV;
    const unsigned nmine = nr < (unsigned)K ? nr : (unsigned)K;  // (nr <= K: later entries were spilled)
    const unsigned nall = nmine + (nsp > (unsigned)tid ? (nsp - 1 - tid) / NT + 1 : 0u);
    // entry e of this thread: its own list, then a strided share of the spill
    auto entry = [&](unsigned e) { return e < nmine ? F.buf[e * NT + tid] : F.ovf[tid + (e - nmine) * NT]; };
    // classify: candidates, peak, extreme
    unsigned ncand = 0, flg = F.novf > (unsigned)OV ? 1u : 0u, kmn = 0xffffffffu;
    unsigned long long am = 0;
    for (unsigned e = 0; e < nall; ++e) {
        const float2 v = entry(e);
        const unsigned kb = __float_as_uint(skey(v.x, v.y));
        if (kb >= HUGEB) flg = 1;
        if (kb - lob <= rng) {
            ++ncand;
            kmn = min(kmn, kb);
        }
        if (kb >= topb) am = max(am, (unsigned long long)__double_as_longlong(np_cabs_f((double)v.x, (double)v.y)));
    }
    for (int o = 16; o; o >>= 1) {
        am = max(am, __shfl_xor_sync(0xffffffffu, am, o));
        kmn = min(kmn, __shfl_xor_sync(0xffffffffu, kmn, o));
    }
    if (lane == 0) {
        atomicMax(&F.amax_b, am);
        atomicMin(&F.kmin, kmn);
    }
    unsigned ntop_any = am != 0 ? 1u : 0u;
    block_sum3<NT>(nzero, below_all, ncand, F.warp_a, F.warp_b, F.warp_c);
    unsigned fl = flg, tp = ntop_any, dummy = 0;
    block_sum3<NT>(fl, tp, dummy, F.warp_a, F.warp_b, F.warp_c);
    PL_T(3)
    const unsigned long long nnz = (unsigned long long)npts - nzero;
    const unsigned below = below_all - nzero;  // lo > 0: every zero counted below
    if (fl) {
        if (tid == 0) fail_seg(list, list_n, seg);
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
        const unsigned nc = ncand;
        if (!(tp >= 1 && below <= r_lo && r_hi < below + nc)) {
            if (tid == 0) fail_seg(list, list_n, seg);
            return;
        }
        const unsigned t = (unsigned)(r_lo - below), t1 = (unsigned)(r_hi - below);
        const unsigned klo = F.kmin;  // smallest candidate key
        const float inv = (float)NBIN / ((float)(hib - klo) + 1.f);
        for (int i = tid; i < NBIN; i += NT) F.u.q.hist[i] = 0;
        __syncthreads();
        for (unsigned e = 0; e < nall; ++e) {
            const float2 v = entry(e);
            const unsigned kb = __float_as_uint(skey(v.x, v.y));
            if (kb - lob <= rng) atomicAdd(&F.u.q.hist[kbin(kb, klo, inv)], 1u);
        }
        __syncthreads();
        {  // exclusive scan of the candidate histogram
            constexpr int B = NBIN / NT > 0 ? NBIN / NT : 1;
            const bool has = tid * B < NBIN;
            unsigned hv[B], tot = 0;
#pragma unroll
            for (int i = 0; i < B; ++i) {
                hv[i] = has ? F.u.q.hist[tid * B + i] : 0u;
                tot += hv[i];
            }
            unsigned incl = tot;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const unsigned y = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += y;
            }
            if (lane == 31) F.warp_a[tid >> 5] = incl;
            __syncthreads();
            unsigned e = incl - tot;
            for (int w = 0; w < (tid >> 5); ++w) e += F.warp_a[w];
            if (has) {
#pragma unroll
                for (int i = 0; i < B; ++i) {
                    if (e <= t && t < e + hv[i]) F.bt = tid * B + i;
                    if (e <= t1 && t1 < e + hv[i]) F.bt1 = tid * B + i;
                    e += hv[i];
                }
            }
            __syncthreads();
            const int wlo = F.bt > 0 ? F.bt - 1 : 0, whi = F.bt1 < NBIN - 1 ? F.bt1 + 1 : NBIN - 1;
            e = incl - tot;
            for (int w = 0; w < (tid >> 5); ++w) e += F.warp_a[w];
            if (has) {
#pragma unroll
                for (int i = 0; i < B; ++i) {
                    if (tid * B + i == wlo) F.woff = e;
                    if (tid * B + i == whi) F.wend = e + hv[i];
                    e += hv[i];
                }
            }
        }
        __syncthreads();
        const int wlo = F.bt > 0 ? F.bt - 1 : 0, whi = F.bt1 < NBIN - 1 ? F.bt1 + 1 : NBIN - 1;
        const unsigned woff = F.woff, wcount = F.wend - F.woff;
        if (wcount > (unsigned)WC) {
            if (tid == 0) fail_seg(list, list_n, seg);
            return;
        }
        PL_T(4)
        for (unsigned e = 0; e < nall; ++e) {
            const float2 v = entry(e);
            const unsigned kb = __float_as_uint(skey(v.x, v.y));
            if (kb - lob <= rng) {
                const int b = kbin(kb, klo, inv);
                if (b >= wlo && b <= whi) F.u.q.w[atomicAdd(&F.wn, 1u)] = np_cabs_f((double)v.x, (double)v.y);
            }
        }
        __syncthreads();
        PL_T(5)
        pick_two<double, NT, WC / NT>(F.u.q.w, (int)wcount, (int)(t - woff), (int)(t1 - woff), F.wsel);
        PL_T(6)
#ifdef PS_TIMING
        if (tid == 0 && (seg == 0 || seg == 100))
            printf("lean seg %d nc=%u wcount=%u spill=%u | bracket %lld stream0 %lld streamed %lld classified %lld hist %lld window %lld picked %lld\n",
                   seg, nc, wcount, F.novf, TL[0], TL[1], TL[2], TL[3], TL[4], TL[5], TL[6]);
#endif
        const double vlo = F.wsel[0], vhi = F.wsel[1];
        const float glo = __uint_as_float(lob), ghi = __uint_as_float(hib);
        const float elo = wlo > 0 ? __uint_as_float(bin_lo(wlo, klo, inv)) : glo;
        const float ehi = whi < NBIN - 1 ? __uint_as_float(bin_lo(whi + 1, klo, inv)) : ghi;
        bool good = true;
        if (elo > 0.f && !(elo >= 0x1p-100f && vlo * vlo > (double)elo * (1.0 + 0x1p-18))) good = false;
        if (ehi <= FLT_MAX && !(vhi * vhi < (double)ehi * (1.0 - 0x1p-18))) good = false;
        if (!good) {
            if (tid == 0) fail_seg(list, list_n, seg);
            return;
        }
        a_max = __longlong_as_double((long long)F.amax_b);
        const double diff = __dsub_rn(vhi, vlo);
        p_tau = gamma >= 0.5 ? __dsub_rn(vhi, __dmul_rn(diff, __dsub_rn(1.0, gamma)))
                             : __dadd_rn(vlo, __dmul_rn(diff, gamma));
    }
    if (tid == 0) finish_result(c, a_max, p_tau, nnz, out, kvec, seg);
}

cudaError_t launch_prescale_fast(const float2* x, int64_t nseg, int64_t npts, double q,
                                 const mxfft_prescale_cfg& c, mxfft_prescale_result* out,
                                 int32_t* kvec, void* ws, int** list_out, int** list_n_out, cudaStream_t st) {
    char* w = reinterpret_cast<char*>(ws);
    SegState* sst = reinterpret_cast<SegState*>(w);
    w += ((int64_t)sizeof(SegState) * nseg + 255) / 256 * 256;
    int* list = reinterpret_cast<int*>(w);
    int* list_n = list + nseg;
    w += ((int64_t)sizeof(int) * (nseg + 1) + 255) / 256 * 256;
    *list_out = list;
    *list_n_out = list_n;
    // the fused kernel streams a segment with ONE CTA: with few segments the
    // grid-wide path (sample / multi-CTA count / select) fills the GPU better
    if (npts <= FUSED_MAX && nseg >= MXFFT_FUSED_MIN_SEG) {
        {
            cudaError_t e = ensure_smem_attr((const void*)k_ps_fused<256, 4096, 1, 256, 1024, 1024>,
                                             (int)sizeof(FusedShared<256, 4096, 256, 1024, 1024>));
            if (e == cudaSuccess)
                e = ensure_smem_attr((const void*)k_ps_fused<256, 4096, 1, 4096, 2048, 1024>,
                                     (int)sizeof(FusedShared<256, 4096, 4096, 2048, 1024>));
            if (e == cudaSuccess)
                e = ensure_smem_attr((const void*)k_ps_fused<512, 4096, 1, 4096, 2048, 1024>,
                                     (int)sizeof(FusedShared<512, 4096, 4096, 2048, 1024>));
            if (e == cudaSuccess)
                e = ensure_smem_attr((const void*)k_ps_fused<512, 8192, 1, 4096, 2048, 2048>,
                                     (int)sizeof(FusedShared<512, 8192, 4096, 2048, 2048>));
            if (e == cudaSuccess && MXFFT_C3_CLUSTER)
                e = ensure_smem_attr(
                    (const void*)k_ps_fused<512, 8192, (MXFFT_C3_CLUSTER > 1 ? MXFFT_C3_CLUSTER : 2), 4096, 2048, 2048>,
                    (int)sizeof(FusedShared<512, 8192, 4096, 2048, 2048>));
            if (e != cudaSuccess) return e;
        }
        cudaError_t e = cudaMemsetAsync(list_n, 0, sizeof(int), st);
        if (e != cudaSuccess) return e;
#if MXFFT_PS_LEAN
        if (npts >= 8192 && npts <= (int64_t(1) << 17) && npts % (npts > 32768 ? 4096 : 2048) == 0) {
            using L512 = LeanShared<512, 12, 1024, 1024>;
            constexpr int NS = MXFFT_PS_LEAN_SMALL_NT;  // threads per CTA for segments <= 2^15 points
            using L256 = LeanShared<NS, 12, 1024, 1024>;
            e = ensure_smem_attr((const void*)k_ps_lean<512, 12, 1024, 1024>, (int)sizeof(L512));
            if (e == cudaSuccess) e = ensure_smem_attr((const void*)k_ps_lean<NS, 12, 1024, 1024>, (int)sizeof(L256));
            if (e != cudaSuccess) return e;
            if (npts > 32768)
                k_ps_lean<512, 12, 1024, 1024><<<(unsigned)nseg, 512, sizeof(L512), st>>>(x, npts, MXFFT_PS_LEAN_S512, q, c, out, kvec,
                                                                                     list, list_n);
            else
                k_ps_lean<NS, 12, 1024, 1024><<<(unsigned)nseg, NS, sizeof(L256), st>>>(x, npts, 1024, q, c, out, kvec,
                                                                                     list, list_n);
            note_launch();
            return cudaGetLastError();
        }
#endif
        const int S = fused_sample_size(npts);
        if (npts < 32768) {  // S = 256: small sample / window / peak buffers, 4 CTAs per SM
            k_ps_fused<256, 4096, 1, 256, 1024, 1024><<<(unsigned)nseg, 256, sizeof(FusedShared<256, 4096, 256, 1024, 1024>), st>>>(
                x, npts, S, q, c, out, kvec, list, list_n);
        } else if (npts <= 32768) {
            k_ps_fused<256, 4096, 1, 4096, 2048, 1024><<<(unsigned)nseg, 256, sizeof(FusedShared<256, 4096, 4096, 2048, 1024>), st>>>(
                x, npts, S, q, c, out, kvec, list, list_n);
        } else if (npts <= (int64_t(1) << 17)) {
            k_ps_fused<512, 4096, 1, 4096, 2048, 1024><<<(unsigned)nseg, 512, sizeof(FusedShared<512, 4096, 4096, 2048, 1024>), st>>>(
                x, npts, S, q, c, out, kvec, list, list_n);
        } else if (nseg * 2 <= 148 * 2 && MXFFT_C3_CLUSTER) {
            // few large segments (C3: 64 x 512^2): a CL-CTA cluster per segment
            // so that CL times as many SMs stream
            constexpr int CLN = MXFFT_C3_CLUSTER > 1 ? MXFFT_C3_CLUSTER : 2;
            auto k = k_ps_fused<512, 8192, CLN, 4096, 2048, 2048>;
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3((unsigned)(nseg * CLN));
            cfg.blockDim = dim3(512);
            cfg.dynamicSmemBytes = sizeof(FusedShared<512, 8192, 4096, 2048, 2048>);
            cfg.stream = st;
            cudaLaunchAttribute attr[1];
            attr[0].id = cudaLaunchAttributeClusterDimension;
            attr[0].val.clusterDim.x = CLN;
            attr[0].val.clusterDim.y = 1;
            attr[0].val.clusterDim.z = 1;
            cfg.attrs = attr;
            cfg.numAttrs = 1;
            cudaError_t e2 = cudaLaunchKernelEx(&cfg, k, x, npts, S, q, c, out, kvec, list, list_n);
            if (e2 != cudaSuccess) return e2;
        } else {  // C3's 512^2 images: ~1.7 % of 2^18 points in the bracket
            k_ps_fused<512, 8192, 1, 4096, 2048, 2048><<<(unsigned)nseg, 512, sizeof(FusedShared<512, 8192, 4096, 2048, 2048>), st>>>(
                x, npts, S, q, c, out, kvec, list, list_n);
        }
        note_launch();
        return cudaGetLastError();
    }
    const int64_t cap = cand_cap(npts);
    float2* cand = reinterpret_cast<float2*>(w);
    float2* top = cand + nseg * cap;
    k_ps_sample<<<(unsigned)nseg, SEL_THREADS, 0, st>>>(x, npts, sample_size(npts), q, sst, list_n);
    note_launch();
    const int cps = (int)((npts + CHUNK - 1) / CHUNK);
    k_ps_count<<<(unsigned)(nseg * cps), CNT_THREADS, 0, st>>>(x, npts, cps, sst, cand, cap, top, TOPCAP);
    note_launch();
    k_ps_select<<<(unsigned)nseg, SEL_THREADS, 0, st>>>(sst, list, list_n, cand, cap, top, q, c, out, kvec);
    note_launch();
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Statistics folded into the first transform pass (mxfft_pipeline_folded).
// The first row pass ran on the UNSCALED input and left, per coil stack, the
// per-warp and per-thread words described at lines_body_tma
// (mxfft_lines.cuh).  One CTA per stack settles k = clip(max(k1, k2))
// (prescale.py:61-73) WITHOUT evaluating p_tau:
//  * k1 = round(log2(target / a_max)) from the largest FP32 key (a_max to
//    2^-23 relative, log2 to 1e-7), unless log2 lands within 1e-6 of a
//    rounding boundary;
//  * k2 <= k1 is PROVEN by counting: k2 = ceil(log2(tau_min / p_tau)) <= k1
//    iff p_tau >= T = tau_min 2^-k1; every np.abs is >= max(|re|, |im|), and
//    a thread whose smallest nonzero max(|re|, |im|) is >= T holds no
//    magnitude below T, so at most 32 F magnitudes lie below T, F = the number
//    of threads with a smaller word.  With nz nonzero points (exact: the
//    words carry the zero counts) and r = floor((nz - 1) tau / 100),
//    32 F <= r puts the order statistic v[r] -- and with it p_tau, which
//    np.percentile interpolates upwards from v[r] -- at or above T;
//  * the unscaled pass equals the scaled one times 2^-k exactly when every
//    v-block exponent stays inside the fast range with and without k (the MX
//    arithmetic is equivariant under powers of two away from its clamps) and
//    the inputs stay FP32-normal under 2^k.
// A stack that fails any of these gets flags = 4 and k = 0: the caller
// (pipeline_resolve) re-runs it through the statistics kernels and the
// standard passes.  Settled rows carry flags = 8 (a_max approximate, p_tau and
// k2 not evaluated, nnz exact).
// ---------------------------------------------------------------------------
// the decision, from the reduced evidence (one thread)
__device__ void fold_finish(unsigned kmx, unsigned hi_u, unsigned lo_u, unsigned rep, unsigned long long zeros,
                            unsigned long long small, unsigned mn, double a_est, int k1, int e_key, bool k1_ok,
                            int64_t stack_points, const mxfft_prescale_cfg& c, mxfft_prescale_result* out,
                            int32_t* kvec, int64_t s) {
    const int hi = (int)hi_u - 128, lo = 128 - (int)lo_u;
    const bool replayed = rep != 0;
    const unsigned long long nnz = (unsigned long long)stack_points - zeros;
    if (kmx < 0x7f800000u && nnz == 0 && !replayed) {  // an all-zero stack: the reference's own formula
        finish_result(c, 0.0, 0.0, 0ull, out, kvec, (int)s);
        return;
    }
    mxfft_prescale_result r;
    r.a_max = r.p_tau = __longlong_as_double(0x7ff8000000000000ll);
    r.k1 = r.k2 = r.k = 0;
    r.flags = 4;
    r.nnz = (int64_t)nnz;
    if (k1_ok && nnz > 0) {
        const double virt = __dmul_rn((double)(nnz - 1), c.tau / 100.0);
        const unsigned long long r_lo = virt >= (double)(nnz - 1) ? nnz - 1 : (unsigned long long)floor(virt);
        const int k = min(max(k1, c.k_min), c.k_max);
        const int e_mu = (int)(mn >> 23) - 127;  // (mn: a lower bound of the smallest nonzero max(|re|, |im|))
        const bool ok = 32ull * small <= r_lo && !replayed && k >= -100 && k <= 100 && lo >= -90 && hi <= 90 &&
                        lo + k >= -90 && hi + k <= 90 && e_mu >= -100 && e_mu + k >= -100 && e_key / 2 + k <= 100;
        if (ok) {
            r.a_max = a_est;
            r.k1 = k1;
            r.k2 = INT_MIN;
            r.k = k;
            r.flags = 8;
        }
    }
    out[s] = r;
    kvec[s] = r.k;
}
// k1 and the threshold T from the largest key (FP64, one thread)
__device__ void fold_k1(unsigned kmx, const mxfft_prescale_cfg& c, double& a_est, int& k1, int& e_key, bool& k1_ok,
                        float& T) {
    a_est = sqrt((double)__uint_as_float(kmx));
    const double L1 = log2(c.target / fmax(a_est, 1e-30));
    const double d1 = fabs(fabs(L1 - trunc(L1)) - 0.5);
    k1 = round_half_away_d(L1);
    e_key = (int)(kmx >> 23) - 127;
    k1_ok = kmx < 0x7f800000u && e_key >= -100 && d1 > 1e-6 && k1 > -200 && k1 < 200;
    // rounded up (and with a margin for the reference's log2 rounding): the count below can only grow
    T = k1_ok ? __double2float_ru(ldexp(c.tau_min, -k1) * (1.0 + 0x1p-20)) : 0.f;
}

// At most 32 registers (launch bounds; the FP64 part spills a little, which does not matter here):
// a 128-thread CTA must fit into the registers the first pass's resident CTAs leave free -- 3 x 128
// threads x 152 registers leave 7168, x 153 (allocated as 160) only 4096 -- or the programmatic
// launch chain first pass -> resolve -> second pass stops overlapping (measured: C2 round trip
// 268 -> 302 us when the resolve CTAs do not fit)
template <int FR_THREADS>
__global__ void __launch_bounds__(FR_THREADS, 2048 / FR_THREADS) k_fold_resolve(const unsigned* __restrict__ acc,
                                                             const unsigned* __restrict__ minw, int64_t stack_points,
                                                             mxfft_prescale_cfg c, mxfft_prescale_result* out,
                                                             int32_t* kvec) {
    pdl_launch_dependents();
    pdl_wait();  // the first pass has finished
    constexpr int NW = FR_THREADS / 32;
    const int64_t s = blockIdx.x;
    const int tid = threadIdx.x, lane = tid & 31, wp = tid >> 5;
    __shared__ unsigned sa[NW], sb[NW], sc[NW], sd[NW];
    __shared__ float s_T;
    // the thread words of the stack (stack_points / 32, a multiple of 512): first batch in flight
    const uint4* w4 = reinterpret_cast<const uint4*>(minw + s * (stack_points / 32));
    const int64_t n4 = stack_points / 128;
    constexpr int PRE = 4;  // 16-byte loads in flight per thread
    uint4 pre[PRE];
#pragma unroll
    for (int j = 0; j < PRE; ++j) {
        const int64_t i = tid + j * FR_THREADS;
        pre[j] = i < n4 ? __ldg(w4 + i) : make_uint4(0xffffffc0u, 0xffffffc0u, 0xffffffc0u, 0xffffffc0u);
    }
    // the warps' words: largest key, exponent range, replay flag
    unsigned kmx = 0, hi_u = 0, lo_u = 0, rep = 0;
    {
        const int64_t nw = stack_points / 1024;  // warp entries of the stack
        const uint2* w = reinterpret_cast<const uint2*>(acc) + s * nw;
        for (int64_t i = tid; i < nw; i += FR_THREADS) {
            const uint2 v = __ldg(w + i);
            kmx = max(kmx, v.x);
            hi_u = max(hi_u, v.y >> 16);
            lo_u = max(lo_u, (v.y >> 4) & 0xfffu);
            rep |= v.y & 1u;
        }
        kmx = __reduce_max_sync(0xffffffffu, kmx);
        hi_u = __reduce_max_sync(0xffffffffu, hi_u);
        lo_u = __reduce_max_sync(0xffffffffu, lo_u);
        rep = __reduce_or_sync(0xffffffffu, rep);
        if (lane == 0) {
            sa[wp] = kmx;
            sb[wp] = hi_u;
            sc[wp] = lo_u;
            sd[wp] = rep;
        }
        __syncthreads();
    }
    // k1 and the threshold T: one thread, in FP64
    double a_est = 0.0;
    int k1 = 0, e_key = 0;
    bool k1_ok = false;
    if (tid == 0) {
        kmx = hi_u = lo_u = rep = 0;
#pragma unroll
        for (int i = 0; i < NW; ++i) {
            kmx = max(kmx, sa[i]);
            hi_u = max(hi_u, sb[i]);
            lo_u = max(lo_u, sc[i]);
            rep |= sd[i];
        }
        float Tt;
        fold_k1(kmx, c, a_est, k1, e_key, k1_ok, Tt);
        s_T = Tt;
    }
    __syncthreads();
    const float T = s_T;
    unsigned zeros = 0, small = 0, mn = 0xffffffffu;
    auto take = [&](unsigned v) {
        const unsigned mb = v & ~63u;
        zeros += v & 63u;
        if (mb != 0xffffffc0u) {
            mn = min(mn, mb);
            small += __uint_as_float(mb) < T;
        }
    };
    for (int64_t i0 = tid;; i0 += PRE * FR_THREADS) {
#pragma unroll
        for (int j = 0; j < PRE; ++j) {
            take(pre[j].x);
            take(pre[j].y);
            take(pre[j].z);
            take(pre[j].w);
        }
        if (i0 + PRE * FR_THREADS >= n4 + tid) break;  // (n4 is a multiple of the batch or smaller than one)
#pragma unroll
        for (int j = 0; j < PRE; ++j) {
            const int64_t i = i0 + (PRE + j) * FR_THREADS;
            pre[j] = i < n4 ? __ldg(w4 + i) : make_uint4(0xffffffc0u, 0xffffffc0u, 0xffffffc0u, 0xffffffc0u);
        }
    }
    zeros = __reduce_add_sync(0xffffffffu, zeros);
    small = __reduce_add_sync(0xffffffffu, small);
    mn = __reduce_min_sync(0xffffffffu, mn);
    __syncthreads();
    if (lane == 0) {
        sa[wp] = zeros;
        sb[wp] = small;
        sc[wp] = mn;
    }
    __syncthreads();
    if (tid != 0) return;
    zeros = small = 0;
    mn = 0xffffffffu;
#pragma unroll
    for (int i = 0; i < NW; ++i) {
        zeros += sa[i];
        small += sb[i];
        mn = min(mn, sc[i]);
    }
    fold_finish(kmx, hi_u, lo_u, rep, zeros, small, mn, a_est, k1, e_key, k1_ok, stack_points, c, out, kvec, s);
}

// Small stacks (<= 2^15 points, C4: one 128^2 image): one WARP per stack, four stacks per CTA --
// no barriers, no shared memory, a quarter of the CTAs (C4: 4096 stacks)
__global__ void __launch_bounds__(128, 16) k_fold_resolve_w(const unsigned* __restrict__ acc,
                                                            const unsigned* __restrict__ minw, int64_t stack_points,
                                                            int64_t nstack, mxfft_prescale_cfg c,
                                                            mxfft_prescale_result* out, int32_t* kvec) {
    pdl_launch_dependents();
    pdl_wait();  // the first pass has finished
    const int lane = threadIdx.x & 31;
    const int64_t s = blockIdx.x * 4ll + (threadIdx.x >> 5);
    if (s >= nstack) return;
    const uint4* w4 = reinterpret_cast<const uint4*>(minw + s * (stack_points / 32));
    const int n4 = (int)(stack_points / 128);  // <= 256: at most 8 per lane
    const int nw = (int)(stack_points / 1024);  // <= 32
    uint4 pre[8];
#pragma unroll
    for (int j = 0; j < 8; ++j)
        pre[j] = lane + 32 * j < n4 ? __ldg(w4 + lane + 32 * j)
                                    : make_uint4(0xffffffc0u, 0xffffffc0u, 0xffffffc0u, 0xffffffc0u);
    unsigned kmx = 0, hi_u = 0, lo_u = 0, rep = 0;
    if (lane < nw) {
        const uint2 v = __ldg(reinterpret_cast<const uint2*>(acc) + s * nw + lane);
        kmx = v.x;
        hi_u = v.y >> 16;
        lo_u = (v.y >> 4) & 0xfffu;
        rep = v.y & 1u;
    }
    kmx = __reduce_max_sync(0xffffffffu, kmx);
    hi_u = __reduce_max_sync(0xffffffffu, hi_u);
    lo_u = __reduce_max_sync(0xffffffffu, lo_u);
    rep = __reduce_or_sync(0xffffffffu, rep);
    double a_est = 0.0;
    int k1 = 0, e_key = 0;
    bool k1_ok = false;
    float T = 0.f;
    if (lane == 0) fold_k1(kmx, c, a_est, k1, e_key, k1_ok, T);
    T = __shfl_sync(0xffffffffu, T, 0);
    unsigned zeros = 0, small = 0, mn = 0xffffffffu;
    auto take = [&](unsigned v) {
        const unsigned mb = v & ~63u;
        zeros += v & 63u;
        if (mb != 0xffffffc0u) {
            mn = min(mn, mb);
            small += __uint_as_float(mb) < T;
        }
    };
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        take(pre[j].x);
        take(pre[j].y);
        take(pre[j].z);
        take(pre[j].w);
    }
    zeros = __reduce_add_sync(0xffffffffu, zeros);
    small = __reduce_add_sync(0xffffffffu, small);
    mn = __reduce_min_sync(0xffffffffu, mn);
    if (lane == 0)
        fold_finish(kmx, hi_u, lo_u, rep, zeros, small, mn, a_est, k1, e_key, k1_ok, stack_points, c, out, kvec, s);
}

// One stack too large for one CTA (C5: 2^28 points): the same decision in three grid-wide steps
// on a per-stack scratch g (8 words, zeroed): [0] largest key, [1] 128 + hi, [2] 128 - lo,
// [3] replay flag, [4] zeros, [5] threads below T, [6] ~(smallest word).
__global__ void __launch_bounds__(256) k_fold_big_a(const unsigned* __restrict__ acc, int64_t stack_points,
                                                    unsigned* g) {
    const int64_t nw = stack_points / 1024;
    const uint2* w = reinterpret_cast<const uint2*>(acc);
    unsigned kmx = 0, hi_u = 0, lo_u = 0, rep = 0;
    for (int64_t i = blockIdx.x * 256ll + threadIdx.x; i < nw; i += gridDim.x * 256ll) {
        const uint2 v = __ldg(w + i);
        kmx = max(kmx, v.x);
        hi_u = max(hi_u, v.y >> 16);
        lo_u = max(lo_u, (v.y >> 4) & 0xfffu);
        rep |= v.y & 1u;
    }
    kmx = __reduce_max_sync(0xffffffffu, kmx);
    hi_u = __reduce_max_sync(0xffffffffu, hi_u);
    lo_u = __reduce_max_sync(0xffffffffu, lo_u);
    rep = __reduce_or_sync(0xffffffffu, rep);
    if ((threadIdx.x & 31) == 0) {
        atomicMax(g, kmx);
        atomicMax(g + 1, hi_u);
        atomicMax(g + 2, lo_u);
        if (rep) atomicOr(g + 3, 1u);
    }
}
__global__ void __launch_bounds__(256) k_fold_big_b(const unsigned* __restrict__ minw, int64_t stack_points,
                                                    mxfft_prescale_cfg c, unsigned* g) {
    __shared__ float s_T;
    if (threadIdx.x == 0) {
        double a_est;
        int k1, e_key;
        bool k1_ok;
        float T;
        fold_k1(g[0], c, a_est, k1, e_key, k1_ok, T);
        s_T = T;
    }
    __syncthreads();
    const float T = s_T;
    const uint4* w4 = reinterpret_cast<const uint4*>(minw);
    const int64_t n4 = stack_points / 128;
    unsigned zeros = 0, small = 0, mn = 0xffffffffu;
    auto take = [&](unsigned v) {
        const unsigned mb = v & ~63u;
        zeros += v & 63u;
        if (mb != 0xffffffc0u) {
            mn = min(mn, mb);
            small += __uint_as_float(mb) < T;
        }
    };
    for (int64_t i = blockIdx.x * 256ll + threadIdx.x; i < n4; i += gridDim.x * 256ll) {
        const uint4 v = __ldg(w4 + i);
        take(v.x);
        take(v.y);
        take(v.z);
        take(v.w);
    }
    zeros = __reduce_add_sync(0xffffffffu, zeros);
    small = __reduce_add_sync(0xffffffffu, small);
    mn = __reduce_min_sync(0xffffffffu, mn);
    if ((threadIdx.x & 31) == 0) {
        atomicAdd(g + 4, zeros);  // (a stack has fewer than 2^32 points: mxfft_pipeline_folded checks)
        atomicAdd(g + 5, small);
        atomicMax(g + 6, ~mn);
    }
}
__global__ void k_fold_big_c(const unsigned* g, int64_t stack_points, mxfft_prescale_cfg c,
                             mxfft_prescale_result* out, int32_t* kvec, int64_t s) {
    double a_est;
    int k1, e_key;
    bool k1_ok;
    float T;
    fold_k1(g[0], c, a_est, k1, e_key, k1_ok, T);
    fold_finish(g[0], g[1], g[2], g[3], g[4], g[5], ~g[6], a_est, k1, e_key, k1_ok, stack_points, c, out, kvec, s);
}

// The grid-wide decision in steps (also the building blocks of a stack split across ranks: the
// caller combines g between the steps -- MAX over g[0..3] after step 0, SUM over g[4..5] and MAX
// over g[6] after step 1 -- mxfft_fold_reduce / mxfft_fold_finish)
cudaError_t launch_fold_reduce(const unsigned* acc, const unsigned* minw, int64_t npoints,
                               const mxfft_prescale_cfg& c, int step, unsigned* g, cudaStream_t st) {
    const int sms = device_attr(cudaDevAttrMultiProcessorCount);
    if (step == 0) {
        cudaError_t e = cudaMemsetAsync(g, 0, 32, st);
        if (e != cudaSuccess) return e;
        k_fold_big_a<<<(unsigned)(2 * sms), 256, 0, st>>>(acc, npoints, g);
    } else {
        k_fold_big_b<<<(unsigned)(8 * sms), 256, 0, st>>>(minw, npoints, c, g);
    }
    note_launch();
    return cudaGetLastError();
}
cudaError_t launch_fold_finish(const unsigned* g, int64_t total_points, const mxfft_prescale_cfg& c,
                               mxfft_prescale_result* out, int32_t* kvec, int64_t s, cudaStream_t st) {
    k_fold_big_c<<<1, 1, 0, st>>>(g, total_points, c, out, kvec, s);
    note_launch();
    return cudaGetLastError();
}

cudaError_t launch_fold_resolve(const unsigned* acc, const unsigned* minw, int64_t nstack, int64_t stack_points,
                                const mxfft_prescale_cfg& c, mxfft_prescale_result* out, int32_t* kvec,
                                unsigned* scratch, cudaStream_t st) {
    if (stack_points > (int64_t(1) << 22)) {  // few huge stacks: grid-wide reduction per stack
        for (int64_t s = 0; s < nstack; ++s) {
            unsigned* g = scratch + 8 * s;
            cudaError_t e = launch_fold_reduce(acc + s * (stack_points / 512), minw + s * (stack_points / 32),
                                               stack_points, c, 0, g, st);
            if (e == cudaSuccess)
                e = launch_fold_reduce(acc + s * (stack_points / 512), minw + s * (stack_points / 32), stack_points, c,
                                       1, g, st);
            if (e == cudaSuccess) e = launch_fold_finish(g, stack_points, c, out, kvec, s, st);
            if (e != cudaSuccess) return e;
        }
        return cudaGetLastError();
    }
    static const int nt_env = getenv("MXFFT_FR_THREADS") ? atoi(getenv("MXFFT_FR_THREADS")) : 0;
    if (stack_points <= 32768 && nt_env != 128) {  // many small stacks: a warp per stack
        cudaError_t e = launch_pdl(k_fold_resolve_w, (unsigned)((nstack + 3) / 4), 128u, 0, st, acc, minw, stack_points,
                                   nstack, c, out, kvec);
        note_launch();
        return e != cudaSuccess ? e : cudaGetLastError();
    }
    // few large stacks: more threads per stack
    // 128 threads: the CTAs then fit next to the first pass's (3 x 128 threads, ~150 registers) and the
    // programmatic launch chain first pass -> resolve -> second pass keeps overlapping (256 threads: C2
    // round trip 270 -> 302 us, C3 310 -> 354 us)
    const int nt = nt_env ? nt_env : 128;
    cudaError_t e = nt == 64 ? launch_pdl(k_fold_resolve<64>, (unsigned)nstack, 64u, 0, st, acc, minw, stack_points,
                                           c, out, kvec) : nt == 256 ? launch_pdl(k_fold_resolve<256>, (unsigned)nstack, 256u, 0, st, acc, minw, stack_points,
                                           c, out, kvec)
                              : launch_pdl(k_fold_resolve<128>, (unsigned)nstack, 128u, 0, st, acc, minw, stack_points,
                                           c, out, kvec);
    note_launch();
    return e != cudaSuccess ? e : cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Building blocks of the global statistics (one segment split over calls or
// ranks; combined on the host, prescale.py compute_prescale_global).
// ---------------------------------------------------------------------------
// nsamples keys (squared magnitudes, FP32) of pseudo-random whole 32-byte
// sectors of the segment: zero -> +inf (excluded), |re|,|im| outside
// [2^-60, 2^60] -> 0 / 2^125 (the count then flags the segment).
__global__ void k_ps_sample_keys(const float2* __restrict__ x, int64_t npts, int64_t nsamples, float* keys) {
    const int64_t nsec = npts / 4;
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < nsamples / 4;
         j += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t h = (uint64_t)j * 2654435761ull;
        const uint64_t sec = (nsec & (nsec - 1)) == 0 ? (h & (uint64_t)(nsec - 1)) : h % (uint64_t)nsec;
        const float4* p = reinterpret_cast<const float4*>(x + sec * 4);
        const float4 a = __ldg(p), b = __ldg(p + 1);
        const float v[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
#pragma unroll
        for (int hh = 0; hh < 4; ++hh) {
            const float re = v[2 * hh], im = v[2 * hh + 1];
            const float m = fmaxf(fabsf(re), fabsf(im));
            float k = __int_as_float(0x7f800000);
            if (m > 0.f) k = (m >= 0x1p-60f && m <= 0x1p60f) ? skey(re, im) : (m < 1.f ? 0.f : 0x1p125f);
            keys[j * 4 + hh] = k;
        }
    }
}

__global__ void k_ps_state_init(SegState* st, float lo, float hi, float top) {
    SegState g;
    g.lo = lo;
    g.hi = hi;
    g.top = top;
    g.pad0 = 0;
    g.nnz = 0;
    g.below = g.ncand = g.ntop = g.flags = 0;
    *st = g;
}

cudaError_t launch_prescale_sample_keys(const float2* x, int64_t npts, int64_t nsamples, float* keys,
                                        cudaStream_t st) {
    const int64_t work = nsamples / 4;
    const unsigned grid = (unsigned)((work + 255) / 256 < 1184 ? (work + 255) / 256 : 1184);
    if (work <= 0) return cudaSuccess;
    k_ps_sample_keys<<<grid, 256, 0, st>>>(x, npts, nsamples, keys);
    note_launch();
    return cudaGetLastError();
}

// One segment (the global statistics' streaming pass): a persistent grid whose
// CTAs walk 4096-point chunks, keep nnz / below in registers, gather candidates
// in a shared-memory buffer that is flushed to global memory in bulk (one
// reservation per flush), and add their totals once at the end.  The
// per-chunk kernel (k_ps_count) issues one same-address atomic per warp and
// chunk, which serialises at ~2.6 ms for a 16384^2 image.
constexpr int CR_BUF = 2048;  // candidates buffered per CTA
constexpr int CR_PER_THREAD = 8;  // complex values per thread per chunk (double-buffered)
constexpr int CR_CHUNK = CNT_THREADS * CR_PER_THREAD;
__global__ void __launch_bounds__(CNT_THREADS, MXFFT_CR_MINB) k_ps_count_range(const float2* __restrict__ x, int64_t npts,
                                                               SegState* st, float2* cand, int64_t cap,
                                                               float2* top, int64_t topcap) {
    __shared__ float2 buf[CR_BUF];
    __shared__ unsigned nbuf, gbase, vend;
    __shared__ unsigned long long s_nnz;
    __shared__ unsigned s_below, s_flags;
    const SegState g = *st;
    if (threadIdx.x == 0) {
        nbuf = 0;
        vend = CR_BUF;
        s_nnz = 0;
        s_below = 0;
        s_flags = 0;
    }
    __syncthreads();
    unsigned long long nnz = 0;
    unsigned below = 0;
    float ksum = 0.f;
    const float4* x4 = reinterpret_cast<const float4*>(x);
    const int64_t npairs = npts / 2, nchunks = (npairs + CR_CHUNK / 2 - 1) / (CR_CHUNK / 2);
    const unsigned lane = threadIdx.x & 31;
    float4 vn[CR_PER_THREAD / 2];  // the next chunk's loads are in flight while this one is classified
    auto load_chunk = [&](int64_t c) {
        const int64_t p0 = c * (CR_CHUNK / 2);
#pragma unroll
        for (int it = 0; it < CR_PER_THREAD / 2; ++it) {
            const int64_t pi = p0 + it * CNT_THREADS + threadIdx.x;
            vn[it] = (c < nchunks && pi < npairs) ? __ldg(x4 + pi) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
    };
    load_chunk(blockIdx.x);
    for (int64_t c = blockIdx.x; c < nchunks; c += gridDim.x) {
        float4 v[CR_PER_THREAD / 2];
#pragma unroll
        for (int it = 0; it < CR_PER_THREAD / 2; ++it) v[it] = vn[it];
        load_chunk(c + gridDim.x);
        unsigned cbits = 0, tbits = 0;
#pragma unroll
        for (int it = 0; it < CR_PER_THREAD / 2; ++it) {
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
        // candidates -> the CTA buffer (warp-aggregated shared atomics)
        {
            const unsigned cnt = __popc(cbits);
            unsigned incl = cnt;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const unsigned y = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= (unsigned)o) incl += y;
            }
            unsigned wbase = 0;
            if (lane == 31 && incl) {
                wbase = atomicAdd(&nbuf, incl);
                // a reservation past the buffer goes to global memory instead;
                // the buffer's valid prefix then ends at the first such base
                if (wbase + incl > (unsigned)CR_BUF) {
                    atomicMin(&vend, wbase);
                    wbase = 0x80000000u | atomicAdd(&st->ncand, incl);
                }
            }
            wbase = __shfl_sync(0xffffffffu, wbase, 31);
            const bool to_global = (wbase & 0x80000000u) != 0;
            unsigned slot = (wbase & 0x7fffffffu) + incl - cnt;
            if (cbits) {
#pragma unroll
                for (int it = 0; it < CR_PER_THREAD / 2; ++it)
#pragma unroll
                    for (int h = 0; h < 2; ++h)
                        if ((cbits >> (2 * it + h)) & 1) {
                            const float2 val = h ? make_float2(v[it].z, v[it].w) : make_float2(v[it].x, v[it].y);
                            if (!to_global) buf[slot] = val;
                            else if (slot < cap) cand[slot] = val;
                            ++slot;
                        }
            }
        }
        if (__any_sync(0xffffffffu, tbits != 0)) {  // peak region: rare, straight to global
            unsigned slot = warp_reserve(__popc(tbits), &st->ntop);
            if (tbits) {
#pragma unroll
                for (int it = 0; it < CR_PER_THREAD / 2; ++it)
#pragma unroll
                    for (int h = 0; h < 2; ++h)
                        if ((tbits >> (2 * it + h)) & 1) {
                            if (slot < topcap) top[slot] = h ? make_float2(v[it].z, v[it].w) : make_float2(v[it].x, v[it].y);
                            ++slot;
                        }
            }
        }
        __syncthreads();
        const unsigned nb_now = nbuf, ve_now = vend;
        // every thread has read the counters (so all take the same flush
        // decision with the same nv) before any warp moves on to the next
        // chunk and reserves new slots
        __syncthreads();
        const unsigned nv = nb_now < ve_now ? nb_now : ve_now;  // valid buffered candidates
        if (nv >= (unsigned)(CR_BUF / 2) || ve_now < (unsigned)CR_BUF) {  // flush
            if (threadIdx.x == 0) gbase = atomicAdd(&st->ncand, nv);
            __syncthreads();
            for (unsigned i = threadIdx.x; i < nv; i += CNT_THREADS)
                if (gbase + i < cap) cand[gbase + i] = buf[i];
            __syncthreads();
            if (threadIdx.x == 0) {
                nbuf = 0;
                vend = CR_BUF;
            }
            __syncthreads();
        }
    }
    {  // final flush (uniform: read after the loop's last barrier)
        const unsigned nv = nbuf < vend ? nbuf : vend;
        if (nv) {
            if (threadIdx.x == 0) gbase = atomicAdd(&st->ncand, nv);
            __syncthreads();
            for (unsigned i = threadIdx.x; i < nv; i += CNT_THREADS)
                if (gbase + i < cap) cand[gbase + i] = buf[i];
        }
    }
    unsigned flags = (ksum <= 0x1p126f) ? 0u : 1u;
    for (int o = 16; o; o >>= 1) {
        nnz += __shfl_xor_sync(0xffffffffu, nnz, o);
        below += __shfl_xor_sync(0xffffffffu, below, o);
        flags |= __shfl_xor_sync(0xffffffffu, flags, o);
    }
    if (lane == 0) {
        atomicAdd(&s_nnz, nnz);
        atomicAdd(&s_below, below);
        if (flags) atomicOr(&s_flags, flags);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        atomicAdd(&st->nnz, s_nnz);
        atomicAdd(&st->below, s_below);
        if (s_flags) atomicOr(&st->flags, s_flags);
    }
}

cudaError_t launch_prescale_count_range(const float2* x, int64_t npts, float lo, float hi, float top,
                                        void* state, float2* cand, int64_t cap, float2* topb,
                                        int64_t topcap, cudaStream_t st) {
    SegState* s = reinterpret_cast<SegState*>(state);
    k_ps_state_init<<<1, 1, 0, st>>>(s, lo, hi, top);
    note_launch();
    const int64_t cps = (npts + CR_CHUNK - 1) / CR_CHUNK;
    if (cps > 0) {
        // a resident (persistent) grid
        const int sms = device_attr(cudaDevAttrMultiProcessorCount);
        int per_sm = 1;
        const cudaError_t e = cached_occupancy((const void*)k_ps_count_range, CNT_THREADS, 0, &per_sm);
        if (e != cudaSuccess) return e;
        const int64_t grid = cps < (int64_t)sms * per_sm ? cps : (int64_t)sms * per_sm;
        k_ps_count_range<<<(unsigned)grid, CNT_THREADS, 0, st>>>(x, npts, s, cand, cap, topb, topcap);
        note_launch();
    }
    return cudaGetLastError();
}

}  // namespace mxfft
