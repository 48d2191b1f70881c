// mxfft_image.cuh -- the fused small-image pipeline (BASELINE configs[3],
// "C4"): ONE 128 x 128 image per CTA, the whole forward / round-trip
// pipeline of roundtrip_pipeline (mri.py:94-107) in one kernel:
//
//   HBM -> shared tile (cp.async, 16-byte chunks, XOR-swizzled; the next
//          image streams in while this one's stores drain, its successor is
//          prefetched into L2 a whole image ahead)
//   statistics on the tile (compute_prescale, prescale.py:61-73): a sampled
//          bracket, one pass that counts and lists bracket candidates, an
//          exact select over a histogram window (np.abs in FP64) -- the
//          algorithm of k_ps_lean -- with an exact in-kernel radix-select
//          fallback; k, the result row and kvec[img] are written here
//   pass 1: rows    (bit-reversed gather from the tile, x 2^k on load)
//   pass 2: columns (transposed gather of pass 1's rows through the tile)
//   [pass 3: rows of F, pass 4: columns -- the inverse transform]
//   store: x 2^-k [x 2^-14] fused, straight from registers to HBM (the last
//          pass's lines are columns of the result: each warp store writes
//          four 64-byte row segments)
//
// Every pass is the line kernel's own register/shared-memory stage code
// (mxfft_lines.cuh: run_stages with T = 4 threads per 128-point line,
// stages 0-4 in registers, stages 5+6 as one radix-4 exchange in the line's
// own row of the tile), so per-stage exponents and codes are those of
// k_mx_lines (pinned bit-exact against the reference).  A block whose
// exponents leave the fast range flags the image; the CTA then recomputes the
// image from HBM with the reference-literal stages (mxfft_generic.cuh).
//
// Shared memory: twiddles (fwd + inv codes, block exponents) | tile 128 KB
// (4 KB aligned) | statistics scratch.  One CTA (512 threads, 16 warps) per SM.
#pragma once
#include <cstdio>

#include "mxfft_lines.cuh"
#include "mxfft_stats.cuh"

namespace mxfft {

#ifndef MXFFT_IM_PF
#define MXFFT_IM_PF 0  // L2 prefetch of coming images: 0 none (measured fastest: 247 vs 259 us per pass with 2), 1 / 2 the next / after-next at the top of an image, 3 the next one pass before its load
#endif

constexpr int IM_N = 128, IM_LT = 2, IM_T = 4, IM_NT = 512, IM_EL = IM_N * IM_N;
constexpr int IM_S = 1024;    // sample points of the bracket
constexpr int IM_K = 8;       // rows of the per-thread candidate lists (+ IM_U2 sink rows)
constexpr int IM_U2 = 8;      // points classified per stream round (a round appends at most this many)
constexpr int IM_OV = 2048;   // shared spill entries
constexpr int IM_WC = 1024;   // exact window capacity
constexpr int IM_BINS = 2048; // sample histogram: key >> 20
constexpr int IM_KM = 2;      // candidate magnitudes kept per thread (the window reuses them)

struct ImageArgs {
    const float2* in;
    float2* out;
    int64_t nimg;
    int npass;  // 2: forward pipeline, 4: round trip
    const unsigned* tw_fwd;
    const unsigned* tw_inv;
    const signed char* twe;
    int trivial01;
    mxfft_prescale_cfg cfg;
    double q;
    mxfft_prescale_result* res;
    int32_t* kvec;
    const int32_t* kin;  // precomputed per-image exponents (k = kin[img / k_group])
    int k_group;
    int stats;           // 1: compute_prescale's statistics in the kernel (res, kvec); 0: k from kin (or 0)
    int first_inverse;   // passes 1-2 use the inverse twiddles (an inverse-only transform)
    int tile_off;  // byte offset of the tile in dynamic shared memory (4 KB aligned in the window)
    // exact replay: reference-literal tables of the plan
    FmtDesc fmt;
    int cpb;
    const double* wcr;
    const double* wci;
    const int* wsexp;
};

struct ImStats {
    union {
        unsigned hist[IM_BINS];  // sample phase
        unsigned whist[IM_NT / 32][256];  // exact path: per-warp radix-digit histograms
        struct {
            unsigned hist[NBIN];
            double w[IM_WC];
        } q;  // select phase
    } u;
    unsigned short buf[(IM_K + IM_U2) * IM_NT];  // per-thread candidate lists (element indices), entry r of thread t at r * NT + t
    unsigned short ovf[IM_OV];
    double cmag[IM_KM * IM_NT];  // exact magnitudes of each thread's first IM_KM candidate entries
    unsigned long long warp_m[IM_NT / 32];
    unsigned warp_a[IM_NT / 32], warp_b[IM_NT / 32], warp_c[IM_NT / 32];
    unsigned sel_t, sel_t1;
    double gamma;
    int state;
    unsigned long long amax_b, nnz64, vsel;
    unsigned snz, smax, flags, kmin, novf, wn, cnt;
    int bsel[2];
    double wsel[3];
    float lo, hi, top;
    int bt, bt1;
    unsigned woff, wend;
    int k, fallback, bad;
};

#ifdef MXFFT_IM_TIMING
__device__ long long g_im_t[16];  // sub-phase clocks of CTA 0 (profiling builds only)
#define IM_ST(i)                                                  \
    if (threadIdx.x == 0 && blockIdx.x == 0) {                    \
        const long long _t = clock64();                           \
        g_im_t[i] += _t - g_im_t[15];                             \
        g_im_t[15] = _t;                                          \
    }
#else
#define IM_ST(i)
#endif

// finish_result (mxfft_stats.cuh: the k rule of prescale.py:70-72, the
// boundary flag, the result row and kvec) returning k
__device__ __forceinline__ int finish_k(const mxfft_prescale_cfg& c, double a_max, double p_tau,
                                        unsigned long long nnz, mxfft_prescale_result* out, int32_t* kvec,
                                        int64_t img) {
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
    out[img] = r;
    if (kvec) kvec[img] = k;
    return k;
}

__device__ __forceinline__ unsigned im_addr(unsigned tile_sh, int e) {
    return tile_sh + 16u * (unsigned)dsw(e >> 1) + 8u * (unsigned)(e & 1);
}

// ---------------------------------------------------------------------------
// statistics: exact fallback.  The thread's 32 exact FP64 magnitudes
// (np.abs, numpy's formula) are computed once and kept in registers as bit
// patterns (positive doubles order like their bits); a radix select over
// 8-bit digits from bit 62 down (per-warp shared histograms, then summed)
// finds the order statistics.  Only for images the sampled path cannot settle
// (extreme ranges, non-finite values, skewed samples).  Leaves the shared
// union dirty (the caller clears it).
// ---------------------------------------------------------------------------
static __device__ __noinline__ void im_stats_exact(unsigned tile_sh, ImStats& F, const ImageArgs& a, int64_t img) {
    const int tid = threadIdx.x, lane = tid & 31, wp = tid >> 5;
    constexpr int NT = IM_NT, PT = IM_EL / NT;  // 32 points per thread
    unsigned long long m[PT];
    bool nonfin = false;
    unsigned long long am = 0;
    unsigned nz = 0;
#pragma unroll
    for (int i = 0; i < PT; ++i) {
        const float2 v = lds64(im_addr(tile_sh, tid + NT * i));
        const bool fin = isfinite(v.x) && isfinite(v.y);
        nonfin |= !fin;
        m[i] = fin ? (unsigned long long)__double_as_longlong(np_cabs_f((double)v.x, (double)v.y)) : 0ull;
        am = m[i] > am ? m[i] : am;
        nz += m[i] != 0;
    }
    for (int o = 16; o; o >>= 1) {
        const unsigned long long t = __shfl_xor_sync(0xffffffffu, am, o);
        am = t > am ? t : am;
        nz += __shfl_xor_sync(0xffffffffu, nz, o);
    }
    const unsigned anynf = __any_sync(0xffffffffu, nonfin);
    __syncthreads();  // the caller's last reads of F are done
    if (lane == 0) {
        F.warp_a[wp] = nz;
        F.warp_b[wp] = anynf;
        reinterpret_cast<unsigned long long*>(F.u.whist[wp])[0] = am;
    }
    __syncthreads();
    unsigned long long nnz = 0, amax = 0;
    unsigned flags = 0;
#pragma unroll
    for (int w = 0; w < NT / 32; ++w) {
        nnz += F.warp_a[w];
        flags |= F.warp_b[w];
        const unsigned long long t = reinterpret_cast<unsigned long long*>(F.u.whist[w])[0];
        amax = t > amax ? t : amax;
    }
    __syncthreads();
    if (flags) {  // non-finite input: the reference raises InvalidValue
        if (tid == 0) {
            mxfft_prescale_result r{};
            r.flags = 1;
            r.nnz = (int64_t)nnz;
            a.res[img] = r;
            if (a.kvec) a.kvec[img] = 0;
            F.k = 0;
        }
        __syncthreads();
        return;
    }
    const double a_max = __longlong_as_double((long long)amax);
    double p_tau = 0.0;
    if (nnz > 0) {
        const double virt = __dmul_rn((double)(nnz - 1), a.q);
        unsigned long long r_lo;
        double gamma;
        bool same;
        if (virt >= (double)(nnz - 1)) {
            r_lo = nnz - 1;
            gamma = __dadd_rn(virt, 1.0);
            same = true;
        } else {
            r_lo = (unsigned long long)floor(virt);
            gamma = __dsub_rn(virt, (double)r_lo);
            same = false;
        }
        // rank r_lo among the nonzero magnitudes (zeros have bit pattern 0)
        unsigned long long prefix = 0, rank = r_lo;
        for (int hi = 63; hi > 0;) {
            const int w = hi < 8 ? hi : 8, lo = hi - w;
            for (int i = lane; i < 256; i += 32) F.u.whist[wp][i] = 0;
            __syncwarp();
#pragma unroll
            for (int i = 0; i < PT; ++i) {
                const unsigned long long b = m[i];
                if (b != 0 && (b >> hi) == prefix) atomicAdd(&F.u.whist[wp][(unsigned)(b >> lo) & ((1u << w) - 1u)], 1u);
            }
            __syncthreads();
            // digit totals, then the digit holding `rank` (warps 0-7 scan 32 digits each)
            unsigned c = 0, incl = 0;
            if (tid < 256) {
#pragma unroll
                for (int w2 = 0; w2 < NT / 32; ++w2) c += F.u.whist[w2][tid];
                incl = c;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const unsigned y = __shfl_up_sync(0xffffffffu, incl, o);
                    if (lane >= o) incl += y;
                }
                if (lane == 31) F.warp_a[wp] = incl;
            }
            __syncthreads();
            if (tid < 256) {
                unsigned long long e0 = incl - c;
                for (int w2 = 0; w2 < wp; ++w2) e0 += F.warp_a[w2];
                if (c && rank >= e0 && rank < e0 + c) {
                    F.vsel = (prefix << w) | (unsigned long long)tid;
                    F.nnz64 = rank - e0;
                }
            }
            __syncthreads();
            prefix = F.vsel;
            rank = F.nnz64;
            hi = lo;
            __syncthreads();
        }
        const double vlo = __longlong_as_double((long long)prefix);
        double vhi = vlo;
        if (!same) {
            // element r_lo + 1: vlo again if it repeats beyond `rank`, else the next larger magnitude
            unsigned cnt_eq = 0;
            unsigned long long nxt = ~0ull;
#pragma unroll
            for (int i = 0; i < PT; ++i) {
                cnt_eq += m[i] == prefix;
                if (m[i] > prefix && m[i] < nxt) nxt = m[i];
            }
            for (int o = 16; o; o >>= 1) {
                cnt_eq += __shfl_xor_sync(0xffffffffu, cnt_eq, o);
                const unsigned long long t = __shfl_xor_sync(0xffffffffu, nxt, o);
                nxt = t < nxt ? t : nxt;
            }
            if (lane == 0) {
                F.warp_a[wp] = cnt_eq;
                reinterpret_cast<unsigned long long*>(F.u.whist[wp])[0] = nxt;
            }
            __syncthreads();
            unsigned ce = 0;
            unsigned long long nx = ~0ull;
#pragma unroll
            for (int w = 0; w < NT / 32; ++w) {
                ce += F.warp_a[w];
                const unsigned long long t = reinterpret_cast<unsigned long long*>(F.u.whist[w])[0];
                nx = t < nx ? t : nx;
            }
            vhi = (rank + 1 < ce) ? vlo : __longlong_as_double((long long)nx);
        }
        const double diff = __dsub_rn(vhi, vlo);
        p_tau = gamma >= 0.5 ? __dsub_rn(vhi, __dmul_rn(diff, __dsub_rn(1.0, gamma)))
                             : __dadd_rn(vlo, __dmul_rn(diff, gamma));
    }
    if (tid == 0) F.k = finish_k(a.cfg, a_max, p_tau, nnz, a.res, a.kvec, img);
    __syncthreads();
}

// ---------------------------------------------------------------------------
// statistics: the sampled path (k_ps_lean's algorithm, restructured for an
// image that is already on chip):
//  1. im_bracket: 1024 hashed sample points of the tile -> a 2048-bin
//     histogram of their FP32 squared-magnitude keys -> the key bracket
//     [lo, hi] around the tau-quantile's rank (+- 8 + 4 sqrt sample ranks) and
//     the peak threshold (the sample maximum);
//  2. im_select, on the 32 values each thread has just gathered for pass 1:
//     counts (nonzero, below lo) and per-thread lists of the bracket / peak
//     candidates (element indices, predicated stores, no atomics), one block
//     reduction, a 512-bin histogram of the candidates over [lo, hi], the
//     window of bins holding the two order statistics, np.abs (FP64) of the
//     window only and counted ranks.  The picks must clear the window edges
//     by more than the FP32 key rounding.
// Anything that does not settle (list / window overflow, ranks outside the
// bracket, extreme or non-finite keys) goes to im_stats_exact.
// ---------------------------------------------------------------------------
static __device__ __noinline__ void im_bracket(unsigned tile_sh, ImStats& F, const ImageArgs& a) {
    constexpr int NT = IM_NT;
    const int tid = threadIdx.x, lane = tid & 31;
    // F.u is all zero here: cleared at kernel start and after every image's statistics
    IM_ST(0)
    unsigned cnt = 0, mx = 0, mn = 0xffffffffu;
#pragma unroll
    for (int u = 0; u < IM_S / NT; ++u) {
        const unsigned j = (unsigned)(tid + u * NT);
        const int e = (int)((j * 2654435761u) >> 18);
        const float2 v = lds64(im_addr(tile_sh, e));
        const float m = fmaxf(fabsf(v.x), fabsf(v.y));
        if (m > 0.f) {
            const float sk = (m >= 0x1p-60f && m <= 0x1p60f) ? skey(v.x, v.y) : (m < 1.f ? 0.f : 0x1p125f);
            const unsigned k = __float_as_uint(sk);
            atomicAdd(&F.u.hist[k >> 20], 1u);
            mx = max(mx, k);
            mn = min(mn, k);
            ++cnt;
        }
    }
    for (int o = 16; o; o >>= 1) {
        cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
        mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    }
    if (lane == 0) {
        F.warp_a[tid >> 5] = cnt;
        F.warp_b[tid >> 5] = mx;
        F.warp_c[tid >> 5] = mn;
    }
    __syncthreads();
    IM_ST(1)
    int n = 0;
    unsigned smax = 0, smin = 0xffffffffu;
#pragma unroll
    for (int w = 0; w < NT / 32; ++w) {
        n += (int)F.warp_a[w];
        smax = max(smax, F.warp_b[w]);
        smin = min(smin, F.warp_c[w]);
    }
    const double rs = (double)(n - 1) * a.q;
    const int d = 8 + (int)(4.0 * sqrt(rs + 1.0));
    const int ilo = (int)floor(rs) - d, ihi = (int)ceil(rs) + 1 + d;
    constexpr int B = IM_BINS / NT;  // 4 consecutive bins per thread
    unsigned hv[B], tot = 0;
#pragma unroll
    for (int i = 0; i < B; ++i) {
        hv[i] = F.u.hist[tid * B + i];
        tot += hv[i];
    }
    unsigned incl = tot;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
    }
    __syncthreads();  // the sample counts in warp_a have been read
    if (lane == 31) F.warp_a[tid >> 5] = incl;
    __syncthreads();
    unsigned base = incl - tot;
    for (int w = 0; w < (tid >> 5); ++w) base += F.warp_a[w];
    // the bins of sample ranks ilo and ihi -> the bracket (one thread finds each)
    if (ilo > 0 && ilo < n && (unsigned)ilo >= base && (unsigned)ilo < base + tot) {
        unsigned e = base;
#pragma unroll
        for (int i = 0; i < B; ++i) {
            if ((unsigned)ilo >= e && (unsigned)ilo < e + hv[i]) F.lo = __uint_as_float(max((unsigned)(tid * B + i) << 20, 1u));
            e += hv[i];
        }
    }
    if (ihi < n && (unsigned)ihi >= base && (unsigned)ihi < base + tot) {
        unsigned e = base;
#pragma unroll
        for (int i = 0; i < B; ++i) {
            if ((unsigned)ihi >= e && (unsigned)ihi < e + hv[i]) F.hi = __uint_as_float((((unsigned)(tid * B + i) + 1u) << 20) - 1u);
            e += hv[i];
        }
    }
    if (tid == 0) {
        if (n == 0) {  // no nonzero sample: everything nonzero is a candidate (-> exact path)
            F.lo = 0x1p-126f;
            F.hi = __int_as_float(0x7f800000);
            F.top = __int_as_float(0x7f800000);
        } else {
            if (ilo <= 0) {  // lo from the sample minimum's bin edge / 2^8 (lo > 0: zeros never qualify)
                const unsigned e = (smin >> 20) << 20;
                const unsigned lob = e > (8u << 23) ? e - (8u << 23) : 0u;
                F.lo = __uint_as_float(lob > 1u ? lob : 1u);
            }
            if (ihi >= n) F.hi = __int_as_float(0x7f800000);
            F.top = __uint_as_float(smax) * (1.f - 0x1p-20f);
        }
        F.novf = 0;
        F.wn = 0;
    }
    __syncthreads();  // every sample bin read
    // the candidate histogram aliases sample bins 0..511
    for (int i = tid; i < NBIN; i += NT) F.u.q.hist[i] = 0;
    __syncthreads();  // bracket published; candidate histogram zeroed
    IM_ST(2)
}

// counts + candidate lists over the thread's 32 gathered values (element
// index of x[j] = ibase + 4 rev5(j)), then the exact selection; k -> F.k, or
// F.fallback = 1 (every thread sees the same values).  The serial steps on
// small data (scan of the candidate histogram, the window's order statistics,
// k) run in warp 0 alone, so the whole selection costs four CTA barriers.
static __device__ __noinline__ void im_select(ImStats& F, const ImageArgs& a, int64_t img, unsigned tile_sh) {
    constexpr int NT = IM_NT;
    constexpr unsigned HUGEB = 0x7e800000u;  // key 2^126: beyond it the exact path decides
    const int tid = threadIdx.x, lane = tid & 31;
    const unsigned lob = __float_as_uint(F.lo), hib = __float_as_uint(F.hi), topb = __float_as_uint(F.top);
    const unsigned rng = hib - lob;
    unsigned nzero = 0, below_all = 0;
    const unsigned row0 = (unsigned)__cvta_generic_to_shared(&F.buf[tid]);
    const unsigned rowK = row0 + (unsigned)(IM_K * NT * 2);
    unsigned wa = row0;
#pragma unroll 1
    for (int g = 0; g < 4; ++g) {
        const unsigned wa0 = wa;
        // chunks tid + NT (4 g + c): 16-byte accesses, conflict-free under dsw
        float2 x[8];
        int xi[8];
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            const int C = tid + NT * (4 * g + c);
            lds128(tile_sh + 16u * (unsigned)dsw(C), x[2 * c], x[2 * c + 1]);
            xi[2 * c] = 2 * C;
            xi[2 * c + 1] = 2 * C + 1;
        }
#pragma unroll
        for (int h = 0; h < 8; ++h) {
            const int j = h;
            const float re = x[j].x, im = x[j].y;
            const unsigned kb = __float_as_uint(skey(re, im));
            const unsigned z = (__float_as_uint(re) | __float_as_uint(im)) & 0x7fffffffu;
            const unsigned d = kb - lob;
            nzero += (z - 1u) >> 31;
            below_all += d >> 31;
            const unsigned short ev = (unsigned short)xi[j];
            asm volatile(
                "{\n\t.reg .pred p, q;\n\t"
                "setp.le.u32 p, %1, %2;\n\t"
                "setp.ge.u32 q, %3, %4;\n\t"
                "or.pred p, p, q;\n\t"
                "@p st.shared.u16 [%0], %5;\n\t"
                "@p add.u32 %0, %0, %6;\n\t}"
                : "+r"(wa)
                : "r"(d), "r"(rng), "r"(kb), "r"(topb), "h"(ev), "n"(NT * 2)
                : "memory");
        }
        if (wa >= rowK) {  // list full: this group's late entries go to the shared spill
            unsigned w2 = wa0;
#pragma unroll
            for (int h = 0; h < 8; ++h) {
                const int j = h;
                const unsigned kb = __float_as_uint(skey(x[j].x, x[j].y));
                if ((kb - lob <= rng) | (kb >= topb)) {
                    if (w2 >= rowK) {
                        const unsigned o = atomicAdd(&F.novf, 1u);
                        if (o < (unsigned)IM_OV) F.ovf[o] = (unsigned short)xi[j];
                    }
                    w2 += NT * 2;
                }
            }
            wa = rowK;
        }
    }
    const unsigned nr = (wa - row0) / (unsigned)(NT * 2);
    __syncthreads();  // lists and spill complete
    IM_ST(4)
    const unsigned nsp = F.novf < (unsigned)IM_OV ? F.novf : (unsigned)IM_OV;
    const unsigned nmine = nr < (unsigned)IM_K ? nr : (unsigned)IM_K;
    const unsigned nall = nmine + (nsp > (unsigned)tid ? (nsp - 1 - tid) / NT + 1 : 0u);
    auto entry = [&](unsigned e) -> float2 {
        const int idx = e < nmine ? F.buf[e * NT + tid] : F.ovf[tid + (e - nmine) * NT];
        return lds64(im_addr(tile_sh, idx));
    };
    // classify this thread's entries: candidate histogram over [lo, hi] and the
    // exact magnitudes of the candidates (kept for the window) and of the peak
    const float inv = (float)NBIN / ((float)rng + 1.f);
    unsigned ncand = 0, flg = F.novf > (unsigned)IM_OV ? 1u : 0u;
    unsigned long long am = 0;
    for (unsigned e = 0; e < nall; ++e) {
        const float2 v = entry(e);
        const unsigned kb = __float_as_uint(skey(v.x, v.y));
        flg |= kb >= HUGEB;
        const bool cand = kb - lob <= rng, top = kb >= topb;
        if (cand | top) {
            const double mag = np_cabs_f((double)v.x, (double)v.y);
            if (top) am = max(am, (unsigned long long)__double_as_longlong(mag));
            if (cand) {
                ++ncand;
                atomicAdd(&F.u.q.hist[kbin(kb, lob, inv)], 1u);
                if (e < IM_KM) F.cmag[e * NT + tid] = mag;
            }
        }
    }
    unsigned tp = am != 0;
    for (int o = 16; o; o >>= 1) {
        nzero += __shfl_xor_sync(0xffffffffu, nzero, o);
        below_all += __shfl_xor_sync(0xffffffffu, below_all, o);
        ncand += __shfl_xor_sync(0xffffffffu, ncand, o);
        flg |= __shfl_xor_sync(0xffffffffu, flg, o);
        tp |= __shfl_xor_sync(0xffffffffu, tp, o);
        const unsigned long long t = __shfl_xor_sync(0xffffffffu, am, o);
        am = t > am ? t : am;
    }
    if (lane == 0) {
        F.warp_a[tid >> 5] = nzero;
        F.warp_b[tid >> 5] = below_all;
        F.warp_c[tid >> 5] = ncand | (flg << 30) | (tp << 31);
        F.warp_m[tid >> 5] = am;
    }
    __syncthreads();  // counts, candidate histogram and peak complete
    IM_ST(5)
    if (tid < 32) {  // warp 0: ranks, the window of bins holding the two order statistics
        unsigned nz = 0, bl = 0, nc = 0, fl = 0, anytop = 0;
        unsigned long long amx = 0;
#pragma unroll
        for (int w = 0; w < NT / 32; ++w) {
            nz += F.warp_a[w];
            bl += F.warp_b[w];
            const unsigned c = F.warp_c[w];
            nc += c & 0x3fffffffu;
            fl |= (c >> 30) & 1u;
            anytop |= c >> 31;
            amx = F.warp_m[w] > amx ? F.warp_m[w] : amx;
        }
        const unsigned long long nnz = (unsigned long long)IM_EL - nz;
        const unsigned below = bl - nz;  // lo > 0: every zero counted below
        int state = fl ? 0 : 1;          // 0: fallback, 1: continue, 2: done (nnz == 0)
        unsigned t = 0, t1 = 0;
        double gamma = 0.0;
        if (state && nnz == 0) state = 2;
        if (state == 1) {
            const double virt = __dmul_rn((double)(nnz - 1), a.q);
            unsigned long long r_lo, r_hi;
            if (virt >= (double)(nnz - 1)) {
                r_lo = r_hi = nnz - 1;
                gamma = __dadd_rn(virt, 1.0);
            } else {
                r_lo = (unsigned long long)floor(virt);
                r_hi = r_lo + 1;
                gamma = __dsub_rn(virt, (double)r_lo);
            }
            if (!(anytop && below <= r_lo && r_hi < below + nc)) state = 0;
            t = (unsigned)(r_lo - below);
            t1 = (unsigned)(r_hi - below);
        }
        if (state == 1) {
            // scan of the 512-bin candidate histogram: 16 consecutive bins per lane
            constexpr int BB = NBIN / 32;
            unsigned tot = 0;
#pragma unroll
            for (int i = 0; i < BB; ++i) tot += F.u.q.hist[lane * BB + i];
            unsigned incl = tot;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const unsigned y = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += y;
            }
            int bt = -1, bt1 = -1;
            unsigned ebt = 0, ebt1 = 0;
            {
                unsigned e = incl - tot;
#pragma unroll
                for (int i = 0; i < BB; ++i) {
                    const unsigned h = F.u.q.hist[lane * BB + i];
                    if (h && e <= t && t < e + h) bt = lane * BB + i, ebt = e;
                    if (h && e <= t1 && t1 < e + h) bt1 = lane * BB + i, ebt1 = e + h;
                    e += h;
                }
            }
            const unsigned lb = __ballot_sync(0xffffffffu, bt >= 0), lb1 = __ballot_sync(0xffffffffu, bt1 >= 0);
            bt = __shfl_sync(0xffffffffu, bt, __ffs(lb) - 1);
            bt1 = __shfl_sync(0xffffffffu, bt1, __ffs(lb1) - 1);
            // window = bins [bt - 1, bt1 + 1]: its offset and end in candidate order
            const int wlo = bt > 0 ? bt - 1 : 0, whi = bt1 < NBIN - 1 ? bt1 + 1 : NBIN - 1;
            unsigned woff = 0, wend = 0;
            {
                unsigned e = incl - tot;
#pragma unroll
                for (int i = 0; i < BB; ++i) {
                    const unsigned h = F.u.q.hist[lane * BB + i];
                    if (lane * BB + i == wlo) woff = e;
                    if (lane * BB + i == whi) wend = e + h;
                    e += h;
                }
            }
            woff = __shfl_sync(0xffffffffu, woff, wlo / BB);
            wend = __shfl_sync(0xffffffffu, wend, whi / BB);
            (void)ebt;
            (void)ebt1;
            if (wend - woff > (unsigned)IM_WC) state = 0;
            if (lane == 0) {
                F.bt = wlo;
                F.bt1 = whi;
                F.woff = woff;
                F.wend = wend;
                F.sel_t = t - woff;
                F.sel_t1 = t1 - woff;
                F.gamma = gamma;
                F.amax_b = amx;
                F.nnz64 = nnz;
            }
        }
        if (lane == 0) {
            F.state = state;
            if (state == 2) {  // no nonzero value: a_max = p_tau = 0
                F.k = finish_k(a.cfg, 0.0, 0.0, 0ull, a.res, a.kvec, img);
            }
        }
    }
    __syncthreads();  // window published
    IM_ST(6)
    if (F.state == 1) {
        const int wlo = F.bt, whi = F.bt1;
        for (unsigned e = 0; e < nall; ++e) {
            const float2 v = entry(e);
            const unsigned kb = __float_as_uint(skey(v.x, v.y));
            if (kb - lob <= rng) {
                const int b = kbin(kb, lob, inv);
                if (b >= wlo && b <= whi)
                    F.u.q.w[atomicAdd(&F.wn, 1u)] = e < IM_KM ? F.cmag[e * NT + tid] : np_cabs_f((double)v.x, (double)v.y);
            }
        }
    }
    __syncthreads();  // window values in place
    IM_ST(7)
    if (tid < 32) {
        int state = F.state;
        if (state == 1) {  // warp 0: counted ranks in the window, guards, k
            const int P = (int)(F.wend - F.woff), r0 = (int)F.sel_t, r1 = (int)F.sel_t1;
            double v0 = 0.0, v1 = 0.0;
            bool f0 = false, f1 = false;
            for (int i = lane; i < P; i += 32) {
                const double v = F.u.q.w[i];
                int r = 0;
                for (int j = 0; j < P; ++j) {
                    const double u = F.u.q.w[j];
                    r += (u < v) | ((u == v) & (j < i));
                }
                if (r == r0) v0 = v, f0 = true;
                if (r == r1) v1 = v, f1 = true;
            }
            const unsigned b0 = __ballot_sync(0xffffffffu, f0), b1 = __ballot_sync(0xffffffffu, f1);
            v0 = __shfl_sync(0xffffffffu, v0, b0 ? __ffs(b0) - 1 : 0);
            v1 = __shfl_sync(0xffffffffu, v1, b1 ? __ffs(b1) - 1 : 0);
            if (lane == 0) {
                const float inv0 = inv;
                const int wlo = F.bt, whi = F.bt1;
                const float elo = wlo > 0 ? __uint_as_float(bin_lo(wlo, lob, inv0)) : __uint_as_float(lob);
                const float ehi = whi < NBIN - 1 ? __uint_as_float(bin_lo(whi + 1, lob, inv0)) : __uint_as_float(hib);
                bool good = b0 && b1;
                if (elo > 0.f && !(elo >= 0x1p-100f && v0 * v0 > (double)elo * (1.0 + 0x1p-18))) good = false;
                if (ehi <= FLT_MAX && !(v1 * v1 < (double)ehi * (1.0 - 0x1p-18))) good = false;
                if (good) {
                    const double a_max = __longlong_as_double((long long)F.amax_b), gamma = F.gamma;
                    const double diff = __dsub_rn(v1, v0);
                    const double p_tau = gamma >= 0.5 ? __dsub_rn(v1, __dmul_rn(diff, __dsub_rn(1.0, gamma)))
                                                      : __dadd_rn(v0, __dmul_rn(diff, gamma));
                    F.k = finish_k(a.cfg, a_max, p_tau, F.nnz64, a.res, a.kvec, img);
                } else {
                    state = 0;
                }
            }
            state = __shfl_sync(0xffffffffu, state, 0);
        }
        if (lane == 0) F.fallback = state == 0;
    }
    __syncthreads();
    IM_ST(9)
}

// ---------------------------------------------------------------------------
// exact replay of a whole image (rare): reload from HBM x 2^kin, run every
// pass with the reference-literal stages in place on the tile (rows, columns,
// rows, columns -- fft_2d twice, fftcore.py:344-353), x 2^kout, store.
// ---------------------------------------------------------------------------
static __device__ __noinline__ void im_replay(const ImageArgs& a, int64_t img, char* tile, int kin, int kout) {
    const int tid = threadIdx.x, nthr = blockDim.x;
    auto acc = [tile](int e) { return reinterpret_cast<float2*>(tile + 16 * dsw(e >> 1) + 8 * (e & 1)); };
    const float2* src = a.in + img * (int64_t)IM_EL;
    __syncthreads();
    for (int e = tid; e < IM_EL; e += nthr) *acc(e) = gscale(src[e], kin);
    __syncthreads();
    const int line = tid >> 2, sub = tid & 3;
    for (int p = 0; p < a.npass; ++p) {
        const bool col = p & 1, inverse = p >= 2;
        auto L = [&](int i) { return acc(col ? i * IM_N + line : line * IM_N + i); };
        for (int i = sub; i < IM_N; i += 4) {  // bit-reversal gather (fftcore.py:262), in place
            const int r = (int)(__brev((unsigned)i) >> (32 - 7));
            if (i < r) {
                const float2 t = *L(i);
                *L(i) = *L(r);
                *L(r) = t;
            }
        }
        __syncthreads();
        for (int s = 0; s < 7; ++s) {
            generic_stage(L, s, IM_N / 2, a.cpb, a.fmt, a.wcr, a.wci, a.wsexp, inverse, sub, 4);
            __syncthreads();
        }
    }
    float2* dst = a.out + img * (int64_t)IM_EL;
    for (int e = tid; e < IM_EL; e += nthr) dst[e] = gscale(*acc(e), kout);
    __syncthreads();
}

template <int ID, int CPB>
__device__ __forceinline__ void im_load_tile(const ImageArgs& a, int64_t img, unsigned tile_sh) {
    const float4* src = reinterpret_cast<const float4*>(a.in + img * (int64_t)IM_EL) + threadIdx.x;
    const int rch = dsw(threadIdx.x);
#pragma unroll
    for (int k = 0; k < IM_EL / 2 / IM_NT; ++k)
        cp_async16(tile_sh + 16u * (unsigned)(rch ^ dsw(IM_NT * k)), src + IM_NT * k, true);
    cp_commit();
}

__device__ __forceinline__ void im_prefetch_l2(const ImageArgs& a, int64_t img) {
    if (threadIdx.x < 4 && img < a.nimg) {
        const char* p = reinterpret_cast<const char*>(a.in + img * (int64_t)IM_EL) + threadIdx.x * (IM_EL * 2);
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "n"(IM_EL * 2) : "memory");
    }
}

template <int ID, int CPB>
__global__ void __launch_bounds__(IM_NT, 1) k_mx_image(ImageArgs a) {
    extern __shared__ __align__(16) char im_smem[];
    const int tid = threadIdx.x;
    unsigned* twf = reinterpret_cast<unsigned*>(im_smem);
    unsigned* twi = twf + IM_N;
    signed char* twe = reinterpret_cast<signed char*>(twi + IM_N);
    char* tile = im_smem + a.tile_off;
    ImStats& F = *reinterpret_cast<ImStats*>(tile + IM_EL * 8);
    const unsigned tile_sh = (unsigned)__cvta_generic_to_shared(tile);
    if (tile_sh & 4095u) __trap();  // the swizzled addressing below relies on it
    for (int i = tid; i < (int)(sizeof(F.u) / 4); i += IM_NT) reinterpret_cast<unsigned*>(&F.u)[i] = 0;  // im_bracket expects zeros
    for (int i = tid; i < IM_N; i += IM_NT) {
        twf[tws(i)] = a.tw_fwd[i];
        twi[tws(i)] = a.tw_inv[i];
        twe[i] = a.twe[i];
    }
    LCtx L;  // the stage context; switched to the inverse twiddles for passes 3-4
    L.tw = twf;
    L.twe = twe;
    L.tw_sh = (unsigned)__cvta_generic_to_shared(twf);
    L.lt = IM_LT;
    L.tl = tid & (IM_T - 1);
    L.c = L.tl;
    L.trivial = a.trivial01;
    L.sigma = 1.f;
    L.slim = 7;
    const int lj = tid >> IM_LT;                                 // this thread's line
    const int rcol = (int)(__brev((unsigned)L.c) >> (32 - IM_LT));
    const int ebase = lj * IM_N;                                  // the line's row of the tile
    // row gather: element ebase + m T + rcol.  The three index fields are
    // bit-disjoint, so dsw (XOR-linear) splits into a per-thread base and a
    // per-m constant < 4096 that can be XORed into the 4 KB-aligned address.
    const unsigned g_row = tile_sh + 16u * (unsigned)(dsw(ebase >> 1) ^ dsw(rcol >> 1)) + 8u * (rcol & 1);
    // column gather: element (m T + rcol) n + lj; the per-m constant spans the
    // whole tile, so it is XORed into the tile-relative offset
    const unsigned g_col = 16u * (unsigned)(dsw((rcol * IM_N) >> 1) ^ dsw(lj >> 1)) + 8u * (lj & 1);
    LDbg dbg;

#ifdef MXFFT_IM_TIMING
    // phase clocks of CTA 0 (profiling builds only): wait, statistics, passes 1-4, store
    long long tsum[8] = {0, 0, 0, 0, 0, 0, 0, 0}, t0 = 0;
    int tn = 0, nfb = 0;
#define IM_T(i)                                   \
    if (tid == 0) {                               \
        const long long t1 = clock64();           \
        tsum[i] += t1 - t0;                       \
        t0 = t1;                                  \
    }
#else
#define IM_T(i)
#endif
    int64_t img = blockIdx.x;
    // the given k of this CTA's next image, loaded an image ahead (its latency
    // then never sits at the top of an image)
    int k_next = (!a.stats && a.kin && img < a.nimg) ? __ldg(a.kin + img / a.k_group) : 0;
    if (img < a.nimg) {
#if MXFFT_IM_PF == 2
        im_prefetch_l2(a, img + gridDim.x);
#endif
        im_load_tile<ID, CPB>(a, img, tile_sh);
    }
    for (; img < a.nimg; img += gridDim.x) {
#ifdef MXFFT_IM_TIMING
        if (tid == 0) t0 = clock64();
        ++tn;
#endif
        cp_wait<0>();
        __syncthreads();  // the tile has landed (and the twiddles are in place)
        IM_T(0)
#if MXFFT_IM_PF == 2
        im_prefetch_l2(a, img + 2 * (int64_t)gridDim.x);
#elif MXFFT_IM_PF == 1
        im_prefetch_l2(a, img + gridDim.x);
#endif
        int k = 0;
        if (!a.stats) {
            k = k_next;
            const int64_t nx = img + gridDim.x;
            if (a.kin && nx < a.nimg) k_next = __ldg(a.kin + nx / a.k_group);
        } else {
            im_bracket(tile_sh, F, a);
            im_select(F, a, img, tile_sh);
            if (F.fallback) {  // block-uniform; the tile is still intact
#ifdef MXFFT_IM_TIMING
                ++nfb;
#endif
                im_stats_exact(tile_sh, F, a, img);
            }
            k = F.k;
        }
        IM_T(1)
        bool bad = false;
        float2 x[32];
        int U, V, P, H;
        // ---- pass 1: rows of 2^k x ----
#pragma unroll
        for (int m = 0; m < 32; ++m) x[rev_c<5>(m)] = lds64(g_row ^ (16u * (unsigned)dsw((m * IM_T) >> 1)));
        // the statistics are done with the shared union: zero it for the next
        // image's sample histogram (many barriers pass before that is read)
        if (a.stats)
            for (int i = tid; i < (int)(sizeof(F.u) / 4); i += IM_NT) reinterpret_cast<unsigned*>(&F.u)[i] = 0;
        scale32<false>(x, k, bad);
        L.tw = a.first_inverse ? twi : twf;
        L.tw_sh = (unsigned)__cvta_generic_to_shared(a.first_inverse ? twi : twf);
        L.sigma = a.first_inverse ? -1.f : 1.f;
        run_stages<ID, CPB, false, IM_LT>(x, U, V, P, H, L, tile_sh, ebase, &dbg, bad);
        publish4(x, tile_sh, ebase, P, H);
#pragma unroll 1
        for (int pass = 1; pass < a.npass; ++pass) {
            __syncthreads();  // every line of the previous pass is in the tile
            IM_T(1 + pass)
#pragma unroll
            for (int m = 0; m < 32; ++m)
                x[rev_c<5>(m)] = lds64(tile_sh + (g_col ^ (16u * (unsigned)dsw((m * IM_T * IM_N) >> 1))));
            __syncthreads();  // all gathered: the rows may be overwritten by the exchanges
#if MXFFT_IM_PF == 3
            if (pass == a.npass - 1) im_prefetch_l2(a, img + gridDim.x);  // the next image, a pass ahead of its load
#endif
            if (pass == 2) {  // the inverse transform (fftcore.py:267-268: conjugated twiddles)
                L.tw = twi;
                L.tw_sh = (unsigned)__cvta_generic_to_shared(twi);
                L.sigma = -1.f;
            }
            run_stages<ID, CPB, false, IM_LT>(x, U, V, P, H, L, tile_sh, ebase, &dbg, bad);
            if (pass + 1 < a.npass) publish4(x, tile_sh, ebase, P, H);
        }
        const int kout = -k - (a.npass == 4 ? 2 * 7 : 0);
        scale32<false>(x, kout, bad);
        const int any_bad = __syncthreads_or(bad);
        IM_T(1 + a.npass)
        if (any_bad) {
            im_replay(a, img, tile, k, kout);
            if (img + gridDim.x < a.nimg) im_load_tile<ID, CPB>(a, img + gridDim.x, tile_sh);
            continue;
        }
        // the tile is free: the next image streams in while this one is stored
        if (img + gridDim.x < a.nimg) im_load_tile<ID, CPB>(a, img + gridDim.x, tile_sh);
        // the lines are columns of the result: x[8q + i] is element P + q H + i of column lj
        {
            float2* dst = a.out + img * (int64_t)IM_EL + lj;
#pragma unroll
            for (int q = 0; q < 4; ++q)
#pragma unroll
                for (int i = 0; i < 8; ++i) dst[(int64_t)(P + q * H + i) * IM_N] = x[8 * q + i];
        }
        IM_T(7)
    }
    cp_wait<0>();
#ifdef MXFFT_IM_TIMING
    if (tid == 0 && blockIdx.x == 0 && tn)
    {
        printf("k_mx_image CTA0 %d images, cycles/image: wait %lld stats %lld p1 %lld p2 %lld p3 %lld p4 %lld store %lld fallbacks %d\n",
               tn, tsum[0] / tn, tsum[1] / tn, tsum[2] / tn, tsum[3] / tn, tsum[4] / tn, tsum[5] / tn, tsum[7] / tn, nfb);
        printf("  stats sub-phases: sample %lld bracket %lld gather %lld select-stream %lld classify %lld scan %lld window %lld rank+k %lld\n",
               g_im_t[1] / tn, g_im_t[2] / tn, 0ll, g_im_t[4] / tn, g_im_t[5] / tn, g_im_t[6] / tn,
               g_im_t[7] / tn, g_im_t[9] / tn);
    }
#endif
#undef IM_T
}

}  // namespace mxfft
