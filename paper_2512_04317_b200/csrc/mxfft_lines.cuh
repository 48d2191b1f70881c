// mxfft_lines.cuh -- the MX-FFT line kernel for sm_100a (the hot path).
//
// One "line" = one 1-D transform of length n (a row, or a column of an n x n
// image).  A line is owned by T = n/32 threads; each thread holds 32 complex
// FP32 values in registers.
//
//   load   : thread c reads its 32 elements straight from HBM in bit-reversed
//            order (fftcore.py:262): position 32c+i <- natural index
//            rev5(i)*T + rev_T(c); a warp's loads cover whole 32B sectors.
//   stages 0..4 run in registers (blocks of cpb butterflies are in-thread, or
//            split over a lane pair for cpb = 32).  Stages 0 and 1 have the
//            twiddles 1 and -i (+i inverse); when the plan's encoded twiddles
//            are exactly those, the MX product reduces to the v-block codes
//            (proved in DESIGN.md) and the multiply/renormalize is skipped.
//   stages >= 5 exchange through shared memory once per stage; thread t takes
//            butterflies [16t, 16t+16) = whole MX blocks.  The layout is an XOR
//            swizzle on 16-byte chunks chosen so that every access pattern
//            (the layout-A write and the u/v runs of every stage) is free of
//            bank conflicts.
//   store  : the last stage writes its u/v runs straight to HBM.
//
// Per butterfly (general stage): FMNMX3 (v amax), 2 FMUL + 2 F2FP (v codes),
// 4 FHFMA (exact mantissa-space products from packed f16 codes), FMNMX3
// (product amax), 2 FMUL + 2 F2FP + 2 HADD2 (requantize), 4 FFMA (decode
// folded into u +- t).  Twiddles live in shared memory as packed f16 codes.
#pragma once
#include "mxfft_common.cuh"
#include "mxfft_generic.cuh"
#include "mxfft_internal.h"
#ifndef MXFFT_WARP_LOCAL_EXCHANGE
#define MXFFT_WARP_LOCAL_EXCHANGE 0  // n >= 2048: warp-level sync for the exchanges that stay inside a warp (measured neutral on C5: 13.91 vs 13.85 ms; off)
#endif
#include <cooperative_groups.h>
#include <type_traits>

#ifndef MXFFT_PAIR_STORE
#define MXFFT_PAIR_STORE 1  // strided copy-out: two adjacent lines per thread, 16-byte stores
#endif
#ifndef MXFFT_BIG_PREFETCH
#define MXFFT_BIG_PREFETCH 1  // n = 8192/16384: bulk L2 prefetch of the next row during this one
#endif
#ifndef MXFFT_KPREF
#define MXFFT_KPREF 1  // load the next group's prescale exponent a group ahead
#endif
#ifndef MXFFT_SHCHAIN
#define MXFFT_SHCHAIN 0  // renormalisation shift by exponent-field carry (non-debug kernels)
#endif
#ifndef MXFFT_PAIR_STAGES
#define MXFFT_PAIR_STAGES 1  // n-specialised kernels: two butterfly stages per shared-memory exchange
#endif
#ifndef MXFFT_PAIR_STORE_MAXLT
#define MXFFT_PAIR_STORE_MAXLT 3  // paired strided copy-out up to n = 32 * 2^LT (n = 512 measured 13 % slower)
#endif
#ifndef MXFFT_CL2
#define MXFFT_CL2 0  // n = 8192/16384 plain row passes: a 2-CTA cluster per line (measured 3.52 vs 2.55 ms: off)
#endif
#ifndef MXFFT_UNROLL_PAIRS
#define MXFFT_UNROLL_PAIRS 0  // unroll the paired-stage loop for LT <= this (compile-time stage indices)
#endif
#ifndef MXFFT_PAIR_BATCH
#define MXFFT_PAIR_BATCH 1  // paired strided copy-out: positions read from shared memory per batch of stores
#endif
#ifndef MXFFT_BATCH_STORE
#define MXFFT_BATCH_STORE 0  // transposed stores: read the whole column run from shared memory first
#endif
#ifndef MXFFT_UNROLL_SMEM
#define MXFFT_UNROLL_SMEM 0  // unroll the shared-memory stages of the n-specialised kernels
#endif
#ifndef MXFFT_TW_FIRST
#define MXFFT_TW_FIRST 0  // paired stages: twiddle loads before the exchange loads (measured: no gain)
#endif
#ifndef MXFFT_LOCAL_STAGES
#define MXFFT_LOCAL_STAGES 5  // unrolled register stages before the shared-memory loop
#endif

namespace mxfft {

// ---------------------------------------------------------------------------
// helpers
// ---------------------------------------------------------------------------
// 16-byte-chunk swizzle of the line data: bit b >= 3 of the chunk index is
// folded into bit (b mod 3) of the bank group, except bit 6 which is folded
// into all three.  Any three consecutive chunk bits (layout-A writes) and the
// bit sets {3,5,6}, {3,4,6}, {3,4,5} (stage-5/6/>=7 runs) map bijectively onto
// the 8 bank groups -> conflict-free 128-bit accesses.
__host__ __device__ __forceinline__ constexpr int dsw(int C) {
    const int x = C >> 3;
    int f = (x ^ (x >> 3) ^ (x >> 6) ^ (x >> 9)) & 7;
    f ^= ((C >> 6) & 1) * 6;
    return C ^ f;
}

// twiddle table swizzle (4-byte entries, 16-byte chunks): stage-s lanes read
// chunks (half + 16t)/4 + k; folding chunk bits 3,4 into bits 0,1 spreads them.
__device__ __forceinline__ int tws(int idx) {
    const int c = idx >> 2;
    return ((c ^ ((c >> 3) & 3)) << 2) | (idx & 3);
}

template <int BITS>
__host__ __device__ constexpr int rev_c(int i) {
    int r = 0;
    for (int b = 0; b < BITS; ++b) r |= ((i >> b) & 1) << (BITS - 1 - b);
    return r;
}

// packed quantize: returns f16x2 codes with lo = q(re), hi = q(im)
template <int ID>
__device__ __forceinline__ unsigned q2h(float re, float im);
template <>
__device__ __forceinline__ unsigned q2h<F_E4M3>(float re, float im) {
    unsigned short p;
    unsigned h;
    asm("cvt.rn.satfinite.e4m3x2.f32 %0, %1, %2;" : "=h"(p) : "f"(im), "f"(re));
    asm("cvt.rn.f16x2.e4m3x2 %0, %1;" : "=r"(h) : "h"(p));
    return h;
}
template <>
__device__ __forceinline__ unsigned q2h<F_E5M2>(float re, float im) {
    unsigned short p;
    unsigned h;
    asm("cvt.rn.satfinite.e5m2x2.f32 %0, %1, %2;" : "=h"(p) : "f"(im), "f"(re));
    asm("cvt.rn.f16x2.e5m2x2 %0, %1;" : "=r"(h) : "h"(p));
    return h;
}
template <>
__device__ __forceinline__ unsigned q2h<F_E2M3>(float re, float im) {
    unsigned short p;
    unsigned h;
    asm("cvt.rn.satfinite.e2m3x2.f32 %0, %1, %2;" : "=h"(p) : "f"(im), "f"(re));
    asm("cvt.rn.f16x2.e2m3x2 %0, %1;" : "=r"(h) : "h"(p));
    return h;
}
template <>
__device__ __forceinline__ unsigned q2h<F_E3M2>(float re, float im) {
    unsigned short p;
    unsigned h;
    asm("cvt.rn.satfinite.e3m2x2.f32 %0, %1, %2;" : "=h"(p) : "f"(im), "f"(re));
    asm("cvt.rn.f16x2.e3m2x2 %0, %1;" : "=r"(h) : "h"(p));
    return h;
}
template <>
__device__ __forceinline__ unsigned q2h<F_E2M1>(float re, float im) {
    unsigned h;
    asm("{\n\t.reg .b8 t;\n\tcvt.rn.satfinite.e2m1x2.f32 t, %1, %2;\n\t"
        "cvt.rn.f16x2.e2m1x2 %0, t;\n\t}"
        : "=r"(h)
        : "f"(im), "f"(re));
    return h;
}

__device__ __forceinline__ float h_lo(unsigned h) {
    return __low2float(*reinterpret_cast<const __half2*>(&h));
}
__device__ __forceinline__ float h_hi(unsigned h) {
    return __high2float(*reinterpret_cast<const __half2*>(&h));
}

// f16x2 -> two FP32 values (exact).  MXFFT_FHFMA_CVT=1 converts on the FMA pipe
// as fma.rn.f32.f16(h, 1.0, -0.0) (FHFMA, full rate) instead of HADD2.F32 on the
// half-rate ALU pipe, which the F2FP packs/unpacks and FMNMX3 already load.
#ifndef MXFFT_FHFMA_CVT
#define MXFFT_FHFMA_CVT 1
#endif
__device__ __forceinline__ void h2f2(unsigned h, float& lo, float& hi) {
#if MXFFT_FHFMA_CVT
    asm("{\n\t.reg .f16 l, u, one;\n\tmov.b32 {l, u}, %2;\n\tmov.b16 one, 0x3C00;\n\t"
        "fma.rn.f32.f16 %0, l, one, 0f80000000;\n\tfma.rn.f32.f16 %1, u, one, 0f80000000;\n\t}"
        : "=f"(lo), "=f"(hi)
        : "r"(h));
#else
    lo = h_lo(h);
    hi = h_hi(h);
#endif
}

// exact mantissa-space complex product of packed f16 codes W = (wr, wi) and
// C = (cr, ci): pr = fl(wr*cr - wi*ci), pi = fl(wr*ci + wi*cr) (fftcore.py:168-169);
// each f16 x f16 product is exact in FP32, one rounding per sum.
__device__ __forceinline__ void cprod(unsigned W, unsigned C, float& pr, float& pi) {
    asm("{\n\t.reg .f16 wl, wh, cl, ch;\n\t.reg .f32 t1, t2;\n\t"
        "mov.b32 {wl, wh}, %2;\n\tmov.b32 {cl, ch}, %3;\n\t"
        "fma.rn.f32.f16 t1, wh, ch, 0f80000000;\n\t"
        "neg.f32 t1, t1;\n\t"
        "fma.rn.f32.f16 %0, wl, cl, t1;\n\t"
        "fma.rn.f32.f16 t2, wh, cl, 0f80000000;\n\t"
        "fma.rn.f32.f16 %1, wl, ch, t2;\n\t}"
        : "=f"(pr), "=f"(pi)
        : "r"(W), "r"(C));
}

// max over the lane pair sharing a 32-butterfly block (pairs always take the
// same branches, so the 2-lane mask is valid even in divergent code)
template <bool PAIR>
__device__ __forceinline__ float pair_max(float a) {
    if (PAIR) {
        const unsigned lane = threadIdx.x & 31;
        a = fmaxf(a, __shfl_xor_sync(3u << (lane & ~1u), a, 1));
    }
    return a;
}

// max over the G consecutive lanes (G = 1, 2, 4) that share one MX block
template <int G>
__device__ __forceinline__ float grp_max(float a) {
    if constexpr (G > 1) {
        const unsigned lane = threadIdx.x & 31;
        const unsigned m = ((1u << G) - 1u) << (lane & ~(unsigned)(G - 1));
        a = fmaxf(a, __shfl_xor_sync(m, a, 1));
        if constexpr (G > 2) a = fmaxf(a, __shfl_xor_sync(m, a, 2));
    }
    return a;
}

struct LDbg {
    int32_t* vexp;
    float* vcodes;
    int32_t* pexp;
    int32_t* pshift;
    float* pcodes;
    int64_t row, rows;
    int m, cpb, stage;
};

__device__ __forceinline__ void dbg_codes(const LDbg& d, int bfly, float a, float b, float c,
                                          float e) {
    if (d.row >= d.rows) return;
    const int64_t o = ((int64_t)d.stage * d.rows + d.row) * d.m + bfly;
    d.vcodes[2 * o] = a;
    d.vcodes[2 * o + 1] = b;
    d.pcodes[2 * o] = c;
    d.pcodes[2 * o + 1] = e;
}
__device__ __forceinline__ void dbg_exps(const LDbg& d, int bfly, int ev, int E, int sh) {
    if (d.row >= d.rows) return;
    const int64_t o = ((int64_t)d.stage * d.rows + d.row) * (d.m / d.cpb) + bfly / d.cpb;
    d.vexp[o] = ev;
    d.pexp[o] = E;
    d.pshift[o] = sh;
}

// ---------------------------------------------------------------------------
// rare path: extreme magnitudes (scale or decode exponent outside FP32's
// normal range).  FP64-assisted, exact; works on a local copy.
// ---------------------------------------------------------------------------
template <int ID, int NB, bool PAIR, bool DBG>
__device__ __noinline__ void mxb_slow(float2* u, float2* v, const unsigned* w, int ew, int ev,
                                      const LDbg* d, int bfly0) {
    using F = HwFmt<ID>;
    const double inv = ldexp(1.0, -ev);
    float pr[NB], pi[NB];
    unsigned cv[NB];
    float ap = 0.f;
    for (int i = 0; i < NB; ++i) {
        cv[i] = q2h<ID>((float)((double)v[i].x * inv), (float)((double)v[i].y * inv));
        cprod(w[i], cv[i], pr[i], pi[i]);
        ap = fmax3(ap, fabsf(pr[i]), fabsf(pi[i]));
    }
    if (PAIR) {
        const unsigned lane = threadIdx.x & 31;
        ap = fmaxf(ap, __shfl_xor_sync(3u << (lane & ~1u), ap, 1));
    }
    const int sh = ap > F::MAXF ? shift_for<F>(ap) : 0;
    const float fac = exp2i(-sh);
    const int E = ew + ev + sh;
    const double sc = ldexp(1.0, E);
    for (int i = 0; i < NB; ++i) {
        const unsigned qp = q2h<ID>(__fmul_rn(pr[i], fac), __fmul_rn(pi[i], fac));
        const float qr = h_lo(qp), qi = h_hi(qp);
        const float tr = (float)((double)qr * sc), ti = (float)((double)qi * sc);
        const float2 uu = u[i];
        u[i] = make_float2(__fadd_rn(uu.x, tr), __fadd_rn(uu.y, ti));
        v[i] = make_float2(__fsub_rn(uu.x, tr), __fsub_rn(uu.y, ti));
        if (DBG) dbg_codes(*d, bfly0 + i, h_lo(cv[i]), h_hi(cv[i]), qr, qi);
    }
    if (DBG && ((bfly0 % d->cpb) == 0)) dbg_exps(*d, bfly0, ev, E, sh);
}

// ---------------------------------------------------------------------------
// general MX block: NB butterflies held by this thread (NB = cpb, or 16 of a
// 32-butterfly block split over a lane pair)
// ---------------------------------------------------------------------------
// block maximum of |re|, |im| over NB complex values as four interleaved
// FMNMX3 chains (dependency depth ~NB/4 + 2 instead of NB)
template <int NB>
__device__ __forceinline__ float amax_c(const float2 (&v)[NB]) {
    constexpr int L = NB < 4 ? NB : 4;
    float m[L];
#pragma unroll
    for (int l = 0; l < L; ++l) m[l] = fmaxf(fabsf(v[l].x), fabsf(v[l].y));
#pragma unroll
    for (int i = L; i < NB; ++i) m[i % L] = fmax3(m[i % L], fabsf(v[i].x), fabsf(v[i].y));
    if (L == 1) return m[0];
    if (L == 2) return fmaxf(m[0], m[1]);
    return fmaxf(fmax3(m[0], m[1], m[2 % L]), m[3 % L]);
}
template <int NB>
__device__ __forceinline__ float amax_2(const float (&a)[NB], const float (&b)[NB]) {
    constexpr int L = NB < 4 ? NB : 4;
    float m[L];
#pragma unroll
    for (int l = 0; l < L; ++l) m[l] = fmaxf(fabsf(a[l]), fabsf(b[l]));
#pragma unroll
    for (int i = L; i < NB; ++i) m[i % L] = fmax3(m[i % L], fabsf(a[i]), fabsf(b[i]));
    if (L == 1) return m[0];
    if (L == 2) return fmaxf(m[0], m[1]);
    return fmaxf(fmax3(m[0], m[1], m[2 % L]), m[3 % L]);
}

// The "replay this group" flag threaded through the stage code is either a
// plain bool or, in the statistics-folding first pass (lines_body_tma<.., ACC>),
// a BadTrack that also records the range of the v-block exponents it saw.
struct BadTrack {
    bool b = false;
    int lo = 127, hi = -127;
    __device__ __forceinline__ BadTrack& operator|=(bool v) {
        b |= v;
        return *this;
    }
    __device__ __forceinline__ operator bool() const { return b; }
};
__device__ __forceinline__ void note_ev(bool&, int) {}
__device__ __forceinline__ void note_ev(BadTrack& t, int ev) {
    t.lo = min(t.lo, ev);
    t.hi = max(t.hi, ev);
}

// floor(log2 am) for the block exponent.  Non-debug kernels read the biased
// exponent field only: a subnormal am then yields -127, which puts ev below
// the fast range, so the group is replayed exactly (replay_lines).
template <bool DBG>
__device__ __forceinline__ int flog2_hot(float am) {
    if constexpr (DBG) return floor_log2f(am);
    return (int)(__float_as_uint(am) >> 23) - 127;  // am >= 0
}

// SLOW: an out-of-range block takes the exact FP64-assisted path inline (as
// the debug kernels do) instead of flagging a replay of the whole group
template <int ID, int NB, int G, bool DBG, bool SLOW = DBG, class BT = bool>
__device__ __forceinline__ void mxb(float2 (&u)[NB], float2 (&v)[NB], const unsigned (&w)[NB],
                                    int ew, const LDbg* d, int bfly0, BT& bad) {
    using F = HwFmt<ID>;
    using Rg = DecodeRange<F>;
    constexpr bool PAIR = G == 2;
    static_assert(!((DBG || SLOW) && G > 2), "the inline exact path splits a block over at most a lane pair");
    const float am = grp_max<G>(amax_c<NB>(v));
    const int ev = am > 0.f ? flog2_hot<DBG || SLOW>(am) - F::EMAX : 0;
    note_ev(bad, ev);
    const float inv = exp2i(-ev);
    unsigned cv[NB];
    float pr[NB], pi[NB];
    const float2 inv2 = make_float2(inv, inv);
#pragma unroll
    for (int i = 0; i < NB; ++i) {
        const float2 vs = __fmul2_rn(v[i], inv2);  // FMUL2: exact power-of-two scaling
        cv[i] = q2h<ID>(vs.x, vs.y);
        cprod(w[i], cv[i], pr[i], pi[i]);
    }
    const float ap = grp_max<G>(amax_2<NB>(pr, pi));
    // ceil(log2(ap / max_finite)) for ap > max_finite, else 0: the mantissa
    // excess over max_finite's carries into the exponent field (exact; NaN and
    // inf give a huge shift, which replays the group)
    const int sh = (DBG || !MXFFT_SHCHAIN) ? (ap > F::MAXF ? shift_for<F>(ap) : 0)
                       : max(0, (int)((__float_as_uint(ap) + (0x7fffffu - F::MM)) >> 23) - 127 - F::EM);
    const int E = ew + ev + sh;
    const bool fast = ((unsigned)(ev + 127) <= 253u) & ((unsigned)(E - Rg::ELO) <= (unsigned)(Rg::EHI - Rg::ELO));
    if constexpr (!DBG && !SLOW) {
        bad |= !fast;  // the group is replayed exactly (replay_lines); keep going
    } else if (__builtin_expect(!fast, 0)) {
        float2 tu[NB], tv[NB];
        unsigned tw[NB];
#pragma unroll
        for (int i = 0; i < NB; ++i) {
            tu[i] = u[i];
            tv[i] = v[i];
            tw[i] = w[i];
        }
        mxb_slow<ID, NB, PAIR, DBG>(tu, tv, tw, ew, ev, d, bfly0);
#pragma unroll
        for (int i = 0; i < NB; ++i) {
            u[i] = tu[i];
            v[i] = tv[i];
        }
        return;
    }
    const float fac = exp2i(-sh);
    const float sc = exp2i(E);
    const float2 fac2 = make_float2(fac, fac), sc2 = make_float2(sc, sc);
#pragma unroll
    for (int i = 0; i < NB; ++i) {
        const float2 ps = __fmul2_rn(make_float2(pr[i], pi[i]), fac2);
        const unsigned qp = q2h<ID>(ps.x, ps.y);
        float qr, qi;
        h2f2(qp, qr, qi);
        const float2 q = make_float2(qr, qi);
        const float2 uu = u[i];
        // decode folded into the butterfly as two FFMA2: u +- q * 2^E
        u[i] = __ffma2_rn(q, sc2, uu);
        v[i] = __ffma2_rn(make_float2(-qr, -qi), sc2, uu);
        if (DBG) dbg_codes(*d, bfly0 + i, h_lo(cv[i]), h_hi(cv[i]), qr, qi);
    }
    if (DBG && ((bfly0 % d->cpb) == 0)) dbg_exps(*d, bfly0, ev, E, sh);
}

// Stages 0/1 with twiddles exactly (2^emax, 0) / (0, -+2^emax) at scale 2^-emax:
// the product block equals the v block shifted by emax, so its codes are the
// v codes (j = 0) or (ci, -cr) * sigma (j = 1) and E = ev.  Returns false when
// the exponents leave the fast range (the caller then runs the general path).
template <int ID, int NB, bool PAIR, int S, bool DBG, class BT>
__device__ __forceinline__ bool trivial_block(float2 (&u)[NB], float2 (&v)[NB], int j0,
                                              float sigma, const LDbg* d, int bfly0, BT& bad) {
    using F = HwFmt<ID>;
    using Rg = DecodeRange<F>;
    const float am = pair_max<PAIR>(amax_c<NB>(v));
    const int ev = am > 0.f ? flog2_hot<DBG>(am) - F::EMAX : 0;
    note_ev(bad, ev);
    const bool ok = (ev >= -127) & (ev <= 126) & (ev >= Rg::ELO) & (ev <= Rg::EHI);
    if (DBG && !ok) return false;  // non-debug kernels finish branch-free and replay
    const float inv = exp2i(-ev), sc = exp2i(ev);
    const float2 inv2 = make_float2(inv, inv), sc2 = make_float2(sc, sc);
    // rotated butterflies: (tr, ti) = (sigma ci, -sigma cr), folded into the
    // scale pair (exact: sigma = +-1) so that no multiply by sigma is issued
    const float2 scr = make_float2(sigma * sc, -sigma * sc);
#pragma unroll
    for (int i = 0; i < NB; ++i) {
        const float2 vs = __fmul2_rn(v[i], inv2);
        const unsigned cv = q2h<ID>(vs.x, vs.y);
        float cr, ci;
        h2f2(cv, cr, ci);
        const bool rot = S == 1 && ((j0 + i) & 1);  // compile-time
        const float2 c = rot ? make_float2(ci, cr) : make_float2(cr, ci);
        const float2 f = rot ? scr : sc2;
        const float2 uu = u[i];
        u[i] = __ffma2_rn(c, f, uu);
        v[i] = __ffma2_rn(make_float2(-c.x, -c.y), f, uu);
        if (DBG) dbg_codes(*d, bfly0 + i, cr, ci, rot ? sigma * ci : cr, rot ? -sigma * cr : ci);
    }
    if (DBG && ((bfly0 % d->cpb) == 0))
        dbg_exps(*d, bfly0, ev, am > 0.f ? ev : -F::EMAX, am > 0.f ? F::EMAX : 0);
    return ok;
}

// One register-resident stage S (half = 2^S <= 16) over the thread's 32 values.
// Stages 0/1 take the trivial-twiddle shortcut (plans always qualify; any
// block outside the fast exponent range goes through the out-of-line exact
// path).  Stages 2..4 run the general block inline.
template <int ID, int CPB, int S, bool DBG, class BT>
__device__ __forceinline__ void local_stage(float2 (&x)[32], const unsigned* tw, const signed char* twe,
                                            int c, bool trivial, float sigma, LDbg* d, BT& bad) {
    constexpr int half = 1 << S;
    constexpr int NB = CPB < 16 ? CPB : 16;
    constexpr bool PAIR = CPB == 32;
    if (DBG) d->stage = S;
#pragma unroll
    for (int k = 0; k < 16 / NB; ++k) {
        float2 ub[NB], vb[NB];
#pragma unroll
        for (int i = 0; i < NB; ++i) {
            const int b = k * NB + i, g = b >> S, j = b & (half - 1);
            ub[i] = x[g * 2 * half + j];
            vb[i] = x[g * 2 * half + half + j];
        }
        const int j0 = (k * NB) & (half - 1);
        const int bfly0 = c * 16 + k * NB;
        if (S <= 1) {
            if constexpr (!DBG) {
                // computed unconditionally (no join to merge registers at); a
                // non-trivial plan or an out-of-range block replays the group
                const bool done = trivial_block<ID, NB, PAIR, S, DBG>(ub, vb, j0, sigma, d, bfly0, bad);
                bad |= !(done & trivial);
            } else if (!(trivial && trivial_block<ID, NB, PAIR, S, DBG>(ub, vb, j0, sigma, d, bfly0, bad))) {
                // exact out-of-line path (also covers plans whose stage-0/1
                // twiddles are not exactly 1 / -i)
                float2 tu[NB], tv[NB];
                unsigned tww[NB];
                float am = 0.f;
#pragma unroll
                for (int i = 0; i < NB; ++i) {
                    tu[i] = ub[i];
                    tv[i] = vb[i];
                    tww[i] = tw[tws(half + ((k * NB + i) & (half - 1)))];
                    am = fmax3(am, fabsf(vb[i].x), fabsf(vb[i].y));
                }
                am = pair_max<PAIR>(am);
                const int ev = am > 0.f ? floor_log2f(am) - HwFmt<ID>::EMAX : 0;
                mxb_slow<ID, NB, PAIR, DBG>(tu, tv, tww, twe[half + j0], ev, d, bfly0);
#pragma unroll
                for (int i = 0; i < NB; ++i) {
                    ub[i] = tu[i];
                    vb[i] = tv[i];
                }
            }
        } else {
            unsigned w[NB];
#pragma unroll
            for (int i = 0; i < NB; ++i) w[i] = tw[tws(half + ((k * NB + i) & (half - 1)))];
            mxb<ID, NB, PAIR ? 2 : 1, DBG>(ub, vb, w, twe[half + j0], d, bfly0, bad);
        }
#pragma unroll
        for (int i = 0; i < NB; ++i) {
            const int b = k * NB + i, g = b >> S, j = b & (half - 1);
            x[g * 2 * half + j] = ub[i];
            x[g * 2 * half + half + j] = vb[i];
        }
    }
}

// power-of-two scaling of the thread's 32 values (apply/undo prescale, 1/n^2):
// one FP32 multiply when 2^e is a normal float, else an exact FP64 product
// rounded once (out of line: never taken for real data).
static __device__ __noinline__ void scale32_slow(float2* x, int e) {
    const double f = ldexp(1.0, e);
    for (int i = 0; i < 32; ++i) x[i] = make_float2((float)((double)x[i].x * f), (float)((double)x[i].y * f));
}

template <bool DBG, class BT>
__device__ __forceinline__ void scale32(float2 (&x)[32], int e, BT& bad) {
    if (!DBG || (e >= -126 && e <= 127)) {
        bad |= !(e >= -126 && e <= 127);  // non-debug kernels replay the group
        const float f = exp2i(e);
        const float2 f2 = make_float2(f, f);
#pragma unroll
        for (int i = 0; i < 32; ++i) x[i] = __fmul2_rn(x[i], f2);
    } else {
        float2 t[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) t[i] = x[i];
        scale32_slow(t, e);
#pragma unroll
        for (int i = 0; i < 32; ++i) x[i] = t[i];
    }
}

// global stores with an explicit state space (a generic ST has to resolve the
// window of every address); MXFFT_STG=0 keeps plain C++ stores
#ifndef MXFFT_STG
#define MXFFT_STG 0  // measured: asm st.global (a "memory" clobber) 73.7 -> 77.5 us on the C2 pass
#endif
__device__ __forceinline__ void stg128(float4* p, float4 v) {
#if MXFFT_STG
    asm volatile("st.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w)
                 : "memory");
#else
    *p = v;
#endif
}
__device__ __forceinline__ void stg64(float2* p, float2 v) {
#if MXFFT_STG
    asm volatile("st.global.v2.f32 [%0], {%1, %2};" ::"l"(p), "f"(v.x), "f"(v.y) : "memory");
#else
    *p = v;
#endif
}

// shared memory accesses by 32-bit shared-window address
__device__ __forceinline__ void sts128(unsigned addr, float2 a, float2 b) {
    asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "f"(a.x), "f"(a.y), "f"(b.x),
                 "f"(b.y)
                 : "memory");
}
__device__ __forceinline__ void lds128(unsigned addr, float2& a, float2& b) {
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(a.x), "=f"(a.y), "=f"(b.x), "=f"(b.y)
                 : "r"(addr)
                 : "memory");
}
__device__ __forceinline__ float2 lds64(unsigned addr) {
    float2 v;
    asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "r"(addr) : "memory");
    return v;
}
__device__ __forceinline__ uint4 lds128u(unsigned addr) {
    uint4 v;
    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "r"(addr)
                 : "memory");
    return v;
}

// A run of 16 complex (8 chunks) starting at element e (multiple of 16) of the
// region at shared address rb: chunk k lives at a0 | (f ^ 16k).
struct Run {
    unsigned a0, f;
};
__device__ __forceinline__ Run mkrun(unsigned rb, int e) {
    const int C0 = e >> 1;
    return {rb + (unsigned)C0 * 16u, (unsigned)(dsw(C0) ^ C0) << 4};
}
__device__ __forceinline__ unsigned radr(const Run& r, int k) { return r.a0 | (r.f ^ (unsigned)(k << 4)); }

// segmented rows input (seg_log2 > 0): the all-to-all receive layout of a
// row-slab transpose, (G, lines, R) with R = 2^seg_log2 -- element q of line c
// lives in segment q / R at offset c R + q mod R
__device__ __forceinline__ int64_t seg_off(const MxLinesArgs& a, int64_t line, int q) {
    const int R = 1 << a.seg_log2;
    return (int64_t)(q >> a.seg_log2) * a.seg_stride + line * R + (q & (R - 1));
}

// prescale-exponent entry of a line: kvec[(line / lines_per_image) / k_group]
// (a shift and no division in the common power-of-two / one-image-per-k case)
__device__ __forceinline__ int64_t k_index(const MxLinesArgs& a, int64_t line) {
    const int64_t img = a.lpi_shift >= 0 ? line >> a.lpi_shift : line / a.lines_per_image;
    return a.k_group == 1 ? img : img / a.k_group;
}

// ---------------------------------------------------------------------------
// kernel body.  The hot variants are specialised on LT = log2(T) (n = 32 T):
// the tile geometry is then compile-time and every swizzled shared address
// below is a per-thread base XOR an immediate (dsw() is linear over XOR, and
// the offsets combined are always bit-disjoint, so dsw(a | b) = dsw(a) ^
// dsw(b)).  LT = -1 instantiates the same code with T taken at run time.
// ---------------------------------------------------------------------------
struct LCtx {
    const unsigned* tw;
    const signed char* twe;
    unsigned tw_sh;  // shared address of the (swizzled) twiddle codes
    int lt, tl, c;
    bool trivial;
    float sigma;
    int slim;
};


__device__ __forceinline__ void lsync(bool big) {
    if (big) __syncthreads(); else __syncwarp();
}

// All butterfly stages of one group.  Registers for stages < 5; stages >= 5
// exchange through the line's region (element e of the buffer at shared
// address rb lives in chunk dsw(e/2), half e&1).  On return x[0..15] sit at
// line positions U.., x[16..31] at V.. .
// One shared-memory stage s >= 5 (thread t takes butterflies [16t, 16t+16)).
template <int ID, int CPB, bool DBG, class BT>
__device__ __forceinline__ void smem_stage(float2 (&x)[32], int& U, int& V, const LCtx& L, unsigned rb,
                                           int ebase, int s, bool big, LDbg* dbg, BT& bad) {
    constexpr int NB = CPB < 16 ? CPB : 16;
    constexpr bool PAIR = CPB == 32;
    {  // publish current values at their positions
        const Run ru = mkrun(rb, ebase + U), rv = mkrun(rb, ebase + V);
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            sts128(radr(ru, k), x[2 * k], x[2 * k + 1]);
            sts128(radr(rv, k), x[16 + 2 * k], x[17 + 2 * k]);
        }
    }
    lsync(big);
    const int half = 1 << s;
    const int b0 = 16 * L.tl;
    const int j0 = b0 & (half - 1);
    U = ((b0 >> s) << (s + 1)) + j0;
    V = U + half;
    {
        const Run ru = mkrun(rb, ebase + U), rv = mkrun(rb, ebase + V);
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            lds128(radr(ru, k), x[2 * k], x[2 * k + 1]);
            lds128(radr(rv, k), x[16 + 2 * k], x[17 + 2 * k]);
        }
    }
    unsigned w16[16];
#pragma unroll
    for (int i = 0; i < 16; i += 4) {
        const uint4 q = lds128u(L.tw_sh + 4u * (unsigned)tws(half + j0 + i));
        w16[i] = q.x;
        w16[i + 1] = q.y;
        w16[i + 2] = q.z;
        w16[i + 3] = q.w;
    }
    if (DBG) dbg->stage = s;
#pragma unroll
    for (int k = 0; k < 16 / NB; ++k) {
        float2 ub[NB], vb[NB];
        unsigned wb[NB];
#pragma unroll
        for (int i = 0; i < NB; ++i) {
            ub[i] = x[k * NB + i];
            vb[i] = x[16 + k * NB + i];
            wb[i] = w16[k * NB + i];
        }
        mxb<ID, NB, PAIR ? 2 : 1, DBG>(ub, vb, wb, L.twe[half + j0 + k * NB], dbg, b0 + k * NB, bad);
#pragma unroll
        for (int i = 0; i < NB; ++i) {
            x[k * NB + i] = ub[i];
            x[16 + k * NB + i] = vb[i];
        }
    }
}

// Two butterfly stages s, s+1 (h = 2^s >= 32) per shared-memory exchange.
// Thread tl owns the radix-4 units [8 tl, 8 tl + 8) of the line: with
// g = 8 tl / h and j0 = 8 tl mod h, x[8k + i] holds line element
// P + k h + i, P = 4 h g + j0 (k < 4, i < 8).  Stage s pairs (x[i], x[8+i]) and
// (x[16+i], x[24+i]) (butterflies j0 + i of groups 2g, 2g+1); stage s+1 pairs
// (x[i], x[16+i]) and (x[8+i], x[24+i]) (butterflies j0 + i and h + j0 + i of
// group g).  Every 8-butterfly set is a whole MX block (cpb 8) or 1/2, 1/4 of
// one shared with the neighbouring lanes (cpb 16, 32: G = cpb/8 lanes, the
// block maxima are reduced with shuffles).  The four runs of 4 chunks are
// conflict-free under dsw() for every n and s (checked by simulation).
__device__ __forceinline__ unsigned run4_addr(unsigned rb, int e) {  // e: multiple of 8
    return rb + 16u * (unsigned)dsw(e >> 1);
}
__device__ __forceinline__ void publish4(const float2 (&x)[32], unsigned rb, int ebase, int P, int h) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const unsigned a = run4_addr(rb, ebase + P + k * h);
#pragma unroll
        for (int c = 0; c < 4; ++c) sts128(a ^ (16u * c), x[8 * k + 2 * c], x[8 * k + 2 * c + 1]);
    }
}
__device__ __forceinline__ void publish2(const float2 (&x)[32], unsigned rb, int ebase, int U, int V) {
    const Run ru = mkrun(rb, ebase + U), rv = mkrun(rb, ebase + V);
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        sts128(radr(ru, k), x[2 * k], x[2 * k + 1]);
        sts128(radr(rv, k), x[16 + 2 * k], x[17 + 2 * k]);
    }
}

// Transposed publish for the TMA store (n = 256 / 512): after the last pair of
// stages x[8k + i] is element 8 tl + (n/4) k + i of line lj; it goes to row
// r = 8T k + T i + tl, column lj of the box [k][i][tl][LPC] (see make_out_map),
// rows of RB = 8 LPC bytes under the TMA swizzle of that row size (16-byte
// chunk index XOR row bits: (r & 7) for 128-byte rows, (r >> 1) & 3 for
// 64-byte rows -- both depend on tl only).  T RB = 1024 for both sizes.
template <int LT>
__device__ __forceinline__ void publish_t(const float2 (&x)[32], unsigned buf, int lj, int tl) {
    constexpr int T = 1 << LT, LPC = 128 >> LT;
    constexpr int RB = LPC >= 16 ? 128 : 8 * LPC;  // bytes per box row
    constexpr int HV = LPC > 16 ? LPC / 16 : 1;    // 128-byte halves per (k, i, tl) (n = 128: 2)
    static_assert(T * HV * RB == 1024, "n = 128 / 256 / 512 only");
    const int r = tl * HV + (lj >> 4) * (HV > 1);  // row within the (k, i) slab; bits above vanish mod 8 rows
    const unsigned sw = RB == 128 ? (unsigned)(r & 7) : (unsigned)((r >> 1) & 3);
    const unsigned base = buf + (((unsigned)(r * RB + (lj & 15) * 8)) ^ (sw << 4));
#pragma unroll
    for (int k = 0; k < 4; ++k)
#pragma unroll
        for (int i = 0; i < 8; ++i)
            asm volatile("st.shared.v2.f32 [%0], {%1, %2};" ::"r"(base + (unsigned)(k * 8192 + i * 1024)),
                         "f"(x[8 * k + i].x), "f"(x[8 * k + i].y)
                         : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void tma_store_4d(const void* map, unsigned smem, int c0, int c1, int c2, int c3) {
    asm volatile(
        "cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%2, %3, %4, %5}], [%1];\n\t"
        "cp.async.bulk.commit_group;" ::"l"(map),
        "r"(smem), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
        : "memory");
}
__device__ __forceinline__ void tma_store_5d(const void* map, unsigned smem, int c0, int c1, int c2, int c3, int c4) {
    asm volatile(
        "cp.async.bulk.tensor.5d.global.shared::cta.bulk_group [%0, {%2, %3, %4, %5, %6}], [%1];\n\t"
        "cp.async.bulk.commit_group;" ::"l"(map),
        "r"(smem), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4)
        : "memory");
}
__device__ __forceinline__ void tma_load_3d(unsigned smem, const void* map, int c0, int c1, int c2, unsigned mbar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem),
        "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(mbar)
        : "memory");
}
__device__ __forceinline__ void mbar_init(unsigned addr, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n\tfence.mbarrier_init.release.cluster;" ::"r"(addr), "r"(count)
                 : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned addr, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(addr), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned addr, unsigned parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "MBW_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra MBW_%=;\n\t}" ::"r"(addr),
        "r"(parity)
        : "memory");
}
// named CTA barriers, split phase: `count` threads in all, some arriving, some waiting
__device__ __forceinline__ void bar_arrive(int id, int count) {
    asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(count) : "memory");
}
__device__ __forceinline__ void bar_sync(int id, int count) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

template <int ID, int CPB, class BT>
__device__ __forceinline__ void pair_stage(float2 (&x)[32], int& P, int& H, const LCtx& L, unsigned rb, int ebase,
                                           int s, bool big, BT& bad) {
    constexpr int G = CPB / 8;  // lanes per MX block
    const int h = 1 << s;
    const int u0 = 8 * L.tl, j0 = u0 & (h - 1);
    P = ((u0 >> s) << (s + 2)) + j0;
    H = h;
    unsigned w0[8], w1[8], w2[8];
#if MXFFT_TW_FIRST
    // the twiddles do not depend on the exchange: their loads go out first
#pragma unroll
    for (int i = 0; i < 8; i += 4) {
        const uint4 q0 = lds128u(L.tw_sh + 4u * (unsigned)tws(h + j0 + i));
        const uint4 q1 = lds128u(L.tw_sh + 4u * (unsigned)tws(2 * h + j0 + i));
        const uint4 q2 = lds128u(L.tw_sh + 4u * (unsigned)tws(3 * h + j0 + i));
        w0[i] = q0.x, w0[i + 1] = q0.y, w0[i + 2] = q0.z, w0[i + 3] = q0.w;
        w1[i] = q1.x, w1[i + 1] = q1.y, w1[i + 2] = q1.z, w1[i + 3] = q1.w;
        w2[i] = q2.x, w2[i + 1] = q2.y, w2[i + 2] = q2.z, w2[i + 3] = q2.w;
    }
#endif
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const unsigned a = run4_addr(rb, ebase + P + k * h);
#pragma unroll
        for (int c = 0; c < 4; ++c) lds128(a ^ (16u * c), x[8 * k + 2 * c], x[8 * k + 2 * c + 1]);
    }
#if !MXFFT_TW_FIRST
#pragma unroll
    for (int i = 0; i < 8; i += 4) {
        const uint4 q0 = lds128u(L.tw_sh + 4u * (unsigned)tws(h + j0 + i));
        const uint4 q1 = lds128u(L.tw_sh + 4u * (unsigned)tws(2 * h + j0 + i));
        const uint4 q2 = lds128u(L.tw_sh + 4u * (unsigned)tws(3 * h + j0 + i));
        w0[i] = q0.x, w0[i + 1] = q0.y, w0[i + 2] = q0.z, w0[i + 3] = q0.w;
        w1[i] = q1.x, w1[i + 1] = q1.y, w1[i + 2] = q1.z, w1[i + 3] = q1.w;
        w2[i] = q2.x, w2[i + 1] = q2.y, w2[i + 2] = q2.z, w2[i + 3] = q2.w;
    }
#endif
    const int e0 = L.twe[h + j0], e1 = L.twe[2 * h + j0], e2 = L.twe[3 * h + j0];
    float2 a[8], b[8], c[8], d[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = x[i], b[i] = x[8 + i], c[i] = x[16 + i], d[i] = x[24 + i];
    // stage s
    mxb<ID, 8, G, false>(a, b, w0, e0, nullptr, 0, bad);
    mxb<ID, 8, G, false>(c, d, w0, e0, nullptr, 0, bad);
    // stage s + 1
    mxb<ID, 8, G, false>(a, c, w1, e1, nullptr, 0, bad);
    mxb<ID, 8, G, false>(b, d, w2, e2, nullptr, 0, bad);
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = a[i], x[8 + i] = b[i], x[16 + i] = c[i], x[24 + i] = d[i];
}

// All butterfly stages of one group.  Registers for stages < 5; stages >= 5
// exchange through the line's region (element e of the buffer at shared
// address rb lives in chunk dsw(e/2), half e&1).  On return x[0..15] sit at
// line positions U.., x[16..31] at V.. (H == 0), or -- after paired stages --
// x[8k..8k+7] at P + k H (H > 0).
struct NoPre {
    __device__ __forceinline__ void operator()() const {}
};
// PRE: called once, just before the group's first write to the exchange region rb
// (n-specialised kernels; the TMA kernel passes its "region is free" barrier)
template <int ID, int CPB, bool DBG, int LT, class PRE = NoPre, class BT = bool>
__device__ __forceinline__ void run_stages(float2 (&x)[32], int& U, int& V, int& P, int& H, const LCtx& L,
                                           unsigned rb, int ebase, LDbg* dbg, BT& bad, PRE pre = PRE()) {
    const int lt = LT >= 0 ? LT : L.lt;
    const bool big = lt > 5;  // a line spans several warps
    constexpr int LOCAL = MXFFT_LOCAL_STAGES;  // unrolled register stages (4 or 5)
    // n-specialised kernels always run every stage (stage-limited launches go to
    // the LT = -1 variant): unconditional register stages leave the compiler no
    // join points at which to shuffle the 32 values back into fixed registers
    constexpr bool FULL = LT >= 0 && !DBG;
    const int lim_loc = FULL ? LOCAL : (L.slim < LOCAL ? L.slim : LOCAL);
    if (lim_loc > 0) local_stage<ID, CPB, 0, DBG>(x, L.tw, L.twe, L.c, L.trivial, L.sigma, dbg, bad);
    if (lim_loc > 1) local_stage<ID, CPB, 1, DBG>(x, L.tw, L.twe, L.c, L.trivial, L.sigma, dbg, bad);
    if (lim_loc > 2) local_stage<ID, CPB, 2, DBG>(x, L.tw, L.twe, L.c, false, L.sigma, dbg, bad);
    if (lim_loc > 3) local_stage<ID, CPB, 3, DBG>(x, L.tw, L.twe, L.c, false, L.sigma, dbg, bad);
    if constexpr (LOCAL > 4)
        if (lim_loc > 4) local_stage<ID, CPB, 4, DBG>(x, L.tw, L.twe, L.c, false, L.sigma, dbg, bad);
    U = 32 * L.c;
    V = U + 16;
    H = 0;
    P = 0;
    // kept rolled: one copy of the stage body keeps the kernel inside the
    // instruction cache (unrolling measured slower)
    const int last = FULL ? lt + 5 : (L.slim < lt + 5 ? L.slim : lt + 5);
#if MXFFT_PAIR_STAGES
    if constexpr (FULL && LOCAL == 5 && LT >= 2) {
        // an odd stage out first (single), then pairs of stages per exchange
        int s = 5;
        pre();
        if (LT & 1) {
            smem_stage<ID, CPB, DBG>(x, U, V, L, rb, ebase, 5, LT > 5, dbg, bad);
            s = 6;
        }
        publish2(x, rb, ebase, U, V);
        lsync(LT > 5);
        pair_stage<ID, CPB>(x, P, H, L, rb, ebase, s, LT > 5, bad);
        if constexpr (LT <= MXFFT_UNROLL_PAIRS) {
#pragma unroll
            for (int s2 = (LT & 1) ? 8 : 7; s2 < LT + 5; s2 += 2) {
                publish4(x, rb, ebase, P, H);
                lsync(LT > 5);
                pair_stage<ID, CPB>(x, P, H, L, rb, ebase, s2, LT > 5, bad);
            }
            return;
        }
#pragma unroll 1
        for (s += 2; s < LT + 5; s += 2) {
            publish4(x, rb, ebase, P, H);
            // the exchange before stages (s, s + 1) stays inside a 2^(s+2)-position chunk, i.e. the
            // 2^(s-3) consecutive threads that own it after the first exchange: one warp for s <= 8
            lsync(LT > 5 && (s > 8 || !MXFFT_WARP_LOCAL_EXCHANGE));
            pair_stage<ID, CPB>(x, P, H, L, rb, ebase, s, LT > 5, bad);
        }
        return;
    }
#endif
#if MXFFT_UNROLL_SMEM
    if constexpr (LT >= 0 && !DBG) {
#pragma unroll
        for (int s = LOCAL; s < LT + 5; ++s)
            if (s < last) smem_stage<ID, CPB, DBG>(x, U, V, L, rb, ebase, s, LT > 5, dbg, bad);
        return;
    }
#endif
#pragma unroll 1
    for (int s = LOCAL; s < last; ++s) smem_stage<ID, CPB, DBG>(x, U, V, L, rb, ebase, s, big, dbg, bad);
}

__device__ __forceinline__ void cp_async16(unsigned dst, const void* src, bool valid) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(valid ? 16 : 0)
                 : "memory");
}
__device__ __forceinline__ void cp_async8(unsigned dst, const void* src, bool valid) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(dst), "l"(src), "r"(valid ? 8 : 0)
                 : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// shared address of the element with swizzled chunk `sch` and half `h`
__device__ __forceinline__ unsigned caddr(unsigned buf, int sch, int h) {
    return buf + 16u * (unsigned)sch + 8u * (unsigned)h;
}

template <int ID, int CPB, bool DBG>
__device__ __forceinline__ void load_twiddles(unsigned* tw, signed char* twe, const MxLinesArgs& a, int n) {
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        tw[tws(i)] = a.tw16[i];
        twe[i] = a.twe[i];
    }
}

template <bool DBG>
__device__ __forceinline__ void init_dbg(LDbg& dbg, const MxLinesArgs& a, int n, int cpb) {
    if (DBG) {
        dbg.vexp = a.d_vexp;
        dbg.vcodes = a.d_vcodes;
        dbg.pexp = a.d_pexp;
        dbg.pshift = a.d_pshift;
        dbg.pcodes = a.d_pcodes;
        dbg.rows = a.total_lines;
        dbg.m = n / 2;
        dbg.cpb = cpb;
    }
}

// Exact replay of `nlines` lines (gl0, gl0 + 1, ...) whose regions start at
// tile elements e0(j): reload each line from HBM into its region and run the
// reference-literal stages (mxfft_generic.cuh) with all threads of the CTA.
// Taken when any block of the group left the fast exponent range (or a
// prescale exponent is not a normal-float power of two); the fast path's
// results for the group are discarded.  The group's input is still intact:
// its stores happen after this point.
static __device__ __noinline__ void replay_lines(const MxLinesArgs& a, int64_t gl0, int nlines, char* tile,
                                                 int lpr_shift, int region, int lpr_mask) {
    const int n = a.n, m = n / 2, tid = threadIdx.x, nthr = blockDim.x;
    for (int j = 0; j < nlines; ++j) {
        const int64_t gl = gl0 + j;
        if (gl >= a.total_lines) break;
        const int e0 = (j >> lpr_shift) * region + (j & lpr_mask) * n;
        auto acc = [tile, e0](int i) {
            const int e = e0 + i;
            return reinterpret_cast<float2*>(tile + 16 * dsw(e >> 1) + 8 * (e & 1));
        };
        int64_t base, es;
        if (a.col_mode) {
            base = (gl >> a.log2n) * (int64_t)n * n + (gl & (n - 1));
            es = n;
        } else {
            base = gl * n;
            es = 1;
        }
        const bool seg = !a.col_mode && a.seg_log2;
        if (!a.col_mode && a.dec) {
            base = (gl >> 1) * (2 * (int64_t)n) + (gl & 1);
            es = 2;
        }
        const int64_t img = gl / a.lines_per_image;
        const int kk = a.kvec ? a.kvec[img / a.k_group] : 0;
        const int kin = a.kin_sign * kk + a.kin_const, kout = a.kout_sign * kk + a.kout_const;
        __syncthreads();
        for (int i = tid; i < n; i += nthr) {
            const int r = (int)(__brev((unsigned)i) >> (32 - a.log2n));
            *acc(i) = gscale(a.in[seg ? seg_off(a, gl, r) : base + (int64_t)r * es], kin);
        }
        __syncthreads();
        const int last = a.stage_limit < a.log2n ? a.stage_limit : a.log2n;
        for (int s = 0; s < last; ++s) {
            generic_stage(acc, s, m, a.cpb, a.fmt, a.wcr, a.wci, a.wsexp, a.inverse != 0, tid, nthr);
            __syncthreads();
        }
        for (int i = tid; i < n; i += nthr) *acc(i) = gscale(*acc(i), kout);
    }
    __syncthreads();
}

// Lines of n <= 4096 (T <= 128 threads per line; 128-thread CTAs): a software
// pipeline per CTA.  While group g computes, group g+1's tile streams into the
// other shared buffer with cp.async (16-byte chunks of contiguous rows, or
// whole row segments of adjacent columns).  Stores leave through the same
// buffer so that HBM sees whole lines: 16-byte chunks of contiguous rows, or
// -- for columns and for rows stored transposed -- LPC adjacent elements of
// each output row.
template <int ID, int CPB, bool DBG, int LT>
__device__ __forceinline__ void lines_body_pipe(const MxLinesArgs& a) {
    constexpr int NT = 128, GEL = NT * 32;  // threads, complex per group tile
    const int lt = LT >= 0 ? LT : a.log2T;
    const int T = 1 << lt, N = 32 * T, LN = lt + 5;
    const int W = T > 32 ? T : 32;         // threads sharing one region
    const int LPC = NT >> lt, LLPC = 7 - lt;  // lines per group
    const int LPR = W >> lt;                  // lines per region
    extern __shared__ float4 smem4[];
    unsigned* tw = reinterpret_cast<unsigned*>(smem4);
    signed char* twe = reinterpret_cast<signed char*>(tw + N);
    const int tid = threadIdx.x;
    pdl_launch_dependents();
    load_twiddles<ID, CPB, DBG>(tw, twe, a, N);
    pdl_wait();  // the plan tables are static; everything below may depend on the kernel before
    LCtx L;
    L.tw = tw;
    L.twe = twe;
    L.tw_sh = (unsigned)__cvta_generic_to_shared(tw);
    L.lt = lt;
    L.tl = tid & (T - 1);
    L.c = L.tl;
    L.trivial = a.trivial01;
    L.sigma = a.inverse ? -1.f : 1.f;
    L.slim = a.stage_limit;
    const int rcol = lt ? (int)(__brev((unsigned)L.c) >> (32 - lt)) : 0;
    const unsigned buf0 = (unsigned)__cvta_generic_to_shared(smem4 + a.tw_chunks);
    char* const tile_g = reinterpret_cast<char*>(smem4 + a.tw_chunks);  // generic view (replay)
    constexpr unsigned BUFSZ = (unsigned)GEL * 8u;
    if (buf0 & 127u) __trap();  // radr() ORs chunk offsets into 128-byte-aligned run bases
    // n = 64 .. 512: the host places both tile buffers on 4 KB boundaries, so a
    // swizzled address (thread base) ^ (constant chunk offset < 256 chunks) is one
    // LOP3 instead of an XOR plus an add
    constexpr bool AX = LT >= 1 && LT <= 4;
    if (AX && (buf0 & 4095u)) __trap();
    // this thread's line inside the buffer (tile element belem(j, q) = line j, position q)
    auto belem = [&](int j, int q) { return (j >> (lt > 5 ? 0 : 5 - lt)) * (W * 32) + (j & (LPR - 1)) * N + q; };
    // the line this thread computes.  n = 256: the two line bits within a warp
    // are swapped so that each half-warp's 64-bit gather loads (two lines)
    // cover all 32 banks (2 wavefronts instead of 4, by simulation and ncu); the
    // 128-bit exchange accesses are one line per quarter-warp either way
    const int lj = (LT == 3) ? (((tid >> 3) & ~3) | (((tid >> 3) & 1) << 1) | (((tid >> 4) & 1))) : (tid >> lt);
    const int ebase = belem(lj, 0);
    // gather: element ebase + m T + rcol -> chunk dsw(ebase/2) ^ dsw(rcol/2) ^ dsw(m T/2)
    const int gch = dsw(ebase >> 1) ^ dsw(rcol >> 1);
    const int gh = rcol & 1;
    // strided (column / transposed) access: line tj of the group, positions tq0 + T k
    const int tj = tid & (LPC - 1), tq0 = tid >> LLPC;
    const int te0 = belem(tj, tq0);
    const int tch = dsw(te0 >> 1);
    const int th = te0 & 1;
#if MXFFT_PAIR_STORE
    // paired strided stores: lines 2 pa, 2 pa + 1 of the group, positions pq0 + 2 T k
    // n <= 256: pa bits 0-2 <- tid bits 0-2, pq0 bit 0 <- tid bit 3, then the
    // remaining pa bits, then pq0: every half-warp reads two positions (both
    // halves of the 16-byte chunks), so its 64-bit reads hit 32 distinct banks
    // (tools/sim_copyout_banks.py); a warp still writes whole 128-byte row segments
    const int phb = 3 - lt > 0 ? 3 - lt : 0;  // pa bits above bit 2 (n <= 256)
    // n = 512 (4 pairs): pa <- tid bits 4-5, pq0 <- tid bits 0-3, 6 (simulated
    // conflict-free; a warp writes 32-byte row segments of 16 rows)
    const int pa = LT >= 0 && LT <= 3 ? ((tid & 7) | (((tid >> 4) & ((1 << phb) - 1)) << 3))
                   : LT == 4          ? ((tid >> 4) & 3)
                                      : tid & ((LPC >> 1) - 1);
    const int pq0 = LT >= 0 && LT <= 3 ? (((tid >> 3) & 1) | ((tid >> (4 + phb)) << 1))
                    : LT == 4          ? ((tid & 15) | ((tid >> 6) << 4))
                                       : tid >> (LLPC > 0 ? LLPC - 1 : 0);
    const int pe0 = belem(2 * pa, pq0), pe1 = belem(2 * pa + 1, pq0);
    const int pch0 = dsw(pe0 >> 1), ph0 = pe0 & 1, pch1 = dsw(pe1 >> 1), ph1 = pe1 & 1;
#endif
    // contiguous access: chunk tid + NT k
    const int rch = dsw(tid);
    const bool strided_out = a.col_mode || a.tstore;
    const int64_t ngroups = (a.total_lines + LPC - 1) / LPC;
    LDbg dbg;
    init_dbg<DBG>(dbg, a, N, CPB);

    // column-mode loads (mxfft_fft_cols / fft2 without workspace) only in the
    // run-time-n variant: the specialised kernels stay small
    const bool col_in = LT < 0 && a.col_mode;
    auto issue_tile = [&](int64_t grp_, unsigned buf) {
        if (a.prof_flags & 1) return;
        const int64_t grp = a.reverse ? ngroups - 1 - grp_ : grp_;
        if (LT < 0 && a.seg_log2) {  // segmented rows (run-time-n variant only): per-chunk addresses
            const int64_t l0 = grp * LPC;
#pragma unroll 4
            for (int k = 0; k < 16; ++k) {
                const int e = 2 * (tid + NT * k);
                const int64_t line = l0 + (e >> (lt + 5));
                const bool ok = line < a.total_lines;
                cp_async16(caddr(buf, rch ^ dsw(NT * k), 0),
                           ok ? (const void*)(a.in + seg_off(a, line, e & (N - 1))) : (const void*)a.in, ok);
            }
        } else if (!col_in) {
            const int64_t base = grp * LPC * (int64_t)N;
            const float4* src = reinterpret_cast<const float4*>(a.in + base) + tid;
            const int64_t lim = (a.total_lines * (int64_t)N - base) / 2;  // chunks left
            if (lim >= NT * 16) {  // whole tile: no per-chunk bounds checks
#pragma unroll
                for (int k = 0; k < 16; ++k) cp_async16(caddr(buf, rch ^ dsw(NT * k), 0), src + NT * k, true);
            } else {
#pragma unroll
                for (int k = 0; k < 16; ++k) {
                    const bool ok = tid + NT * k < lim;
                    cp_async16(caddr(buf, rch ^ dsw(NT * k), 0), ok ? (const void*)(src + NT * k) : (const void*)a.in,
                               ok);
                }
            }
        } else {
            const int64_t gl = grp * LPC + tj;
            const bool ok = gl < a.total_lines;
            const int64_t img = gl >> LN;
            const float2* src = a.in + (ok ? img * (int64_t)N * N + (int64_t)tq0 * N + (gl & (N - 1)) : 0);
#pragma unroll 8
            for (int k = 0; k < 32; ++k)
                cp_async8(caddr(buf, tch ^ dsw((T * k) >> 1), th ^ ((T * k) & 1)),
                          ok ? src + (int64_t)k * T * N : src, ok);
        }
    };

    auto body = [&](const int64_t grp, const unsigned bcur, const int kk) {
        const int64_t line = grp * LPC + lj;
        const int kin = a.kin_const + a.kin_sign * kk, kout = a.kout_const + a.kout_sign * kk;
        if (DBG) dbg.row = line;

        // bit-reversed gather (fftcore.py:262): x[rev5(m)] <- line element m*T + rev_T(c)
        float2 x[32];
        bool bad = false;
#pragma unroll
        for (int m = 0; m < 32; ++m)
            x[rev_c<5>(m)] = AX ? lds64(caddr(bcur, gch, gh) ^ (16u * (unsigned)dsw((m * T) >> 1)))
                                : lds64(caddr(bcur, gch ^ dsw((m * T) >> 1), lt ? gh : (m & 1)));
        if (a.prof_flags & 1) {  // profiling without loads: synthetic in-range data
#pragma unroll
            for (int m = 0; m < 32; ++m)
                x[m] = make_float2((float)((tid * 37 + m * 11) & 255) * 0.01f, (float)((tid * 13 + m * 7) & 127) * 0.01f);
        }
        if (kin) scale32<DBG>(x, kin, bad);

        int U, V, P, H;
        run_stages<ID, CPB, DBG, LT>(x, U, V, P, H, L, bcur, ebase, &dbg, bad);

        // publish (undo_prescale / 1/n^2 fused), then coalesced stores
        if (kout) scale32<DBG>(x, kout, bad);
        if (!DBG && __syncthreads_or(bad)) {
            replay_lines(a, grp * LPC, LPC, tile_g + (bcur - buf0), lt > 5 ? 0 : 5 - lt, W * 32, LPR - 1);
        } else if (H > 0) {
            publish4(x, bcur, ebase, P, H);
        } else {
            publish2(x, bcur, ebase, U, V);
        }
        __syncthreads();
        if (a.prof_flags & 2) {
        } else if (!strided_out) {
            const int64_t base = grp * LPC * (int64_t)N;
            float4* dst = reinterpret_cast<float4*>(a.out + base) + tid;
            const int64_t lim = (a.total_lines * (int64_t)N - base) / 2;
#pragma unroll
            for (int k = 0; k < 16; ++k) {
                if (tid + NT * k < lim) {
                    float2 p0, p1;
                    lds128(caddr(bcur, rch ^ dsw(NT * k), 0), p0, p1);
                    stg128(dst + NT * k, make_float4(p0.x, p0.y, p1.x, p1.y));
                }
            }
#if MXFFT_PAIR_STORE
        } else if (LT >= 0 && LT <= MXFFT_PAIR_STORE_MAXLT && (grp + 1) * LPC <= a.total_lines) {
            // two adjacent output columns per thread: one 16-byte store per position
            const int64_t gl = grp * LPC + 2 * pa;
            const int64_t img = gl >> LN;
            float4* dst = reinterpret_cast<float4*>(a.out + img * (int64_t)N * N + (int64_t)pq0 * N + (gl & (N - 1)));
            const int64_t rs = (int64_t)T * N;  // 2 T rows, in float4 units
            // shared-memory reads in batches of PB positions ahead of their stores,
            // so that no store waits on the load just before it
            constexpr int PB = MXFFT_PAIR_BATCH;
#pragma unroll
            for (int k0 = 0; k0 < 16; k0 += PB) {
                float4 o[PB];
#pragma unroll
                for (int k = 0; k < PB; ++k) {
                    const unsigned c16 = 16u * (unsigned)dsw(T * (k0 + k));
                    const float2 v0 = AX ? lds64(caddr(bcur, pch0, ph0) ^ c16) : lds64(caddr(bcur, pch0 ^ dsw(T * (k0 + k)), ph0));
                    const float2 v1 = AX ? lds64(caddr(bcur, pch1, ph1) ^ c16) : lds64(caddr(bcur, pch1 ^ dsw(T * (k0 + k)), ph1));
                    o[k] = make_float4(v0.x, v0.y, v1.x, v1.y);
                }
#pragma unroll
                for (int k = 0; k < PB; ++k) stg128(dst + (k0 + k) * rs, o[k]);
            }
#endif
        } else {  // columns, or rows stored transposed: line gl -> column (gl mod n) of image gl/n
            const int64_t gl = grp * LPC + tj;
            if (gl < a.total_lines) {
                const int64_t img = gl >> LN;
                float2* dst = a.out + img * (int64_t)N * N + (int64_t)tq0 * N + (gl & (N - 1));
#if MXFFT_BATCH_STORE
                // all shared-memory reads first: each store then finds its data ready
                float2 o[32];
#pragma unroll
                for (int k = 0; k < 32; ++k) o[k] = lds64(caddr(bcur, tch ^ dsw((T * k) >> 1), th ^ ((T * k) & 1)));
#pragma unroll
                for (int k = 0; k < 32; ++k) stg64(dst + (int64_t)k * T * N, o[k]);
#else
#pragma unroll
                for (int k = 0; k < 32; ++k)
                    stg64(dst + (int64_t)k * T * N, lds64(caddr(bcur, tch ^ dsw((T * k) >> 1), th ^ ((T * k) & 1))));
#endif
            }
        }
    };
    // iteration "grp - gridDim.x" only issues the first tile (one issue site)
    int cur = 1;
    int kk_nxt = 0;  // kvec entry of this thread's line in the next group, loaded a group ahead
    for (int64_t grp_it = (int64_t)blockIdx.x - gridDim.x; grp_it < ngroups; grp_it += gridDim.x) {
        const int64_t nxt = grp_it + gridDim.x;
        const unsigned bcur = buf0 + (unsigned)cur * BUFSZ, bnxt = buf0 + (unsigned)(cur ^ 1) * BUFSZ;
        cur ^= 1;
        __syncthreads();  // the other buffer's previous readers are done
        if (nxt < ngroups) issue_tile(nxt, bnxt);
        cp_commit();
#if MXFFT_KPREF
        const int kk = kk_nxt;
        if (a.kvec && nxt < ngroups) {
            const int64_t nl = (a.reverse ? ngroups - 1 - nxt : nxt) * LPC + lj;
            kk_nxt = nl < a.total_lines ? __ldg(a.kvec + k_index(a, nl)) : 0;
        }
#endif
        if (grp_it < 0) continue;
        const int64_t grp = a.reverse ? ngroups - 1 - grp_it : grp_it;
        cp_wait<1>();     // this thread's copies of group grp have landed
        __syncthreads();  // ... and everybody's
#if !MXFFT_KPREF
        const int64_t l0 = grp * LPC + lj;
        const int kk = a.kvec && l0 < a.total_lines ? a.kvec[k_index(a, l0)] : 0;
#endif
        body(grp, bcur, kk);
    }
    cp_wait<0>();
}

// ---------------------------------------------------------------------------
// Evidence for compute_prescale gathered by a first pass on the unscaled input
// (mxfft_pipeline_folded; see lines_body_tma below for the word formats).
// `grp` is the CTA's group (TMA kernel) or line (one-line-per-CTA kernel): its
// threads each hold 32 points, so thread words sit at grp * blockDim + tid and
// warp words at 2 (grp * warps + warp).
// ---------------------------------------------------------------------------
template <int NT>
__device__ __forceinline__ void fold_points(const float2 (&x)[32], const MxLinesArgs& a, int64_t grp) {
    const int tid = threadIdx.x;
    constexpr int nt = NT;
    unsigned acc_key = 0, mn_all = 0xffffffffu;
#pragma unroll
    for (int m = 0; m < 32; ++m) {
        const float re = x[m].x, im = x[m].y;
        acc_key = max(acc_key, __float_as_uint(fmaf(re, re, im * im)));  // NaN / inf compare largest
        mn_all = min(mn_all, __float_as_uint(fmaxf(fabsf(re), fabsf(im))));
    }
    unsigned zeros = 0, nzb = mn_all;
    if (__builtin_expect(mn_all == 0u, 0)) {  // the thread holds zero points: count them, skip them
        unsigned acc_min = 0xffffffffu;
#pragma unroll
        for (int m = 0; m < 32; ++m) {
            const unsigned ub = __float_as_uint(fmaxf(fabsf(x[m].x), fabsf(x[m].y)));
            zeros += ub == 0u;
            acc_min = min(acc_min, ub - 1u);  // zero -> 2^32 - 1
        }
        nzb = acc_min + 1u;  // 0: every point is zero
    }
    a.minw[grp * nt + tid] = (nzb ? (nzb & ~63u) : 0xffffffc0u) | zeros;
    acc_key = __reduce_max_sync(0xffffffffu, acc_key);
    if ((tid & 31) == 0) a.acc[(grp * (nt >> 5) + (tid >> 5)) * 2] = acc_key;
}
template <int NT>
__device__ __forceinline__ void fold_range(const BadTrack& bad, const MxLinesArgs& a, int64_t grp) {
    const int tid = threadIdx.x;
    constexpr int nt = NT;
    const int hi_ = __reduce_max_sync(0xffffffffu, bad.hi), lo_ = __reduce_min_sync(0xffffffffu, bad.lo);
    const unsigned b_ = __ballot_sync(0xffffffffu, bad.b);
    if ((tid & 31) == 0)
        a.acc[(grp * (nt >> 5) + (tid >> 5)) * 2 + 1] =
            ((unsigned)(128 + hi_) << 16) | ((unsigned)(128 - lo_) << 4) | (b_ ? 1u : 0u);
}

// ---------------------------------------------------------------------------
// n = 256 / 512 row passes stored transposed (the two passes of mxfft_fft2):
// the group leaves with ONE TMA tensor store (make_out_map, mxfft_lines.cu).
// Two 32 KB buffers with fixed roles: X receives the group tiles (cp.async,
// the next group's tile is issued as soon as this group is in registers), Y is
// the exchange region of the shared-memory stages and then holds the group in
// output order ([k][i][tl][LPC] rows under the TMA swizzle, publish_t) for the
// store.  Thread 0 waits for the previous store's reads of Y after the
// gather, so that latency hides behind the gather instead of sitting at the
// top of the group.  A group with a block outside the fast exponent range is
// replayed exactly into Y and written by a plain loop.
// ---------------------------------------------------------------------------
//
// ACC (the first pass of mxfft_pipeline_folded): the pass runs on the UNSCALED
// input and leaves, without atomics,
//  * per warp and group two words in a.acc (group g, warp w at 2 (4 g + w)):
//    the largest FP32 key re^2 + im^2 of the warp's points (bit pattern;
//    >= 0x7f800000: non-finite or overflow), and (128 + hi) << 16 |
//    (128 - lo) << 4 | replayed, [lo, hi] the range of the v-block exponents
//    of every stage;
//  * per thread and group one word in a.minw (group g, thread t at 128 g + t):
//    the bit pattern of the smallest nonzero max(|re|, |im|) of the thread's
//    32 points with its low 6 bits replaced by the thread's count of zero
//    points (0xffffffc0 | 32: all zero).
// k_fold_resolve (mxfft_prescale_fast.cu) turns them into k or sends the stack
// to the standard path.
template <int ID, int CPB, int LT, bool ACC = false>
__device__ __forceinline__ void lines_body_tma(const MxLinesArgs& a) {
    static_assert(LT >= 2 && LT <= 4, "n = 128 / 256 / 512");
    constexpr int NT = 128, GEL = NT * 32, T = 1 << LT, N = 32 * T, LN = LT + 5;
    constexpr int W = 32, LPC = NT >> LT, LPR = W >> LT;
    extern __shared__ float4 smem4[];
    unsigned* tw = reinterpret_cast<unsigned*>(smem4);
    signed char* twe = reinterpret_cast<signed char*>(tw + N);
    const int tid = threadIdx.x;
    pdl_launch_dependents();
    load_twiddles<ID, CPB, false>(tw, twe, a, N);
    pdl_wait();  // the plan tables are static; everything below may depend on the kernel before
    LCtx L;
    L.tw = tw;
    L.twe = twe;
    L.tw_sh = (unsigned)__cvta_generic_to_shared(tw);
    L.lt = LT;
    // Thread -> (line lj of the group, thread tl of the line): a line's T threads are consecutive
    // lanes of one warp (warp-level exchanges), ordered so that every half-warp of the 64-bit
    // gather from X (chunk index XOR line & 7) and of the 64-bit stores of publish_t touches 16
    // distinct 8-byte bank pairs (ncu: no excess shared-memory wavefronts).
    //  n = 128: warp w takes lines 8 w + {0, 3, 5, 6 | 1, 2, 4, 7} (even / odd parity): a half-warp's
    //           four lines have distinct l >> 1 (gather) and no pair (l, l ^ 4) (publish);
    //  n = 256: warp w takes lines b + {0, 5 | 1, 4}, b = 2 (w & 1) + 8 (w >> 1): a half-warp's two
    //           lines differ in bit 2 (gather) and in bit 0 (publish);
    //  n = 512: warp w takes lines 2 w, 2 w + 1; a half-warp is threads 0-7 of one line and 8-15 of
    //           the other (even / odd rcol = the two halves of a 16-byte chunk in both patterns).
    const int lane = tid & 31, wj = (lane >> 3) & 3, g3 = (lane >> 2) & 3;
    const int lj = LT == 2   ? (8 * (tid >> 5) + 2 * g3 + ((__popc(g3) & 1) ^ (lane >> 4)))
                   : LT == 3 ? (2 * ((tid >> 5) & 1) + 8 * (tid >> 6) + 4 * (wj & 1) + ((wj & 1) ^ (wj >> 1)))
                             : (2 * (tid >> 5) + (wj & 1));
    L.tl = LT == 4 ? ((lane & 7) + 8 * ((wj & 1) ^ (lane >> 4))) : (tid & (T - 1));
    L.c = L.tl;
    L.trivial = a.trivial01;
    L.sigma = a.inverse ? -1.f : 1.f;
    L.slim = a.stage_limit;
    const int rcol = (int)(__brev((unsigned)L.c) >> (32 - LT));
    constexpr unsigned BUFSZ = (unsigned)GEL * 8u;
    const unsigned bx = (unsigned)__cvta_generic_to_shared(smem4 + a.tw_chunks), by = bx + BUFSZ;
    char* const y_g = reinterpret_cast<char*>(smem4 + a.tw_chunks) + BUFSZ;  // generic view of Y (replay)
    if (bx & 4095u) __trap();  // swizzled addresses are formed with XOR / OR on 4 KB-aligned buffers
    // the tile's mbarrier sits in the padding behind the twiddle tables (5 n bytes used of tw_chunks * 16)
    const unsigned mbar = (unsigned)__cvta_generic_to_shared(twe + N);
    if (tid == 0) mbar_init(mbar, 1);
    auto belem = [&](int j, int q) { return (j >> (5 - LT)) * (W * 32) + (j & (LPR - 1)) * N + q; };
    // the line's slot in Y (the exchange region): natural thread order for n <= 256, the layout
    // the swizzled exchange patterns were derived for (two lines per quarter-warp at n = 128);
    // n = 512: the line itself (its threads are two separate runs of 8 lanes)
    const int ebase = belem(LT == 4 ? lj : tid >> LT, 0);
    // X holds [segment q / 16][line][16 elements] with the 16-byte chunk index XOR (line & 7):
    // element m T + rcol -> segment (m T) / 16, chunk ((m T mod 16) + rcol) / 2 ^ (line & 7)
    const unsigned gaddr = bx + (unsigned)lj * 128u + ((unsigned)((rcol >> 1) ^ (lj & 7)) << 4) + 8u * (rcol & 1);
    const int64_t ngroups = a.total_lines / LPC;  // whole groups (total_lines is a multiple of n)
    LDbg dbg;

    auto issue_tile = [&](int64_t grp_) {  // thread 0 only
        const int64_t grp = a.reverse ? ngroups - 1 - grp_ : grp_;
        mbar_expect_tx(mbar, BUFSZ);
        tma_load_3d(bx, &a.in_map, 0, (int)(grp * LPC), 0, mbar);
    };
    auto k_of = [&](int64_t grp_) {
        const int64_t nl = (a.reverse ? ngroups - 1 - grp_ : grp_) * LPC + lj;
        return a.kvec ? __ldg(a.kvec + k_index(a, nl)) : 0;
    };

    int64_t grp_it = blockIdx.x;
    int kk_nxt = 0;
    unsigned phase = 0;
    __syncthreads();  // the mbarrier is initialised (and the twiddles are in place)
    if (grp_it < ngroups) {
        if (tid == 0) issue_tile(grp_it);
        kk_nxt = k_of(grp_it);
    }
    for (; grp_it < ngroups; grp_it += gridDim.x) {
        const int64_t nxt = grp_it + gridDim.x;
        const int64_t grp = a.reverse ? ngroups - 1 - grp_it : grp_it;
        const int kk = kk_nxt;
        mbar_wait(mbar, phase);  // the tile is in X
        phase ^= 1u;
        float2 x[32];
        typename std::conditional<ACC, BadTrack, bool>::type bad{};
#pragma unroll
        for (int m = 0; m < 32; ++m) {
            constexpr int MS = 16 / T;  // values of m per 128-byte segment (chunk step T / 2)
            const unsigned ad = (gaddr ^ ((unsigned)(m & (MS - 1)) * (T * 8u))) + (unsigned)(m / MS) * (LPC * 128u);
            x[rev_c<5>(m)] = lds64(ad);
        }
        if constexpr (ACC) fold_points<NT>(x, a, grp);
        if (nxt < ngroups) kk_nxt = k_of(nxt);
        // n <= 256: split barriers instead of one __syncthreads.  Only warp 0 waits for every
        // warp's gather (barrier 1: X is in registers, free for the next tile) before thread 0
        // issues the next load; the others just arrive and go on to the register stages.  Warp 0
        // then arrives on barrier 2 (thread 0 has seen the previous group's store finish reading
        // Y), which the other warps pass just before their first write to Y, five stages later.
        // (Measured: C4 pass 192.3 -> 188.8 us, C2 62.7 -> 62.1; n = 512 71.8 -> 72.3, so it keeps
        // the plain barrier.)
        constexpr bool SPLIT = LT <= 3;
        if (!SPLIT) {
            if (tid == 0) bulk_wait_read0();  // the previous group's store has read Y
            __syncthreads();                  // X is in registers: free for the next tile; Y is free
            if (tid == 0 && nxt < ngroups) issue_tile(nxt);
        } else if (tid < 32) {
            if (tid == 0) bulk_wait_read0();
            __syncwarp();
            bar_sync(1, NT);
            if (tid == 0 && nxt < ngroups) issue_tile(nxt);
            bar_arrive(2, NT);
        } else {
            bar_arrive(1, NT);
        }
        const int kin = a.kin_const + a.kin_sign * kk, kout = a.kout_const + a.kout_sign * kk;
        if (kin) scale32<false>(x, kin, bad);
        int U, V, P, H;
        auto y_free = [tid]() {
            if (SPLIT && tid >= 32) bar_sync(2, NT);
        };
        run_stages<ID, CPB, false, LT>(x, U, V, P, H, L, by, ebase, &dbg, bad, y_free);
        if (kout) scale32<false>(x, kout, bad);
        const int64_t gl = grp * LPC;  // first line of the group: column gl mod n of image gl / n
        if constexpr (ACC) fold_range<NT>(bad, a, grp);
        if (__syncthreads_or(bad)) {
            replay_lines(a, gl, LPC, y_g, 5 - LT, W * 32, LPR - 1);
            float2* dst = a.out + (gl >> LN) * (int64_t)N * N + (gl & (N - 1));
            for (int e = tid; e < GEL; e += NT) {
                const int el = belem(e & (LPC - 1), e >> (7 - LT));
                dst[(int64_t)(e >> (7 - LT)) * N + (e & (LPC - 1))] =
                    *reinterpret_cast<const float2*>(y_g + 16 * dsw(el >> 1) + 8 * (el & 1));
            }
            continue;  // (the next group's barrier orders these reads before any write to Y)
        }
        publish_t<LT>(x, by, lj, L.tl);
        fence_proxy_async();
        __syncthreads();
        if (tid == 0) {
            if constexpr (LPC > 16) tma_store_5d(&a.out_map, by, 0, (int)(gl & (N - 1)) >> 4, 0, 0, (int)(gl >> LN) * 4);
            else tma_store_4d(&a.out_map, by, (int)(gl & (N - 1)), 0, 0, (int)(gl >> LN) * 4);
        }
    }
    if (tid == 0) bulk_wait0();
}

template <int ID, int CPB, int LT, bool ACC = false>
__global__ void __launch_bounds__(128, MXFFT_LINES_MINB) k_mx_lines_tma(const __grid_constant__ MxLinesArgs a) {
    lines_body_tma<ID, CPB, LT, ACC>(a);
}

// Lines of n = 8192/16384 (T = 256/512; one line per CTA): direct loads from
// HBM (whole sectors per warp), no prefetch (a second 128 KB buffer would not
// fit next to the twiddle table).
template <int ID, int CPB, bool DBG, int LT, bool ACC = false>
__device__ __forceinline__ void lines_body_direct(const MxLinesArgs& a) {
    const int lt = LT >= 0 ? LT : a.log2T;
    const int T = 1 << lt, N = 32 * T;
    extern __shared__ float4 smem4[];
    unsigned* tw = reinterpret_cast<unsigned*>(smem4);
    signed char* twe = reinterpret_cast<signed char*>(tw + N);
    const int tid = threadIdx.x;
    load_twiddles<ID, CPB, DBG>(tw, twe, a, N);
    LCtx L;
    L.tw = tw;
    L.twe = twe;
    L.tw_sh = (unsigned)__cvta_generic_to_shared(tw);
    L.lt = lt;
    L.tl = tid & (T - 1);
    L.c = (int)(__brev((unsigned)L.tl) >> (32 - lt));  // owned chunk: consecutive lanes load consecutive elements
    L.trivial = a.trivial01;
    L.sigma = a.inverse ? -1.f : 1.f;
    L.slim = a.stage_limit;
    const int rcol = L.tl;
    const unsigned rb = (unsigned)__cvta_generic_to_shared(smem4 + a.tw_chunks);
    if (rb & 127u) __trap();
    const int ebase = 0;
    const int64_t ngroups = a.total_lines;
    LDbg dbg;
    init_dbg<DBG>(dbg, a, N, CPB);
    __syncthreads();
    for (int64_t grp = blockIdx.x; grp < ngroups; grp += gridDim.x) {
        const int64_t line = grp;
        const int64_t img = line / a.lines_per_image;
        int64_t base, es, obase, oes;
        if (a.col_mode) {
            base = img * (int64_t)N * N + (line - img * N);
            es = N;
        } else if (a.dec) {  // half (line & 1) of row line >> 1, decimated: x[2q + h]
            base = (line >> 1) * (2 * (int64_t)N) + (line & 1);
            es = 2;
        } else {
            base = line * N;
            es = 1;
        }
        if (a.tstore) {
            obase = img * (int64_t)N * N + (line - img * N);
            oes = N;
        } else if (a.dec) {  // the halves' outputs are plain rows of N (half h of a 2N-row at h N)
            obase = line * N;
            oes = 1;
        } else {
            obase = base;
            oes = es;
        }
        const int kk = a.kvec ? a.kvec[img / a.k_group] : 0;
        const int kin = a.kin_sign * kk + a.kin_const;
        const int kout = a.kout_sign * kk + a.kout_const;
        if (DBG) dbg.row = line;
        float2 x[32];
        typename std::conditional<ACC, BadTrack, bool>::type bad{};
        if (a.seg_log2 && !a.col_mode) {  // segmented rows: element m T + rcol of the line
#pragma unroll
            for (int m = 0; m < 32; ++m) x[rev_c<5>(m)] = __ldg(a.in + seg_off(a, line, m * T + rcol));
            if (kin) scale32<DBG>(x, kin, bad);
        } else {
            const float2* src = a.in + base + (int64_t)rcol * es;
            const int64_t stride = (int64_t)T * es;
#pragma unroll
            for (int m = 0; m < 32; ++m) x[rev_c<5>(m)] = __ldg(src + m * stride);
            if (kin) scale32<DBG>(x, kin, bad);
        }
        if constexpr (ACC) fold_points<(LT >= 0 ? (1 << (LT >= 0 ? LT : 0)) : 1)>(x, a, grp);  // (the folded first pass runs unscaled: kin == 0; ACC kernels have a compile-time LT)
#if MXFFT_BIG_PREFETCH
        // while this line computes, its successor (a contiguous row) streams into
        // L2, so the next load phase hits L2 instead of waiting on HBM
        if (!a.col_mode && a.seg_log2 && grp + gridDim.x < ngroups && tid < (N >> a.seg_log2)) {
            // the next line's segments, one per thread
            const char* nx = reinterpret_cast<const char*>(a.in + seg_off(a, grp + gridDim.x, tid << a.seg_log2));
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(nx), "r"(8u << a.seg_log2) : "memory");
        } else if (!a.col_mode && !a.seg_log2 && tid < 4 && grp + gridDim.x < ngroups && (!a.dec || !(grp & 1))) {
            // (decimated halves: the even line of a pair prefetches the whole row)
            const int64_t nl = grp + gridDim.x;
            const char* nx = reinterpret_cast<const char*>(a.in + (a.dec ? (nl >> 1) * 2 * (int64_t)N : nl * (int64_t)N));
            const unsigned part = (unsigned)N * (a.dec ? 4u : 2u);  // bytes per prefetching thread
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(nx + (size_t)tid * part), "r"(part)
                         : "memory");
        }
#endif
        int U, V, P, H;
        run_stages<ID, CPB, DBG, LT>(x, U, V, P, H, L, rb, ebase, &dbg, bad);
        if (kout) scale32<DBG>(x, kout, bad);
        if constexpr (ACC) fold_range<(LT >= 0 ? (1 << (LT >= 0 ? LT : 0)) : 1)>(bad, a, grp);
        if (!DBG && __syncthreads_or(bad)) {
            char* tile = reinterpret_cast<char*>(smem4 + a.tw_chunks);
            replay_lines(a, line, 1, tile, 0, N, 0);
            for (int i = tid; i < N; i += blockDim.x)
                a.out[obase + (int64_t)i * oes] = *reinterpret_cast<const float2*>(tile + 16 * dsw(i >> 1) + 8 * (i & 1));
            __syncthreads();
            continue;
        }
        if (H > 0) {  // paired-stage layout: x[8k..8k+7] at P + k H
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                float2* dk = a.out + obase + (int64_t)(P + k * H) * oes;
                if (oes == 1) {
#pragma unroll
                    for (int i = 0; i < 8; i += 2)
                        stg128(reinterpret_cast<float4*>(dk + i),
                               make_float4(x[8 * k + i].x, x[8 * k + i].y, x[8 * k + i + 1].x, x[8 * k + i + 1].y));
                } else {
#pragma unroll
                    for (int i = 0; i < 8; ++i) stg64(dk + i * oes, x[8 * k + i]);
                }
            }
            __syncthreads();
            continue;
        }
        float2* du = a.out + obase + (int64_t)U * oes;
        float2* dv = a.out + obase + (int64_t)V * oes;
        if (oes == 1) {
#pragma unroll
            for (int i = 0; i < 16; i += 2) {
                *reinterpret_cast<float4*>(du + i) = make_float4(x[i].x, x[i].y, x[i + 1].x, x[i + 1].y);
                *reinterpret_cast<float4*>(dv + i) =
                    make_float4(x[16 + i].x, x[16 + i].y, x[17 + i].x, x[17 + i].y);
            }
        } else {
#pragma unroll
            for (int i = 0; i < 16; ++i) {
                du[i * oes] = x[i];
                dv[i * oes] = x[16 + i];
            }
        }
        __syncthreads();
    }
}

// ---------------------------------------------------------------------------
// n = 8192 / 16384 plain row passes on a 2-CTA cluster per line.  The first
// L-1 stages of a radix-2 DIT transform on bit-reversed input act on the two
// contiguous halves independently, and half r of the bit-reversed line is the
// (n/2)-point transform of the decimated sequence x[2m + r] (the MX block and
// twiddle structure of stages < L-1 do not depend on n: blocks never straddle
// the halves, and the stage tables are the plan's own prefix).  So CTA r runs
// the n/2-point kernel on x[r::2] with 256 (or 128) threads, both CTAs publish
// their halves to shared memory, and the last stage (butterflies j and
// n/2 + j) reads u from CTA 0 and v from CTA 1 through distributed shared
// memory; CTA r takes j in [r n/4, (r+1) n/4).  Half a line plus the n/2
// twiddle entries fit twice per SM, so one CTA's loads and stores overlap the
// other's arithmetic (the one-CTA-per-line kernel cannot).  A line with any
// block outside the fast exponent range is recomputed by both CTAs with the
// reference-literal stages over the cluster's shared memory.
// ---------------------------------------------------------------------------
__device__ __forceinline__ float2 lds64_cluster(unsigned addr) {
    float2 v;
    asm volatile("ld.shared::cluster.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "r"(addr) : "memory");
    return v;
}
__device__ __forceinline__ void lds128_cluster(unsigned addr, float2& a, float2& b) {
    asm volatile("ld.shared::cluster.v4.f32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(a.x), "=f"(a.y), "=f"(b.x), "=f"(b.y)
                 : "r"(addr)
                 : "memory");
}
__device__ __forceinline__ unsigned map_cluster(unsigned addr, unsigned rank) {
    unsigned r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
    return r;
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// exact recomputation of one line over the cluster's two regions (rare path)
static __device__ __noinline__ void replay_line_cl2(const MxLinesArgs& a, int64_t line, char* reg0, char* reg1,
                                                    int rank, int kin, int kout) {
    const int n = a.n, m = n / 2, nthr = 2 * blockDim.x, tid = rank * blockDim.x + threadIdx.x;
    auto acc = [reg0, reg1, m](int i) {
        const int e = i < m ? i : i - m;
        char* r = i < m ? reg0 : reg1;
        return reinterpret_cast<float2*>(r + 16 * dsw(e >> 1) + 8 * (e & 1));
    };
    const int64_t base = line * n;
    cluster_sync_all();  // both CTAs are done with their regions' normal contents
    for (int i = tid; i < n; i += nthr) {
        const int r = (int)(__brev((unsigned)i) >> (32 - a.log2n));
        *acc(i) = gscale(a.in[base + r], kin);
    }
    cluster_sync_all();
    for (int st = 0; st < a.log2n; ++st) {
        generic_stage(acc, st, m, a.cpb, a.fmt, a.wcr, a.wci, a.wsexp, a.inverse != 0, tid, nthr);
        cluster_sync_all();
    }
    for (int i = tid; i < n; i += nthr) a.out[base + i] = gscale(*acc(i), kout);
    cluster_sync_all();
}

template <int ID, int CPB, int LT>  // LT: log2 of the threads per CTA (n / 64)
__device__ __forceinline__ void lines_body_cl2(const MxLinesArgs& a) {
    constexpr int T = 1 << LT, NH = 32 * T;  // threads per CTA, points per half line
    constexpr int NB = CPB < 16 ? CPB : 16;
    constexpr bool PAIR = CPB == 32;
    const int n = 2 * NH;
    extern __shared__ float4 smem4[];
    unsigned* tw = reinterpret_cast<unsigned*>(smem4);
    signed char* twe = reinterpret_cast<signed char*>(tw + NH);
    const int tid = threadIdx.x;
    const unsigned rank = cooperative_groups::this_cluster().block_rank();
    load_twiddles<ID, CPB, false>(tw, twe, a, NH);  // stages < L-1: the plan table's prefix
    LCtx L;
    L.tw = tw;
    L.twe = twe;
    L.tw_sh = (unsigned)__cvta_generic_to_shared(tw);
    L.lt = LT;
    L.tl = tid;
    L.c = (int)(__brev((unsigned)tid) >> (32 - LT));
    L.trivial = a.trivial01;
    L.sigma = a.inverse ? -1.f : 1.f;
    L.slim = a.stage_limit;
    const unsigned rb = (unsigned)__cvta_generic_to_shared(smem4 + a.tw_chunks);
    if (rb & 127u) __trap();
    char* const reg_mine = reinterpret_cast<char*>(smem4 + a.tw_chunks);
    char* const reg_other = static_cast<char*>(cooperative_groups::this_cluster().map_shared_rank(
        static_cast<void*>(reg_mine), rank ^ 1u));
    char* const reg0 = rank ? reg_other : reg_mine;
    char* const reg1 = rank ? reg_mine : reg_other;
    const unsigned rb_u = map_cluster(rb, 0);  // CTA 0's region (u of the last stage)
    const unsigned rb_v = map_cluster(rb, 1);  // CTA 1's region (v)
    int& bad_flag = *reinterpret_cast<int*>(reg_mine + NH * 8);  // just past the region
    const int64_t nclusters = gridDim.x / 2, cl = blockIdx.x / 2;
    const int j0 = (int)rank * (NH / 2) + 16 * tid;  // last-stage butterflies of this thread
    LDbg dbg;
    __syncthreads();
    for (int64_t line = cl; line < a.total_lines; line += nclusters) {
        const int kk = a.kvec ? a.kvec[k_index(a, line)] : 0;
        const int kin = a.kin_sign * kk + a.kin_const, kout = a.kout_sign * kk + a.kout_const;
        float2 x[32];
        bool bad = false;
        {
            // decimated half: sub-index m T + tid <- natural element 2 (m T + tid) + rank
            const float2* src = a.in + line * n + rank + 2 * tid;
#pragma unroll
            for (int m = 0; m < 32; ++m) x[rev_c<5>(m)] = __ldg(src + (int64_t)m * 2 * T);
            if (kin) scale32<false>(x, kin, bad);
        }
#if MXFFT_BIG_PREFETCH
        if (tid < 2 && line + nclusters < a.total_lines) {  // this CTA's half of the next row into L2
            const char* nx = reinterpret_cast<const char*>(a.in + (line + nclusters) * n);
            const unsigned part = (unsigned)n * 2u;  // n * 8 bytes / 4 parts
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(nx + (size_t)(2 * rank + tid) * part),
                         "r"(part)
                         : "memory");
        }
#endif
        int U, V, P, H;
        run_stages<ID, CPB, false, LT>(x, U, V, P, H, L, rb, 0, &dbg, bad);
        if (H > 0) publish4(x, rb, 0, P, H);
        else publish2(x, rb, 0, U, V);
        cluster_sync_all();  // both halves published
        // last stage: butterflies j0 .. j0+15, u from CTA 0's half, v from CTA 1's
        float2 u[16], v[16];
        {
            const Run ru = mkrun(rb_u, j0), rv = mkrun(rb_v, j0);
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                lds128_cluster(ru.a0 + (ru.f ^ (unsigned)(k << 4)), u[2 * k], u[2 * k + 1]);
                lds128_cluster(rv.a0 + (rv.f ^ (unsigned)(k << 4)), v[2 * k], v[2 * k + 1]);
            }
        }
        unsigned w16[16];
        {
            const uint4* wp = reinterpret_cast<const uint4*>(a.tw16 + NH + j0);
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const uint4 q = __ldg(wp + i);
                w16[4 * i] = q.x, w16[4 * i + 1] = q.y, w16[4 * i + 2] = q.z, w16[4 * i + 3] = q.w;
            }
        }
#pragma unroll
        for (int k = 0; k < 16 / NB; ++k) {
            float2 ub[NB], vb[NB];
            unsigned wb[NB];
#pragma unroll
            for (int i = 0; i < NB; ++i) ub[i] = u[k * NB + i], vb[i] = v[k * NB + i], wb[i] = w16[k * NB + i];
            mxb<ID, NB, PAIR ? 2 : 1, false>(ub, vb, wb, __ldg(a.twe + NH + j0 + k * NB), nullptr, 0, bad);
#pragma unroll
            for (int i = 0; i < NB; ++i) u[k * NB + i] = ub[i], v[k * NB + i] = vb[i];
        }
        if (kout) {  // undo_prescale / 1/n^2 (a power of two; non-normal factors replay)
            bad |= !(kout >= -126 && kout <= 127);
            const float f = exp2i(kout);
            const float2 f2 = make_float2(f, f);
#pragma unroll
            for (int i = 0; i < 16; ++i) u[i] = __fmul2_rn(u[i], f2), v[i] = __fmul2_rn(v[i], f2);
        }
        const int mine = __syncthreads_or(bad);
        if (tid == 0) bad_flag = mine;
        cluster_sync_all();  // last-stage reads of both regions done; flags visible
        const int other = *static_cast<volatile int*>(
            cooperative_groups::this_cluster().map_shared_rank(&bad_flag, rank ^ 1u));
        if (mine | other) {
            replay_line_cl2(a, line, reg0, reg1, (int)rank, kin, kout);
            continue;
        }
        float2* du = a.out + line * n + j0;
        float2* dv = du + NH;
#pragma unroll
        for (int i = 0; i < 16; i += 2) {
            *reinterpret_cast<float4*>(du + i) = make_float4(u[i].x, u[i].y, u[i + 1].x, u[i + 1].y);
            *reinterpret_cast<float4*>(dv + i) = make_float4(v[i].x, v[i].y, v[i + 1].x, v[i + 1].y);
        }
    }
    cluster_sync_all();  // no CTA leaves while its partner may still read its region
}

template <int ID, int CPB, int LT>
__global__ void __launch_bounds__(1 << LT, 2) k_mx_lines_cl2(const __grid_constant__ MxLinesArgs a) {
    lines_body_cl2<ID, CPB, LT>(a);
}

template <int ID, int CPB, bool DBG, int LT>
__global__ void __launch_bounds__(128, MXFFT_LINES_MINB) k_mx_lines(const __grid_constant__ MxLinesArgs a) {
    lines_body_pipe<ID, CPB, DBG, LT>(a);
}

template <int ID, int CPB, bool DBG, int LT, bool ACC = false>
__global__ void __launch_bounds__(512, 1) k_mx_lines_big(const __grid_constant__ MxLinesArgs a) {
    lines_body_direct<ID, CPB, DBG, LT, ACC>(a);
}

// ---------------------------------------------------------------------------
// launch
// ---------------------------------------------------------------------------
template <int ID, int CPB, bool DBG, int LT, bool BIGK>
static cudaError_t launch_t(const MxLinesArgs& a, size_t smem, cudaStream_t st) {
    const int nt = BIGK ? (1 << a.log2T) : 128;
    void (*k)(MxLinesArgs);
    if constexpr (BIGK) k = k_mx_lines_big<ID, CPB, DBG, LT>;
    else k = k_mx_lines<ID, CPB, DBG, LT>;
    // per (device, kernel, threads, shared memory): the run-time-n variants
    // (LT = -1) serve several n with different tiles
    cudaError_t e = ensure_smem_attr((const void*)k, 227 * 1024);
    if (e != cudaSuccess) return e;
    const int sms = device_attr(cudaDevAttrMultiProcessorCount);
    int occ = 1;
    e = cached_occupancy((const void*)k, nt, smem, &occ);
    if (e != cudaSuccess) return e;
    const int lines_per_cta = nt >> a.log2T;
    const int64_t groups = (a.total_lines + lines_per_cta - 1) / lines_per_cta;
    const int per_sm = g_lines_ctas_per_sm > 0 && g_lines_ctas_per_sm < occ ? g_lines_ctas_per_sm : occ;
    const int64_t cap = (int64_t)sms * per_sm;
    const int grid = (int)(groups < cap ? groups : cap);
    if constexpr (BIGK) {
        k<<<grid, nt, smem, st>>>(a);
    } else {
        e = launch_pdl(k, (unsigned)grid, (unsigned)nt, smem, st, a);
        if (e != cudaSuccess) return e;
    }
    note_launch();
    return cudaGetLastError();
}

template <int ID, int CPB, int LT, bool ACC = false>
static cudaError_t launch_tma(const MxLinesArgs& a, size_t smem, cudaStream_t st) {
    void (*k)(MxLinesArgs) = k_mx_lines_tma<ID, CPB, LT, ACC>;
    cudaError_t e = ensure_smem_attr((const void*)k, 227 * 1024);
    if (e != cudaSuccess) return e;
    const int sms = device_attr(cudaDevAttrMultiProcessorCount);
    int occ = 1;
    e = cached_occupancy((const void*)k, 128, smem, &occ);
    if (e != cudaSuccess) return e;
    const int64_t groups = a.total_lines / (128 >> LT);
    const int per_sm = g_lines_ctas_per_sm > 0 && g_lines_ctas_per_sm < occ ? g_lines_ctas_per_sm : occ;
    const int64_t cap = (int64_t)sms * per_sm;
    e = launch_pdl(k, (unsigned)(groups < cap ? groups : cap), 128u, smem, st, a);
    if (e != cudaSuccess) return e;
    note_launch();
    return cudaGetLastError();
}

template <int ID, int CPB, int LT>
static cudaError_t launch_cl2(const MxLinesArgs& a0, cudaStream_t st) {
    MxLinesArgs a = a0;
    constexpr int NH = 32 << LT;
    a.tw_chunks = ((NH * 5 + 1023) / 1024) * 64;
    const size_t smem = (size_t)a.tw_chunks * 16 + (size_t)NH * 8 + 128;
    auto k = k_mx_lines_cl2<ID, CPB, LT>;
    {
        cudaError_t e = ensure_smem_attr((const void*)k, (int)smem);
        if (e != cudaSuccess) return e;
    }
    const int sms = device_attr(cudaDevAttrMultiProcessorCount);
    const int64_t nclusters = a.total_lines < sms ? a.total_lines : sms;  // two CTAs per SM
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(2 * nclusters));
    cfg.blockDim = dim3(1u << LT);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaError_t e = cudaLaunchKernelEx(&cfg, k, a);
    note_launch();
    return e != cudaSuccess ? e : cudaGetLastError();
}

// Specialised (compile-time n) variants: block sizes 16/32/64 (cpb 8..32),
// n <= 4096.  Everything else -- smaller blocks, n = 8192/16384 and the
// debug-capture kernels (test instrumentation, n <= 4096 only) -- runs the
// same code with n taken at run time.
template <int ID, int CPB, bool DBG>
static cudaError_t disp_lt(const MxLinesArgs& a, size_t smem, cudaStream_t st) {
    if (a.log2T > 7) {
        if constexpr (!DBG) {
            // n = 8192 / 16384 specialised (every stage, unconditional register stages)
            if constexpr (CPB >= 8) {
#if MXFFT_CL2
                if (!a.col_mode && !a.tstore && a.stage_limit >= a.log2n && a.prof_flags == 0) {
                    if (a.log2T == 8) return launch_cl2<ID, CPB, 7>(a, st);
                    if (a.log2T == 9) return launch_cl2<ID, CPB, 8>(a, st);
                }
#endif
                if (!a.col_mode && a.stage_limit >= a.log2n) {
                    if (a.log2T == 8) return launch_t<ID, CPB, false, 8, true>(a, smem, st);
                    if (a.log2T == 9) return launch_t<ID, CPB, false, 9, true>(a, smem, st);
                }
            }
            return launch_t<ID, CPB, false, -1, true>(a, smem, st);
        }
        return cudaErrorInvalidValue;
    }
    if constexpr (!DBG && CPB >= 8) {
        if (a.col_mode || a.seg_log2 || a.stage_limit < a.log2n) return launch_t<ID, CPB, DBG, -1, false>(a, smem, st);
        if (a.tma_out && a.log2T == 2) return launch_tma<ID, CPB, 2>(a, smem, st);
        if (a.tma_out && a.log2T == 3) return launch_tma<ID, CPB, 3>(a, smem, st);
        if (a.tma_out && a.log2T == 4) return launch_tma<ID, CPB, 4>(a, smem, st);
        switch (a.log2T) {
            case 0: return launch_t<ID, CPB, DBG, 0, false>(a, smem, st);
            case 1: return launch_t<ID, CPB, DBG, 1, false>(a, smem, st);
            case 2: return launch_t<ID, CPB, DBG, 2, false>(a, smem, st);
            case 3: return launch_t<ID, CPB, DBG, 3, false>(a, smem, st);
            case 4: return launch_t<ID, CPB, DBG, 4, false>(a, smem, st);
            case 5: return launch_t<ID, CPB, DBG, 5, false>(a, smem, st);
            case 6: return launch_t<ID, CPB, DBG, 6, false>(a, smem, st);
            case 7: return launch_t<ID, CPB, DBG, 7, false>(a, smem, st);
        }
        return cudaErrorInvalidValue;
    } else {
        return launch_t<ID, CPB, DBG, -1, false>(a, smem, st);
    }
}

// one line per CTA with the prescale evidence: the 8192-point decimated half rows of an n = 16384
// split pass (LT = 8) and plain n = 16384 rows (LT = 9, the slab passes of a distributed image)
template <int ID, int CPB, int LT>
static cudaError_t launch_big_acc(const MxLinesArgs& a, size_t smem, cudaStream_t st) {
    void (*k)(MxLinesArgs) = k_mx_lines_big<ID, CPB, false, LT, true>;
    cudaError_t e = ensure_smem_attr((const void*)k, 227 * 1024);
    if (e != cudaSuccess) return e;
    const int sms = device_attr(cudaDevAttrMultiProcessorCount);
    int occ = 1;
    e = cached_occupancy((const void*)k, 1 << LT, smem, &occ);
    if (e != cudaSuccess) return e;
    const int64_t cap = (int64_t)sms * occ;
    k<<<(unsigned)(a.total_lines < cap ? a.total_lines : cap), 1 << LT, smem, st>>>(a);
    note_launch();
    return cudaGetLastError();
}

// statistics-folding first pass (the TMA kernel, or the 8192-point half rows; instantiated in lines_acc_<fmt>.cu)
template <int ID>
static cudaError_t disp_acc(const MxLinesArgs& a, int cpb, size_t smem, cudaStream_t st) {
    if (!a.acc || !a.minw) return cudaErrorInvalidValue;
    if (a.log2T == 8 && a.dec && !a.col_mode && !a.tstore && a.stage_limit >= a.log2n) {
        if (cpb == 8) return launch_big_acc<ID, 8, 8>(a, smem, st);
        if (cpb == 16) return launch_big_acc<ID, 16, 8>(a, smem, st);
        if (cpb == 32) return launch_big_acc<ID, 32, 8>(a, smem, st);
        return cudaErrorInvalidValue;
    }
    if (a.log2T == 9 && !a.dec && !a.col_mode && !a.tstore && !a.seg_log2 && a.stage_limit >= a.log2n) {
        if (cpb == 8) return launch_big_acc<ID, 8, 9>(a, smem, st);
        if (cpb == 16) return launch_big_acc<ID, 16, 9>(a, smem, st);
        if (cpb == 32) return launch_big_acc<ID, 32, 9>(a, smem, st);
        return cudaErrorInvalidValue;
    }
    if (!a.tma_out) return cudaErrorInvalidValue;
#define MXFFT_ACC_CASE(C, L) \
    if (cpb == C && a.log2T == L) return launch_tma<ID, C, L, true>(a, smem, st);
    MXFFT_ACC_CASE(8, 2) MXFFT_ACC_CASE(8, 3) MXFFT_ACC_CASE(8, 4)
    MXFFT_ACC_CASE(16, 2) MXFFT_ACC_CASE(16, 3) MXFFT_ACC_CASE(16, 4)
    MXFFT_ACC_CASE(32, 2) MXFFT_ACC_CASE(32, 3) MXFFT_ACC_CASE(32, 4)
#undef MXFFT_ACC_CASE
    return cudaErrorInvalidValue;
}

template <int ID, bool DBG>
static cudaError_t disp_cpb(const MxLinesArgs& a, int cpb, size_t smem, cudaStream_t st) {
    switch (cpb) {
        case 1: return disp_lt<ID, 1, DBG>(a, smem, st);
        case 2: return disp_lt<ID, 2, DBG>(a, smem, st);
        case 4: return disp_lt<ID, 4, DBG>(a, smem, st);
        case 8: return disp_lt<ID, 8, DBG>(a, smem, st);
        case 16: return disp_lt<ID, 16, DBG>(a, smem, st);
        case 32: return disp_lt<ID, 32, DBG>(a, smem, st);
    }
    return cudaErrorInvalidValue;
}

}  // namespace mxfft
