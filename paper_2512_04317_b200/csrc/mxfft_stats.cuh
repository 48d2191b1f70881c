// mxfft_stats.cuh -- device helpers of the exact prescale statistics
// (compute_prescale, prescale.py:61-73) shared by the statistics kernels
// (mxfft_prescale_fast.cu) and the fused small-image kernel (mxfft_image.cuh):
// numpy's |z|, the FP32 squared-magnitude key, counted-rank / bitonic order
// statistics, the candidate histogram bins, and the k rule.
#pragma once
#include <cfloat>

#include "../../include/mxfft_b200.h"
#include "mxfft_common.cuh"

namespace mxfft {

constexpr int NBIN = 512;  // candidate histogram bins of the select phase

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
struct Limits;
template <>
struct Limits<unsigned> {
    static __device__ __forceinline__ unsigned max() { return 0xffffffffu; }
    static __device__ __forceinline__ unsigned shfl_xor(unsigned v, int j) { return __shfl_xor_sync(0xffffffffu, v, j); }
};
template <>
struct Limits<double> {
    static __device__ __forceinline__ double max() { return DBL_MAX; }
    static __device__ __forceinline__ double shfl_xor(double v, int j) { return __shfl_xor_sync(0xffffffffu, v, j); }
};

// Block-wide ascending bitonic sort of a[0..P) (P <= NT * SLOTS) with the
// elements in registers: element i = tid + NT * s lives in slot s of thread
// tid (pads past P sort last).  Compare-exchange distance j < 32: warp shuffle;
// j >= NT: between two slots of the same thread; otherwise through shared
// memory.  SLOTS is exact (sort_block picks it), so no slot is predicated off.
template <typename T, int NT, int SLOTS>
__device__ void reg_bitonic_sort(T* a, int P) {
    constexpr int PE = NT * SLOTS;
    const int tid = threadIdx.x;
    T r[SLOTS];
#pragma unroll
    for (int s = 0; s < SLOTS; ++s) {
        const int i = tid + NT * s;
        r[s] = i < P ? a[i] : Limits<T>::max();
    }
#pragma unroll 1
    for (int k = 2; k <= PE; k <<= 1) {
#pragma unroll 1
        for (int j = k >> 1; j > 0; j >>= 1) {
            if (j >= NT) {
#pragma unroll
                for (int jb = 1; jb < SLOTS; jb <<= 1) {  // compile-time slot pairs
                    if (jb != j / NT) continue;
#pragma unroll
                    for (int s = 0; s < SLOTS; ++s) {
                        const int sp = s ^ jb;
                        if (sp > s) {
                            const bool asc = ((tid + NT * s) & k) == 0;
                            const T x = r[s], y = r[sp];
                            if ((x > y) == asc) {
                                r[s] = y;
                                r[sp] = x;
                            }
                        }
                    }
                }
            } else if (j >= 32) {
                __syncthreads();
#pragma unroll
                for (int s = 0; s < SLOTS; ++s) a[tid + NT * s] = r[s];
                __syncthreads();
#pragma unroll
                for (int s = 0; s < SLOTS; ++s) {
                    const int i = tid + NT * s, l = i ^ j;
                    const T y = a[l];
                    const bool asc = (i & k) == 0, low = i < l;
                    // the lower index keeps the min when ascending
                    r[s] = (low == asc) ? (y < r[s] ? y : r[s]) : (y > r[s] ? y : r[s]);
                }
            } else {
#pragma unroll
                for (int s = 0; s < SLOTS; ++s) {
                    const int i = tid + NT * s;
                    const T y = Limits<T>::shfl_xor(r[s], j);
                    const bool asc = (i & k) == 0, low = (i & j) == 0;
                    r[s] = (low == asc) ? (y < r[s] ? y : r[s]) : (y > r[s] ? y : r[s]);
                }
            }
        }
    }
    __syncthreads();
#pragma unroll
    for (int s = 0; s < SLOTS; ++s)
        if (tid + NT * s < P) a[tid + NT * s] = r[s];
    __syncthreads();
}

// Order statistics without sorting: the elements of rank r0, r1, r2 of
// a[0..P) (ascending; ties broken by index, so ranks are a permutation) go to
// out[0..2] (a rank < 0 is skipped).  Each element's rank is counted against
// broadcast shared-memory reads -- no barriers between phases.
template <typename T, int NT>
__device__ void rank_select(const T* a, int P, int r0, int r1, int r2, T* out) {
    for (int i = threadIdx.x; i < P; i += NT) {
        const T v = a[i];
        int r = 0;
        int j = 0;
        for (; j + 4 <= P; j += 4) {
            const T u0 = a[j], u1 = a[j + 1], u2 = a[j + 2], u3 = a[j + 3];
            r += (u0 < v) | ((u0 == v) & (j < i));
            r += (u1 < v) | ((u1 == v) & (j + 1 < i));
            r += (u2 < v) | ((u2 == v) & (j + 2 < i));
            r += (u3 < v) | ((u3 == v) & (j + 3 < i));
        }
        for (; j < P; ++j) {
            const T u = a[j];
            r += (u < v) | ((u == v) & (j < i));
        }
        if (r == r0) out[0] = v;
        if (r == r1) out[1] = v;
        if (r == r2) out[2] = v;
    }
    __syncthreads();
}

template <typename T, int NT, int MAXS>
__device__ void sort_block(T* a, int P);

// The elements of rank r0 and r1 of a[0..P) -> out[0], out[1]: counted ranks
// for small P (P^2 / NT compares, no barriers), a register sort beyond.
template <typename T, int NT, int MAXS>
__device__ void pick_two(T* a, int P, int r0, int r1, T* out) {
    if (P <= 2 * NT) {
        rank_select<T, NT>(a, P, r0, r1, -1, out);
        return;
    }
    sort_block<T, NT, MAXS>(a, P);
    if (threadIdx.x == 0) {
        out[0] = a[r0];
        out[1] = a[r1];
    }
    __syncthreads();
}

// sort a[0..P), P <= NT * MAXS, with the smallest power-of-two slot count
template <typename T, int NT, int MAXS>
__device__ void sort_block(T* a, int P) {
    if (P <= NT || MAXS == 1) return reg_bitonic_sort<T, NT, 1>(a, P);
    if (P <= 2 * NT || MAXS == 2) return reg_bitonic_sort<T, NT, (MAXS < 2 ? MAXS : 2)>(a, P);
    if (P <= 4 * NT || MAXS == 4) return reg_bitonic_sort<T, NT, (MAXS < 4 ? MAXS : 4)>(a, P);
    if (P <= 8 * NT || MAXS == 8) return reg_bitonic_sort<T, NT, (MAXS < 8 ? MAXS : 8)>(a, P);
    return reg_bitonic_sort<T, NT, MAXS>(a, P);
}

__device__ __forceinline__ int round_half_away_d(double v) {
    return v >= 0 ? (int)floor(__dadd_rn(v, 0.5)) : (int)ceil(__dsub_rn(v, 0.5));
}

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

// k (prescale.py:61-73) from a_max / p_tau; flags bit 1 marks a log2 within a
// few ulps of a rounding boundary (the host re-checks it)
__device__ inline void finish_result(const mxfft_prescale_cfg& c, double a_max, double p_tau, unsigned long long nnz,
                              mxfft_prescale_result* out, int32_t* kvec, int seg) {
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

// block-wide sum of three counters (all threads get the totals)
template <int NT>
__device__ __forceinline__ void block_sum3(unsigned& a, unsigned& b, unsigned& c, unsigned* wa, unsigned* wb,
                                           unsigned* wc) {
    const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
    for (int o = 16; o; o >>= 1) {
        a += __shfl_xor_sync(0xffffffffu, a, o);
        b += __shfl_xor_sync(0xffffffffu, b, o);
        c += __shfl_xor_sync(0xffffffffu, c, o);
    }
    __syncthreads();
    if (lane == 0) {
        wa[wp] = a;
        wb[wp] = b;
        wc[wp] = c;
    }
    __syncthreads();
    a = b = c = 0;
#pragma unroll
    for (int i = 0; i < NT / 32; ++i) {
        a += wa[i];
        b += wb[i];
        c += wc[i];
    }
}

}  // namespace mxfft
