// mxfft_laststage.cu -- the last butterfly stage of a long row pass, fused
// into the tiled transpose that follows it.
//
// For n >= 16384 (C5) a row is too long to share an SM with a second line, so
// mxfft_fft2 splits each row pass in two:
//  1. stages 0 .. L-2 of a radix-2 DIT transform on bit-reversed input act on
//     the two halves independently, and half h is the n/2-point transform of
//     the decimated sequence x[2q + h] with the same per-stage twiddles and MX
//     block layout (fftcore.py:264-281: blocks never straddle the halves) --
//     the n/2-point line kernel runs them, two CTAs per SM;
//  2. this kernel: stage L-1 pairs column j with j + n/2 (butterfly j, blocks
//     of cpb consecutive j) and the transposed store of fft_2d's rows.T
//     (fftcore.py:352) follows in the same pass over the data.
// A tile is 32 rows x 64 butterflies: the u tile (columns j0 .. j0+63) and the
// v tile (columns n/2 + j0 ..), each staged in shared memory with an XOR
// swizzle that keeps the row loads, the per-thread block reads and the
// transposed reads free of bank conflicts; thread t takes row t / 8 and
// butterflies 8 (t mod 8) .. +7 (an MX block spans G = cpb / 8 lanes).  The
// MX arithmetic is the line kernel's own block code (mxb), with the exact
// FP64-assisted path inline for blocks outside the fast exponent range.
#include "mxfft_lines.cuh"

namespace mxfft {

int g_split_last_stage = 1;

#ifndef MXFFT_LS_MINB
#define MXFFT_LS_MINB 3  // CTAs per SM the register budget is sized for (2: 118 regs, 3.22 ms per C5 pass; 3: 75 regs, 3.10 ms)
#endif

struct LastArgs {
    const float2* in;
    float2* out;
    int n, log2n;
    int64_t batch;
    const unsigned* tw16;
    const signed char* twe;
    const int32_t* kvec;
    int k_group, kout_sign, kout_const, kin_sign;
};

constexpr int LS_R = 32, LS_C = 64;  // tile rows x butterflies

// swizzled slot of element (row r, column c) of a 32 x 64 tile (8-byte slots)
__device__ __forceinline__ int ls_slot(int r, int c) { return r * LS_C + (c ^ ((c >> 3) & 7) ^ ((r >> 1) & 15)); }

template <int ID, int G>
__global__ void __launch_bounds__(256, MXFFT_LS_MINB) k_last_stage_t(LastArgs a) {
    __shared__ float2 tu[LS_R * LS_C], tv[LS_R * LS_C];
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const int n = a.n, hn = n >> 1;
    const int tiles_r = n / LS_R, tiles_c = hn / LS_C;
    const int64_t per = (int64_t)tiles_r * tiles_c, ntiles = per * a.batch;
    const int r = tid >> 3, cb = (tid & 7) * 8;  // compute mapping
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const int64_t b = t / per;
        const int rem = (int)(t - b * per);
        const int i0 = (rem / tiles_c) * LS_R, j0 = (rem % tiles_c) * LS_C;
        const float2* xb = a.in + b * (int64_t)n * n;
        float2* yb = a.out + b * (int64_t)n * n;
        // rows i0 .. i0+31: columns j0 + 2l, +1 (u) and hn + j0 + 2l, +1 (v)
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int rr = w + 8 * q;
            const float2* src = xb + (int64_t)(i0 + rr) * n + j0 + 2 * lane;
            const float4 pu = __ldg(reinterpret_cast<const float4*>(src));
            const float4 pv = __ldg(reinterpret_cast<const float4*>(src + hn));
            tu[ls_slot(rr, 2 * lane)] = make_float2(pu.x, pu.y);
            tu[ls_slot(rr, 2 * lane + 1)] = make_float2(pu.z, pu.w);
            tv[ls_slot(rr, 2 * lane)] = make_float2(pv.x, pv.y);
            tv[ls_slot(rr, 2 * lane + 1)] = make_float2(pv.z, pv.w);
        }
        __syncthreads();
        {
            float2 u[8], v[8];
            unsigned wc[8];
            const int j = j0 + cb;
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                u[i] = tu[ls_slot(r, cb + i)];
                v[i] = tv[ls_slot(r, cb + i)];
                wc[i] = __ldg(a.tw16 + hn + j + i);
            }
            const int ew = __ldg(a.twe + hn + j);
            bool bad = false;
            const int kk = a.kvec ? __ldg(a.kvec + b / a.k_group) : 0;
            const int kin = a.kin_sign * kk;  // (the folded pipeline scales here: stages 0 .. L-2 ran unscaled)
            if (kin) {
                if (kin >= -126 && kin <= 127) {
                    const float f = exp2i(kin);
                    const float2 f2 = make_float2(f, f);
#pragma unroll
                    for (int i = 0; i < 8; ++i) u[i] = __fmul2_rn(u[i], f2), v[i] = __fmul2_rn(v[i], f2);
                } else {
#pragma unroll
                    for (int i = 0; i < 8; ++i) u[i] = gscale(u[i], kin), v[i] = gscale(v[i], kin);
                }
            }
            mxb<ID, 8, G, false, true>(u, v, wc, ew, nullptr, 0, bad);
            const int kout = a.kout_sign * kk + a.kout_const;
            if (kout) {
                if (kout >= -126 && kout <= 127) {
                    const float f = exp2i(kout);
                    const float2 f2 = make_float2(f, f);
#pragma unroll
                    for (int i = 0; i < 8; ++i) u[i] = __fmul2_rn(u[i], f2), v[i] = __fmul2_rn(v[i], f2);
                } else {
#pragma unroll
                    for (int i = 0; i < 8; ++i) u[i] = gscale(u[i], kout), v[i] = gscale(v[i], kout);
                }
            }
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                tu[ls_slot(r, cb + i)] = u[i];
                tv[ls_slot(r, cb + i)] = v[i];
            }
        }
        __syncthreads();
        // transposed stores: output row j0 + c (u) / hn + j0 + c (v), elements i0 + 2m, +1
        {
            const int m = lane & 15;
            const bool isv = lane >= 16;
            const float2* tile = isv ? tv : tu;
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const int c = w * 8 + q;
                const float2 e0 = tile[ls_slot(2 * m, c)], e1 = tile[ls_slot(2 * m + 1, c)];
                float2* dst = yb + (int64_t)((isv ? hn : 0) + j0 + c) * n + i0 + 2 * m;
                *reinterpret_cast<float4*>(dst) = make_float4(e0.x, e0.y, e1.x, e1.y);
            }
        }
        __syncthreads();
    }
}

bool last_stage_ok(const Plan& p) {
    return p.n >= 16384 && p.fmt.id != F_GENERIC && (p.cpb == 8 || p.cpb == 16);
}

template <int ID>
static cudaError_t launch_ls(const LastArgs& a, int cpb, cudaStream_t st) {
    const int sms = device_attr(cudaDevAttrMultiProcessorCount);
    int occ = 1;
    void (*k)(LastArgs) = cpb == 16 ? k_last_stage_t<ID, 2> : k_last_stage_t<ID, 1>;
    cudaError_t e = cached_occupancy((const void*)k, 256, 0, &occ);
    if (e != cudaSuccess) return e;
    const int64_t ntiles = (int64_t)(a.n / LS_R) * (a.n / 2 / LS_C) * a.batch;
    const int64_t cap = (int64_t)sms * occ;
    k<<<(unsigned)(ntiles < cap ? ntiles : cap), 256, 0, st>>>(a);
    note_launch();
    return cudaGetLastError();
}

cudaError_t run_last_stage_transpose(const Plan& p, const LastStagePass& lp, cudaStream_t st) {
    LastArgs a{};
    a.in = reinterpret_cast<const float2*>(lp.in);
    a.out = reinterpret_cast<float2*>(lp.out);
    a.n = p.n;
    a.log2n = p.log2n;
    a.batch = lp.batch;
    a.tw16 = lp.inverse ? p.d_tw16_inv : p.d_tw16_fwd;
    a.twe = p.d_twe8;
    a.kvec = lp.kvec;
    a.k_group = lp.k_group > 0 ? lp.k_group : 1;
    a.kout_sign = lp.kout_sign;
    a.kout_const = lp.kout_const;
    a.kin_sign = lp.kin_sign;
    if (lp.batch <= 0) return cudaSuccess;
    switch (p.fmt.id) {
        case F_E4M3: return launch_ls<F_E4M3>(a, p.cpb, st);
        case F_E5M2: return launch_ls<F_E5M2>(a, p.cpb, st);
        case F_E2M3: return launch_ls<F_E2M3>(a, p.cpb, st);
        case F_E3M2: return launch_ls<F_E3M2>(a, p.cpb, st);
        case F_E2M1: return launch_ls<F_E2M1>(a, p.cpb, st);
    }
    return cudaErrorInvalidValue;
}

}  // namespace mxfft
