// Issue-rate probe for the instruction kinds of the MX butterfly on sm_100a:
// cycles per warp-instruction per SMSP, 8 independent chains per thread,
// W warps per SMSP.  Also pairs of kinds, to see which share a pipe.
// usage: ./pipes3
#include <cstdio>
#include <cuda_fp16.h>
#define N_IT 2048

enum { PACK, UNPACK, FMNMX3, FMNMX, FFMA, FFMA2, FMUL2, FHFMA, PRMT, LOP3, IMAD, SHF, VIMNMX3, HMNMX2, PACKBF, IADD3, Q2H, NK };
static const char* NAMES[NK] = {"F2FP pack e4m3x2<-f32", "F2FP unpack f16x2<-e4m3x2", "FMNMX3", "FMNMX", "FFMA",
                                "FFMA2", "FMUL2", "FHFMA", "PRMT", "LOP3", "IMAD", "SHF", "VIMNMX3.u16x2", "HMNMX2",
                                "F2FP pack bf16x2<-f32", "IADD3", "pack+unpack (2 instr)"};

template <int KIND>
__device__ __forceinline__ void op(unsigned& r, unsigned long long& rr, unsigned s1, unsigned s2) {
    if (KIND == PACK) {
        unsigned short p;
        asm volatile("cvt.rn.satfinite.e4m3x2.f32 %0, %1, %2;" : "=h"(p) : "f"(__uint_as_float(r)), "f"(__uint_as_float(s1)));
        r = p;
    }
    if (KIND == UNPACK) {
        asm volatile("cvt.rn.f16x2.e4m3x2 %0, %1;" : "=r"(r) : "h"((unsigned short)r));
    }
    if (KIND == Q2H) {
        unsigned short p;
        asm volatile("cvt.rn.satfinite.e4m3x2.f32 %0, %1, %2;" : "=h"(p) : "f"(__uint_as_float(r)), "f"(__uint_as_float(s1)));
        asm volatile("cvt.rn.f16x2.e4m3x2 %0, %1;" : "=r"(r) : "h"(p));
    }
    if (KIND == FMNMX3)
        asm volatile("{.reg .f32 a, b, c; mov.b32 a, %0; mov.b32 b, %1; mov.b32 c, %2; max.f32 a, a, b, c; mov.b32 %0, a;}"
                     : "+r"(r) : "r"(s1), "r"(s2));
    if (KIND == FMNMX)
        asm volatile("{.reg .f32 a, b; mov.b32 a, %0; mov.b32 b, %1; max.f32 a, a, b; mov.b32 %0, a;}" : "+r"(r) : "r"(s1));
    if (KIND == FFMA)
        asm volatile("{.reg .f32 a, b, c; mov.b32 a, %0; mov.b32 b, %1; mov.b32 c, %2; fma.rn.f32 a, a, b, c; mov.b32 %0, a;}"
                     : "+r"(r) : "r"(s1), "r"(s2));
    if (KIND == FFMA2)
        asm volatile("{.reg .b64 b; mov.b64 b, {%1, %2}; fma.rn.f32x2 %0, %0, b, b;}" : "+l"(rr) : "r"(s1), "r"(s2));
    if (KIND == FMUL2)
        asm volatile("{.reg .b64 b; mov.b64 b, {%1, %2}; mul.rn.f32x2 %0, %0, b;}" : "+l"(rr) : "r"(s1), "r"(s2));
    if (KIND == FHFMA)
        asm volatile("{.reg .f16 l, h; .reg .f32 a; mov.b32 {l, h}, %1; mov.b32 a, %0; fma.rn.f32.f16 a, l, h, a; mov.b32 %0, a;}"
                     : "+r"(r) : "r"(s1));
    if (KIND == PRMT) asm volatile("prmt.b32 %0, %0, %1, 0x7250;" : "+r"(r) : "r"(s1));
    if (KIND == LOP3) asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(r) : "r"(s1), "r"(s2));
    if (KIND == IMAD) asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(r) : "r"(s1), "r"(s2));
    if (KIND == SHF) asm volatile("shf.l.wrap.b32 %0, %0, %1, 7;" : "+r"(r) : "r"(s1));
    if (KIND == VIMNMX3) r = __vimax3_u16x2(r, s1, s2);
    if (KIND == HMNMX2) asm volatile("max.f16x2 %0, %0, %1;" : "+r"(r) : "r"(s1));
    if (KIND == PACKBF)
        asm volatile("{.reg .f32 a, b; mov.b32 a, %0; mov.b32 b, %1; cvt.rz.bf16x2.f32 %0, a, b;}" : "+r"(r) : "r"(s1));
    if (KIND == IADD3) asm volatile("{.reg .u32 t; add.u32 t, %0, %1; add.u32 %0, t, %2;}" : "+r"(r) : "r"(s1), "r"(s2));
}

// NA ops of kind A and NB ops of kind B per chain step, interleaved
template <int A, int B, int NA, int NB>
__global__ void k(unsigned* out, long long* cyc) {
    unsigned h[8];
    unsigned long long hh[8];
    for (int i = 0; i < 8; ++i) {
        h[i] = 0x3c003c00u + threadIdx.x * 17 + i;
        hh[i] = 0x3f8000003f800000ull + threadIdx.x + i;
    }
    unsigned g[8];
    unsigned long long gg[8];
    for (int i = 0; i < 8; ++i) g[i] = h[i] ^ 0x1234u, gg[i] = hh[i] + 5;
    const unsigned s1 = 0x3f800100u + threadIdx.x, s2 = 0x3f900000u;
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < N_IT; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
#pragma unroll
            for (int a = 0; a < NA; ++a) op<A>(h[i], hh[i], s1, s2);
#pragma unroll
            for (int b = 0; b < NB; ++b) op<B>(g[i], gg[i], s1, s2);
        }
    }
    long long t1 = clock64();
    unsigned s = 0;
    for (int i = 0; i < 8; ++i) s += h[i] + g[i] + (unsigned)hh[i] + (unsigned)gg[i] + (unsigned)(hh[i] >> 32) + (unsigned)(gg[i] >> 32);
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int A, int B, int NA, int NB>
void run(unsigned* d, long long* c, int threads) {
    for (int r = 0; r < 2; ++r) k<A, B, NA, NB><<<148, threads>>>(d, c);
    cudaDeviceSynchronize();
    long long h[148];
    cudaMemcpy(h, c, sizeof(h), cudaMemcpyDeviceToHost);
    double cy = 0;
    for (int i = 0; i < 148; ++i) cy += h[i];
    cy /= 148;
    const double wps = threads / 128.0;
    const double steps = wps * N_IT * 8;
    if (NB == 0)
        printf("%-28s x%d  W=%2.0f: %.2f cycles per warp-op per SMSP\n", NAMES[A], NA, wps, cy / (steps * NA));
    else
        printf("%-28s x%d + %-28s x%d  W=%2.0f: %.2f cycles per step per SMSP\n", NAMES[A], NA, NAMES[B], NB, wps,
               cy / steps);
}

template <int A>
void single(unsigned* d, long long* c) {
    run<A, A, 1, 0>(d, c, 512);
    run<A, A, 1, 0>(d, c, 1024);
}

int main() {
    unsigned* d;
    long long* c;
    cudaMalloc(&d, 148 * 1024 * 4);
    cudaMalloc(&c, 148 * 8);
    single<PACK>(d, c);
    single<UNPACK>(d, c);
    single<FMNMX3>(d, c);
    single<FMNMX>(d, c);
    single<FFMA>(d, c);
    single<FFMA2>(d, c);
    single<FMUL2>(d, c);
    single<FHFMA>(d, c);
    single<PRMT>(d, c);
    single<LOP3>(d, c);
    single<IMAD>(d, c);
    single<SHF>(d, c);
    single<VIMNMX3>(d, c);
    single<HMNMX2>(d, c);
    single<PACKBF>(d, c);
    single<IADD3>(d, c);
    single<Q2H>(d, c);
    run<Q2H, FFMA, 1, 1>(d, c, 1024);
    run<Q2H, FFMA, 1, 2>(d, c, 1024);
    run<Q2H, FFMA, 1, 3>(d, c, 1024);
    run<Q2H, FFMA, 1, 4>(d, c, 1024);
    run<Q2H, FMNMX3, 2, 1>(d, c, 1024);
    run<Q2H, FMNMX3, 1, 1>(d, c, 1024);
    // which kinds share a pipe: A x1 + B x1 per step (sum of singles = shared, max = independent)
    run<PACK, UNPACK, 1, 1>(d, c, 1024);
    run<PACK, FMNMX3, 1, 1>(d, c, 1024);
    run<UNPACK, FMNMX3, 1, 1>(d, c, 1024);
    run<PACK, LOP3, 1, 1>(d, c, 1024);
    run<UNPACK, LOP3, 1, 1>(d, c, 1024);
    run<PACK, FFMA, 1, 1>(d, c, 1024);
    run<UNPACK, FFMA, 1, 1>(d, c, 1024);
    run<PACK, FHFMA, 1, 1>(d, c, 1024);
    run<FMNMX3, FFMA, 1, 1>(d, c, 1024);
    run<FMNMX3, LOP3, 1, 1>(d, c, 1024);
    run<FFMA, FHFMA, 1, 1>(d, c, 1024);
    run<FFMA2, FHFMA, 1, 1>(d, c, 1024);
    run<FFMA2, FFMA, 1, 1>(d, c, 1024);
    run<IMAD, FFMA, 1, 1>(d, c, 1024);
    run<IMAD, LOP3, 1, 1>(d, c, 1024);
    run<PRMT, LOP3, 1, 1>(d, c, 1024);
    run<PRMT, FFMA, 1, 1>(d, c, 1024);
    run<PACK, PRMT, 1, 1>(d, c, 1024);
    run<PACK, IMAD, 1, 1>(d, c, 1024);
    // the butterfly's mix: 2 pack + 2 unpack + 2 FMNMX3 against 10 FMA-pipe ops
    run<PACK, FFMA, 2, 5>(d, c, 1024);
    return 0;
}
