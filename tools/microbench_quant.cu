// Microbenchmark: throughput of the hardware F2FP minifloat pack/unpack versus
// a software RNE quantizer on the FMA/ALU pipes (sm_100a).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mbq tools/microbench_quant.cu
#include <cstdio>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

constexpr int ILP = 8;
constexpr int ITERS = 4096;

__device__ __forceinline__ void hwq(float a, float b, float& qa, float& qb) {
    unsigned short p;
    unsigned h;
    asm volatile("cvt.rn.satfinite.e4m3x2.f32 %0, %1, %2;" : "=h"(p) : "f"(a), "f"(b));
    asm volatile("cvt.rn.f16x2.e4m3x2 %0, %1;" : "=r"(h) : "h"(p));
    __half2 hv = *reinterpret_cast<__half2*>(&h);
    qa = __high2float(hv);
    qb = __low2float(hv);
}

// software RNE onto E4M3 (value grid with binade floor at EMIN=-6, M=3), clamp 448
__device__ __forceinline__ float swq(float y) {
    unsigned b = __float_as_uint(y) & 0x7f800000u;
    b = max(b, (unsigned)(127 - 6) << 23);
    float c = __uint_as_float(b + ((23u - 3u) << 23) + 0x400000u);
    float q = __fsub_rn(__fadd_rn(y, c), c);
    return fminf(fmaxf(q, -448.f), 448.f);
}

// variant with DPX viaddmax: max(bits&mask + K, EMB + K)
__device__ __forceinline__ float swq2(float y) {
    int b = (int)(__float_as_uint(y) & 0x7f800000u);
    int c = __viaddmax_s32(b, (int)(((23u - 3u) << 23) + 0x400000u), (int)((((127u - 6u) << 23)) + ((23u - 3u) << 23) + 0x400000u));
    float cf = __int_as_float(c);
    float q = __fsub_rn(__fadd_rn(y, cf), cf);
    return fminf(fmaxf(q, -448.f), 448.f);
}

template <int MODE>
__global__ void kbench(float* out, float seed) {
    float x[ILP], y[ILP];
#pragma unroll
    for (int i = 0; i < ILP; ++i) {
        x[i] = seed * (threadIdx.x + 1 + i) * 0.37f;
        y[i] = seed * (threadIdx.x + 3 + i) * 0.91f;
    }
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int i = 0; i < ILP; ++i) {
            if (MODE == 0) {  // FFMA baseline: 2 FFMA per pair
                x[i] = __fmaf_rn(x[i], 1.0001f, 0.5f);
                y[i] = __fmaf_rn(y[i], 0.9999f, 0.25f);
            } else if (MODE == 1) {  // HW pack+unpack (+2 HADD2.F32) per pair, + 2 FFMA perturb
                float qa, qb;
                hwq(x[i], y[i], qa, qb);
                x[i] = __fmaf_rn(qa, 1.0001f, 0.5f);
                y[i] = __fmaf_rn(qb, 0.9999f, 0.25f);
            } else if (MODE == 2) {  // SW quantizer on both + 2 FFMA perturb
                x[i] = __fmaf_rn(swq(x[i]), 1.0001f, 0.5f);
                y[i] = __fmaf_rn(swq(y[i]), 0.9999f, 0.25f);
            } else if (MODE == 3) {
                x[i] = __fmaf_rn(swq2(x[i]), 1.0001f, 0.5f);
                y[i] = __fmaf_rn(swq2(y[i]), 0.9999f, 0.25f);
            } else if (MODE == 4) {  // HW pack only (packed result fed back through an int op)
                unsigned short p;
                asm volatile("cvt.rn.satfinite.e4m3x2.f32 %0, %1, %2;" : "=h"(p) : "f"(x[i]), "f"(y[i]));
                x[i] = __fmaf_rn(x[i], 1.0001f, (float)(p & 1));
                y[i] = __fmaf_rn(y[i], 0.9999f, 0.25f);
            }
        }
    }
    float s = 0;
#pragma unroll
    for (int i = 0; i < ILP; ++i) s += x[i] + y[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int MODE>
float run(float* d, int blocks, int threads) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    kbench<MODE><<<blocks, threads>>>(d, 1.0f);
    cudaEventRecord(a);
    kbench<MODE><<<blocks, threads>>>(d, 1.0f);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    return ms;
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int clk;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    const int threads = 256, blocks = sms * 8;
    float* d;
    cudaMalloc(&d, sizeof(float) * blocks * threads);
    const double pairs = (double)blocks * threads * ITERS * ILP;  // value pairs processed
    const char* names[] = {"FFMA baseline (2 FFMA/pair)", "HW F2FP pack+unpack+2cvt (+2 FFMA)/pair",
                           "SW quantizer x2 (+2 FFMA)/pair", "SW quantizer (viaddmax) x2 (+2 FFMA)/pair",
                           "HW F2FP pack only (+2 FFMA)/pair"};
    float ms[5] = {run<0>(d, blocks, threads), run<1>(d, blocks, threads), run<2>(d, blocks, threads),
                   run<3>(d, blocks, threads), run<4>(d, blocks, threads)};
    for (int m = 0; m < 5; ++m) {
        double per_sm_clk = pairs / (ms[m] * 1e-3) / sms / (clk * 1e3);
        printf("%-45s %8.3f ms  %7.2f pairs/clk/SM (at %d MHz nominal)\n", names[m], ms[m], per_sm_clk, clk / 1000);
    }
    return 0;
}
