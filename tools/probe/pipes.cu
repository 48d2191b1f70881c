// Throughput probe: warp-instructions per cycle per SM for the instruction
// kinds of the MX butterfly (FFMA, FMUL, FHFMA (mixed f16*f16+f32), HADD2.F32,
// F2FP pack/unpack, FMNMX3, LOP3), 8 independent chains per thread, 4 warps per
// SMSP.  usage: ./pipes
#include <cstdio>
#include <cuda_fp16.h>
#define N_IT 4096
template <int KIND>
__global__ void k(float* out, long long* cyc) {
    float a[8];
    unsigned h[8];
    for (int i = 0; i < 8; ++i) { a[i] = threadIdx.x * 0.001f + i; h[i] = 0x3c003c00u + i; }
    const float b = 1.0001f, c = 0.999f;
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < N_IT; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if (KIND == 0) asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(a[i]) : "f"(b), "f"(a[(i + 1) & 7]));
            if (KIND == 1) asm volatile("mul.rn.f32 %0, %0, %1;" : "+f"(a[i]) : "f"(a[(i + 3) & 7]));
            if (KIND == 2) asm volatile("{.reg .f16 l, hh; mov.b32 {l, hh}, %1; fma.rn.f32.f16 %0, l, hh, %0;}" : "+f"(a[i]) : "r"(h[i]));
            if (KIND == 3) asm volatile("{.reg .f16 l, hh; mov.b32 {l, hh}, %1; cvt.f32.f16 %0, hh;}" : "=f"(a[i]) : "r"(h[(i + it) & 7]));
            if (KIND == 4) { unsigned short p; asm volatile("cvt.rn.satfinite.e4m3x2.f32 %0, %1, %2;" : "=h"(p) : "f"(a[i]), "f"(a[(i+1)&7])); asm volatile("cvt.rn.f16x2.e4m3x2 %0, %1;" : "=r"(h[i]) : "h"(p)); }
            if (KIND == 5) asm volatile("max.f32 %0, %0, %1;" : "+f"(a[i]) : "f"(a[(i + 5) & 7]));
            if (KIND == 6) asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(h[i]) : "r"(h[(i + 1) & 7]), "r"(h[(i + 2) & 7]));
            if (KIND == 7) asm volatile("fma.rn.f32 %0, %1, %2, %0;" : "+f"(a[i]) : "f"(a[(i + 1) & 7]), "f"(a[(i + 2) & 7]));
        }
    }
    long long t1 = clock64();
    float s = 0; for (int i = 0; i < 8; ++i) s += a[i] + (float)h[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
template <int KIND>
void run(const char* name, float* d, long long* c) {
    k<KIND><<<148, 512>>>(d, c);
    cudaDeviceSynchronize();
    k<KIND><<<148, 512>>>(d, c);
    long long h[148];
    cudaMemcpy(h, c, sizeof(h), cudaMemcpyDeviceToHost);
    double cy = 0; for (int i = 0; i < 148; ++i) cy += h[i]; cy /= 148;
    // per SMSP: 4 warps x N_IT x 8 instructions (+ unpack for KIND 4 counted as 2)
    double instr = 4.0 * N_IT * 8 * (KIND == 4 ? 2 : 1);
    printf("%-34s %.3f warp-instr/cycle/SMSP (%.2f cycles each)\n", name, instr / cy, cy / instr);
}
int main() {
    float* d; long long* c;
    cudaMalloc(&d, 148 * 512 * 4); cudaMalloc(&c, 148 * 8);
    run<0>("FFMA (a*imm-ish reg + reg)", d, c);
    run<7>("FFMA 3-reg", d, c);
    run<1>("FMUL", d, c);
    run<2>("FHFMA f16*f16+f32", d, c);
    run<3>("HADD2.F32 / cvt f16->f32", d, c);
    run<4>("F2FP pack + unpack (pair)", d, c);
    run<5>("FMNMX", d, c);
    run<6>("LOP3", d, c);
    return 0;
}
