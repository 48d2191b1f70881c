// Throughput of the conversion instructions of the MX butterfly, as
// dependent chains (8 per thread, 4 warps per SMSP) so ptxas cannot drop them.
#include <cstdio>
#define N_IT 2048
template <int KIND>
__global__ void k(unsigned* out, long long* cyc) {
    unsigned h[8];
    for (int i = 0; i < 8; ++i) h[i] = 0x3c003c00u + threadIdx.x * 17 + i;
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < N_IT; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if (KIND == 0)  // F2FP pack (e4m3x2 from two f32)
                asm volatile("{.reg .b16 p; cvt.rn.satfinite.e4m3x2.f32 p, %0, %0; mov.b32 %0, {p, p};}" : "+r"(h[i]));
            if (KIND == 1)  // F2FP unpack (e4m3x2 -> f16x2)
                asm volatile("{.reg .b16 p, q; mov.b32 {p, q}, %0; cvt.rn.f16x2.e4m3x2 %0, p;}" : "+r"(h[i]));
            if (KIND == 2)  // HADD2.F32 (f16 -> f32)
                asm volatile("{.reg .f16 l, hh; .reg .f32 f; mov.b32 {l, hh}, %0; cvt.f32.f16 f, hh; mov.b32 %0, f;}" : "+r"(h[i]));
            if (KIND == 3)  // FMNMX3 style: max of 3
                asm volatile("{.reg .f32 a, b; mov.b32 a, %0; max.f32 b, a, %1; max.f32 b, b, %2; mov.b32 %0, b;}" : "+r"(h[i]) : "f"(1.0f), "f"(2.0f));
            if (KIND == 4)  // FFMA dependent
                asm volatile("{.reg .f32 a; mov.b32 a, %0; fma.rn.f32 a, a, a, a; mov.b32 %0, a;}" : "+r"(h[i]));
        }
    }
    long long t1 = clock64();
    unsigned s = 0; for (int i = 0; i < 8; ++i) s += h[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
template <int KIND>
void run(const char* name, unsigned* d, long long* c) {
    for (int r = 0; r < 2; ++r) k<KIND><<<148, 512>>>(d, c);
    cudaDeviceSynchronize();
    long long h[148];
    cudaMemcpy(h, c, sizeof(h), cudaMemcpyDeviceToHost);
    double cy = 0; for (int i = 0; i < 148; ++i) cy += h[i]; cy /= 148;
    printf("%-28s %.2f cycles per warp-op per SMSP\n", name, cy / (4.0 * N_IT * 8));
}
int main() {
    unsigned* d; long long* c;
    cudaMalloc(&d, 148 * 512 * 4); cudaMalloc(&c, 148 * 8);
    run<0>("F2FP pack e4m3x2", d, c);
    run<1>("F2FP unpack e4m3x2->f16x2", d, c);
    run<2>("HADD2.F32 (cvt f16->f32)", d, c);
    run<3>("FMNMX3 (max of 3)", d, c);
    run<4>("FFMA", d, c);
    return 0;
}
