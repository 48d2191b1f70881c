#include <cstdio>
#include <cuda_fp16.h>
__global__ void k(float* out) {
    float c[4] = {0.0287f, 83.2667f, 1.0f + 1.0f/4096, -0.013f};
    unsigned short a16[4] = {0x3c00 /*1*/, 0x4000 /*2*/, 0x2c00 /*2^-4*/, 0x1c00 /*2^-8*/};
    unsigned short b16 = 0x2400; // 2^-6
    for (int i = 0; i < 4; ++i) {
        float d;
        asm("{\n\t.reg .f16 a, b;\n\tmov.b16 a, %1;\n\tmov.b16 b, %2;\n\tfma.rn.f32.f16 %0, a, b, %3;\n\t}"
            : "=f"(d) : "h"(a16[i]), "h"(b16), "f"(c[i]));
        float ref = __fmaf_rn(__half2float(__ushort_as_half(a16[i])), __half2float(__ushort_as_half(b16)), c[i]);
        out[2*i] = d; out[2*i+1] = ref;
    }
    // packed variant like dec_h
    unsigned q = (0x4000u << 16) | 0x3c00u;  // lo = 1, hi = 2
    float2 u = make_float2(0.0287f, 83.2667f);
    float r0, r1, r2, r3;
    unsigned short sp = 0x2400, sn = 0xa400;
    asm("{\n\t.reg .f16 ql, qh, a, b;\n\t"
        "mov.b32 {ql, qh}, %4;\n\tmov.b16 a, %5;\n\tmov.b16 b, %6;\n\t"
        "fma.rn.f32.f16 %0, ql, a, %7;\n\t"
        "fma.rn.f32.f16 %1, qh, a, %8;\n\t"
        "fma.rn.f32.f16 %2, ql, b, %7;\n\t"
        "fma.rn.f32.f16 %3, qh, b, %8;\n\t}"
        : "=f"(r0), "=f"(r1), "=f"(r2), "=f"(r3) : "r"(q), "h"(sp), "h"(sn), "f"(u.x), "f"(u.y));
    out[8] = r0; out[9] = u.x + 1.f/64; out[10] = r1; out[11] = u.y + 2.f/64;
    out[12] = r2; out[13] = u.x - 1.f/64; out[14] = r3; out[15] = u.y - 2.f/64;
}
int main() {
    float* d; cudaMalloc(&d, 64 * 4); k<<<1, 1>>>(d); float h[16]; cudaMemcpy(h, d, 64, cudaMemcpyDeviceToHost);
    for (int i = 0; i < 8; ++i) printf("got %.9g  ref %.9g\n", h[2*i], h[2*i+1]);
    return 0;
}
