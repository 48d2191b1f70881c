// Probe: is fma.rn.f32.f16 exact for subnormal f16 operands (2^-24..2^-15)?
// Compares against FP64 for every power-of-two scale E in [-24, 15] and many
// codes / addends; prints the number of mismatches per E.
#include <cstdio>
#include <cuda_fp16.h>
__global__ void k(int* bad, int n) {
    const int E = (int)blockIdx.x - 24;  // -24..15
    unsigned short s16 = E >= -14 ? (unsigned short)((E + 15) << 10) : (unsigned short)(1u << (E + 24));
    int nb = 0;
    for (int t = threadIdx.x; t < n; t += blockDim.x) {
        // code: f16 with 4 significant bits, random-ish exponent in [-9, 8]
        unsigned h = (unsigned)t * 2654435761u;
        int ce = (int)((h >> 8) % 18) - 9;
        int cm = (h >> 4) & 7;
        float cf = ldexpf(1.0f + cm / 8.0f, ce) * ((h & 1) ? -1.f : 1.f);
        __half ch = __float2half_rn(cf);
        unsigned short cb = __half_as_ushort(ch);
        float u = __int_as_float((int)(h * 747796405u) & 0x7f7fffff) ;  // finite
        u = ldexpf(frexpf(u, &ce), (int)((h >> 12) % 60) - 40);
        float d;
        asm("{\n\t.reg .f16 a, b;\n\tmov.b16 a, %1;\n\tmov.b16 b, %2;\n\tfma.rn.f32.f16 %0, a, b, %3;\n\t}"
            : "=f"(d) : "h"(cb), "h"(s16), "f"(u));
        const float ref = __fmaf_rn(__half2float(ch), ldexpf(1.f, E), u);
        if (__float_as_int(d) != __float_as_int(ref)) ++nb;
    }
    atomicAdd(&bad[blockIdx.x], nb);
}
int main() {
    int* d; cudaMalloc(&d, 64 * 4); cudaMemset(d, 0, 256);
    k<<<40, 256>>>(d, 1 << 20);
    int h[40]; cudaMemcpy(h, d, 160, cudaMemcpyDeviceToHost);
    for (int i = 0; i < 40; ++i) printf("E=%d mismatches=%d\n", i - 24, h[i]);
    return 0;
}
