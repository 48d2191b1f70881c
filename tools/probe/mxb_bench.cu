// Compute roofline of the MX butterfly block: runs the line kernel's own
// general block (mxb, NB = 16) and stage-0/1 block (trivial_block) on
// register data in a loop, 4 warps per SMSP on every SM, and reports cycles
// per butterfly per SMSP.  usage: ./mxb_bench
#include <cstdio>
#include "../../paper_2512_04317_b200/csrc/mxfft_lines.cuh"
using namespace mxfft;
#define ITERS 512
__device__ __forceinline__ void dec_h(unsigned q, unsigned short sp, unsigned short sn, float2 u,
                                      float2& uo, float2& vo) {
    asm("{\n\t.reg .f16 ql, qh, a, b;\n\t"
        "mov.b32 {ql, qh}, %4;\n\tmov.b16 a, %5;\n\tmov.b16 b, %6;\n\t"
        "fma.rn.f32.f16 %0, ql, a, %7;\n\t"
        "fma.rn.f32.f16 %1, qh, a, %8;\n\t"
        "fma.rn.f32.f16 %2, ql, b, %7;\n\t"
        "fma.rn.f32.f16 %3, qh, b, %8;\n\t}"
        : "=&f"(uo.x), "=&f"(uo.y), "=&f"(vo.x), "=&f"(vo.y)
        : "r"(q), "h"(sp), "h"(sn), "f"(u.x), "f"(u.y));
}
// mxb with the decode as mixed f16 FMAs (no f16->f32 conversions); no fallback
template <int ID, int NB>
__device__ __forceinline__ void mxb_h(float2 (&u)[NB], float2 (&v)[NB], const unsigned (&w)[NB], int ew, bool& bad) {
    using F = HwFmt<ID>;
    const float am = amax_c<NB>(v);
    const int ev = am > 0.f ? floor_log2f(am) - F::EMAX : 0;
    const float inv = exp2i(-ev);
    unsigned cv[NB];
    float pr[NB], pi[NB];
#pragma unroll
    for (int i = 0; i < NB; ++i) {
        cv[i] = q2h<ID>(v[i].x * inv, v[i].y * inv);
        cprod(w[i], cv[i], pr[i], pi[i]);
    }
    const float ap = amax_2<NB>(pr, pi);
    const int sh = ap > F::MAXF ? shift_for<F>(ap) : 0;
    const int E = ew + ev + sh;
    bad |= !((unsigned)(E + 24) <= 39u) | (ev < -127);
    const float fac = exp2i(-sh);
    const unsigned short sp = (unsigned short)(E >= -14 ? (E + 15) << 10 : 1 << (E + 24)), sn = sp | 0x8000;
#pragma unroll
    for (int i = 0; i < NB; ++i) {
        const unsigned qp = q2h<ID>(pr[i] * fac, pi[i] * fac);
        const float2 uu = u[i];
        dec_h(qp, sp, sn, uu, u[i], v[i]);
    }
}
template <int MODE>
__global__ void k(float* out, long long* cyc, unsigned wseed) {
    float2 u[16], v[16];
    unsigned w[16];
    for (int i = 0; i < 16; ++i) {
        u[i] = make_float2(0.01f * (threadIdx.x + i), -0.02f * i);
        v[i] = make_float2(0.03f * i - 0.1f, 0.001f * threadIdx.x);
        w[i] = wseed + 0x00010001u * i;
    }
    bool bad = false;
    LDbg* d = nullptr;
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < ITERS; ++it) {
        if (MODE == 0) mxb<F_E4M3, 16, false, false>(u, v, w, -8, d, 0, bad);
        else if (MODE == 1) trivial_block<F_E4M3, 16, false, 1, false>(u, v, 0, 1.f, d, 0);
        else if (MODE == 2) mxb_h<F_E4M3, 16>(u, v, w, -8, bad);
        // keep magnitudes bounded: swap roles and rescale
#pragma unroll
        for (int i = 0; i < 16; ++i) { float2 t = u[i]; u[i] = make_float2(v[i].x * 0.5f, v[i].y * 0.5f); v[i] = t; }
    }
    long long t1 = clock64();
    float s = bad;
    for (int i = 0; i < 16; ++i) s += u[i].x + v[i].y;
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
template <int MODE>
void run(const char* name, float* d, long long* c) {
    for (int rep = 0; rep < 2; ++rep) k<MODE><<<148, 512>>>(d, c, 0x3c003800u);
    cudaDeviceSynchronize();
    long long h[148];
    cudaMemcpy(h, c, sizeof(h), cudaMemcpyDeviceToHost);
    double cy = 0; for (int i = 0; i < 148; ++i) cy += h[i]; cy /= 148;
    // per SMSP: 4 warps x ITERS x 16 butterflies x 32 lanes
    const double bf = 4.0 * ITERS * 16;
    printf("%-28s %.2f cycles per warp-butterfly per SMSP\n", name, cy / bf);
}
int main() {
    float* d; long long* c;
    cudaMalloc(&d, 148 * 512 * 4); cudaMalloc(&c, 148 * 8);
    run<0>("general block (mxb)", d, c);
    run<1>("stage-1 block (trivial)", d, c);
    run<2>("general block, f16 decode", d, c);
    run<3>("harness only (swap/rescale)", d, c);
    return 0;
}
