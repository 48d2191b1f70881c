// mxfft_common.cuh -- shared device code for the B200-native MX-FFT (sm_100a).
//
// Element formats, the reference FP64 quantizer (minifloat.py:105-120), and the
// hardware quantizers built on sm_100a's F2FP.SATFINITE packs: cvt.rn.satfinite
// .{e4m3,e5m2,e2m3,e3m2,e2m1}x2.f32 (RNE + saturation) and the matching
// cvt.rn.f16x2.*x2 unpacks.  The MX transform carries FP32 (fftcore.py:7-12),
// so every quantized value is handed back as an exact FP32 "code" (a decoded
// element-format real, exactly like the reference's MxBlock.codes).
#pragma once

#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace mxfft {

enum Policy { POL_IEEE = 0, POL_EXTENDED = 1, POL_FINITE = 2 };
enum FmtId { F_E4M3 = 0, F_E5M2 = 1, F_E2M3 = 2, F_E3M2 = 3, F_E2M1 = 4, F_GENERIC = 5 };

// Runtime format descriptor with the derived constants of MinifloatFormat
// (minifloat.py:56-81) and the product-dtype rule of fftcore.py:163.
struct FmtDesc {
    int ebits, mbits, policy, bias;
    int emin, emax;
    double max_finite;
    int prod_f32;  // 1: mantissa products in FP32, 0: FP64 (wide test formats)
    int id;        // FmtId
};

__host__ __device__ inline FmtDesc make_fmt(int ebits, int mbits, int policy, int bias) {
    FmtDesc f;
    f.ebits = ebits;
    f.mbits = mbits;
    f.policy = policy;
    f.bias = bias;
    f.emin = 1 - bias;
    int top = (1 << ebits) - 1;
    if (policy == POL_IEEE) top -= 1;
    f.emax = top - bias;
    int m = 1 << mbits;
    int frac = (policy == POL_EXTENDED) ? m + (m - 2) : m + (m - 1);
    double mf = (double)frac;
    int sh = f.emax - mbits;
    // ldexp without <cmath> host/device ambiguity
    if (sh >= 0)
        for (int i = 0; i < sh; ++i) mf *= 2.0;
    else
        for (int i = 0; i < -sh; ++i) mf *= 0.5;
    f.max_finite = mf;
    f.prod_f32 = 2 * (f.emax + 1) <= 126;
    f.id = F_GENERIC;
    if (ebits == 4 && mbits == 3 && policy == POL_EXTENDED && bias == 7) f.id = F_E4M3;
    if (ebits == 5 && mbits == 2 && policy == POL_IEEE && bias == 15) f.id = F_E5M2;
    if (ebits == 2 && mbits == 3 && policy == POL_FINITE && bias == 1) f.id = F_E2M3;
    if (ebits == 3 && mbits == 2 && policy == POL_FINITE && bias == 3) f.id = F_E3M2;
    if (ebits == 2 && mbits == 1 && policy == POL_FINITE && bias == 1) f.id = F_E2M1;
    return f;
}

// ---------------------------------------------------------------------------
// Reference quantizer, FP64, literal restatement of minifloat.py:114-120:
// binade max(floor(log2|x|), emin), step 2^(eb-M), rint (half-even), clip.
// ---------------------------------------------------------------------------
__device__ __forceinline__ double quantize_ref(double x, const FmtDesc& f) {
    int e;
    frexp(fabs(x), &e);
    int eb = e - 1;
    eb = eb < f.emin ? f.emin : eb;
    double step = ldexp(1.0, eb - f.mbits);
    double q = rint(x / step) * step;
    q = fmin(q, f.max_finite);
    q = fmax(q, -f.max_finite);
    return q;
}

// block_scales (mxblock.py:27-38) as an exponent: log2 of the shared scale.
__device__ __forceinline__ int block_scale_exp(double amax, const FmtDesc& f) {
    if (!(amax > 0.0)) return 0;
    int e;
    frexp(amax, &e);
    int se = e - 1 - f.emax;
    se = se < -1022 ? -1022 : (se > 1023 ? 1023 : se);
    return se;
}

// ---------------------------------------------------------------------------
// FP32 bit helpers
// ---------------------------------------------------------------------------
// floor(log2 x) for finite x > 0, subnormals included (frexp semantics).
__device__ __forceinline__ int floor_log2f(float x) {
    unsigned b = __float_as_uint(x) & 0x7fffffffu;
    int e = (int)(b >> 23);
    return e ? e - 127 : (31 - __clz(b)) - 149;
}

// 2^e as a normal float; valid for e in [-126, 127].
__device__ __forceinline__ float exp2i(int e) { return __int_as_float((e + 127) << 23); }

__device__ __forceinline__ float fmax3(float a, float b, float c) { return fmaxf(fmaxf(a, b), c); }

// ---------------------------------------------------------------------------
// Hardware quantizers.  q2(a, b) rounds both inputs onto the format grid
// (RNE, saturating at +-max_finite) and returns the decoded codes as FP32.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void unpack_f16x2(unsigned h, float& hi, float& lo) {
    __half2 hv = *reinterpret_cast<__half2*>(&h);
    lo = __low2float(hv);
    hi = __high2float(hv);
}

template <int ID>
struct HwFmt;

// EM / MM: floor(log2 max_finite) and its FP32 mantissa field (for the exact
// integer renormalization shift, see shift_for()).  ELO/EHI: range of the
// product exponent E for which code * 2^E is an exact normal FP32 value.
template <>
struct HwFmt<F_E4M3> {
    static constexpr int EMAX = 8, EMIN = -6, M = 3, EM = 8;
    static constexpr unsigned MM = 0x600000u;
    static constexpr float MAXF = 448.0f;
    __device__ static __forceinline__ void q2(float a, float b, float& qa, float& qb) {
        unsigned short p;
        unsigned h;
        asm("cvt.rn.satfinite.e4m3x2.f32 %0, %1, %2;" : "=h"(p) : "f"(a), "f"(b));
        asm("cvt.rn.f16x2.e4m3x2 %0, %1;" : "=r"(h) : "h"(p));
        unpack_f16x2(h, qa, qb);
    }
};
template <>
struct HwFmt<F_E5M2> {
    static constexpr int EMAX = 15, EMIN = -14, M = 2, EM = 15;
    static constexpr unsigned MM = 0x600000u;
    static constexpr float MAXF = 57344.0f;
    __device__ static __forceinline__ void q2(float a, float b, float& qa, float& qb) {
        unsigned short p;
        unsigned h;
        asm("cvt.rn.satfinite.e5m2x2.f32 %0, %1, %2;" : "=h"(p) : "f"(a), "f"(b));
        asm("cvt.rn.f16x2.e5m2x2 %0, %1;" : "=r"(h) : "h"(p));
        unpack_f16x2(h, qa, qb);
    }
};
template <>
struct HwFmt<F_E2M3> {
    static constexpr int EMAX = 2, EMIN = 0, M = 3, EM = 2;
    static constexpr unsigned MM = 0x700000u;
    static constexpr float MAXF = 7.5f;
    __device__ static __forceinline__ void q2(float a, float b, float& qa, float& qb) {
        unsigned short p;
        unsigned h;
        asm("cvt.rn.satfinite.e2m3x2.f32 %0, %1, %2;" : "=h"(p) : "f"(a), "f"(b));
        asm("cvt.rn.f16x2.e2m3x2 %0, %1;" : "=r"(h) : "h"(p));
        unpack_f16x2(h, qa, qb);
    }
};
template <>
struct HwFmt<F_E3M2> {
    static constexpr int EMAX = 4, EMIN = -2, M = 2, EM = 4;
    static constexpr unsigned MM = 0x600000u;
    static constexpr float MAXF = 28.0f;
    __device__ static __forceinline__ void q2(float a, float b, float& qa, float& qb) {
        unsigned short p;
        unsigned h;
        asm("cvt.rn.satfinite.e3m2x2.f32 %0, %1, %2;" : "=h"(p) : "f"(a), "f"(b));
        asm("cvt.rn.f16x2.e3m2x2 %0, %1;" : "=r"(h) : "h"(p));
        unpack_f16x2(h, qa, qb);
    }
};
template <>
struct HwFmt<F_E2M1> {
    static constexpr int EMAX = 2, EMIN = 0, M = 1, EM = 2;
    static constexpr unsigned MM = 0x400000u;
    static constexpr float MAXF = 6.0f;
    __device__ static __forceinline__ void q2(float a, float b, float& qa, float& qb) {
        unsigned h;
        asm("{\n\t.reg .b8 t;\n\tcvt.rn.satfinite.e2m1x2.f32 t, %1, %2;\n\t"
            "cvt.rn.f16x2.e2m1x2 %0, t;\n\t}"
            : "=r"(h)
            : "f"(a), "f"(b));
        unpack_f16x2(h, qa, qb);
    }
};

// Smallest s >= 1 with amax <= MAXF * 2^s, for normal amax > MAXF.  Equal to
// the reference's ceil(log2(amax / max_finite)) (fftcore.py:175): with
// amax = (1+fa) 2^ea and MAXF = (1+fm) 2^em, s = ea - em + [fa > fm].
template <class F>
__device__ __forceinline__ int shift_for(float amax) {
    unsigned b = __float_as_uint(amax);
    int ea = (int)(b >> 23) - 127;
    return ea - F::EM + ((b & 0x7fffffu) > F::MM ? 1 : 0);
}

template <class F>
struct DecodeRange {
    // c * 2^E exact & normal for every nonzero code c (|c| >= 2^(EMIN-M)) and
    // |c| * 2^E < 2^128 for |c| <= MAXF < 2^(EMAX+1).
    static constexpr int ELO = -126 - (F::EMIN - F::M);
    static constexpr int EHI = 127 - F::EMAX - 1;
};

// Twiddle table entry layout used by the kernels (built at plan time from the
// encoded plan, one entry per (stage, j < half)): codes in FP32 code space and
// the exponent of the block that butterfly j belongs to.
struct TwEntry {
    float wr, wi;
};

// launch bookkeeping (gpu_launches)
void note_launch(int n = 1);

// Programmatic dependent launch (mxfft_pdl): the transform kernels signal
// griddepcontrol.launch_dependents when they start and pass
// griddepcontrol.wait before their first access to data that an earlier kernel
// may have produced (or may still read), so the next kernel's launch, shared
// memory set-up and twiddle loads overlap the tail of this one.
extern int g_pdl;
__device__ __forceinline__ void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
template <class... Par, class... Arg>
inline cudaError_t launch_pdl(void (*k)(Par...), unsigned grid, unsigned block, size_t smem, cudaStream_t st,
                              Arg&&... a) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(block);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = g_pdl ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, k, static_cast<Par>(a)...);
}

// Per-device launch setup (mxfft_capi.cu), thread-safe and keyed by the
// current device, so a second GPU in the same process gets its own attributes
// and grid sizes:
//  - ensure_smem_attr: raise kernel k's dynamic shared memory limit to
//    smem_max bytes (once per (k, device));
//  - cached_occupancy: CTAs per SM of k at (nt threads, smem bytes), cached per
//    (k, device, nt, smem);
//  - device_attr: an attribute of the current device, cached.
cudaError_t ensure_smem_attr(const void* k, int smem_max);
cudaError_t cached_occupancy(const void* k, int nt, size_t smem, int* occ);
int device_attr(cudaDeviceAttr a);

}  // namespace mxfft
