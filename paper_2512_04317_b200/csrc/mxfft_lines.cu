// mxfft_lines.cu -- dispatch of the line kernel (kernels in mxfft_lines.cuh,
// instantiated per element format in lines_<fmt>.cu).
#include "mxfft_common.cuh"
#include "mxfft_internal.h"

#ifndef MXFFT_REVERSE_PASSES
#define MXFFT_REVERSE_PASSES 1  // fft2: every second pass walks its groups backwards (L2 reuse)
#endif

namespace mxfft {

cudaError_t run_mx_lines_e4m3(const MxLinesArgs&, int, size_t, cudaStream_t);
cudaError_t run_mx_lines_e4m3_dbg(const MxLinesArgs&, int, size_t, cudaStream_t);
cudaError_t run_mx_lines_e5m2(const MxLinesArgs&, int, size_t, cudaStream_t);
cudaError_t run_mx_lines_e5m2_dbg(const MxLinesArgs&, int, size_t, cudaStream_t);
cudaError_t run_mx_lines_e2m3(const MxLinesArgs&, int, size_t, cudaStream_t);
cudaError_t run_mx_lines_e2m3_dbg(const MxLinesArgs&, int, size_t, cudaStream_t);
cudaError_t run_mx_lines_e3m2(const MxLinesArgs&, int, size_t, cudaStream_t);
cudaError_t run_mx_lines_e3m2_dbg(const MxLinesArgs&, int, size_t, cudaStream_t);
cudaError_t run_mx_lines_e2m1(const MxLinesArgs&, int, size_t, cudaStream_t);
cudaError_t run_mx_lines_e2m1_dbg(const MxLinesArgs&, int, size_t, cudaStream_t);

cudaError_t run_mx_lines_acc_e4m3(const MxLinesArgs&, int, size_t, cudaStream_t);
cudaError_t run_mx_lines_acc_e5m2(const MxLinesArgs&, int, size_t, cudaStream_t);
cudaError_t run_mx_lines_acc_e2m3(const MxLinesArgs&, int, size_t, cudaStream_t);
cudaError_t run_mx_lines_acc_e3m2(const MxLinesArgs&, int, size_t, cudaStream_t);
cudaError_t run_mx_lines_acc_e2m1(const MxLinesArgs&, int, size_t, cudaStream_t);

static cudaError_t disp_fmt(const MxLinesArgs& a, int id, int cpb, size_t smem, bool dbg,
                            cudaStream_t st) {
    if (dbg) switch (id) {
        case F_E4M3: return run_mx_lines_e4m3_dbg(a, cpb, smem, st);
        case F_E5M2: return run_mx_lines_e5m2_dbg(a, cpb, smem, st);
        case F_E2M3: return run_mx_lines_e2m3_dbg(a, cpb, smem, st);
        case F_E3M2: return run_mx_lines_e3m2_dbg(a, cpb, smem, st);
        case F_E2M1: return run_mx_lines_e2m1_dbg(a, cpb, smem, st);
    }
    else switch (id) {
        case F_E4M3: return run_mx_lines_e4m3(a, cpb, smem, st);
        case F_E5M2: return run_mx_lines_e5m2(a, cpb, smem, st);
        case F_E2M3: return run_mx_lines_e2m3(a, cpb, smem, st);
        case F_E3M2: return run_mx_lines_e3m2(a, cpb, smem, st);
        case F_E2M1: return run_mx_lines_e2m1(a, cpb, smem, st);
    }
    return cudaErrorInvalidValue;
}

#ifndef MXFFT_TMA_STORE
#define MXFFT_TMA_STORE 1  // n = 128 / 256 / 512 transposed-store row passes on the TMA kernel (k_mx_lines_tma)
#endif
int g_tma_store = MXFFT_TMA_STORE;

// Tensor map of a transposed store (rows of n x n images stored as columns):
// `out` seen as (batch n) rows of n complex64.  After the last radix-4 pair of
// stages, thread tl of a line holds positions 8 tl + (n/4) k + i (k < 4, i < 8),
// so the rows are split as (k, tl, i) and the box [k][i][tl][LPC columns] lands
// in shared memory with the T threads of one store instruction on consecutive
// 128-byte (64-byte) rows: under the 128B (64B) swizzle the warp's 8-byte
// stores are free of bank conflicts.  Returns false when the driver's encoder
// is unavailable or refuses the map (the kernel then keeps its own copy-out).
typedef CUresult (*encode_t)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static encode_t tensor_map_encoder() {
    static encode_t enc = nullptr;
    static bool tried = false;
    if (!tried) {
        tried = true;
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            enc = reinterpret_cast<encode_t>(fn);
        else
            (void)cudaGetLastError();
    }
    return enc;
}

// Tensor map of the group tiles (LPC contiguous rows of n complex64): rows are
// cut into 128-byte segments of 16 elements and the box is [segment][line][16],
// so under the 128B swizzle the 16-byte chunk index is XORed with the LINE
// index: the bit-reversed gather of a warp (elements m T + rcol of 4 (2) lines)
// then reads 32 distinct 8-byte bank pairs per half-warp (lines_body_tma).
static bool make_in_map(MxLinesArgs& a) {
    encode_t enc = tensor_map_encoder();
    if (!enc) return false;
    const cuuint64_t n = (cuuint64_t)a.n, T = n / 32, lpc = 128 / T;
    const cuuint64_t dims[3] = {16, (cuuint64_t)a.total_lines, n / 16};
    const cuuint64_t strides[2] = {n * 8, 128};  // bytes: one line, one segment
    const cuuint32_t box[3] = {16, (cuuint32_t)lpc, (cuuint32_t)(n / 16)};
    const cuuint32_t es[3] = {1, 1, 1};
    const CUresult r = enc(&a.in_map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<float2*>(a.in), dims, strides,
                           box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

static bool make_out_map(MxLinesArgs& a) {
    encode_t enc = tensor_map_encoder();
    if (!enc) return false;
    const cuuint64_t n = (cuuint64_t)a.n, T = n / 32, lpc = 128 / T;
    const cuuint64_t batch = (cuuint64_t)(a.total_lines / a.n);
    const cuuint64_t row = n * 8;  // bytes
    CUresult r;
    if (lpc <= 16) {
        const cuuint64_t dims[4] = {n, T, 8, 4 * batch};
        const cuuint64_t strides[3] = {8 * row, row, (n / 4) * row};  // 8 rows, 1 row, n/4 rows
        const cuuint32_t box[4] = {(cuuint32_t)lpc, (cuuint32_t)T, 8, 4};
        const cuuint32_t es[4] = {1, 1, 1, 1};
        const CUtensorMapSwizzle sw = lpc * 8 == 128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B;
        r = enc(&a.out_map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, a.out, dims, strides, box, es,
                CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    } else {
        // n = 128: 32 columns per group = two 128-byte halves of a box row: [k][i][tl][half][16]
        const cuuint64_t dims[5] = {16, n / 16, T, 8, 4 * batch};
        const cuuint64_t strides[4] = {128, 8 * row, row, (n / 4) * row};
        const cuuint32_t box[5] = {16, (cuuint32_t)(lpc / 16), (cuuint32_t)T, 8, 4};
        const cuuint32_t es[5] = {1, 1, 1, 1, 1};
        r = enc(&a.out_map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 5, a.out, dims, strides, box, es,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    }
    return r == CUDA_SUCCESS;
}

int g_profile_stage_limit = -1;
int g_profile_flags = 0;
int g_lines_ctas_per_sm = 0;  // 0: occupancy (see mxfft_lines_ctas_per_sm)

bool mx_lines_ok(const Plan& p) {
    if (p.fmt.id == F_GENERIC) return false;
    if (p.cpb > 32 || (p.cpb & (p.cpb - 1))) return false;
    if (p.log2n < 5 || p.log2n > 14) return false;
    const int T = p.n >> 5;
    if (p.cpb == 32 && T > 32) return false;  // lane-pair blocks need both halves in one warp
    return true;
}

cudaError_t run_mx_lines(const Plan& p, const LinePass& lp, cudaStream_t st) {
    MxLinesArgs a{};
    a.in = reinterpret_cast<const float2*>(lp.in);
    a.out = reinterpret_cast<float2*>(lp.out);
    a.n = p.n;
    a.log2n = p.log2n;
    a.log2T = p.log2n - 5;
    a.col_mode = lp.col_mode;
    a.tstore = lp.tstore;
    a.lines_per_image = lp.col_mode ? p.n : lp.lines_per_image;
    a.total_lines = lp.col_mode ? lp.batch * p.n : lp.total_lines;
    a.tw16 = lp.inverse ? p.d_tw16_inv : p.d_tw16_fwd;
    a.twe = p.d_twe8;
    a.trivial01 = p.trivial01;
    a.inverse = lp.inverse;
    a.kvec = lp.kvec;
    a.k_group = lp.k_group > 0 ? lp.k_group : 1;
    a.reverse = lp.reverse && MXFFT_REVERSE_PASSES;
    a.seg_log2 = lp.seg_log2;
    a.seg_stride = lp.seg_stride;
    a.dec = lp.dec;
    a.lpi_shift = -1;
    if (a.lines_per_image > 0 && (a.lines_per_image & (a.lines_per_image - 1)) == 0)
        for (a.lpi_shift = 0; (1 << a.lpi_shift) < a.lines_per_image; ++a.lpi_shift) {
        }
    a.kin_sign = lp.kin_sign;
    a.kout_sign = lp.kout_sign;
    a.kout_const = lp.kout_const;
    a.kin_const = lp.kin_const;
    a.stage_limit = lp.stage_limit >= 0 ? lp.stage_limit : p.log2n;
    if (lp.stage_limit < 0 && g_profile_stage_limit >= 0 && g_profile_stage_limit < p.log2n)
        a.stage_limit = g_profile_stage_limit;  // profiling knob (mxfft_profile_stage_limit)
    a.fmt = p.fmt;
    a.cpb = p.cpb;
    a.wcr = p.d_wcr;
    a.wci = p.d_wci;
    a.wsexp = p.d_wsexp;
    a.prof_flags = g_profile_flags;
    a.d_vexp = lp.d_vexp;
    a.d_vcodes = lp.d_vcodes;
    a.d_pexp = lp.d_pexp;
    a.d_pshift = lp.d_pshift;
    a.d_pcodes = lp.d_pcodes;
    const int T = p.n >> 5;
    const int nt = T <= 128 ? 128 : T;
    // twiddle prefix rounded up to 1 KB: the data regions must stay 128-byte
    // aligned (run addresses are formed with OR, see radr())
    a.tw_chunks = ((p.n * 5 + 1023) / 1024) * 64;
    if (nt == 128 && T >= 2 && T <= 16) {
        // n = 64 .. 512: pad the twiddle prefix so that the tile buffers start on a
        // 4 KB boundary of the shared window (dynamic shared memory begins after
        // the per-block reserved area); the kernels rely on it (see AX)
        const int reserved = device_attr(cudaDevAttrReservedSharedMemoryPerBlock);
        while ((reserved + a.tw_chunks * 16) % 4096) a.tw_chunks += 64;
    }
    // 128-thread kernels double-buffer their group tile (cp.async pipeline)
#ifndef MXFFT_NBUF
#define MXFFT_NBUF 2
#endif
    const size_t nbuf = nt == 128 ? MXFFT_NBUF : 1;
    const size_t smem = (size_t)a.tw_chunks * 16 + nbuf * (size_t)nt * 32 * sizeof(float2);
    const bool dbg = lp.d_vexp != nullptr;
    a.tma_out = 0;
    if (g_tma_store && !dbg && a.tstore && !a.col_mode && !a.seg_log2 && !a.dec && p.cpb >= 8 &&
        a.log2T >= 2 && a.log2T <= 4 && a.stage_limit >= a.log2n && a.lines_per_image == a.n &&
        a.total_lines % a.n == 0 && a.prof_flags == 0 && (reinterpret_cast<uintptr_t>(a.out) & 15) == 0 &&
        (reinterpret_cast<uintptr_t>(a.in) & 15) == 0)
        a.tma_out = make_out_map(a) && make_in_map(a) ? 1 : 0;
    a.acc = lp.acc;
    a.minw = lp.minw;
    if (a.acc) {  // statistics-folding first pass: the TMA kernel only (mxfft_pipeline_folded checks first)
        if (!a.minw || a.kin_sign || a.kin_const || a.reverse || dbg) return cudaErrorInvalidValue;
        switch (p.fmt.id) {
            case F_E4M3: return run_mx_lines_acc_e4m3(a, p.cpb, smem, st);
            case F_E5M2: return run_mx_lines_acc_e5m2(a, p.cpb, smem, st);
            case F_E2M3: return run_mx_lines_acc_e2m3(a, p.cpb, smem, st);
            case F_E3M2: return run_mx_lines_acc_e3m2(a, p.cpb, smem, st);
            case F_E2M1: return run_mx_lines_acc_e2m1(a, p.cpb, smem, st);
        }
        return cudaErrorInvalidValue;
    }
    return disp_fmt(a, p.fmt.id, p.cpb, smem, dbg, st);
}

}  // namespace mxfft
