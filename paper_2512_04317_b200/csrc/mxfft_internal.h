// mxfft_internal.h -- library-internal types shared by the .cu translation units.
#pragma once

#include <cuda.h>  // CUtensorMap (the encoder is fetched with cudaGetDriverEntryPoint: no libcuda link)
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/mxfft_b200.h"
#include "mxfft_common.cuh"

namespace mxfft {

// Encoded plan (FftPlan, fftcore.py:84-117), resident on the device.
struct Plan {
    int n, log2n, block_size, cpb;
    FmtDesc fmt;
    // full tables, reference layout: codes (stages, n/2), scale exponents (stages, n/2/cpb)
    double* d_wcr = nullptr;
    double* d_wci = nullptr;
    int* d_wsexp = nullptr;
    // kernel tables, entry half + j (j < half = 2^s) for stage s; entry 0 unused:
    unsigned* d_tw16_fwd = nullptr;  // packed f16x2 codes (lo = re, hi = im)
    unsigned* d_tw16_inv = nullptr;  // conjugated twiddles (fftcore.py:267-268)
    signed char* d_twe8 = nullptr;   // log2 scale of the block holding butterfly j
    int trivial01 = 0;  // stage 0/1 twiddles are exactly 1 and -i at scale 2^-emax
    int device = 0;     // the tables live on this device; transforms must run there
    // n >= 16384: the plan of the first log2(n) - 1 stages on n/2-point halves
    // (kernel tables alias this plan's; reference-layout rows copied), used by
    // mxfft_fft2's split passes (decimated half rows + last stage fused into
    // the transpose, mxfft_laststage.cu)
    Plan* half = nullptr;
};

// the last butterfly stage of an n-point row pass fused into the tiled
// transpose that follows it (mxfft_laststage.cu): in = rows after stage L-2,
// out = transposed rows after stage L-1 [x 2^kout]
struct LastStagePass {
    const void* in;
    void* out;
    int64_t batch;
    int inverse;
    const int32_t* kvec;
    int k_group, kout_sign, kout_const;
    int kin_sign = 0;  // x 2^(kin_sign k) on load (the folded pipeline's first pass)
};
bool last_stage_ok(const Plan& p);
cudaError_t run_last_stage_transpose(const Plan& p, const LastStagePass& lp, cudaStream_t st);
extern int g_split_last_stage;

// One pass of 1-D transforms over a set of lines.
struct LinePass {
    const void* in = nullptr;
    void* out = nullptr;
    int col_mode = 0;            // 0: lines are contiguous rows; 1: columns of n x n images
    int tstore = 0;              // rows of n x n images, stored transposed (out[i][q][r] = line r, elem q)
    int64_t img_elems = 0;       // complex elements per image
    int lines_per_image = 1;     // rows mode: lines per image (for k lookup)
    int64_t total_lines = 0;     // rows mode: number of lines
    int64_t batch = 0;           // cols mode: number of images
    int inverse = 0;
    const int32_t* kvec = nullptr;
    int k_group = 1;
    int kin_sign = 0, kout_sign = 0, kout_const = 0, kin_const = 0;
    int stage_limit = -1;
    int reverse = 0;  // walk the groups last to first (the previous pass's latest output is still in L2)
    int seg_log2 = 0;  // rows mode, > 0: element q of line c is in[(q >> seg_log2) * seg_stride + c * 2^seg_log2 + (q & mask)]
    int64_t seg_stride = 0;
    int dec = 0;  // rows mode: line L is half (L & 1) of row L >> 1 of length 2n, decimated (x[2q + h])
    unsigned* acc = nullptr;  // statistics-folding first pass: two words per warp and group (total points / 512 words)
    unsigned* minw = nullptr;  // ... and one word per thread and group (total points / 32 words)
    int32_t* d_vexp = nullptr;
    float* d_vcodes = nullptr;
    int32_t* d_pexp = nullptr;
    int32_t* d_pshift = nullptr;
    float* d_pcodes = nullptr;
};

// arguments of the fast line kernel (mxfft_lines.cu)
struct MxLinesArgs {
    const float2* in;
    float2* out;
    int n, log2n, log2T, col_mode, tstore;
    int lines_per_image;
    int64_t total_lines;
    const unsigned* tw16;
    const signed char* twe;
    int trivial01, inverse;
    const int32_t* kvec;
    int k_group, kin_sign, kout_sign, kout_const, kin_const, stage_limit;
    int lpi_shift;  // log2(lines_per_image) when it is a power of two, else -1
    int reverse;    // group order last to first
    int seg_log2;   // segmented input (the all-to-all receive layout), 0 = off
    int64_t seg_stride;
    int dec;        // decimated halves of rows twice as long (the first L-1 stages of an L-stage row)
    int prof_flags;  // profiling only: bit 0 skip tile loads, bit 1 skip stores
    int tw_chunks;
    // exact replay (replay_lines): reference-literal tables of the plan
    FmtDesc fmt;
    int cpb;
    const double* wcr;
    const double* wci;
    const int* wsexp;
    int32_t* d_vexp;
    float* d_vcodes;
    int32_t* d_pexp;
    int32_t* d_pshift;
    float* d_pcodes;
    // transposed stores through TMA (n = 256 / 512 specialised kernels): one
    // cp.async.bulk.tensor store per group from a tile published in output order
    int tma_out;
    unsigned* acc;  // statistics-folding first pass (lines_body_tma<.., ACC>), else nullptr
    unsigned* minw;
    alignas(64) CUtensorMap out_map;
    alignas(64) CUtensorMap in_map;  // group tiles in gather order ([segment][line][16 elements], make_in_map)
};

// arguments of the generic reference-literal kernel (mxfft_fft.cu)
struct GenericArgs {
    const float2* in;
    float2* out;
    int n, log2n, cpb;
    FmtDesc fmt;
    const double* wcr;
    const double* wci;
    const int* wsexp;
    int inverse, col_mode;
    int64_t img_elems;
    int lines_per_image;
    const int32_t* kvec;
    int k_group, kin_sign, kout_sign, kout_const, kin_const;
};

extern int g_profile_stage_limit;
extern int g_lines_ctas_per_sm;
extern int g_profile_flags;  // < 0: off (see mxfft_profile_stage_limit)
bool mx_lines_ok(const Plan& p);
// fused small-image pipeline (mxfft_image.cu)
bool mx_image_ok(const Plan& p);
// mode 0 forward, 1 inverse, 2 round trip (x 1/n^2); kin: precomputed k (no
// statistics in the kernel), else the statistics run in the kernel (res, kvec)
cudaError_t run_mx_image(const Plan& p, const void* x, void* y, int64_t nimg, int mode,
                         const mxfft_prescale_cfg& cfg, mxfft_prescale_result* res, int32_t* kvec,
                         const int32_t* kin, int k_group, cudaStream_t st);
extern int g_tma_store;    // n = 256 / 512 transposed stores through TMA (mxfft_tma_store)
extern int g_fused_image;  // mxfft_fft2 runs n = 128 batches on the fused image kernel (mxfft_fused_image)
cudaError_t run_mx_lines(const Plan& p, const LinePass& lp, cudaStream_t st);
cudaError_t run_lines(const Plan& p, const LinePass& lp, cudaStream_t st);

// codec kernels (mxfft_codec.cu)
cudaError_t launch_quantize_f64(const double* x, double* out, int64_t n, const FmtDesc& f,
                                int32_t* d_nonfinite, cudaStream_t st);
cudaError_t launch_encode_f64(const double* v, int64_t nblocks, int block_len, const FmtDesc& f,
                              double* codes, double* scales, int* scale_exp, int32_t* d_nonfinite,
                              cudaStream_t st);
cudaError_t launch_decode_f64(const double* codes, const double* scales, int64_t nblocks,
                              int block_len, double* out, cudaStream_t st);
cudaError_t plan_encode(Plan& p, const double* d_tw, cudaStream_t st);
cudaError_t launch_cabs(const void* x, int is_c128, int64_t n, double* out, cudaStream_t st);
cudaError_t launch_transpose_c64(const void* x, void* y, int64_t batch, int n, cudaStream_t st,
                                 int64_t ldx = 0, int64_t bsx = 0);
cudaError_t launch_metrics(const double* r, const double* t, int64_t h, int64_t w, int do_ssim, const double* win,
                           double c1, double c2, double* out, cudaStream_t st);
cudaError_t launch_fp16_rows(const void* x, int x_is_c128, void* y, int64_t batch, int n, const void* tw,
                             int inverse, int* nonfinite, cudaStream_t st);
cudaError_t launch_f64_rows(const void* x, void* y, int64_t batch, int n, const void* tw, int inverse,
                            cudaStream_t st);
cudaError_t launch_prescale_sample_keys(const float2* x, int64_t npts, int64_t nsamples, float* keys,
                                        cudaStream_t st);
cudaError_t launch_prescale_count_range(const float2* x, int64_t npts, float lo, float hi, float top,
                                        void* state, float2* cand, int64_t cap, float2* topb,
                                        int64_t topcap, cudaStream_t st);
cudaError_t launch_fold_resolve(const unsigned* acc, const unsigned* minw, int64_t nstack, int64_t stack_points,
                                const mxfft_prescale_cfg& c, mxfft_prescale_result* out, int32_t* kvec,
                                unsigned* scratch, cudaStream_t st);
cudaError_t launch_fold_reduce(const unsigned* acc, const unsigned* minw, int64_t npoints,
                               const mxfft_prescale_cfg& c, int step, unsigned* g, cudaStream_t st);
cudaError_t launch_fold_finish(const unsigned* g, int64_t total_points, const mxfft_prescale_cfg& c,
                               mxfft_prescale_result* out, int32_t* kvec, int64_t s, cudaStream_t st);
cudaError_t launch_rss(const void* x, int is_c128, int64_t groups, int coils, int64_t npix,
                       double* out, cudaStream_t st, const int32_t* kvec = nullptr, int ksign = 0,
                       int econst = 0);
cudaError_t launch_prescale_apply_c128(const void* x, void* y, int64_t seg_points, int64_t nseg,
                                       const int32_t* kvec, cudaStream_t st);
cudaError_t launch_scale(const void* x, void* y, int64_t n, int dtype, double f, cudaStream_t st);
cudaError_t launch_mx_multiply(const void* v, const double* wcr, const double* wci, const double* ws, int64_t rows,
                               int m, int cpb, const FmtDesc& f, void* wv, const void* u, void* y0, void* y1,
                               int32_t* nonfinite, cudaStream_t st);
cudaError_t launch_selftest_hwq(const FmtDesc& f, unsigned long long* mism, unsigned* first_bad,
                                cudaStream_t st);

}  // namespace mxfft
