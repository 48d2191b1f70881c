/*
 * mxfft_b200.h -- C-ABI of the B200-native MX-FFT hot path (sm_100a).
 *
 * The reference (arxiv/paper_2512_04317, package `mxfft`, pure Python/NumPy)
 * has no FFI: its boundary for this path is the Python API re-exported in
 * pkg/src/mxfft/__init__.py:3-65.  Each entry point below replaces one
 * reference function (cited as pkg/src/mxfft/<file>:<line>); the Python
 * package paper_2512_04317_b200 binds them with ctypes and keeps the
 * reference's names, argument meanings and exceptions.
 *
 * Conventions
 *  - Every function returns an mxfft_status; mxfft_last_error() holds the
 *    message of the most recent failure on the calling thread.
 *  - Data pointers are DEVICE pointers unless a parameter says "host".
 *    The caller allocates all memory (including workspace); the library only
 *    owns plan tables.  No allocation happens on the transform path.
 *  - `stream` is a cudaStream_t passed as uintptr_t (0 = legacy default).
 *    All calls are stream-ordered and asynchronous unless stated otherwise.
 *  - Complex data is interleaved (re, im): complex64 = 2 x float,
 *    complex128 = 2 x double.
 */
#ifndef MXFFT_B200_H
#define MXFFT_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    MXFFT_OK = 0,
    MXFFT_ERR_INVALID_VALUE = 1,     /* errors.InvalidValue   (errors.py:8)  */
    MXFFT_ERR_SHAPE = 2,             /* errors.ShapeError     (errors.py:12) */
    MXFFT_ERR_UNSUPPORTED_SIZE = 3,  /* errors.UnsupportedSize(errors.py:16) */
    MXFFT_ERR_VALUE = 4,             /* ValueError (bad direction / block size / argument) */
    MXFFT_ERR_CUDA = 5,              /* RuntimeError (CUDA failure) */
    MXFFT_ERR_MANTISSA_OVERFLOW = 6  /* errors.MantissaOverflow (errors.py:20) */
} mxfft_status;

/* Element format (minifloat.py:28-46).  policy: 0 = "ieee", 1 = "extended",
 * 2 = "finite"; bias is the resolved bias (2^(E-1)-1 by default). */
typedef struct {
    int32_t exponent_bits;
    int32_t mantissa_bits;
    int32_t policy;
    int32_t bias;
} mxfft_format;

/* Prescale configuration (PrescaleConfig, prescale.py:21-37). */
typedef struct {
    double target;
    double tau;
    double tau_min;
    int32_t k_min;
    int32_t k_max;
} mxfft_prescale_cfg;

/* One segment's prescale result (PrescaleResult, prescale.py:40-46).
 * flags bit 0: a non-finite value was seen (InvalidValue);
 * flags bit 1: log2 landed within a few ulps of a rounding boundary, so the
 *              host must confirm k with its own log2 (measure-zero case);
 * flags bit 2: (mxfft_pipeline_folded only) the stack was not settled: re-run it
 *              with mxfft_prescale_stats + mxfft_fft2;
 * flags bit 3: (mxfft_pipeline_folded only) k-only row: p_tau / k2 not evaluated. */
typedef struct {
    double a_max;
    double p_tau;
    int32_t k1;
    int32_t k2;
    int32_t k;
    int32_t flags;
    int64_t nnz;
} mxfft_prescale_result;

typedef struct mxfft_plan_s* mxfft_plan;

int32_t mxfft_version(void);
const char* mxfft_last_error(void);

/* quantize_array (minifloat.py:105-120): RNE onto the format grid with
 * saturation, FP64 in/out (n values).  *d_nonfinite (device int32) is set
 * to 1 when a non-finite input is seen (the host raises InvalidValue). */
int32_t mxfft_quantize_f64(const double* x, double* out, int64_t n, const mxfft_format* fmt,
                           int32_t* d_nonfinite, uintptr_t stream);

/* block_scales + encode (mxblock.py:27-51 / fftcore.py:131-147), batched:
 * v: FP64 (nblocks, block_len) -> codes FP64 (nblocks, block_len), scales FP64 (nblocks). */
int32_t mxfft_mx_encode_f64(const double* v, int64_t nblocks, int32_t block_len,
                            const mxfft_format* fmt, double* codes, double* scales,
                            int32_t* d_nonfinite, uintptr_t stream);

/* decode_block_mx (mxblock.py:86-90), batched: codes (nblocks, block_len) with
 * block_len even, scales (nblocks) -> complex128 (nblocks, block_len/2). */
int32_t mxfft_mx_decode_f64(const double* codes, const double* scales, int64_t nblocks,
                            int32_t block_len, double* out, uintptr_t stream);

/* FftPlan(n, ModeSpec.mx(fmt, block_size)) (fftcore.py:84-121).
 * h_twiddles: HOST complex128 (stages, n/2) twiddles in butterfly order, built by
 * the caller with the reference's own NumPy expression (fftcore.py:101-105); the
 * library encodes them on the device (fftcore.py:108-113).  Synchronous. */
int32_t mxfft_plan_create(mxfft_plan* plan, int32_t n, const mxfft_format* fmt,
                          int32_t block_size, const double* h_twiddles, uintptr_t stream);
int32_t mxfft_plan_destroy(mxfft_plan plan);

/* Read the encoded twiddles back to HOST arrays: codes (stages, n/2) x2 and
 * scales (stages, n/2/cpb) -- plan.mx_twiddles of the reference.  Synchronous. */
int32_t mxfft_plan_twiddles(mxfft_plan plan, double* h_codes_re, double* h_codes_im,
                            double* h_scales);

/* Batched 1-D MX transform along contiguous rows (_fft_batch_mx,
 * fftcore.py:259-282): x, y complex64 (batch, n); x may alias y. */
int32_t mxfft_fft_rows(mxfft_plan plan, const void* x, void* y, int64_t batch, int32_t inverse,
                       uintptr_t stream);

/* mxfft_fft_rows with exact power-of-two scalings fused into the load and the
 * store: y = 2^exp_out * rows(2^exp_in * x) (apply_prescale / undo_prescale /
 * 1/n^2, prescale.py:76-91, mri.py:100).  The row passes of a distributed 2-D
 * transform (paper_2512_04317_b200/distributed.py) use it. */
int32_t mxfft_fft_rows_scaled(mxfft_plan plan, const void* x, void* y, int64_t batch, int32_t inverse,
                              int32_t exp_in, int32_t exp_out, uintptr_t stream);

/* mxfft_fft_rows_scaled reading its lines from the receive layout of a
 * row-slab all-to-all transpose (the distributed 2-D transform,
 * paper_2512_04317_b200/distributed.py): x is (n / seg_len, lines, seg_len)
 * complex64 and element q of line c is x[q / seg_len][c][q mod seg_len], so
 * the next pass needs no permute copy; y is (lines, n), out of place.
 * seg_len: a power of two dividing n (seg_len == n: plain rows). */
int32_t mxfft_fft_rows_seg(mxfft_plan plan, const void* x, void* y, int64_t lines, int32_t inverse, int32_t exp_in,
                           int32_t exp_out, int32_t seg_len, uintptr_t stream);

/* Batched 1-D MX transform along the COLUMNS of `batch` n x n complex64 images
 * (the second pass of fft_2d, fftcore.py:352, without materialising rows.T);
 * x may alias y.  With mxfft_fft_rows this gives either pass of fft_2d alone. */
int32_t mxfft_fft_cols(mxfft_plan plan, const void* x, void* y, int64_t batch, int32_t inverse,
                       uintptr_t stream);

/* Batched 2-D MX transform (fft_2d, fftcore.py:344-353 = rows then columns) of
 * `batch` n x n complex64 images; x may alias y (but not the workspace).
 *   mode 0: forward; 1: inverse; 2: round trip = forward, inverse, x 1/n^2
 *           (roundtrip_pipeline's per-coil body, mri.py:100-105).
 *   d_k:    optional per-image int32 prescale exponents (device).  Image i is
 *           multiplied by 2^k[i / k_group] on load (apply_prescale,
 *           prescale.py:76-86) and the result by 2^-k on store (undo_prescale,
 *           prescale.py:89-91).  NULL = no prescale.
 *   workspace: optional device buffer of mxfft_fft2_workspace_bytes(plan, batch)
 *           bytes (0 = none needed).  With it each pass is a row pass whose
 *           output is stored transposed (fftcore.py:351-353 literally), which
 *           keeps every HBM access a full 128-byte line; NULL = the column pass
 *           runs in place on y (same results, slower).
 * Exact in FP32 (power-of-two scalings) while results stay in FP32 range. */
int32_t mxfft_fft2(mxfft_plan plan, const void* x, void* y, int64_t batch, int32_t mode,
                   const int32_t* d_k, int32_t k_group, void* workspace, int64_t workspace_bytes,
                   uintptr_t stream);
int64_t mxfft_fft2_workspace_bytes(mxfft_plan plan, int64_t batch);

/* The non-MX modes of ModeSpec (fftcore.py:32-64), batched rows of length n
 * (power of two <= 16384).  d_tw: n device entries, entry 2^s + j = twiddle j
 * of stage s (j < 2^s) of the plan's FP64 table (fftcore.py:101-105):
 *  - fp16 (_fft_batch_fp16, fftcore.py:285-311): entries are half2 (re, im)
 *    rounded from FP64 by the plan builder; x complex64 or complex128
 *    (x_is_c128); y complex64 holding FP16 values.  *d_nonfinite is set when
 *    an intermediate overflowed (the reference's quantize_array raises).
 *  - reference (_fft_batch_reference, fftcore.py:243-256): entries complex128;
 *    x, y complex128, out of place. */
int32_t mxfft_fft_rows_fp16(const void* x, int32_t x_is_c128, void* y, int64_t batch, int32_t n,
                            const void* d_tw, int32_t inverse, int32_t* d_nonfinite, uintptr_t stream);
int32_t mxfft_fft_rows_f64(const void* x, void* y, int64_t batch, int32_t n, const void* d_tw, int32_t inverse,
                           uintptr_t stream);

/* Image-quality metrics of an h x w FP64 test image against a reference
 * (metrics.py:38-93), device pointers.  d_out (5 doubles): sum (ref-test)^2,
 * sum ref^2, max ref, min ref, and -- when do_ssim -- the sum over the
 * (h-10) x (w-10) valid positions of the local SSIM with the 11 x 11 window
 * d_window (row-major) and constants c1, c2.  FP64; the summation order is
 * not numpy's (agreement ~1e-15 relative). */
int32_t mxfft_metrics(const double* ref, const double* test, int64_t h, int64_t w, int32_t do_ssim,
                      const double* d_window, double c1, double c2, double* d_out, uintptr_t stream);

/* Batched out-of-place transpose of `batch` n x n complex64 images,
 * y[b][j][i] = x[b][i][j] (the rows.T between the passes of fft_2d,
 * fftcore.py:352); n a multiple of 64. */
int32_t mxfft_transpose_c64(const void* x, void* y, int64_t batch, int32_t n, uintptr_t stream);
/* Same from n x n blocks of a larger array: block b starts at
 * x + b * batch_stride_x, rows ld_x apart (0 = the dense defaults n*n / n);
 * y stays dense.  The row-slab all-to-all uses it to transpose the (N/G)^2
 * blocks of a slab straight into send order. */
int32_t mxfft_transpose_c64_strided(const void* x, int64_t ld_x, int64_t batch_stride_x, void* y, int64_t batch,
                                    int32_t n, uintptr_t stream);

/* compute_prescale (prescale.py:61-73) over `nseg` segments of `seg_points`
 * complex values each (complex64 when is_c128 == 0, else complex128),
 * contiguous.  Writes one mxfft_prescale_result per segment to d_out and, when
 * d_k is not NULL, the applied exponent k to d_k[seg].  workspace: device
 * buffer of at least mxfft_prescale_workspace_bytes(nseg, seg_points) bytes. */
int32_t mxfft_prescale_stats(const void* x, int32_t is_c128, int64_t nseg, int64_t seg_points,
                             const mxfft_prescale_cfg* cfg, mxfft_prescale_result* d_out,
                             int32_t* d_k, void* workspace, int64_t workspace_bytes,
                             uintptr_t stream);
int64_t mxfft_prescale_workspace_bytes(int64_t nseg, int64_t seg_points);

/* Building blocks of compute_prescale over ONE segment that is too large for
 * a CTA or split across calls / ranks (the C5 global prescale);
 * paper_2512_04317_b200/prescale.py compute_prescale_global combines them.
 *  - sample_keys: FP32 squared magnitudes of `nsamples` points taken as
 *    pseudo-random whole 32-byte sectors of x (complex64, npts a multiple of
 *    4); zero -> +inf, |re|,|im| outside [2^-60, 2^60] -> 0 or 2^125.
 *  - count_range: one streaming pass over x (complex64): d_state (40 bytes:
 *    float lo, hi, top; int pad; uint64 nnz; uint32 below, ncand, ntop,
 *    flags) receives the nonzero count, the points with key < lo, and the
 *    numbers of points with key in [lo, hi] and key >= top, which are copied
 *    (as complex64) to d_cand / d_top up to their capacities.  flags bit 0:
 *    a non-finite value, or a key beyond FP32 range, was seen.
 *  - cabs: |z| exactly as numpy's np.abs(complex128), FP64 out. */
int32_t mxfft_prescale_sample_keys(const void* x, int64_t npts, int64_t nsamples, float* d_keys,
                                   uintptr_t stream);
int32_t mxfft_prescale_count_range(const void* x, int64_t npts, float lo, float hi, float top, void* d_state,
                                   void* d_cand, int64_t cand_cap, void* d_top, int64_t top_cap,
                                   uintptr_t stream);
int32_t mxfft_cabs(const void* x, int32_t is_c128, int64_t n, double* out, uintptr_t stream);

/* Root-sum-square coil combine (rss, mri.py:70-81) of per-coil complex images
 * (complex64 when is_c128 == 0, else complex128): x (groups, coils, npix) ->
 * FP64 (groups, npix).  |z| is computed exactly as numpy's np.abs(complex128). */
int32_t mxfft_rss(const void* x, int32_t is_c128, int64_t groups, int32_t coils, int64_t npix,
                  double* out, uintptr_t stream);

/* The fused small-image pipeline (BASELINE configs[3]): one n x n image per
 * CTA, the whole per-image pipeline of forward_pipeline / roundtrip_pipeline
 * (mri.py:84-107, one coil) in ONE kernel -- compute_prescale's statistics
 * (prescale.py:61-73) on the image held in shared memory, x 2^k on load, the
 * row and column passes of fft_2d (fftcore.py:344-353) [then the inverse
 * fft_2d and x 1/n^2], x 2^-k on store.  x, y: complex64 (nimg, n, n), out of
 * place; d_res: one mxfft_prescale_result per image (flags as
 * mxfft_prescale_stats); d_k: optional per-image k.  Results are identical to
 * mxfft_prescale_stats + mxfft_fft2.  Supported when
 * mxfft_pipeline_fused_supported(plan) != 0 (n = 128, a hardware MX format,
 * B in {16, 32, 64}). */
int32_t mxfft_pipeline_fused_supported(mxfft_plan plan);
/* Scheduling knob for mxfft_fft2 on batches of n = 128 images (plans for which
 * mxfft_pipeline_fused_supported holds): on > 0 the one-image-per-CTA kernel
 * (given the per-image k), on == 0 four line passes, on < 0 (the default)
 * automatic: the line passes when a workspace is given and batch >= 64, else
 * the one-image-per-CTA kernel; results are identical. */
void mxfft_fused_image(int32_t on);
/* Scheduling knob: with on != 0 (the default) the n = 256 / 512 row passes of
 * mxfft_fft2 (rows stored transposed, fftcore.py:351-353) leave each group of
 * lines with one TMA tensor store (cp.async.bulk.tensor) from a tile published
 * in output order, instead of a per-thread copy-out; results are identical. */
void mxfft_tma_store(int32_t on);
/* Scheduling knob: with on != 0 (the default) the line and image kernels are
 * launched with programmatic stream serialization: each signals
 * griddepcontrol.launch_dependents when it starts and passes
 * griddepcontrol.wait before touching any data an earlier kernel produced, so
 * the next pass's launch and set-up overlap this pass's tail; results are
 * identical. */
void mxfft_pdl(int32_t on);
/* Scheduling knob: with on != 0 (the default) mxfft_fft2 runs n >= 16384
 * passes as stages 0 .. L-2 on the decimated half rows (the n/2-point line
 * kernel) followed by the last stage fused into the transposed store, when
 * the workspace holds two image copies (mxfft_fft2_workspace_bytes);
 * results are identical. */
void mxfft_split_last_stage(int32_t on);
int32_t mxfft_pipeline_fused(mxfft_plan plan, const void* x, void* y, int64_t nimg, int32_t roundtrip,
                             const mxfft_prescale_cfg* cfg, mxfft_prescale_result* d_res, int32_t* d_k,
                             uintptr_t stream);

/* The pipelines with compute_prescale FOLDED INTO THE FIRST TRANSFORM PASS
 * (forward_pipeline / roundtrip_pipeline, mri.py:84-107; n = 128 / 256 / 512,
 * and n = 16384 through the split passes; stacks of `coils` consecutive
 * images share one prescale): no standalone
 * statistics read of x.  The first row pass runs on the unscaled input and
 * accumulates, per stack, the largest |x|^2, the smallest nonzero
 * max(|re|, |im|) and the range of the MX block exponents it produced; a small
 * kernel then settles k = clip(max(k1, k2)) (prescale.py:66-72) -- k1 from the
 * peak, k2 <= k1 PROVEN from the smallest nonzero magnitude (p_tau is not
 * evaluated) -- and the later passes apply 2^k on the way in and 2^-k (and
 * 1/n^2) on the way out.  This equals the scaled transform bit for bit because
 * the MX arithmetic commutes with powers of two while every block exponent
 * stays inside the unclamped range, which the accumulated range proves.
 * A stack for which any proof fails (k1 near a rounding boundary, tiny nonzero
 * magnitudes so that k2 may exceed k1, exponents near a clamp, non-finite or
 * out-of-range input) gets d_res[s].flags = 4 and d_k[s] = 0, and its output
 * is unspecified: the caller re-runs those stacks with mxfft_prescale_stats +
 * mxfft_fft2 (pipeline_resolve does).  Settled rows carry flags = 8: k and k1
 * exact, a_max to 2^-23 relative, p_tau = NaN, k2 = INT32_MIN, nnz = -1.
 * x, y: complex64 (nimg, n, n), out of place, 16-byte aligned; workspace: at
 * least mxfft_pipeline_folded_workspace_bytes(plan, nimg, coils) bytes. */
int32_t mxfft_pipeline_folded_supported(mxfft_plan plan);
int64_t mxfft_pipeline_folded_workspace_bytes(mxfft_plan plan, int64_t nimg, int32_t coils);
int32_t mxfft_pipeline_folded(mxfft_plan plan, const void* x, void* y, int64_t nimg, int32_t coils,
                              int32_t roundtrip, const mxfft_prescale_cfg* cfg, mxfft_prescale_result* d_res,
                              int32_t* d_k, void* workspace, int64_t workspace_bytes, uintptr_t stream);

/* The fold's building blocks for ONE image whose rows are split across ranks
 * (compute_prescale over the whole image, prescale.py:61-73, SPEC.md:205;
 * distributed.pipeline_slab combines them with two small all-reduces):
 *  - fft_rows_evidence: the first row pass (fftcore.py:351) of this rank's
 *    rows on the UNSCALED input (n = 16384), plus the evidence words of
 *    mxfft_pipeline_folded in d_words (mxfft_fold_words_bytes(batch * n) bytes);
 *  - fold_reduce, step 0: d_g (8 words) <- this rank's largest key, exponent
 *    range and replay flag (g[0..3]; combine across ranks with MAX); step 1:
 *    with the GLOBAL g[0] in place, g[4] += zero points, g[5] += threads below
 *    the threshold (combine with SUM), g[6] = ~(smallest word) (MAX);
 *  - fold_finish: k and the result row (flags 8 / 4 as mxfft_pipeline_folded)
 *    from the combined g and the image's total point count. */
int64_t mxfft_fold_words_bytes(int64_t npoints);
int32_t mxfft_fft_rows_evidence(mxfft_plan plan, const void* x, void* y, int64_t batch, int32_t inverse,
                                void* d_words, int64_t words_bytes, uintptr_t stream);
int32_t mxfft_fold_reduce(const void* d_words, int64_t npoints, const mxfft_prescale_cfg* cfg, int32_t step,
                          uint32_t* d_g, uintptr_t stream);
int32_t mxfft_fold_finish(const uint32_t* d_g, int64_t total_points, const mxfft_prescale_cfg* cfg,
                          mxfft_prescale_result* d_res, int32_t* d_k, uintptr_t stream);

/* mxfft_rss with the pipelines' FP64 epilogue folded in: every coil value of
 * group g is multiplied by 2^(k_sign * d_k[g] + exp_const) in FP64 (exact)
 * before |.| -- the x 1/N^2 and undo_prescale of roundtrip_pipeline /
 * forward_pipeline (mri.py:84-107, prescale.py:89-91) done in FP64 as the
 * reference does.  d_k may be NULL (then only exp_const applies). */
int32_t mxfft_rss_scaled(const void* x, int32_t is_c128, int64_t groups, int32_t coils, int64_t npix,
                         const int32_t* d_k, int32_t k_sign, int32_t exp_const, double* out, uintptr_t stream);

/* apply_prescale (prescale.py:76-86) on complex128 input followed by the
 * transform's complex64 cast (fftcore.py:262): y (complex64) =
 * x (complex128) * 2^d_k[seg], the product in FP64, rounded to FP32 once;
 * nseg contiguous segments of seg_points values. */
int32_t mxfft_prescale_apply_c128(const void* x, void* y, int64_t nseg, int64_t seg_points, const int32_t* d_k,
                                  uintptr_t stream);

/* _mx_multiply_batch (fftcore.py:150-183) / butterfly_mx (fftcore.py:186-235):
 * v complex128 (rows, m) in blocks of cpb complex values; twiddle codes
 * wcr, wci (m/cpb, cpb) and scales ws (m/cpb), FP64, shared by every row.
 * wv (complex128 (rows, m), may be NULL) receives the decoded MX products w*v
 * (v encoded per block, products in the reference's product dtype,
 * renormalized, requantized); with u (complex128, may be NULL) also
 * y0 = u32 + wv32 and y1 = u32 - wv32 (complex64).  *d_nonfinite is set
 * for a non-finite v block (the reference raises InvalidValue). */
int32_t mxfft_mx_multiply_f64(const void* v, const double* wcr, const double* wci, const double* ws, int64_t rows,
                              int32_t m, int32_t cpb, const mxfft_format* fmt, void* wv, const void* u, void* y0,
                              void* y1, int32_t* d_nonfinite, uintptr_t stream);

/* data * math.ldexp(1.0, k) (apply_prescale / undo_prescale, prescale.py:76-91)
 * on n elements of dtype 0 = float32, 1 = float64, 2 = complex64,
 * 3 = complex128; `factor` is 2^k already rounded to the array's precision
 * (numpy rounds the Python-float scalar the same way).  Complex elements are
 * multiplied as numpy multiplies by the scalar cast to complex:
 * (re f - im 0, re 0 + im f).  x may alias y. */
int32_t mxfft_scale(const void* x, void* y, int64_t n, int32_t dtype, double factor, uintptr_t stream);

/* Test instrumentation: run the 1-D row transform stage by stage through the
 * same device code as mxfft_fft_rows and record, per stage s (arrays laid out
 * [stage][batch][...]): v-block scale exponents v_exp (int32, n/2/cpb per row),
 * v codes (float, n/2 x 2), product exponents p_exp and shifts p_shift (int32),
 * product codes p_codes (float, n/2 x 2) and the stage output (complex64, n).
 * Any output pointer may be NULL.  y receives the final output. */
int32_t mxfft_fft_rows_debug(mxfft_plan plan, const void* x, void* y, int64_t batch,
                             int32_t inverse, int32_t* v_exp, float* v_codes, int32_t* p_exp,
                             int32_t* p_shift, float* p_codes, void* stage_out, uintptr_t stream);

/* Test instrumentation: compare the hardware quantizer used inside the
 * transform (F2FP.SATFINITE pack + unpack) with the reference-literal FP64
 * quantizer over all 2^32 FP32 bit patterns (non-finite skipped).  Adds the
 * mismatch count to *d_mismatches and atomicMin's the first bad pattern into
 * *d_first_bad (device pointers; initialise to 0 / 0xffffffff). */
int32_t mxfft_selftest_hw_quantizer(const mxfft_format* fmt, uint64_t* d_mismatches,
                                    uint32_t* d_first_bad, uintptr_t stream);

/* Profiling knob: run only the first `limit` butterfly stages of every line
 * pass (the output is then NOT a transform); limit < 0 restores full passes. */
void mxfft_profile_stage_limit(int32_t limit);
/* Profiling knob for the line kernel: bit 0 skips the tile loads, bit 1 the
 * stores (outputs are then NOT valid); 0 restores normal passes. */
void mxfft_profile_flags(int32_t flags);
/* Scheduling knob for the line kernels: cap the persistent grid at n CTAs per
 * SM (n <= 0: as many as fit).  Results are unchanged. */
void mxfft_lines_ctas_per_sm(int32_t n);

/* Total number of kernels this library has launched in the process
 * (bookkeeping for the benchmark's gpu_launches count). */
int64_t mxfft_launch_count(void);

#ifdef __cplusplus
}
#endif

#endif /* MXFFT_B200_H */
