// mxfft_capi.cu -- extern "C" entry points declared in include/mxfft_b200.h.
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <tuple>

#include "../../include/mxfft_b200.h"
#include "mxfft_common.cuh"
#include "mxfft_internal.h"

namespace mxfft {
static std::atomic<long long> g_launches{0};
#ifndef MXFFT_PDL
#define MXFFT_PDL 1
#endif
int g_pdl = MXFFT_PDL;
void note_launch(int n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

static std::mutex g_attr_mu;
static std::map<std::tuple<const void*, int, int>, int> g_smem_attr;          // (k, dev, -) -> limit set
static std::map<std::tuple<const void*, int, int, size_t>, int> g_occ;       // (k, dev, nt, smem) -> CTAs/SM
static std::map<std::pair<int, int>, int> g_dev_attr;                        // (dev, attr) -> value

cudaError_t ensure_smem_attr(const void* k, int smem_max) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    std::lock_guard<std::mutex> g(g_attr_mu);
    auto key = std::make_tuple(k, dev, 0);
    auto it = g_smem_attr.find(key);
    if (it != g_smem_attr.end() && it->second >= smem_max) return cudaSuccess;
    e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_max);
    if (e == cudaSuccess) g_smem_attr[key] = smem_max;
    return e;
}

cudaError_t cached_occupancy(const void* k, int nt, size_t smem, int* occ) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    std::lock_guard<std::mutex> g(g_attr_mu);
    auto key = std::make_tuple(k, dev, nt, smem);
    auto it = g_occ.find(key);
    if (it != g_occ.end()) {
        *occ = it->second;
        return cudaSuccess;
    }
    int o = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, k, nt, smem);
    if (e != cudaSuccess) return e;
    o = o < 1 ? 1 : o;
    g_occ[key] = o;
    *occ = o;
    return cudaSuccess;
}

int device_attr(cudaDeviceAttr a) {
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> g(g_attr_mu);
    auto key = std::make_pair(dev, (int)a);
    auto it = g_dev_attr.find(key);
    if (it != g_dev_attr.end()) return it->second;
    int v = 0;
    cudaDeviceGetAttribute(&v, a, dev);
    g_dev_attr[key] = v;
    return v;
}
cudaError_t plan_encode(Plan& p, const double* d_tw, cudaStream_t st);
cudaError_t launch_prescale(const void* x, int is_c128, int64_t nseg, int64_t npts,
                            const mxfft_prescale_cfg& c, mxfft_prescale_result* out, int32_t* kvec,
                            void* ws, int64_t ws_bytes, cudaStream_t st);
int64_t prescale_fast_ws_bytes(int64_t nseg, int64_t npts);
bool prescale_fast_ok(int64_t npts);
}  // namespace mxfft

using namespace mxfft;

struct mxfft_plan_s {
    Plan p;
};

static thread_local std::string g_err;

static int32_t fail(int32_t code, const std::string& msg) {
    g_err = msg;
    return code;
}

static int32_t cuda_fail(cudaError_t e, const char* where) {
    return fail(MXFFT_ERR_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

#define CK(call, where)                                   \
    do {                                                  \
        cudaError_t _e = (call);                          \
        if (_e != cudaSuccess) return cuda_fail(_e, where); \
    } while (0)

static bool check_fmt(const mxfft_format* f, std::string& why) {
    if (!f) {
        why = "null format";
        return false;
    }
    if (f->exponent_bits < 2) {
        why = "exponent_bits must be >= 2";
        return false;
    }
    if (f->mantissa_bits < 1) {
        why = "mantissa_bits must be >= 1";
        return false;
    }
    if (f->policy < 0 || f->policy > 2) {
        why = "unknown policy";
        return false;
    }
    if (f->exponent_bits > 11 || f->mantissa_bits > 52) {
        why = "format wider than FP64 is not supported";
        return false;
    }
    return true;
}

static FmtDesc desc_of(const mxfft_format* f) {
    return make_fmt(f->exponent_bits, f->mantissa_bits, f->policy, f->bias);
}

// a plan's tables live on the device it was created on
static int32_t check_plan(mxfft_plan plan) {
    if (!plan) return fail(MXFFT_ERR_VALUE, "null plan");
    int dev = -1;
    cudaGetDevice(&dev);
    if (dev != plan->p.device)
        return fail(MXFFT_ERR_VALUE, "plan was created on device " + std::to_string(plan->p.device) +
                                         ", current device is " + std::to_string(dev));
    return MXFFT_OK;
}
#define CHECK_PLAN(plan)                            \
    do {                                            \
        const int32_t _c = check_plan(plan);        \
        if (_c != MXFFT_OK) return _c;              \
    } while (0)

static int ilog2(int64_t n) {
    int s = 0;
    while ((int64_t(1) << s) < n) ++s;
    return s;
}

extern "C" {

int32_t mxfft_version(void) { return 1; }

const char* mxfft_last_error(void) { return g_err.c_str(); }

int64_t mxfft_launch_count(void) { return g_launches.load(); }

void mxfft_profile_stage_limit(int32_t limit) { mxfft::g_profile_stage_limit = limit; }
void mxfft_profile_flags(int32_t flags) { mxfft::g_profile_flags = flags; }
void mxfft_lines_ctas_per_sm(int32_t n) { mxfft::g_lines_ctas_per_sm = n < 0 ? 0 : n; }

int32_t mxfft_quantize_f64(const double* x, double* out, int64_t n, const mxfft_format* fmt,
                           int32_t* d_nonfinite, uintptr_t stream) {
    std::string why;
    if (!check_fmt(fmt, why)) return fail(MXFFT_ERR_VALUE, why);
    if (n < 0) return fail(MXFFT_ERR_SHAPE, "negative length");
    CK(launch_quantize_f64(x, out, n, desc_of(fmt), d_nonfinite, (cudaStream_t)stream),
       "quantize_f64");
    return MXFFT_OK;
}

int32_t mxfft_mx_encode_f64(const double* v, int64_t nblocks, int32_t block_len,
                            const mxfft_format* fmt, double* codes, double* scales,
                            int32_t* d_nonfinite, uintptr_t stream) {
    std::string why;
    if (!check_fmt(fmt, why)) return fail(MXFFT_ERR_VALUE, why);
    if (block_len < 1 || nblocks < 0) return fail(MXFFT_ERR_SHAPE, "block must be non-empty");
    CK(launch_encode_f64(v, nblocks, block_len, desc_of(fmt), codes, scales, nullptr, d_nonfinite,
                         (cudaStream_t)stream),
       "mx_encode_f64");
    return MXFFT_OK;
}

int32_t mxfft_mx_decode_f64(const double* codes, const double* scales, int64_t nblocks,
                            int32_t block_len, double* out, uintptr_t stream) {
    if (block_len % 2 != 0) return fail(MXFFT_ERR_SHAPE, "complex block length must be even");
    CK(launch_decode_f64(codes, scales, nblocks, block_len, out, (cudaStream_t)stream),
       "mx_decode_f64");
    return MXFFT_OK;
}

int32_t mxfft_plan_create(mxfft_plan* plan, int32_t n, const mxfft_format* fmt,
                          int32_t block_size, const double* h_twiddles, uintptr_t stream) {
    if (!plan) return fail(MXFFT_ERR_VALUE, "null plan pointer");
    *plan = nullptr;
    if (n < 2 || (n & (n - 1)))
        return fail(MXFFT_ERR_UNSUPPORTED_SIZE,
                    "transform length must be a power of two >= 2, got " + std::to_string(n));
    if (block_size < 2 || block_size % 2)
        return fail(MXFFT_ERR_VALUE, "block_size must be an even integer >= 2");
    std::string why;
    if (!check_fmt(fmt, why)) return fail(MXFFT_ERR_VALUE, why);
    const int m = n / 2;
    const int cpb = std::min(block_size / 2, m);  // fftcore.py:109
    if (m % cpb != 0)
        return fail(MXFFT_ERR_VALUE, "block_size/2 must divide n/2 (fftcore.py:139-141 reshape)");
    auto* h = new mxfft_plan_s;
    Plan& p = h->p;
    p.n = n;
    p.log2n = ilog2(n);
    p.block_size = block_size;
    p.cpb = cpb;
    p.fmt = desc_of(fmt);
    cudaGetDevice(&p.device);
    const int st = p.log2n;
    const int nb = m / cpb;
    cudaStream_t s = (cudaStream_t)stream;
    double* d_tw = nullptr;
    cudaError_t e;
    if ((e = cudaMalloc(&p.d_wcr, sizeof(double) * st * m)) != cudaSuccess ||
        (e = cudaMalloc(&p.d_wci, sizeof(double) * st * m)) != cudaSuccess ||
        (e = cudaMalloc(&p.d_wsexp, sizeof(int) * st * nb)) != cudaSuccess ||
        (e = cudaMalloc(&p.d_tw16_fwd, sizeof(unsigned) * n)) != cudaSuccess ||
        (e = cudaMalloc(&p.d_tw16_inv, sizeof(unsigned) * n)) != cudaSuccess ||
        (e = cudaMalloc(&p.d_twe8, n)) != cudaSuccess ||
        (e = cudaMalloc(&d_tw, sizeof(double) * 2 * st * m)) != cudaSuccess ||
        (e = cudaMemcpyAsync(d_tw, h_twiddles, sizeof(double) * 2 * st * m,
                             cudaMemcpyHostToDevice, s)) != cudaSuccess ||
        (e = plan_encode(p, d_tw, s)) != cudaSuccess || (e = cudaStreamSynchronize(s)) != cudaSuccess) {
        cudaFree(d_tw);
        mxfft_plan_destroy(h);
        return cuda_fail(e, "plan_create");
    }
    cudaFree(d_tw);
    if (mx_lines_ok(p) && last_stage_ok(p)) {
        // the n/2-point plan of the first L-1 stages (split row passes of
        // mxfft_fft2): kernel tables are the prefix of this plan's; the
        // reference-layout rows (exact replays) are copied
        Plan* hp = new Plan;
        *hp = p;
        hp->half = nullptr;
        hp->n = n / 2;
        hp->log2n = p.log2n - 1;
        const int hm = n / 4, hnb = hm / p.cpb;
        hp->d_wcr = hp->d_wci = nullptr;
        hp->d_wsexp = nullptr;
        if ((e = cudaMalloc(&hp->d_wcr, sizeof(double) * hp->log2n * hm)) != cudaSuccess ||
            (e = cudaMalloc(&hp->d_wci, sizeof(double) * hp->log2n * hm)) != cudaSuccess ||
            (e = cudaMalloc(&hp->d_wsexp, sizeof(int) * hp->log2n * hnb)) != cudaSuccess ||
            (e = cudaMemcpy2D(hp->d_wcr, sizeof(double) * hm, p.d_wcr, sizeof(double) * m, sizeof(double) * hm,
                              hp->log2n, cudaMemcpyDeviceToDevice)) != cudaSuccess ||
            (e = cudaMemcpy2D(hp->d_wci, sizeof(double) * hm, p.d_wci, sizeof(double) * m, sizeof(double) * hm,
                              hp->log2n, cudaMemcpyDeviceToDevice)) != cudaSuccess ||
            (e = cudaMemcpy2D(hp->d_wsexp, sizeof(int) * hnb, p.d_wsexp, sizeof(int) * nb, sizeof(int) * hnb,
                              hp->log2n, cudaMemcpyDeviceToDevice)) != cudaSuccess) {
            cudaFree(hp->d_wcr);
            cudaFree(hp->d_wci);
            cudaFree(hp->d_wsexp);
            delete hp;
            mxfft_plan_destroy(h);
            return cuda_fail(e, "plan_create (half plan)");
        }
        p.half = hp;
    }
    *plan = h;
    return MXFFT_OK;
}

int32_t mxfft_plan_destroy(mxfft_plan plan) {
    if (!plan) return MXFFT_OK;
    Plan& p = plan->p;
    if (p.half) {  // (its kernel tables alias this plan's)
        cudaFree(p.half->d_wcr);
        cudaFree(p.half->d_wci);
        cudaFree(p.half->d_wsexp);
        delete p.half;
        p.half = nullptr;
    }
    cudaFree(p.d_wcr);
    cudaFree(p.d_wci);
    cudaFree(p.d_wsexp);
    cudaFree(p.d_tw16_fwd);
    cudaFree(p.d_tw16_inv);
    cudaFree(p.d_twe8);
    delete plan;
    return MXFFT_OK;
}

int32_t mxfft_plan_twiddles(mxfft_plan plan, double* h_codes_re, double* h_codes_im,
                            double* h_scales) {
    CHECK_PLAN(plan);
    const Plan& p = plan->p;
    const int m = p.n / 2, nb = m / p.cpb, st = p.log2n;
    CK(cudaMemcpy(h_codes_re, p.d_wcr, sizeof(double) * st * m, cudaMemcpyDeviceToHost), "plan_twiddles");
    CK(cudaMemcpy(h_codes_im, p.d_wci, sizeof(double) * st * m, cudaMemcpyDeviceToHost), "plan_twiddles");
    int* tmp = new int[st * nb];
    cudaError_t e = cudaMemcpy(tmp, p.d_wsexp, sizeof(int) * st * nb, cudaMemcpyDeviceToHost);
    if (e == cudaSuccess)
        for (int i = 0; i < st * nb; ++i) h_scales[i] = std::ldexp(1.0, tmp[i]);
    delete[] tmp;
    if (e != cudaSuccess) return cuda_fail(e, "plan_twiddles");
    return MXFFT_OK;
}

int32_t mxfft_fft_rows(mxfft_plan plan, const void* x, void* y, int64_t batch, int32_t inverse,
                       uintptr_t stream) {
    CHECK_PLAN(plan);
    if (batch < 0) return fail(MXFFT_ERR_SHAPE, "negative batch");
    if (batch == 0) return MXFFT_OK;
    LinePass lp;
    lp.in = x;
    lp.out = y;
    lp.col_mode = 0;
    lp.lines_per_image = 1;
    lp.total_lines = batch;
    lp.img_elems = plan->p.n;
    lp.inverse = inverse ? 1 : 0;
    CK(run_lines(plan->p, lp, (cudaStream_t)stream), "fft_rows");
    return MXFFT_OK;
}

int32_t mxfft_fft_rows_scaled(mxfft_plan plan, const void* x, void* y, int64_t batch, int32_t inverse,
                              int32_t exp_in, int32_t exp_out, uintptr_t stream) {
    CHECK_PLAN(plan);
    if (batch < 0) return fail(MXFFT_ERR_SHAPE, "negative batch");
    if (batch == 0) return MXFFT_OK;
    LinePass lp;
    lp.in = x;
    lp.out = y;
    lp.lines_per_image = 1;
    lp.total_lines = batch;
    lp.img_elems = plan->p.n;
    lp.inverse = inverse ? 1 : 0;
    lp.kin_const = exp_in;
    lp.kout_const = exp_out;
    CK(run_lines(plan->p, lp, (cudaStream_t)stream), "fft_rows_scaled");
    return MXFFT_OK;
}

int32_t mxfft_fft_rows_seg(mxfft_plan plan, const void* x, void* y, int64_t lines, int32_t inverse, int32_t exp_in,
                           int32_t exp_out, int32_t seg_len, uintptr_t stream) {
    CHECK_PLAN(plan);
    if (lines < 0) return fail(MXFFT_ERR_SHAPE, "negative batch");
    if (lines == 0) return MXFFT_OK;
    const int n = plan->p.n;
    if (seg_len < 2 || (seg_len & (seg_len - 1)) || seg_len > n || n % seg_len)
        return fail(MXFFT_ERR_SHAPE, "seg_len must be a power of two dividing n");
    if (x == y) return fail(MXFFT_ERR_VALUE, "segmented rows are out of place");
    LinePass lp;
    lp.in = x;
    lp.out = y;
    lp.lines_per_image = 1;
    lp.total_lines = lines;
    lp.img_elems = n;
    lp.inverse = inverse ? 1 : 0;
    lp.kin_const = exp_in;
    lp.kout_const = exp_out;
    lp.seg_log2 = ilog2(seg_len);
    lp.seg_stride = lines * (int64_t)seg_len;
    if (seg_len < n) {
        if (!mx_lines_ok(plan->p)) return fail(MXFFT_ERR_VALUE, "segmented rows need a line-kernel plan");
        CK(run_mx_lines(plan->p, lp, (cudaStream_t)stream), "fft_rows_seg");
    } else {
        lp.seg_log2 = 0;  // one segment: plain rows
        CK(run_lines(plan->p, lp, (cudaStream_t)stream), "fft_rows_seg");
    }
    return MXFFT_OK;
}

int32_t mxfft_fft_cols(mxfft_plan plan, const void* x, void* y, int64_t batch, int32_t inverse,
                       uintptr_t stream) {
    CHECK_PLAN(plan);
    if (batch < 0) return fail(MXFFT_ERR_SHAPE, "negative batch");
    if (batch == 0) return MXFFT_OK;
    LinePass lp;
    lp.in = x;
    lp.out = y;
    lp.col_mode = 1;
    lp.img_elems = (int64_t)plan->p.n * plan->p.n;
    lp.lines_per_image = plan->p.n;
    lp.total_lines = batch * plan->p.n;
    lp.batch = batch;
    lp.inverse = inverse ? 1 : 0;
    CK(run_lines(plan->p, lp, (cudaStream_t)stream), "fft_cols");
    return MXFFT_OK;
}

int64_t mxfft_fft2_workspace_bytes(mxfft_plan plan, int64_t batch) {
    if (!plan || batch <= 0 || !mx_lines_ok(plan->p)) return 0;
    // split row passes (n >= 16384) stage the half-row outputs in a second image buffer
    const int64_t copies = plan->p.half ? 2 : 1;
    return copies * batch * (int64_t)plan->p.n * plan->p.n * 8;
}

void mxfft_split_last_stage(int32_t on) { mxfft::g_split_last_stage = on ? 1 : 0; }

int32_t mxfft_fft2(mxfft_plan plan, const void* x, void* y, int64_t batch, int32_t mode,
                   const int32_t* d_k, int32_t k_group, void* workspace, int64_t workspace_bytes,
                   uintptr_t stream) {
    CHECK_PLAN(plan);
    if (mode < 0 || mode > 2) return fail(MXFFT_ERR_VALUE, "mode must be 0 (forward), 1 (inverse) or 2 (round trip)");
    if (batch < 0) return fail(MXFFT_ERR_SHAPE, "negative batch");
    if (batch == 0) return MXFFT_OK;
    const Plan& p = plan->p;
    cudaStream_t s = (cudaStream_t)stream;
    // n = 128: automatic choice (g_fused_image < 0) = the four TMA line passes when the
    // caller gave the transposed-store workspace and the batch fills the GPU (measured
    // 806 vs 862 us for 4096 images), else the one-image-per-CTA kernel (one launch, no
    // workspace)
    const bool want_fused = g_fused_image < 0 ? (workspace == nullptr || batch < 64) : g_fused_image != 0;
    if (want_fused && mx_image_ok(p)) {
        // n = 128: one image per CTA, every pass in shared memory (exact replays
        // re-read an image from x before any of its outputs is written, so x
        // may alias y here too)
        const mxfft_prescale_cfg dummy{1.0, 1.0, 1.0, 0, 0};
        CK(run_mx_image(p, x, y, batch, mode, dummy, nullptr, nullptr, d_k, k_group > 0 ? k_group : 1, s),
           "fft2 (fused image kernel)");
        return MXFFT_OK;
    }
    const int64_t nn = (int64_t)p.n * p.n;
    const int npass = mode == 2 ? 4 : 2;
    if (p.half && g_split_last_stage && workspace && workspace_bytes >= 2 * batch * nn * 8) {
        // n >= 16384: every pass = stages 0 .. L-2 on the decimated half rows
        // (the n/2-point line kernel, two CTAs per SM) + the last stage fused
        // into the transposed store.  x -> W2 -> W1 [-> W2 -> W1 -> W2 -> W1] -> W2 -> y
        float2* w1 = reinterpret_cast<float2*>(workspace);
        float2* w2 = w1 + batch * nn;
        for (int pass = 0; pass < npass; ++pass) {
            const bool inv = mode == 1 || (mode == 2 && pass >= 2);
            const bool last = pass == npass - 1;
            LinePass lp;
            lp.in = pass == 0 ? x : (const void*)w1;
            lp.out = w2;
            lp.dec = 1;
            lp.lines_per_image = 2 * p.n;
            lp.total_lines = batch * 2 * (int64_t)p.n;
            lp.img_elems = nn;
            lp.inverse = inv;
            lp.kvec = d_k;
            lp.k_group = k_group > 0 ? k_group : 1;
            if (pass == 0 && d_k) lp.kin_sign = 1;
            CK(run_mx_lines(*p.half, lp, s), "fft2 (half rows)");
            LastStagePass ls;
            ls.in = w2;
            ls.out = last ? y : (void*)w1;
            ls.batch = batch;
            ls.inverse = inv;
            ls.kvec = d_k;
            ls.k_group = k_group > 0 ? k_group : 1;
            ls.kout_sign = last && d_k ? -1 : 0;
            ls.kout_const = last && mode == 2 ? -2 * p.log2n : 0;
            CK(run_last_stage_transpose(p, ls, s), "fft2 (last stage + transpose)");
        }
        return MXFFT_OK;
    }
    // With a workspace every pass is a row pass that stores its lines transposed
    // (rows.T of fft_2d, fftcore.py:351-353): x -> ws -> y [-> ws -> y].  Both
    // reads and writes then move whole 128-byte lines.  Without one, the
    // second pass walks the columns in place.
    const int64_t need = mxfft_fft2_workspace_bytes(plan, batch);
    const bool tpose = workspace && need > 0;
    if (workspace && need > 0 && workspace_bytes < need)
        return fail(MXFFT_ERR_VALUE, "fft2 workspace too small");
    // n >= 4096 (one line per group or CTA): a transposed store would scatter
    // 8-byte elements over n rows, so those passes store plain rows and a tiled
    // transpose kernel follows: x -> y -T-> ws -> ws -T-> y [-> y -T-> ws -> ws -T-> y]
    const bool split_t = tpose && p.n >= 4096;  // measured: 4096 split 3.2 vs 5.2 ms per 2^28-point pass; 2048 tstore wins
    for (int pass = 0; pass < npass; ++pass) {
        LinePass lp;
        if (split_t) {
            lp.in = pass == 0 ? x : ((pass & 1) ? workspace : y);
            lp.out = (pass & 1) ? workspace : y;
        } else if (tpose) {
            lp.in = pass == 0 ? x : ((pass & 1) ? workspace : y);
            lp.out = (pass & 1) ? y : workspace;
            lp.tstore = 1;
        } else {
            lp.in = pass == 0 ? x : y;
            lp.out = y;
            lp.col_mode = pass & 1;
        }
        lp.img_elems = nn;
        lp.lines_per_image = p.n;
        lp.total_lines = batch * p.n;
        lp.batch = batch;
        lp.inverse = mode == 1 || (mode == 2 && pass >= 2);
        lp.reverse = !split_t && (pass & 1);  // read the previous pass's output newest first
        lp.kvec = d_k;
        lp.k_group = k_group > 0 ? k_group : 1;
        if (pass == 0 && d_k) lp.kin_sign = 1;
        if (pass == npass - 1) {
            if (d_k) lp.kout_sign = -1;
            if (mode == 2) lp.kout_const = -2 * p.log2n;  // x 1/n^2 (mri.py:100)
        }
        CK(run_lines(p, lp, s), "fft2");
        if (split_t)
            CK(launch_transpose_c64(lp.out, (pass & 1) ? y : workspace, batch, p.n, s), "fft2 transpose");
    }
    return MXFFT_OK;
}

static bool pow2_len(int32_t n) { return n >= 2 && n <= 16384 && !(n & (n - 1)); }

int32_t mxfft_fft_rows_fp16(const void* x, int32_t x_is_c128, void* y, int64_t batch, int32_t n,
                            const void* d_tw, int32_t inverse, int32_t* d_nonfinite, uintptr_t stream) {
    if (batch < 0) return fail(MXFFT_ERR_SHAPE, "negative batch");
    if (!pow2_len(n)) return fail(MXFFT_ERR_UNSUPPORTED_SIZE, "fp16 rows: n must be a power of two in [2, 16384]");
    CK(launch_fp16_rows(x, x_is_c128, y, batch, n, d_tw, inverse, d_nonfinite, (cudaStream_t)stream), "fft_rows_fp16");
    return MXFFT_OK;
}

int32_t mxfft_fft_rows_f64(const void* x, void* y, int64_t batch, int32_t n, const void* d_tw, int32_t inverse,
                           uintptr_t stream) {
    if (batch < 0) return fail(MXFFT_ERR_SHAPE, "negative batch");
    if (!pow2_len(n)) return fail(MXFFT_ERR_UNSUPPORTED_SIZE, "f64 rows: n must be a power of two in [2, 16384]");
    if (x == y) return fail(MXFFT_ERR_VALUE, "f64 rows are out of place (bit-reversed gather)");
    CK(launch_f64_rows(x, y, batch, n, d_tw, inverse, (cudaStream_t)stream), "fft_rows_f64");
    return MXFFT_OK;
}

int32_t mxfft_metrics(const double* ref, const double* test, int64_t h, int64_t w, int32_t do_ssim,
                      const double* d_window, double c1, double c2, double* d_out, uintptr_t stream) {
    if (h < 0 || w < 0) return fail(MXFFT_ERR_SHAPE, "negative image size");
    if (do_ssim && (h < 11 || w < 11)) return fail(MXFFT_ERR_SHAPE, "image smaller than the 11x11 SSIM window");
    CK(launch_metrics(ref, test, h, w, do_ssim, d_window, c1, c2, d_out, (cudaStream_t)stream), "metrics");
    return MXFFT_OK;
}

int32_t mxfft_transpose_c64(const void* x, void* y, int64_t batch, int32_t n, uintptr_t stream) {
    return mxfft_transpose_c64_strided(x, 0, 0, y, batch, n, stream);
}

int32_t mxfft_transpose_c64_strided(const void* x, int64_t ld_x, int64_t batch_stride_x, void* y, int64_t batch,
                                    int32_t n, uintptr_t stream) {
    if (batch < 0 || n <= 0) return fail(MXFFT_ERR_SHAPE, "bad transpose shape");
    if (n % 64) return fail(MXFFT_ERR_UNSUPPORTED_SIZE, "transpose needs n to be a multiple of 64");
    if (x == y) return fail(MXFFT_ERR_VALUE, "transpose is out of place");
    if (ld_x != 0 && ld_x < n) return fail(MXFFT_ERR_SHAPE, "source row stride below n");
    CK(launch_transpose_c64(x, y, batch, n, (cudaStream_t)stream, ld_x, batch_stride_x), "transpose");
    return MXFFT_OK;
}

int64_t mxfft_prescale_workspace_bytes(int64_t nseg, int64_t seg_points) {
    // sampled fast path for complex64 segments; 0 means "exact kernel only"
    if (nseg <= 0 || !prescale_fast_ok(seg_points) || (seg_points & 1)) return 0;
    return prescale_fast_ws_bytes(nseg, seg_points);
}

int32_t mxfft_prescale_stats(const void* x, int32_t is_c128, int64_t nseg, int64_t seg_points,
                             const mxfft_prescale_cfg* cfg, mxfft_prescale_result* d_out,
                             int32_t* d_k, void* workspace, int64_t workspace_bytes,
                             uintptr_t stream) {
    if (!cfg) return fail(MXFFT_ERR_VALUE, "null config");
    if (nseg < 0 || seg_points < 0) return fail(MXFFT_ERR_SHAPE, "negative size");
    if (nseg == 0) return MXFFT_OK;
    if (seg_points > (int64_t)0x7fffffff) return fail(MXFFT_ERR_UNSUPPORTED_SIZE, "segment too large");
    if (seg_points & 1) workspace = nullptr;  // fast path reads complex pairs
    CK(launch_prescale(x, is_c128, nseg, seg_points, *cfg, d_out, d_k, workspace, workspace_bytes,
                       (cudaStream_t)stream),
       "prescale_stats");
    return MXFFT_OK;
}

int32_t mxfft_cabs(const void* x, int32_t is_c128, int64_t n, double* out, uintptr_t stream) {
    if (n < 0) return fail(MXFFT_ERR_SHAPE, "negative size");
    CK(launch_cabs(x, is_c128, n, out, (cudaStream_t)stream), "cabs");
    return MXFFT_OK;
}

int32_t mxfft_prescale_sample_keys(const void* x, int64_t npts, int64_t nsamples, float* d_keys,
                                   uintptr_t stream) {
    if (npts < 4 || (npts & 3)) return fail(MXFFT_ERR_SHAPE, "sampling needs a multiple of 4 points");
    if (nsamples < 0 || (nsamples & 3)) return fail(MXFFT_ERR_VALUE, "nsamples must be a multiple of 4");
    CK(launch_prescale_sample_keys(reinterpret_cast<const float2*>(x), npts, nsamples, d_keys,
                                   (cudaStream_t)stream),
       "prescale_sample_keys");
    return MXFFT_OK;
}

int32_t mxfft_prescale_count_range(const void* x, int64_t npts, float lo, float hi, float top, void* d_state,
                                   void* d_cand, int64_t cand_cap, void* d_top, int64_t top_cap,
                                   uintptr_t stream) {
    if (npts < 0 || (npts & 1)) return fail(MXFFT_ERR_SHAPE, "count needs an even number of points");
    CK(launch_prescale_count_range(reinterpret_cast<const float2*>(x), npts, lo, hi, top, d_state,
                                   reinterpret_cast<float2*>(d_cand), cand_cap, reinterpret_cast<float2*>(d_top),
                                   top_cap, (cudaStream_t)stream),
       "prescale_count_range");
    return MXFFT_OK;
}

int32_t mxfft_rss(const void* x, int32_t is_c128, int64_t groups, int32_t coils, int64_t npix,
                  double* out, uintptr_t stream) {
    if (coils < 1) return fail(MXFFT_ERR_SHAPE, "need at least one coil");
    CK(launch_rss(x, is_c128, groups, coils, npix, out, (cudaStream_t)stream), "rss");
    return MXFFT_OK;
}

void mxfft_fused_image(int32_t on) { mxfft::g_fused_image = on < 0 ? -1 : (on ? 1 : 0); }
void mxfft_tma_store(int32_t on) { mxfft::g_tma_store = on ? 1 : 0; }
void mxfft_pdl(int32_t on) { mxfft::g_pdl = on ? 1 : 0; }

int32_t mxfft_pipeline_fused_supported(mxfft_plan plan) { return plan && mx_image_ok(plan->p) ? 1 : 0; }

int32_t mxfft_pipeline_fused(mxfft_plan plan, const void* x, void* y, int64_t nimg, int32_t roundtrip,
                             const mxfft_prescale_cfg* cfg, mxfft_prescale_result* d_res, int32_t* d_k,
                             uintptr_t stream) {
    CHECK_PLAN(plan);
    if (!cfg) return fail(MXFFT_ERR_VALUE, "null config");
    if (nimg < 0) return fail(MXFFT_ERR_SHAPE, "negative batch");
    if (!mx_image_ok(plan->p))
        return fail(MXFFT_ERR_UNSUPPORTED_SIZE, "the fused pipeline needs n = 128, a hardware MX format and B in {16, 32, 64}");
    if (!d_res) return fail(MXFFT_ERR_VALUE, "null result rows");
    if (x == y) return fail(MXFFT_ERR_VALUE, "the fused pipeline is out of place (exact replays re-read the input)");
    CK(run_mx_image(plan->p, x, y, nimg, roundtrip ? 2 : 0, *cfg, d_res, d_k, nullptr, 1, (cudaStream_t)stream),
       "pipeline_fused");
    return MXFFT_OK;
}

// ---- statistics folded into the first pass (n = 128 / 256 / 512 on the TMA line kernel;
// n = 16384 on the split passes' half-row kernel) ----
static bool fold_ok_tma(const Plan& p) {
    return mxfft::g_tma_store && mx_lines_ok(p) && p.cpb >= 8 && p.log2n >= 7 && p.log2n <= 9;
}
static bool fold_ok_split(const Plan& p) {
    return p.half && mxfft::g_split_last_stage && mx_lines_ok(p) && p.cpb >= 8 && p.log2n == 14;
}
static bool fold_ok(const Plan& p) { return fold_ok_tma(p) || fold_ok_split(p); }
int32_t mxfft_pipeline_folded_supported(mxfft_plan plan) { return plan && fold_ok(plan->p) ? 1 : 0; }

int64_t mxfft_pipeline_folded_workspace_bytes(mxfft_plan plan, int64_t nimg, int32_t coils) {
    if (!plan || nimg <= 0 || coils < 1 || !fold_ok(plan->p)) return 0;
    const int64_t nn = (int64_t)plan->p.n * plan->p.n, nstack = nimg / coils;
    const int64_t copies = fold_ok_split(plan->p) ? 2 : 1;
    // scratch image(s) + warp words + thread words + the big-stack reduction scratch
    return copies * nimg * nn * 8 + nimg * nn / 512 * 4 + nimg * nn / 32 * 4 + ((nstack * 32 + 255) / 256) * 256;
}

int32_t mxfft_pipeline_folded(mxfft_plan plan, const void* x, void* y, int64_t nimg, int32_t coils,
                              int32_t roundtrip, const mxfft_prescale_cfg* cfg, mxfft_prescale_result* d_res,
                              int32_t* d_k, void* workspace, int64_t workspace_bytes, uintptr_t stream) {
    CHECK_PLAN(plan);
    if (!cfg) return fail(MXFFT_ERR_VALUE, "null config");
    if (nimg < 0 || coils < 1 || nimg % coils) return fail(MXFFT_ERR_SHAPE, "the batch is not a whole number of coil stacks");
    if (nimg == 0) return MXFFT_OK;
    const Plan& p = plan->p;
    if (!fold_ok(p))
        return fail(MXFFT_ERR_UNSUPPORTED_SIZE, "the folded pipeline needs n in {128, 256, 512, 16384}, a hardware MX format and B in {16, 32, 64}");
    if (!d_res || !d_k) return fail(MXFFT_ERR_VALUE, "null result rows / k vector");
    if (x == y) return fail(MXFFT_ERR_VALUE, "the folded pipeline is out of place (flagged stacks are re-run from the input)");
    if (!workspace || workspace_bytes < mxfft_pipeline_folded_workspace_bytes(plan, nimg, coils))
        return fail(MXFFT_ERR_VALUE, "folded pipeline workspace too small");
    if ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(y) | reinterpret_cast<uintptr_t>(workspace)) & 15)
        return fail(MXFFT_ERR_VALUE, "the folded pipeline needs 16-byte aligned buffers");
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t nn = (int64_t)p.n * p.n, nstack = nimg / coils;
    if ((int64_t)coils * nn >= (int64_t(1) << 32)) return fail(MXFFT_ERR_UNSUPPORTED_SIZE, "coil stack too large");
    const bool split = fold_ok_split(p);
    unsigned* acc = reinterpret_cast<unsigned*>(reinterpret_cast<char*>(workspace) + (split ? 2 : 1) * nimg * nn * 8);
    unsigned* minw = acc + nimg * nn / 512;
    unsigned* scratch = minw + nimg * nn / 32;
    const int npass = roundtrip ? 4 : 2;
    if (split) {
        // n = 16384: every pass = the 8192-point line kernel on the decimated half rows (the first
        // one with the evidence) + the last stage fused into the transposed store (see mxfft_fft2)
        float2* w1 = reinterpret_cast<float2*>(workspace);
        float2* w2 = w1 + nimg * nn;
        for (int pass = 0; pass < npass; ++pass) {
            const bool inv = roundtrip && pass >= 2;
            const bool last = pass == npass - 1;
            LinePass lp;
            lp.in = pass == 0 ? x : (const void*)w1;
            lp.out = w2;
            lp.dec = 1;
            lp.lines_per_image = 2 * p.n;
            lp.total_lines = nimg * 2 * (int64_t)p.n;
            lp.img_elems = nn;
            lp.inverse = inv;
            lp.k_group = coils;
            if (pass == 0) {
                lp.acc = acc;
                lp.minw = minw;
            }
            // (x 2^k happens at the load of the first pass's last-stage kernel, once k is known:
            // stages 0 .. 12 of the first row pass are the unscaled, range-tracked ones)
            CK(run_mx_lines(*p.half, lp, s), "pipeline_folded (half rows)");
            if (pass == 0)
                CK(launch_fold_resolve(acc, minw, nstack, coils * nn, *cfg, d_res, d_k, scratch, s),
                   "pipeline_folded (resolve)");
            LastStagePass ls;
            ls.in = w2;
            ls.out = last ? y : (void*)w1;
            ls.batch = nimg;
            ls.inverse = inv;
            ls.kvec = d_k;
            ls.k_group = coils;
            ls.kin_sign = pass == 0 ? 1 : 0;
            ls.kout_sign = last ? -1 : 0;
            ls.kout_const = last && roundtrip ? -2 * p.log2n : 0;
            CK(run_last_stage_transpose(p, ls, s), "pipeline_folded (last stage + transpose)");
        }
        return MXFFT_OK;
    }
    for (int pass = 0; pass < npass; ++pass) {
        LinePass lp;
        lp.in = pass == 0 ? x : ((pass & 1) ? workspace : y);
        lp.out = (pass & 1) ? y : workspace;
        lp.tstore = 1;
        lp.img_elems = nn;
        lp.lines_per_image = p.n;
        lp.total_lines = nimg * p.n;
        lp.batch = nimg;
        lp.inverse = roundtrip && pass >= 2;
        lp.reverse = pass & 1;
        lp.kvec = d_k;
        lp.k_group = coils;
        if (pass == 0) {
            lp.kvec = nullptr;  // unscaled; the pass gathers the evidence
            lp.acc = acc;
            lp.minw = minw;
        }
        if (pass == 1) lp.kin_sign = 1;  // x 2^k on the way in (exact: see k_fold_resolve)
        if (pass == npass - 1) {
            lp.kout_sign = -1;
            if (roundtrip) lp.kout_const = -2 * p.log2n;  // x 1/n^2 (mri.py:100)
        }
        CK(run_mx_lines(p, lp, s), "pipeline_folded");
        if (pass == 0)
            CK(launch_fold_resolve(acc, minw, nstack, coils * nn, *cfg, d_res, d_k, scratch, s),
               "pipeline_folded (resolve)");
    }
    return MXFFT_OK;
}

// ---- the fold's building blocks for one image split across ranks (distributed.pipeline_slab) ----
int64_t mxfft_fold_words_bytes(int64_t npoints) {
    return npoints > 0 && npoints % 1024 == 0 ? npoints / 512 * 4 + npoints / 32 * 4 : 0;
}

int32_t mxfft_fft_rows_evidence(mxfft_plan plan, const void* x, void* y, int64_t batch, int32_t inverse,
                                void* d_words, int64_t words_bytes, uintptr_t stream) {
    CHECK_PLAN(plan);
    const Plan& p = plan->p;
    if (batch <= 0) return fail(MXFFT_ERR_SHAPE, "need at least one row");
    if (!(mx_lines_ok(p) && p.cpb >= 8 && p.log2n == 14))
        return fail(MXFFT_ERR_UNSUPPORTED_SIZE, "rows with evidence need n = 16384, a hardware MX format and B in {16, 32, 64}");
    if (x == y) return fail(MXFFT_ERR_VALUE, "rows with evidence are out of place");
    const int64_t npoints = batch * (int64_t)p.n;
    if (!d_words || words_bytes < mxfft_fold_words_bytes(npoints)) return fail(MXFFT_ERR_VALUE, "evidence buffer too small");
    LinePass lp;
    lp.in = x;
    lp.out = y;
    lp.lines_per_image = 1;
    lp.total_lines = batch;
    lp.img_elems = p.n;
    lp.inverse = inverse ? 1 : 0;
    lp.acc = reinterpret_cast<unsigned*>(d_words);
    lp.minw = lp.acc + npoints / 512;
    CK(run_mx_lines(p, lp, (cudaStream_t)stream), "fft_rows_evidence");
    return MXFFT_OK;
}

int32_t mxfft_fold_reduce(const void* d_words, int64_t npoints, const mxfft_prescale_cfg* cfg, int32_t step,
                          uint32_t* d_g, uintptr_t stream) {
    if (!cfg || !d_words || !d_g) return fail(MXFFT_ERR_VALUE, "null argument");
    if (npoints <= 0 || npoints % 1024 || npoints >= (int64_t(1) << 32)) return fail(MXFFT_ERR_SHAPE, "bad point count");
    if (step != 0 && step != 1) return fail(MXFFT_ERR_VALUE, "step must be 0 or 1");
    const unsigned* acc = reinterpret_cast<const unsigned*>(d_words);
    CK(launch_fold_reduce(acc, acc + npoints / 512, npoints, *cfg, step, d_g, (cudaStream_t)stream), "fold_reduce");
    return MXFFT_OK;
}

int32_t mxfft_fold_finish(const uint32_t* d_g, int64_t total_points, const mxfft_prescale_cfg* cfg,
                          mxfft_prescale_result* d_res, int32_t* d_k, uintptr_t stream) {
    if (!cfg || !d_g || !d_res || !d_k) return fail(MXFFT_ERR_VALUE, "null argument");
    if (total_points <= 0 || total_points >= (int64_t(1) << 32)) return fail(MXFFT_ERR_SHAPE, "bad point count");
    CK(launch_fold_finish(d_g, total_points, *cfg, d_res, d_k, 0, (cudaStream_t)stream), "fold_finish");
    return MXFFT_OK;
}

int32_t mxfft_rss_scaled(const void* x, int32_t is_c128, int64_t groups, int32_t coils, int64_t npix,
                         const int32_t* d_k, int32_t k_sign, int32_t exp_const, double* out, uintptr_t stream) {
    if (coils < 1) return fail(MXFFT_ERR_SHAPE, "need at least one coil");
    if (groups < 0 || npix < 0) return fail(MXFFT_ERR_SHAPE, "negative size");
    CK(launch_rss(x, is_c128, groups, coils, npix, out, (cudaStream_t)stream, d_k, k_sign, exp_const), "rss_scaled");
    return MXFFT_OK;
}

int32_t mxfft_prescale_apply_c128(const void* x, void* y, int64_t nseg, int64_t seg_points, const int32_t* d_k,
                                  uintptr_t stream) {
    if (nseg < 0 || seg_points < 0) return fail(MXFFT_ERR_SHAPE, "negative size");
    if (!d_k) return fail(MXFFT_ERR_VALUE, "null k vector");
    CK(launch_prescale_apply_c128(x, y, seg_points, nseg, d_k, (cudaStream_t)stream), "prescale_apply_c128");
    return MXFFT_OK;
}

int32_t mxfft_mx_multiply_f64(const void* v, const double* wcr, const double* wci, const double* ws, int64_t rows,
                              int32_t m, int32_t cpb, const mxfft_format* fmt, void* wv, const void* u, void* y0,
                              void* y1, int32_t* d_nonfinite, uintptr_t stream) {
    std::string why;
    if (!check_fmt(fmt, why)) return fail(MXFFT_ERR_VALUE, why);
    if (rows < 0 || m < 0) return fail(MXFFT_ERR_SHAPE, "negative size");
    if (cpb < 1 || m % cpb) return fail(MXFFT_ERR_SHAPE, "cpb must divide m (fftcore.py:139-141 reshape)");
    if (u && (!y0 || !y1)) return fail(MXFFT_ERR_VALUE, "butterfly outputs missing");
    CK(launch_mx_multiply(v, wcr, wci, ws, rows, m, cpb, desc_of(fmt), wv, u, y0, y1, d_nonfinite,
                          (cudaStream_t)stream),
       "mx_multiply_f64");
    return MXFFT_OK;
}

int32_t mxfft_scale(const void* x, void* y, int64_t n, int32_t dtype, double factor, uintptr_t stream) {
    if (n < 0) return fail(MXFFT_ERR_SHAPE, "negative size");
    if (dtype < 0 || dtype > 3) return fail(MXFFT_ERR_VALUE, "dtype must be 0 (f32), 1 (f64), 2 (c64) or 3 (c128)");
    CK(launch_scale(x, y, n, dtype, factor, (cudaStream_t)stream), "scale");
    return MXFFT_OK;
}

int32_t mxfft_fft_rows_debug(mxfft_plan plan, const void* x, void* y, int64_t batch,
                             int32_t inverse, int32_t* v_exp, float* v_codes, int32_t* p_exp,
                             int32_t* p_shift, float* p_codes, void* stage_out, uintptr_t stream) {
    CHECK_PLAN(plan);
    const Plan& p = plan->p;
    if (!mx_lines_ok(p)) return fail(MXFFT_ERR_VALUE, "debug capture needs a line-kernel plan");
    if (p.n > 4096) return fail(MXFFT_ERR_UNSUPPORTED_SIZE, "debug capture supports n <= 4096");
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t m = p.n / 2, nb = m / p.cpb, st = p.log2n;
    // scratch for any dump array the caller did not ask for
    int32_t *ve = v_exp, *pe = p_exp, *ps = p_shift;
    float *vc = v_codes, *pc = p_codes;
    void* scratch[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};
    const size_t nbx = sizeof(int32_t) * st * batch * nb, ncx = sizeof(float) * 2 * st * batch * m;
    if (!ve) { CK(cudaMalloc(&scratch[0], nbx), "debug"); ve = (int32_t*)scratch[0]; }
    if (!pe) { CK(cudaMalloc(&scratch[1], nbx), "debug"); pe = (int32_t*)scratch[1]; }
    if (!ps) { CK(cudaMalloc(&scratch[2], nbx), "debug"); ps = (int32_t*)scratch[2]; }
    if (!vc) { CK(cudaMalloc(&scratch[3], ncx), "debug"); vc = (float*)scratch[3]; }
    if (!pc) { CK(cudaMalloc(&scratch[4], ncx), "debug"); pc = (float*)scratch[4]; }
    LinePass lp;
    lp.in = x;
    lp.out = y;
    lp.col_mode = 0;
    lp.lines_per_image = 1;
    lp.total_lines = batch;
    lp.img_elems = p.n;
    lp.inverse = inverse ? 1 : 0;
    lp.d_vexp = ve;
    lp.d_vcodes = vc;
    lp.d_pexp = pe;
    lp.d_pshift = ps;
    lp.d_pcodes = pc;
    cudaError_t e = run_lines(p, lp, s);
    if (e == cudaSuccess && stage_out) {
        for (int k = 0; k < st && e == cudaSuccess; ++k) {
            LinePass l2 = lp;
            l2.d_vexp = nullptr;
            l2.d_vcodes = nullptr;
            l2.d_pexp = nullptr;
            l2.d_pshift = nullptr;
            l2.d_pcodes = nullptr;
            l2.stage_limit = k + 1;
            l2.out = reinterpret_cast<float2*>(stage_out) + (int64_t)k * batch * p.n;
            e = run_lines(p, l2, s);
        }
    }
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    for (void* q : scratch) cudaFree(q);
    if (e != cudaSuccess) return cuda_fail(e, "fft_rows_debug");
    return MXFFT_OK;
}

}  // extern "C"

extern "C" int32_t mxfft_selftest_hw_quantizer(const mxfft_format* fmt, uint64_t* d_mismatches,
                                               uint32_t* d_first_bad, uintptr_t stream) {
    std::string why;
    if (!check_fmt(fmt, why)) return fail(MXFFT_ERR_VALUE, why);
    FmtDesc f = desc_of(fmt);
    if (f.id == F_GENERIC) return fail(MXFFT_ERR_VALUE, "format has no hardware quantizer");
    CK(launch_selftest_hwq(f, reinterpret_cast<unsigned long long*>(d_mismatches), d_first_bad,
                           (cudaStream_t)stream),
       "selftest_hw_quantizer");
    return MXFFT_OK;
}
