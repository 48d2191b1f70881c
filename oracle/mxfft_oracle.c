/*
 * mxfft_oracle.c -- CPU restatement of the reference MX-FFT hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the checker the CUDA product is
 * compared against; it is never linked into, loaded by, or called from the
 * product package (paper_2512_04317_b200/).  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference leg may load it.
 *
 * Every function restates one reference function (paths relative to
 * /root/reference/pkg/src/mxfft/).  Arithmetic is literal: FP64 quantization,
 * FP32 mantissa products, FP32 butterfly sums, compiled with
 * -ffp-contract=off so that no FMA contraction changes a rounding.
 *
 * Pinned against the reference itself: the fixtures in tests/golden/ were produced by
 * importing the reference package (tests/golden/make_golden.py) and
 * tests/test_oracle_golden.py checks this file bit-for-bit against them.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ */
/* Element format: minifloat.py:28-85                                  */
/* ------------------------------------------------------------------ */
enum { POL_IEEE = 0, POL_EXTENDED = 1, POL_FINITE = 2 };

typedef struct {
    int ebits, mbits, policy, bias;
    int emin, emax;
    double max_finite;
} orc_fmt;

static orc_fmt make_fmt(int ebits, int mbits, int policy, int bias) {
    orc_fmt f;
    f.ebits = ebits;
    f.mbits = mbits;
    f.policy = policy;
    f.bias = bias; /* caller passes the resolved bias (minifloat.py:45-46) */
    f.emin = 1 - bias; /* minifloat.py:57-59 */
    int top = (1 << ebits) - 1; /* minifloat.py:61-67 */
    if (policy == POL_IEEE) top -= 1;
    f.emax = top - bias;
    int m = 1 << mbits; /* minifloat.py:69-77 */
    int frac = (policy == POL_EXTENDED) ? m + (m - 2) : m + (m - 1);
    f.max_finite = ldexp((double)frac, f.emax - mbits);
    return f;
}

void orc_format_info(int ebits, int mbits, int policy, int bias, int* emin, int* emax,
                     double* max_finite, double* min_subnormal) {
    orc_fmt f = make_fmt(ebits, mbits, policy, bias);
    *emin = f.emin;
    *emax = f.emax;
    *max_finite = f.max_finite;
    *min_subnormal = ldexp(1.0, f.emin - f.mbits); /* minifloat.py:79-81 */
}

/* quantize_array, minifloat.py:105-120: RNE at binade max(floor(log2|x|), emin),
 * np.round (half-even) == rint under the default rounding mode, then clip. */
static inline double q1(double x, const orc_fmt* f) {
    int e;
    frexp(fabs(x), &e);
    int eb = e - 1;
    if (eb < f->emin) eb = f->emin;
    double step = ldexp(1.0, eb - f->mbits);
    double q = rint(x / step) * step;
    if (q > f->max_finite) q = f->max_finite;
    if (q < -f->max_finite) q = -f->max_finite;
    return q;
}

/* returns 0, or 1 when a non-finite input was seen (minifloat.py:112-113) */
int orc_quantize_array(const double* x, double* out, long n, int ebits, int mbits, int policy,
                       int bias) {
    orc_fmt f = make_fmt(ebits, mbits, policy, bias);
    for (long i = 0; i < n; i++)
        if (!isfinite(x[i])) return 1;
    for (long i = 0; i < n; i++) out[i] = q1(x[i], &f);
    return 0;
}

/* block_scales, mxblock.py:27-38 */
static inline double block_scale(double amax, const orc_fmt* f) {
    if (!(amax > 0)) return 1.0;
    int e;
    frexp(amax, &e);
    int se = e - 1 - f->emax;
    if (se < -1022) se = -1022;
    if (se > 1023) se = 1023;
    return ldexp(1.0, se);
}

void orc_block_scales(const double* amax, double* out, long n, int ebits, int mbits, int policy,
                      int bias) {
    orc_fmt f = make_fmt(ebits, mbits, policy, bias);
    for (long i = 0; i < n; i++) out[i] = block_scale(amax[i], &f);
}

/* _encode_blocks_batch, fftcore.py:131-147.  vr/vi: (batch, m); codes: (batch, m);
 * scales: (batch, m/cpb).  One shared scale per cpb complex values. */
static void encode_blocks(const double* vr, const double* vi, long batch, long m, int cpb,
                          const orc_fmt* f, double* cr, double* ci, double* scales) {
    long nb = m / cpb;
    for (long b = 0; b < batch; b++)
        for (long k = 0; k < nb; k++) {
            const double* r = vr + b * m + k * cpb;
            const double* im = vi + b * m + k * cpb;
            double amax = 0.0;
            for (int j = 0; j < cpb; j++) {
                double a = fabs(r[j]), c = fabs(im[j]);
                double mx = a > c ? a : c; /* np.maximum */
                if (mx > amax) amax = mx;
            }
            double s = block_scale(amax, f);
            double inv = 1.0 / s; /* exact: reciprocal of a power of two */
            for (int j = 0; j < cpb; j++) {
                cr[b * m + k * cpb + j] = q1(r[j] * inv, f);
                ci[b * m + k * cpb + j] = q1(im[j] * inv, f);
            }
            scales[b * nb + k] = s;
        }
}

void orc_encode_blocks(const double* vr, const double* vi, long batch, long m, int cpb, int ebits,
                       int mbits, int policy, int bias, double* cr, double* ci, double* scales) {
    orc_fmt f = make_fmt(ebits, mbits, policy, bias);
    encode_blocks(vr, vi, batch, m, cpb, &f, cr, ci, scales);
}

/* Optional per-stage capture of the MX multiply (test instrumentation). */
typedef struct {
    int32_t* v_exp;   /* log2 of the v-block scale, (batch, nb) */
    double* v_codes;  /* (batch, m, 2) interleaved re/im codes */
    int32_t* p_exp;   /* log2 of s_out (product block scale after renorm), (batch, nb) */
    double* p_codes;  /* (batch, m, 2) product codes */
    int32_t* p_shift; /* renormalization shift, (batch, nb) */
} orc_mul_dump;

static inline int ilog2_pow2(double s) {
    int e;
    frexp(s, &e);
    return e - 1;
}

/* _mx_multiply_batch, fftcore.py:150-183.  Returns wv cast to complex64
 * (the caller casts, fftcore.py:279). */
static void mx_multiply(const double* vr, const double* vi, long batch, long m, const double* wcr,
                        const double* wci, const double* ws, int cpb, const orc_fmt* f,
                        float* wv_re, float* wv_im, const orc_mul_dump* d, double* scratch) {
    long nb = m / cpb;
    double* cvr = scratch;
    double* cvi = scratch + batch * m;
    double* sv = scratch + 2 * batch * m;
    encode_blocks(vr, vi, batch, m, cpb, f, cvr, cvi, sv);
    int use_f32 = 2 * (f->emax + 1) <= 126; /* fftcore.py:163 */
    double* pr64 = malloc(sizeof(double) * cpb);
    double* pi64 = malloc(sizeof(double) * cpb);
    float* pr32 = malloc(sizeof(float) * cpb);
    float* pi32 = malloc(sizeof(float) * cpb);
    for (long b = 0; b < batch; b++)
        for (long k = 0; k < nb; k++) {
            double s_out = ws[k] * sv[b * nb + k]; /* fftcore.py:170 */
            double amax = 0.0;
            for (int j = 0; j < cpb; j++) {
                long t = k * cpb + j;
                long i = b * m + t;
                if (use_f32) {
                    float xr = (float)wcr[t], xi = (float)wci[t];
                    float yr = (float)cvr[i], yi = (float)cvi[i];
                    pr32[j] = xr * yr - xi * yi; /* fftcore.py:168 */
                    pi32[j] = xr * yi + xi * yr; /* fftcore.py:169 */
                    float a = fabsf(pr32[j]), c = fabsf(pi32[j]);
                    double mx = (double)(a > c ? a : c);
                    if (mx > amax) amax = mx;
                } else {
                    double xr = wcr[t], xi = wci[t], yr = cvr[i], yi = cvi[i];
                    pr64[j] = xr * yr - xi * yi;
                    pi64[j] = xr * yi + xi * yr;
                    double a = fabs(pr64[j]), c = fabs(pi64[j]);
                    double mx = a > c ? a : c;
                    if (mx > amax) amax = mx;
                }
            }
            int shift = 0;
            if (amax > f->max_finite) { /* fftcore.py:173-179 */
                shift = (int)ceil(log2(amax / f->max_finite));
                if (use_f32) {
                    float fac = ldexpf(1.0f, -shift);
                    for (int j = 0; j < cpb; j++) {
                        pr32[j] = pr32[j] * fac;
                        pi32[j] = pi32[j] * fac;
                    }
                } else {
                    double fac = ldexp(1.0, -shift);
                    for (int j = 0; j < cpb; j++) {
                        pr64[j] = pr64[j] * fac;
                        pi64[j] = pi64[j] * fac;
                    }
                }
                s_out = s_out * ldexp(1.0, shift);
            }
            for (int j = 0; j < cpb; j++) {
                long i = b * m + k * cpb + j;
                double pr = use_f32 ? (double)pr32[j] : pr64[j];
                double pi = use_f32 ? (double)pi32[j] : pi64[j];
                double c_r = q1(pr, f), c_i = q1(pi, f); /* fftcore.py:180-181 */
                /* fftcore.py:182 then .astype(complex64) at fftcore.py:279 */
                wv_re[i] = (float)(c_r * s_out);
                wv_im[i] = (float)(c_i * s_out);
                if (d && d->p_codes) {
                    d->p_codes[2 * i] = c_r;
                    d->p_codes[2 * i + 1] = c_i;
                }
                if (d && d->v_codes) {
                    d->v_codes[2 * i] = cvr[i];
                    d->v_codes[2 * i + 1] = cvi[i];
                }
            }
            if (d && d->v_exp) d->v_exp[b * nb + k] = ilog2_pow2(sv[b * nb + k]);
            if (d && d->p_exp) d->p_exp[b * nb + k] = ilog2_pow2(s_out);
            if (d && d->p_shift) d->p_shift[b * nb + k] = shift;
        }
    free(pr64); free(pi64); free(pr32); free(pi32);
}

/* ------------------------------------------------------------------ */
/* Plan: fftcore.py:84-117                                             */
/* ------------------------------------------------------------------ */
static int log2i(long n) {
    int s = 0;
    while ((1L << s) < n) s++;
    return s;
}

static long bitrev(long i, int bits) { /* _bit_reversal, fftcore.py:67-77 */
    long r = 0;
    for (int b = 0; b < bits; b++) {
        r = (r << 1) | (i & 1);
        i >>= 1;
    }
    return r;
}

/* Encode the plan's per-stage twiddles (fftcore.py:108-113).  tw: FP64 complex,
 * (stages, n/2) interleaved, in butterfly order -- produced by the host with the
 * reference's own NumPy expression (fftcore.py:101-105).
 * Outputs: wcr/wci (stages, n/2), ws (stages, n/2/cpb). */
void orc_encode_twiddles(const double* tw, int n, int cpb, int ebits, int mbits, int policy,
                         int bias, double* wcr, double* wci, double* ws) {
    orc_fmt f = make_fmt(ebits, mbits, policy, bias);
    int stages = log2i(n);
    long m = n / 2;
    double* re = malloc(sizeof(double) * m);
    double* im = malloc(sizeof(double) * m);
    for (int s = 0; s < stages; s++) {
        for (long j = 0; j < m; j++) {
            re[j] = tw[2 * (s * m + j)];
            im[j] = tw[2 * (s * m + j) + 1];
        }
        encode_blocks(re, im, 1, m, cpb, &f, wcr + s * m, wci + s * m, ws + s * (m / cpb));
    }
    free(re);
    free(im);
}

/* Per-stage dump of a whole transform (test instrumentation).  Arrays are laid
 * out [stage][batch][...]; any pointer may be NULL. */
typedef struct {
    int32_t* v_exp;
    double* v_codes;
    int32_t* p_exp;
    double* p_codes;
    int32_t* p_shift;
    float* stage_out; /* [stage][batch][n][2] */
} orc_fft_dump;

/* _fft_batch_mx, fftcore.py:259-282 (with the dispatch checks of _fft_batch,
 * fftcore.py:321-326, done by the caller).  x: complex128 (batch, n) interleaved;
 * y: complex64 (batch, n) interleaved. */
int orc_fft_batch_mx(const double* x, long batch, int n, int block_size, int ebits, int mbits,
                     int policy, int bias, const double* wcr, const double* wci, const double* ws,
                     int inverse, float* y, const orc_fft_dump* dump) {
    orc_fmt f = make_fmt(ebits, mbits, policy, bias);
    int stages = log2i(n);
    long m = n / 2;
    int cpb = block_size / 2 < m ? block_size / 2 : (int)m; /* fftcore.py:109 */
    long nb = m / cpb;
    float* yr = malloc(sizeof(float) * batch * n);
    float* yi = malloc(sizeof(float) * batch * n);
    double* vr = malloc(sizeof(double) * batch * m);
    double* vi = malloc(sizeof(double) * batch * m);
    float* wvr = malloc(sizeof(float) * batch * m);
    float* wvi = malloc(sizeof(float) * batch * m);
    double* wci_s = malloc(sizeof(double) * m);
    double* scratch = malloc(sizeof(double) * (2 * batch * m + batch * nb));
    if (!yr || !yi || !vr || !vi || !wvr || !wvi || !wci_s || !scratch) return 2;
    /* fftcore.py:262: bit-reversal gather, complex128 -> complex64 */
    for (long b = 0; b < batch; b++)
        for (long i = 0; i < n; i++) {
            long src = bitrev(i, stages);
            yr[b * n + i] = (float)x[2 * (b * n + src)];
            yi[b * n + i] = (float)x[2 * (b * n + src) + 1];
        }
    for (int s = 0; s < stages; s++) {
        long half = 1L << s;
        const double* wr_s = wcr + s * m;
        const double* wi_s = wci + s * m;
        for (long j = 0; j < m; j++) wci_s[j] = inverse ? -wi_s[j] : wi_s[j]; /* fftcore.py:267-268 */
        /* fftcore.py:269-272: v in (group, j) order */
        for (long b = 0; b < batch; b++)
            for (long t = 0; t < m; t++) {
                long g = t / half, j = t % half;
                long pv = g * 2 * half + half + j;
                vr[b * m + t] = (double)yr[b * n + pv];
                vi[b * m + t] = (double)yi[b * n + pv];
            }
        orc_mul_dump md = {0};
        const orc_mul_dump* mdp = NULL;
        if (dump) {
            md.v_exp = dump->v_exp ? dump->v_exp + (long)s * batch * nb : NULL;
            md.v_codes = dump->v_codes ? dump->v_codes + (long)s * batch * m * 2 : NULL;
            md.p_exp = dump->p_exp ? dump->p_exp + (long)s * batch * nb : NULL;
            md.p_codes = dump->p_codes ? dump->p_codes + (long)s * batch * m * 2 : NULL;
            md.p_shift = dump->p_shift ? dump->p_shift + (long)s * batch * nb : NULL;
            mdp = &md;
        }
        mx_multiply(vr, vi, batch, m, wr_s, wci_s, ws + s * nb, cpb, &f, wvr, wvi, mdp, scratch);
        /* fftcore.py:280-281: y = [u + t | u - t] in FP32 */
        for (long b = 0; b < batch; b++)
            for (long t = 0; t < m; t++) {
                long g = t / half, j = t % half;
                long pu = g * 2 * half + j, pv = pu + half;
                float ur = yr[b * n + pu], ui = yi[b * n + pu];
                float tr = wvr[b * m + t], ti = wvi[b * m + t];
                yr[b * n + pu] = ur + tr;
                yi[b * n + pu] = ui + ti;
                yr[b * n + pv] = ur - tr;
                yi[b * n + pv] = ui - ti;
            }
        if (dump && dump->stage_out)
            for (long b = 0; b < batch; b++)
                for (long i = 0; i < n; i++) {
                    long o = ((long)s * batch + b) * n + i;
                    dump->stage_out[2 * o] = yr[b * n + i];
                    dump->stage_out[2 * o + 1] = yi[b * n + i];
                }
    }
    for (long i = 0; i < batch * n; i++) {
        y[2 * i] = yr[i];
        y[2 * i + 1] = yi[i];
    }
    free(yr); free(yi); free(vr); free(vi); free(wvr); free(wvi); free(wci_s); free(scratch);
    return 0;
}

/* fft_2d, fftcore.py:344-353: rows, then columns of the transposed rows.
 * x: complex128 (n, n); y: complex64 (n, n) (the reference returns the same
 * values widened to complex128). */
int orc_fft2_mx(const double* x, int n, int block_size, int ebits, int mbits, int policy, int bias,
                const double* wcr, const double* wci, const double* ws, int inverse, float* y) {
    long nn = (long)n * n;
    float* rows = malloc(sizeof(float) * 2 * nn);
    double* t = malloc(sizeof(double) * 2 * nn);
    float* cols = malloc(sizeof(float) * 2 * nn);
    if (!rows || !t || !cols) return 2;
    int rc = orc_fft_batch_mx(x, n, n, block_size, ebits, mbits, policy, bias, wcr, wci, ws,
                              inverse, rows, NULL);
    if (rc) return rc;
    for (long i = 0; i < n; i++)
        for (long j = 0; j < n; j++) { /* np.ascontiguousarray(rows.T) */
            t[2 * (j * n + i)] = rows[2 * (i * n + j)];
            t[2 * (j * n + i) + 1] = rows[2 * (i * n + j) + 1];
        }
    rc = orc_fft_batch_mx(t, n, n, block_size, ebits, mbits, policy, bias, wcr, wci, ws, inverse,
                          cols, NULL);
    for (long i = 0; i < n; i++)
        for (long j = 0; j < n; j++) { /* cols.T */
            y[2 * (j * n + i)] = cols[2 * (i * n + j)];
            y[2 * (j * n + i) + 1] = cols[2 * (i * n + j) + 1];
        }
    free(rows); free(t); free(cols);
    return rc;
}

/* ------------------------------------------------------------------ */
/* Prescale: prescale.py:18-91                                         */
/* ------------------------------------------------------------------ */
#define ORC_EPS 1e-30 /* prescale.py:18 */

/* np.abs(complex128) as numpy 2.3.5 computes it on FMA3/AVX2/AVX-512 hosts
 * (CDOUBLE_absolute SIMD loop: larger * sqrt(fma(r, r, 1)), r = smaller/larger;
 * pinned bit-exact against np.abs by tests/test_oracle_golden.py). */
static inline double np_cabs(double re, double im) {
    double a = fabs(re), b = fabs(im);
    double larger = a > b ? a : b;
    double smaller = b < a ? b : a;
    if (larger == 0.0) return 0.0;
    double r = smaller / larger;
    return sqrt(fma(r, r, 1.0)) * larger;
}

static int cmp_double(const void* a, const void* b) {
    double x = *(const double*)a, y = *(const double*)b;
    return (x > y) - (x < y);
}

/* np.percentile(nz, tau), method 'linear' (numpy 2.3.5 _quantile / _lerp). */
static double np_percentile_linear(double* v, long n, double tau) {
    qsort(v, n, sizeof(double), cmp_double);
    double q = tau / 100.0;
    double virt = (double)(n - 1) * q;
    long prev, next;
    double gamma;
    if (virt >= (double)(n - 1)) {
        prev = next = n - 1;
        gamma = virt + 1.0; /* numpy sets previous index to -1 before gamma */
    } else {
        prev = (long)floor(virt);
        next = prev + 1;
        gamma = virt - (double)prev;
    }
    double a = v[prev], b = v[next];
    double diff = b - a;
    double r = a + diff * gamma;
    if (gamma >= 0.5) r = b - diff * (1.0 - gamma);
    return r;
}

static int round_half_away(double v) { /* prescale.py:49-50 */
    return v >= 0 ? (int)floor(v + 0.5) : (int)ceil(v - 0.5);
}

/* compute_prescale, prescale.py:61-73.  x: interleaved complex128 (n values) when
 * is_complex, else real FP64.  Returns 1 when a non-finite value was seen. */
int orc_compute_prescale(const double* x, long n, int is_complex, double target, double tau,
                         double tau_min, int k_min, int k_max, double* a_max_out,
                         double* p_tau_out, int* k1_out, int* k2_out, int* k_out) {
    long tot = is_complex ? 2 * n : n;
    for (long i = 0; i < tot; i++)
        if (!isfinite(x[i])) return 1;
    double* nz = malloc(sizeof(double) * (n > 0 ? n : 1));
    double a_max = 0.0;
    long cnt = 0;
    for (long i = 0; i < n; i++) {
        double m = is_complex ? np_cabs(x[2 * i], x[2 * i + 1]) : fabs(x[i]);
        if (m > a_max) a_max = m;
        if (m > 0) nz[cnt++] = m;
    }
    double p_tau = cnt ? np_percentile_linear(nz, cnt, tau) : 0.0;
    free(nz);
    int k1 = round_half_away(log2(target / (a_max > ORC_EPS ? a_max : ORC_EPS)));
    int k2 = (int)ceil(log2(tau_min / (p_tau > ORC_EPS ? p_tau : ORC_EPS)));
    int k = k1 > k2 ? k1 : k2;
    if (k < k_min) k = k_min;
    if (k > k_max) k = k_max;
    *a_max_out = a_max;
    *p_tau_out = p_tau;
    *k1_out = k1;
    *k2_out = k2;
    *k_out = k;
    return 0;
}

/* ------------------------------------------------------------------ */
/* Pipelines: mri.py:84-107 (one coil stack, C coils of n x n)         */
/* ------------------------------------------------------------------ */

/* forward (roundtrip=0) or round trip (roundtrip=1).  x: complex128 (C, n, n).
 * out: complex128 (C, n, n) after undo_prescale; rss: FP64 (n, n). */
int orc_pipeline(const double* x, int coils, int n, int block_size, int ebits, int mbits,
                 int policy, int bias, const double* wcr, const double* wci, const double* ws,
                 double target, double tau, double tau_min, int k_min, int k_max, int roundtrip,
                 double* out, double* rss, int* k_out) {
    long nn = (long)n * n;
    double a_max, p_tau;
    int k1, k2, k;
    int rc = orc_compute_prescale(x, coils * nn, 1, target, tau, tau_min, k_min, k_max, &a_max,
                                  &p_tau, &k1, &k2, &k);
    if (rc) return rc;
    *k_out = k;
    double g = ldexp(1.0, k), ug = ldexp(1.0, -k);
    double norm = 1.0 / ((double)n * (double)n); /* mri.py:100 */
    double* xs = malloc(sizeof(double) * 2 * nn);
    float* f1 = malloc(sizeof(float) * 2 * nn);
    double* mid = malloc(sizeof(double) * 2 * nn);
    float* f2 = malloc(sizeof(float) * 2 * nn);
    for (int c = 0; c < coils; c++) {
        const double* xc = x + 2 * c * nn;
        for (long i = 0; i < 2 * nn; i++) xs[i] = xc[i] * g; /* apply_prescale */
        rc = orc_fft2_mx(xs, n, block_size, ebits, mbits, policy, bias, wcr, wci, ws, 0, f1);
        if (rc) break;
        double* oc = out + 2 * c * nn;
        if (!roundtrip) {
            for (long i = 0; i < 2 * nn; i++) oc[i] = (double)f1[i] * ug; /* undo_prescale */
        } else {
            for (long i = 0; i < 2 * nn; i++) mid[i] = (double)f1[i];
            rc = orc_fft2_mx(mid, n, block_size, ebits, mbits, policy, bias, wcr, wci, ws, 1, f2);
            if (rc) break;
            for (long i = 0; i < 2 * nn; i++) oc[i] = ((double)f2[i] * norm) * ug;
        }
    }
    /* rss, mri.py:70-81: sqrt(sum_c |T_c|^2), coils summed in order */
    if (!rc)
        for (long i = 0; i < nn; i++) {
            double acc = 0.0;
            for (int c = 0; c < coils; c++) {
                double m = np_cabs(out[2 * (c * nn + i)], out[2 * (c * nn + i) + 1]);
                double sq = m * m;
                acc = c == 0 ? sq : acc + sq;
            }
            rss[i] = sqrt(acc);
        }
    free(xs); free(f1); free(mid); free(f2);
    return rc;
}

/* np.abs(complex128) restated, exposed so tests can pin it against numpy */
void orc_cabs(const double* x, long n, double* out) {
    for (long i = 0; i < n; i++) out[i] = np_cabs(x[2 * i], x[2 * i + 1]);
}
