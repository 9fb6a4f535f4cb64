/*
 * oracle/svd2_oracle.c -- TEST INFRASTRUCTURE, NOT THE PRODUCT.
 *
 * A plain-C, one-lane-at-a-time restatement of the reference's batched 2x2
 * SVD (lanesvd 0.1.0, /root/reference/pkg/src/lanesvd).  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
 * may load it, and only as the checker or the timed CPU baseline.  The CUDA
 * product never links or calls this file.
 *
 * Parity pin: tests/golden/ holds outputs of the reference itself (imported
 * in the build container by tests/golden/make_golden.py) -- per-lane input
 * and output bit patterns plus SHA-256 digests of whole output trains for the
 * BASELINE configs.  tests/test_oracle_golden.py checks this file against all
 * of them bit for bit, and against the reference's own known-answer tests.
 *
 * Arithmetic follows the reference operation by operation: IEEE binary64,
 * round-to-nearest-even, every fused multiply-add explicit through fma(),
 * no contraction (build with -ffp-contract=off, never -ffast-math).
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef uint64_t u64;

static inline u64 b_(double x) { u64 u; memcpy(&u, &x, 8); return u; }
static inline double d_(u64 u) { double x; memcpy(&x, &u, 8); return x; }

#define SIGN_BIT 0x8000000000000000ULL
/* lanes.py:41-47 */
#define O_DBL_MAX 1.7976931348623157e+308
#define O_TRUE_MIN 4.9406564584124654e-324
/* svd2.py:52-59 */
#define O_HEADROOM 1021.0
#define O_SQRT_DBL_MAX 1.34078079299425956e+154

/* ---- lane primitives (lanes.py) ------------------------------------- */

/* lanes.py:102-108: a where a < b, else b (second wins on tie / NaN) */
static inline double rmin(double a, double b) { return a < b ? a : b; }
/* lanes.py:111-114 */
static inline double rmax(double a, double b) { return a > b ? a : b; }
/* lanes.py:117-119: b where mask, a elsewhere */
static inline double sel(int m, double a, double b) { return m ? b : a; }
/* lanes.py:169-206: sign-bit algebra on raw patterns */
static inline double fabs_(double x) { return d_(b_(x) & ~SIGN_BIT); }
static inline double neg_(double x) { return d_(b_(x) ^ SIGN_BIT); }
static inline double sgn_(double x) { return d_(b_(x) & SIGN_BIT); }
static inline double xor_(double a, double b) { return d_(b_(a) ^ b_(b)); }
static inline double or_(double a, double b) { return d_(b_(a) | b_(b)); }
/* lanes.py:86-95 */
static inline double fma_(double a, double b, double c) { return fma(a, b, c); }
static inline double fnma_(double a, double b, double c) { return fma(-a, b, c); }

/* lanes.py:126-140: floor(log2|a|) via frexp; 0 -> -inf, inf -> +inf, NaN
 * propagates. */
static double getexp(double a)
{
    if (isnan(a)) return a;
    if (isinf(a)) return INFINITY;
    if (a == 0.0) return -INFINITY;
    int e;
    (void)frexp(a, &e);
    return (double)e - 1.0;
}

/* lanes.py:143-159: a * 2**floor(e) with one rounding (ldexp); shifts
 * clipped to +-4500; non-finite e -> a * exp2(e). */
static double scalef(double a, double e)
{
    double ef = floor(e);
    if (isfinite(ef)) {
        double sh = ef < -4500.0 ? -4500.0 : (ef > 4500.0 ? 4500.0 : ef);
        return ldexp(a, (int)sh);
    }
    return a * exp2(ef);
}

/* lanes.py:213-227 */
static double hypot_lane(double a, double b)
{
    double aa = fabs_(a), ab = fabs_(b);
    double big = rmax(aa, ab);
    double small = rmin(aa, ab);
    double q = small / rmax(big, O_TRUE_MIN);
    return big * sqrt(fma_(q, q, 1.0));
}

/* lanes.py:230-232: two roundings */
static inline double invsqrt_lane(double a) { return 1.0 / sqrt(a); }

/* lanes.py:235-245 */
static inline void cmul(double ar, double ai, double br, double bi,
                        double *re, double *im)
{
    *re = fma_(ar, br, neg_(ai * bi));
    *im = fma_(ar, bi, ai * br);
}

/* lanes.py:248-259 */
static inline void phase_from_parts(double re, double im, double mag,
                                    double *c, double *s)
{
    *c = or_(rmin(fabs_(re) / mag, 1.0), sgn_(re));
    *s = im / rmax(mag, O_TRUE_MIN);
}

/* ---- per-lane state (svd2.py:62-127) -------------------------------- */

typedef struct {
    /* inputs: e[t][0] re, e[t][1] im; t = 11, 21, 12, 22 (layout.py:3-10) */
    double shift;
    int swap_c, swap_r;
    double ph1r, ph1i, ph2r, ph2i;   /* row phases (real: sign patterns) */
    double dtr, dti, dhr, dhi;       /* r12 phase (conj, for V), r22 phase */
    double g_tan, g_cos, r11, r12, r22;
    double l_tan, l_sec2, l_cos, r_tan, r_sec2, r_cos;
    double smax, smin;
    double u[4][2], v[4][2];         /* (re, im) in order 11, 21, 12, 22 */
} lane_t;

/* svd2.py:134-160: joint power-of-two scaling; pairwise relaxed-min tree */
static double compute_scale(const double *p, int np_, double *out)
{
    double m[8];
    for (int i = 0; i < np_; i++) m[i] = O_HEADROOM - getexp(p[i]);
    int len = np_;
    while (len > 1) {
        for (int i = 0; i < len; i += 2) m[i / 2] = rmin(m[i], m[i + 1]);
        len /= 2;
    }
    double shift = rmin(O_DBL_MAX, m[0]);
    for (int i = 0; i < np_; i++) out[i] = scalef(p[i], shift);
    return shift;
}

static inline void swap_sel(int mask, double *a, double *b)
{
    double na = sel(mask, *a, *b), nb = sel(mask, *b, *a);
    *a = na; *b = nb;
}

/* svd2.py:306-343 */
static void triangular_svd(lane_t *L)
{
    double x = rmax(L->r12 / L->r11, 0.0);
    double y = rmax(L->r22 / L->r11, 0.0);
    double num = scalef(rmin(x, y), 1.0) * rmax(x, y);
    double den = fma_(x - y, x + y, 1.0);
    double tan2 = or_(rmin(rmax(num / den, 0.0), O_SQRT_DBL_MAX), -0.0);
    L->l_tan = tan2 / (1.0 + sqrt(fma_(tan2, tan2, 1.0)));
    L->l_sec2 = fma_(L->l_tan, L->l_tan, 1.0);
    L->l_cos = invsqrt_lane(L->l_sec2);
    L->r_tan = fma_(y, L->l_tan, neg_(x));
    L->r_sec2 = fma_(L->r_tan, L->r_tan, 1.0);
    L->r_cos = invsqrt_lane(L->r_sec2);
    double cc = L->l_cos * L->r_cos;
    L->smax = (cc * L->r_sec2) * L->r11;
    L->smin = (cc * L->l_sec2) * L->r22;
}

/* svd2.py:350-369 (_assemble_v) and 372-375 (_finish_u) */
static void assemble_v(lane_t *L, int cplx)
{
    double cr = L->r_cos;
    double sr = cr * L->r_tan;
    double v[4][2];
    if (!cplx) {
        v[0][0] = cr;                          /* v11 */
        v[2][0] = sr;                          /* v12 */
        v[1][0] = xor_(sr, xor_(L->dtr, -0.0)); /* v21 */
        v[3][0] = xor_(cr, L->dtr);            /* v22 */
        v[0][1] = v[1][1] = v[2][1] = v[3][1] = 0.0;
    } else {
        v[0][0] = cr; v[0][1] = 0.0;
        v[2][0] = sr; v[2][1] = 0.0;
        v[1][0] = neg_(sr * L->dtr); v[1][1] = neg_(sr * L->dti);
        v[3][0] = cr * L->dtr; v[3][1] = cr * L->dti;
    }
    for (int k = 0; k < 2; k++) {
        swap_sel(L->swap_c, &v[0][k], &v[1][k]);
        swap_sel(L->swap_c, &v[2][k], &v[3][k]);
    }
    memcpy(L->v, v, sizeof v);
}

static void finish_u(lane_t *L, double pre[4][2])
{
    for (int k = 0; k < 2; k++) {
        swap_sel(L->swap_r, &pre[0][k], &pre[1][k]);
        swap_sel(L->swap_r, &pre[2][k], &pre[3][k]);
    }
    memcpy(L->u, pre, sizeof L->u);
}

/* svd2.py:378-424 (tangent form) */
static void assemble_uv(lane_t *L, int cplx)
{
    double mt = neg_(L->g_tan);
    double gt = L->g_tan, lt = L->l_tan;
    double c = L->g_cos * L->l_cos;
    double pre[4][2];
    if (!cplx) {
        double d = L->dhr;
        double core11 = fma_(xor_(mt, d), lt, 1.0);
        double core12 = lt + xor_(gt, d);
        double core21 = gt + xor_(lt, d);
        double core22 = fma_(mt, lt, xor_(1.0, d));
        pre[0][0] = xor_(c * core11, L->ph1r);
        pre[2][0] = xor_(c * core12, L->ph1r);
        pre[1][0] = xor_(c * core21, xor_(L->ph2r, -0.0));
        pre[3][0] = xor_(c * core22, L->ph2r);
        pre[0][1] = pre[1][1] = pre[2][1] = pre[3][1] = 0.0;
    } else {
        double t = mt * lt;
        double dr = L->dhr, di = L->dhi;
        double i11r = fma_(dr, t, 1.0), i11i = di * t;
        double i21r = fma_(dr, lt, gt), i21i = di * lt;
        double i12r = fma_(dr, gt, lt), i12i = di * gt;
        double i22r = fma_(mt, lt, dr), i22i = di;
        double p[4][2];
        cmul(L->ph1r, L->ph1i, i11r, i11i, &p[0][0], &p[0][1]);
        cmul(L->ph2r, L->ph2i, i21r, i21i, &p[1][0], &p[1][1]);
        cmul(L->ph1r, L->ph1i, i12r, i12i, &p[2][0], &p[2][1]);
        cmul(L->ph2r, L->ph2i, i22r, i22i, &p[3][0], &p[3][1]);
        pre[0][0] = c * p[0][0]; pre[0][1] = c * p[0][1];
        pre[1][0] = neg_(c * p[1][0]); pre[1][1] = neg_(c * p[1][1]);
        pre[2][0] = c * p[2][0]; pre[2][1] = c * p[2][1];
        pre[3][0] = c * p[3][0]; pre[3][1] = c * p[3][1];
    }
    finish_u(L, pre);
    assemble_v(L, cplx);
}

/* svd2.py:427-474 (sine form) */
static void assemble_uv_sine(lane_t *L, int cplx)
{
    double sin_g = L->g_cos * L->g_tan;
    double sin_l = L->l_cos * L->l_tan;
    double cc = L->g_cos * L->l_cos;
    double ss = sin_g * sin_l;
    double cs = L->g_cos * sin_l;
    double sc = sin_g * L->l_cos;
    double pre[4][2];
    if (!cplx) {
        double d = L->dhr;
        double core11 = cc - xor_(ss, d);
        double core12 = cs + xor_(sc, d);
        double core21 = sc + xor_(cs, d);
        double core22 = xor_(cc, d) - ss;
        pre[0][0] = xor_(core11, L->ph1r);
        pre[2][0] = xor_(core12, L->ph1r);
        pre[1][0] = xor_(core21, xor_(L->ph2r, -0.0));
        pre[3][0] = xor_(core22, L->ph2r);
        pre[0][1] = pre[1][1] = pre[2][1] = pre[3][1] = 0.0;
    } else {
        double dr = L->dhr, di = L->dhi;
        double i11r = fnma_(dr, ss, cc), i11i = neg_(di * ss);
        double i12r = fma_(dr, sc, cs), i12i = di * sc;
        double i21r = fma_(dr, cs, sc), i21i = di * cs;
        double i22r = fma_(dr, cc, neg_(ss)), i22i = di * cc;
        double p[4][2];
        cmul(L->ph1r, L->ph1i, i11r, i11i, &p[0][0], &p[0][1]);
        cmul(L->ph2r, L->ph2i, i21r, i21i, &p[1][0], &p[1][1]);
        cmul(L->ph1r, L->ph1i, i12r, i12i, &p[2][0], &p[2][1]);
        cmul(L->ph2r, L->ph2i, i22r, i22i, &p[3][0], &p[3][1]);
        pre[0][0] = p[0][0]; pre[0][1] = p[0][1];
        pre[1][0] = neg_(p[1][0]); pre[1][1] = neg_(p[1][1]);
        pre[2][0] = p[2][0]; pre[2][1] = p[2][1];
        pre[3][0] = p[3][0]; pre[3][1] = p[3][1];
    }
    finish_u(L, pre);
    assemble_v(L, cplx);
}

/* svd2.py:521-570 for one lane.  a[t][0..1] = (re, im) of entry t in the
 * order e11, e21, e12, e22. */
static void svd2_lane(lane_t *L, double a[4][2], int cplx, int sine_form)
{
    /* phase 1: svd2.py:134-160 (component order e11r,e11i,e21r,...) */
    double p[8], s[8];
    int np_ = cplx ? 8 : 4;
    for (int t = 0; t < 4; t++) {
        if (cplx) { p[2 * t] = a[t][0]; p[2 * t + 1] = a[t][1]; }
        else p[t] = a[t][0];
    }
    L->shift = compute_scale(p, np_, s);
    double e[4][2];
    for (int t = 0; t < 4; t++) {
        e[t][0] = cplx ? s[2 * t] : s[t];
        e[t][1] = cplx ? s[2 * t + 1] : 0.0;
    }
    /* column norms: svd2.py:167-182 */
    double m[4];
    for (int t = 0; t < 4; t++)
        m[t] = cplx ? hypot_lane(e[t][0], e[t][1]) : fabs_(e[t][0]);
    double n1 = hypot_lane(m[0], m[1]);
    double n2 = hypot_lane(m[2], m[3]);
    /* column pivot: svd2.py:193-208 */
    int sc = n1 < n2;
    for (int k = 0; k < 2; k++) {
        swap_sel(sc, &e[0][k], &e[2][k]);
        swap_sel(sc, &e[1][k], &e[3][k]);
    }
    swap_sel(sc, &m[0], &m[2]);
    swap_sel(sc, &m[1], &m[3]);
    swap_sel(sc, &n1, &n2);
    /* row sort: svd2.py:211-224 */
    int sr = m[0] < m[1];
    for (int k = 0; k < 2; k++) {
        swap_sel(sr, &e[0][k], &e[1][k]);
        swap_sel(sr, &e[2][k], &e[3][k]);
    }
    swap_sel(sr, &m[0], &m[1]);
    swap_sel(sr, &m[2], &m[3]);
    L->swap_c = sc;
    L->swap_r = sr;
    /* left phase reduce: svd2.py:227-250 */
    double b11 = m[0], b21 = m[1];
    double f12r, f12i = 0.0, f22r, f22i = 0.0;
    if (!cplx) {
        L->ph1r = sgn_(e[0][0]); L->ph1i = 0.0;
        L->ph2r = sgn_(e[1][0]); L->ph2i = 0.0;
        f12r = xor_(e[2][0], L->ph1r);
        f22r = xor_(e[3][0], L->ph2r);
    } else {
        phase_from_parts(e[0][0], e[0][1], m[0], &L->ph1r, &L->ph1i);
        phase_from_parts(e[1][0], e[1][1], m[1], &L->ph2r, &L->ph2i);
        cmul(L->ph1r, neg_(L->ph1i), e[2][0], e[2][1], &f12r, &f12i);
        cmul(L->ph2r, neg_(L->ph2i), e[3][0], e[3][1], &f22r, &f22i);
    }
    /* givens: svd2.py:253-276 */
    double mt = rmax(b21 / b11, 0.0);
    double cg = invsqrt_lane(fma_(mt, mt, 1.0));
    L->r11 = n1;
    double g12r = cg * fma_(mt, f22r, f12r);
    double g22r = cg * fnma_(mt, f12r, f22r);
    double g12i = 0.0, g22i = 0.0;
    if (cplx) {
        g12i = cg * fma_(mt, f22i, f12i);
        g22i = cg * fnma_(mt, f12i, f22i);
    }
    L->g_tan = neg_(mt);
    L->g_cos = cg;
    /* phase fix: svd2.py:279-299 */
    if (!cplx) {
        double sg12 = sgn_(g12r);
        double w = xor_(g22r, sg12);
        L->r12 = fabs_(g12r);
        L->r22 = fabs_(w);
        L->dtr = sg12; L->dti = 0.0;
        L->dhr = sgn_(w); L->dhi = 0.0;
    } else {
        double c12, s12, wr, wi;
        L->r12 = hypot_lane(g12r, g12i);
        phase_from_parts(g12r, g12i, L->r12, &c12, &s12);
        cmul(c12, neg_(s12), g22r, g22i, &wr, &wi);
        L->r22 = hypot_lane(wr, wi);
        phase_from_parts(wr, wi, L->r22, &L->dhr, &L->dhi);
        L->dtr = c12; L->dti = neg_(s12);
    }
    triangular_svd(L);
    if (sine_form) assemble_uv_sine(L, cplx);
    else assemble_uv(L, cplx);
}

/* svd2.py:481-514 */
static void backscale(double smax, double smin, double shift, int mode,
                      double *omax, double *omin, double *oshift)
{
    if (mode == 0) { *omax = smax; *omin = smin; *oshift = shift; return; }
    double neg_s = neg_(shift);
    double bs_max = scalef(smax, neg_s);
    double bs_min = scalef(smin, neg_s);
    if (mode == 2) { *omax = bs_max; *omin = bs_min; *oshift = -0.0; return; }
    double e_max = getexp(smax) - shift;
    double e_min = getexp(smin) - shift;
    int ok = (e_max <= 1023.0) && ((smin == 0.0) || (e_min >= -1022.0));
    *omax = sel(ok, smax, bs_max);
    *omin = sel(ok, smin, bs_min);
    *oshift = sel(ok, shift, -0.0);
}

/* ---- batch entry points ---------------------------------------------- */

typedef struct {
    int64_t lo, hi;
    int cplx, mode, sine;
    const double *const *re, *const *im;
    double *const *ure, *const *uim, *const *vre, *const *vim;
    double *smax, *smin, *shift;
    double *const *states;   /* optional: 16 (real) / 20 (complex) trains */
} job_t;

static void run_range(const job_t *J)
{
    for (int64_t k = J->lo; k < J->hi; k++) {
        double a[4][2];
        for (int t = 0; t < 4; t++) {
            a[t][0] = J->re[t][k];
            a[t][1] = J->cplx ? J->im[t][k] : 0.0;
        }
        lane_t L;
        svd2_lane(&L, a, J->cplx, J->sine);
        for (int t = 0; t < 4; t++) {
            J->ure[t][k] = L.u[t][0];
            J->vre[t][k] = L.v[t][0];
            if (J->cplx) { J->uim[t][k] = L.u[t][1]; J->vim[t][k] = L.v[t][1]; }
        }
        backscale(L.smax, L.smin, L.shift, J->mode,
                  &J->smax[k], &J->smin[k], &J->shift[k]);
        if (J->states) {
            /* driver.py:193-216 train order */
            int i = 0;
            J->states[i++][k] = L.shift;
            J->states[i++][k] = L.swap_c ? 1.0 : 0.0;
            J->states[i++][k] = L.swap_r ? 1.0 : 0.0;
            J->states[i++][k] = L.ph1r; if (J->cplx) J->states[i++][k] = L.ph1i;
            J->states[i++][k] = L.ph2r; if (J->cplx) J->states[i++][k] = L.ph2i;
            J->states[i++][k] = L.dtr;  if (J->cplx) J->states[i++][k] = L.dti;
            J->states[i++][k] = L.dhr;  if (J->cplx) J->states[i++][k] = L.dhi;
            J->states[i++][k] = L.g_tan;
            J->states[i++][k] = L.g_cos;
            J->states[i++][k] = L.r11;
            J->states[i++][k] = L.r12;
            J->states[i++][k] = L.r22;
            J->states[i++][k] = L.l_tan;
            J->states[i++][k] = L.r_tan;
            J->states[i++][k] = L.smax;
            J->states[i++][k] = L.smin;
        }
    }
}

static void *thread_main(void *arg) { run_range((const job_t *)arg); return NULL; }

/* driver.py:134-146: contiguous 8-lane-aligned slabs, one per worker */
static int run_threads(job_t base, int64_t n, int threads)
{
    if (threads < 1) threads = 1;
    int64_t chunks = (n + 7) / 8;
    if (threads > chunks) threads = chunks ? (int)chunks : 1;
    if (threads == 1) { base.lo = 0; base.hi = n; run_range(&base); return 0; }
    pthread_t *tid = malloc(sizeof(pthread_t) * threads);
    job_t *jobs = malloc(sizeof(job_t) * threads);
    int64_t q = chunks / threads, r = chunks % threads, lo = 0;
    for (int w = 0; w < threads; w++) {
        int64_t width = (q + (w < r ? 1 : 0)) * 8;
        jobs[w] = base;
        jobs[w].lo = lo;
        jobs[w].hi = lo + width < n ? lo + width : n;
        lo += width;
        pthread_create(&tid[w], NULL, thread_main, &jobs[w]);
    }
    for (int w = 0; w < threads; w++) pthread_join(tid[w], NULL);
    free(tid);
    free(jobs);
    return 0;
}

int oracle_svd2_real(int64_t n, const double *const a[4], double *const u[4],
                     double *const v[4], double *smax, double *smin,
                     double *shift, int backscale_mode, int sine_form,
                     int threads, double *const *states)
{
    if (n < 0 || backscale_mode < 0 || backscale_mode > 2) return 1;
    job_t J = {0, 0, 0, backscale_mode, sine_form, a, NULL, u, NULL, v, NULL,
               smax, smin, shift, states};
    return run_threads(J, n, threads);
}

int oracle_svd2_complex(int64_t n, const double *const re[4],
                        const double *const im[4], double *const ure[4],
                        double *const uim[4], double *const vre[4],
                        double *const vim[4], double *smax, double *smin,
                        double *shift, int backscale_mode, int sine_form,
                        int threads, double *const *states)
{
    if (n < 0 || backscale_mode < 0 || backscale_mode > 2) return 1;
    job_t J = {0, 0, 1, backscale_mode, sine_form, re, im, ure, uim, vre, vim,
               smax, smin, shift, states};
    return run_threads(J, n, threads);
}

/* elementwise probes for the primitive-level known-answer tests */
double oracle_getexp(double a) { return getexp(a); }
double oracle_scalef(double a, double e) { return scalef(a, e); }
double oracle_hypot(double a, double b) { return hypot_lane(a, b); }
double oracle_invsqrt(double a) { return invsqrt_lane(a); }
void oracle_backscale(int64_t n, const double *smax, const double *smin,
                      const double *shift, int mode, double *omax,
                      double *omin, double *oshift)
{
    for (int64_t k = 0; k < n; k++)
        backscale(smax[k], smin[k], shift[k], mode, &omax[k], &omin[k],
                  &oshift[k]);
}

/* vectorised probes for the GPU arithmetic tests */
void oracle_hypot_vec(int64_t n, const double *a, const double *b, double *out)
{
    for (int64_t k = 0; k < n; k++) out[k] = hypot_lane(a[k], b[k]);
}

/* lanes.py:262-270 polar(): magnitude and unit phase */
void oracle_phase_vec(int64_t n, const double *re, const double *im,
                      double *c, double *s)
{
    for (int64_t k = 0; k < n; k++) {
        double mag = hypot_lane(re[k], im[k]);
        phase_from_parts(re[k], im[k], mag, &c[k], &s[k]);
    }
}
