// b2s_verify.cu -- batch quality metrics in double-double on the GPU.
//
// Device port of lanesvd.verify.metrics (verify.py:355-477): per lane, in
// the domain the stored values live in (A if the lane was backscaled, else
// 2^shift A), exactly normalised by 2^-getexp(smax), the relative residual
// rho = |U S V* - A|_F / |A|_F and the unitarity defects delta = |U*U - I|_F,
// eta = |V*V - I|_F in double-double (~106 bits), and the condition number
// kappa = smax / smin as an exact (double-double mantissa, integer exponent)
// pair.  Every double-double operation is the reference's own sequence of
// IEEE operations (verify.py:42-169), so per-lane values are bit-identical to
// the reference and the exact maxima below reproduce its Metrics.
//
// Reduction: per block, exact lexicographic maxima -- (hi, then lo among
// equal hi) for rho / delta / eta, (exponent, hi, lo) for kappa -- written as
// one partial record per block; the host folds the partials the same way
// (the maximum over a union is the maximum of the parts).
#include "../../include/b2s.h"
#include "b2s_common.cuh"
#include "b2s_lane.cuh"

namespace b2s {
namespace dd {

struct DD {
  double hi, lo;
};

__device__ __forceinline__ DD from(double x) { return {x, 0.0}; }

// verify.py:55-58
__device__ __forceinline__ void two_sum(double a, double b, double& s, double& e) {
  s = __dadd_rn(a, b);
  const double bb = __dsub_rn(s, a);
  e = __dadd_rn(__dsub_rn(a, __dsub_rn(s, bb)), __dsub_rn(b, bb));
}

// verify.py:61-64
__device__ __forceinline__ void quick_two_sum(double a, double b, double& s, double& e) {
  s = __dadd_rn(a, b);
  e = __dsub_rn(b, __dsub_rn(s, a));
}

// verify.py:67-69
__device__ __forceinline__ void two_prod(double a, double b, double& p, double& e) {
  p = __dmul_rn(a, b);
  e = __fma_rn(a, b, -p);
}

// verify.py:72-78
__device__ __forceinline__ DD add(DD a, DD b) {
  double s1, s2, t1, t2;
  two_sum(a.hi, b.hi, s1, s2);
  two_sum(a.lo, b.lo, t1, t2);
  s2 = __dadd_rn(s2, t1);
  quick_two_sum(s1, s2, s1, s2);
  s2 = __dadd_rn(s2, t2);
  DD r;
  quick_two_sum(s1, s2, r.hi, r.lo);
  return r;
}

__device__ __forceinline__ DD neg(DD a) { return {-a.hi, -a.lo}; }
__device__ __forceinline__ DD sub(DD a, DD b) { return add(a, neg(b)); }

// verify.py:90-93
__device__ __forceinline__ DD mul(DD a, DD b) {
  double p1, p2;
  two_prod(a.hi, b.hi, p1, p2);
  p2 = __dadd_rn(p2, __dadd_rn(__dmul_rn(a.hi, b.lo), __dmul_rn(a.lo, b.hi)));
  DD r;
  quick_two_sum(p1, p2, r.hi, r.lo);
  return r;
}

// verify.py:96-100
__device__ __forceinline__ DD mul_f(DD a, double b) {
  double p1, p2;
  two_prod(a.hi, b, p1, p2);
  p2 = __dadd_rn(p2, __dmul_rn(a.lo, b));
  DD r;
  quick_two_sum(p1, p2, r.hi, r.lo);
  return r;
}

// verify.py:103-106
__device__ __forceinline__ DD add_f(DD a, double b) {
  double s1, s2;
  two_sum(a.hi, b, s1, s2);
  s2 = __dadd_rn(s2, a.lo);
  DD r;
  quick_two_sum(s1, s2, r.hi, r.lo);
  return r;
}

// verify.py:114-124
__device__ __forceinline__ DD div(DD a, DD b) {
  const double q1 = __ddiv_rn(a.hi, b.hi);
  DD r = sub(a, mul_f(b, q1));
  const double q2 = __ddiv_rn(r.hi, b.hi);
  r = sub(r, mul_f(b, q2));
  const double q3 = __ddiv_rn(r.hi, b.hi);
  DD s;
  quick_two_sum(q1, q2, s.hi, s.lo);
  return add_f(s, q3);
}

// verify.py:127-136
__device__ __forceinline__ DD sqrt(DD a) {
  const double x = __ddiv_rn(1.0, __dsqrt_rn(a.hi));
  const double ax = __dmul_rn(a.hi, x);
  DD axx;
  two_prod(ax, ax, axx.hi, axx.lo);
  const double corr = __dmul_rn(sub(a, axx).hi, __dmul_rn(x, 0.5));
  DD r;
  quick_two_sum(ax, corr, r.hi, r.lo);
  if (a.hi == 0.0) r = {0.0, 0.0};
  return r;
}

// verify.py:145-147 with k = 1 or 2 (exact power-of-two scaling)
__device__ __forceinline__ DD scalb(DD a, double k) { return {scalef_dev(a.hi, k), scalef_dev(a.lo, k)}; }

struct CD {
  DD re, im;
};

__device__ __forceinline__ CD cfrom(double re, double im) { return {from(re), from(im)}; }
__device__ __forceinline__ CD conj(CD a) { return {a.re, neg(a.im)}; }
__device__ __forceinline__ CD cadd(CD a, CD b) { return {add(a.re, b.re), add(a.im, b.im)}; }
__device__ __forceinline__ CD csub(CD a, CD b) { return {sub(a.re, b.re), sub(a.im, b.im)}; }
// verify.py:196-199
__device__ __forceinline__ CD cmul(CD a, CD b) {
  return {sub(mul(a.re, b.re), mul(a.im, b.im)), add(mul(a.re, b.im), mul(a.im, b.re))};
}
__device__ __forceinline__ CD cmul_dd(CD a, DD s) { return {mul(a.re, s), mul(a.im, s)}; }
__device__ __forceinline__ DD abs2(CD a) { return add(mul(a.re, a.re), mul(a.im, a.im)); }

// verify.py:384-392
__device__ __forceinline__ DD gram_deviation(CD c11, CD c21, CD c12, CD c22) {
  const DD one = from(1.0);
  const DD g11 = sub(add(abs2(c11), abs2(c21)), one);
  const DD g22 = sub(add(abs2(c12), abs2(c22)), one);
  const CD g12 = cadd(cmul(conj(c11), c12), cmul(conj(c21), c22));
  const DD s = add(add(mul(g11, g11), mul(g22, g22)), scalb(abs2(g12), 1.0));
  return sqrt(s);
}

// Spectral-norm companion of gram_deviation (an extension for the
// north-star tolerance report): |G|_2 of the Hermitian
// G = C*C - I is |tr G| / 2 + sqrt(((g11 - g22) / 2)^2 + |g12|^2).
__device__ __forceinline__ DD gram_deviation2(CD c11, CD c21, CD c12, CD c22) {
  const DD one = from(1.0);
  const DD g11 = sub(add(abs2(c11), abs2(c21)), one);
  const DD g22 = sub(add(abs2(c12), abs2(c22)), one);
  const CD g12 = cadd(cmul(conj(c11), c12), cmul(conj(c21), c22));
  DD half_tr = scalb(add(g11, g22), -1.0);
  if (half_tr.hi < 0.0) half_tr = neg(half_tr);
  const DD half_df = scalb(sub(g11, g22), -1.0);
  return add(half_tr, sqrt(add(mul(half_df, half_df), abs2(g12))));
}

}  // namespace dd

// Per-block partial: rho, delta, eta (hi, lo), kappa (d, qhi, qlo), kappa
// infinite flag, excluded-lane count, then the spectral-norm delta2, eta2
// (hi, lo).
constexpr int kPartial = 17;

struct Acc {
  double rho_hi, rho_lo, del_hi, del_lo, eta_hi, eta_lo, kd, kq_hi, kq_lo, kinf, bad;
  double d2_hi, d2_lo, e2_hi, e2_lo;
  double over_f, over_2;     // lanes with max(rho, delta, eta) > 8 eps (Frobenius / 2-norm)
};

// Lexicographic maximum helpers (NaN in hi propagates, like numpy.max).
__device__ __forceinline__ void max_dd(double& mh, double& ml, double h, double l) {
  if (h != h || mh != mh) {
    if (h != h) { mh = h; ml = l; }
    return;
  }
  if (h > mh || (h == mh && l > ml)) { mh = h; ml = l; }
}

__device__ __forceinline__ void max_kappa(Acc& a, double d, double h, double l) {
  if (d > a.kd || (d == a.kd && (h > a.kq_hi || (h == a.kq_hi && l > a.kq_lo)))) {
    a.kd = d; a.kq_hi = h; a.kq_lo = l;
  }
}

__device__ __forceinline__ void merge(Acc& a, const Acc& b) {
  max_dd(a.rho_hi, a.rho_lo, b.rho_hi, b.rho_lo);
  max_dd(a.del_hi, a.del_lo, b.del_hi, b.del_lo);
  max_dd(a.eta_hi, a.eta_lo, b.eta_hi, b.eta_lo);
  max_kappa(a, b.kd, b.kq_hi, b.kq_lo);
  a.kinf = fmax(a.kinf, b.kinf);
  a.bad += b.bad;
  max_dd(a.d2_hi, a.d2_lo, b.d2_hi, b.d2_lo);
  max_dd(a.e2_hi, a.e2_lo, b.e2_hi, b.e2_lo);
  a.over_f += b.over_f;
  a.over_2 += b.over_2;
}

__device__ __forceinline__ Acc acc_identity() {
  const double ninf = -__longlong_as_double(0x7FF0000000000000ll);
  return {ninf, ninf, ninf, ninf, ninf, ninf, ninf, ninf, ninf, 0.0, 0.0, ninf, ninf, ninf, ninf, 0.0, 0.0};
}

struct MetricArgs {
  int64_t n;
  int cplx;
  const double* ar[4];
  const double* ai[4];
  const double* ur[4];
  const double* ui[4];
  const double* vr[4];
  const double* vi[4];
  const double *smax, *smin, *shift;
  double* partial;              // [gridDim.x][kPartial]
  double *lane_rho, *lane_delta, *lane_eta;   // optional per-lane hi parts
};

// verify.py:395-477 for one lane.
__device__ Acc lane_metrics(const MetricArgs& M, int64_t i) {
  using namespace dd;
  Acc r = acc_identity();
  double smax = M.smax[i], smin = M.smin[i];
  const double shift = M.shift[i];
  const bool performed = shift == 0.0 && (bits(shift) & kSign);
  const double eff = performed ? 0.0 : shift;
  const bool bad = !(isfinite(smax) && isfinite(smin));
  const double g = (smax > 0.0 && !bad) ? getexp_dev(smax) : 0.0;
  CD a[4], u[4], v[4];
  for (int t = 0; t < 4; t++) {
    const double re = scalef_dev(scalef_dev(M.ar[t][i], eff), -g);
    const double im = M.cplx ? scalef_dev(scalef_dev(M.ai[t][i], eff), -g) : 0.0;
    a[t] = cfrom(re, im);
    u[t] = cfrom(M.ur[t][i], M.cplx ? M.ui[t][i] : 0.0);
    v[t] = cfrom(M.vr[t][i], M.cplx ? M.vi[t][i] : 0.0);
  }
  const DD s1 = from(bad ? 0.0 : scalef_dev(smax, -g));
  const DD s2 = from(bad ? 0.0 : scalef_dev(smin, -g));
  const CD w[4] = {cmul_dd(u[0], s1), cmul_dd(u[1], s1), cmul_dd(u[2], s2), cmul_dd(u[3], s2)};
  DD num2 = from(0.0), den2 = from(0.0);
  const int ij[4][2] = {{0, 0}, {1, 0}, {0, 1}, {1, 1}};
  for (int t = 0; t < 4; t++) {
    const int ii = ij[t][0], jj = ij[t][1];
    const CD rec = cadd(cmul(w[ii], conj(v[jj])), cmul(w[2 + ii], conj(v[2 + jj])));
    num2 = add(num2, abs2(csub(rec, a[t])));
    den2 = add(den2, abs2(a[t]));
  }
  DD rho = sqrt(div(num2, den2));
  const bool drop = bad || !isfinite(rho.hi);
  rho = drop ? DD{0.0, 0.0} : DD{rmax(rho.hi, 0.0), rho.lo};
  const DD delta = gram_deviation(u[0], u[1], u[2], u[3]);
  const DD eta = gram_deviation(v[0], v[1], v[2], v[3]);
  r.rho_hi = rho.hi; r.rho_lo = rho.lo;
  r.del_hi = delta.hi; r.del_lo = delta.lo;
  r.eta_hi = eta.hi; r.eta_lo = eta.lo;
  r.bad = bad ? 1.0 : 0.0;
  const DD d2 = gram_deviation2(u[0], u[1], u[2], u[3]);
  const DD e2 = gram_deviation2(v[0], v[1], v[2], v[3]);
  r.d2_hi = d2.hi; r.d2_lo = d2.lo;
  r.e2_hi = e2.hi; r.e2_lo = e2.lo;
  // north_star's 8-eps gate per lane (eps = 2^-52), exact on the DD values
  const double tol = 0x1p-49;
  auto over = [&](const DD& x) { return x.hi > tol || (x.hi == tol && x.lo > 0.0); };
  const bool of = over(rho) || over(delta) || over(eta);
  const bool o2 = over(rho) || over(d2) || over(e2);
  r.over_f = of ? 1.0 : 0.0;
  r.over_2 = o2 ? 1.0 : 0.0;
  if (bad || smin == 0.0) {
    r.kinf = 1.0;
  } else {
    const double e1 = getexp_dev(smax), e2 = getexp_dev(smin);
    DD q = div(from(scalef_dev(smax, -e1)), from(scalef_dev(smin, -e2)));
    double d = e1 - e2;
    if (q.hi < 1.0) {
      q = scalb(q, 1.0);
      d -= 1.0;
    }
    r.kd = d; r.kq_hi = q.hi; r.kq_lo = q.lo;
  }
  if (M.lane_rho) M.lane_rho[i] = rho.hi;
  if (M.lane_delta) M.lane_delta[i] = delta.hi;
  if (M.lane_eta) M.lane_eta[i] = eta.hi;
  return r;
}

constexpr int kMBlock = 128;

__global__ void __launch_bounds__(kMBlock) k_metrics(const MetricArgs M) {
  __shared__ Acc part[kMBlock / 32];
  Acc acc = acc_identity();
  for (int64_t i = (int64_t)blockIdx.x * kMBlock + threadIdx.x; i < M.n; i += (int64_t)gridDim.x * kMBlock)
    merge(acc, lane_metrics(M, i));
  // warp reduction
  for (int off = 16; off; off >>= 1) {
    Acc o;
    double* po = reinterpret_cast<double*>(&o);
    double* pa = reinterpret_cast<double*>(&acc);
    #pragma unroll
    for (int k = 0; k < kPartial; k++) po[k] = __shfl_down_sync(0xFFFFFFFFu, pa[k], off);
    merge(acc, o);
  }
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < kMBlock / 32; w++) merge(acc, part[w]);
    const double* pa = reinterpret_cast<const double*>(&acc);
    for (int k = 0; k < kPartial; k++) M.partial[(size_t)blockIdx.x * kPartial + k] = pa[k];
  }
}

// ---------------------------------------------------------------------------
// lanesvd.verify.oracle_svd2 (verify.py:259-352): the closed-form reference
// SVD in double-double, independent of the pipeline phases -- per lane an
// exact power-of-two prescale by the largest component's exponent, the Gram
// matrix's eigensystem with the cancellation-free discriminant, smin from
// |det| / smax, the right vectors from the better-conditioned Gram row, the
// left vectors as their images (the unitary completion when smin / smax <
// 1e-25).  The same double-double operation sequence as the reference, so
// every output word is bit-identical.  Output trains (36): smax hi/lo, smin
// hi/lo, then u11 u21 u12 u22 v11 v21 v12 v22 as re.hi re.lo im.hi im.lo.
// ---------------------------------------------------------------------------
struct OracleArgs {
  int64_t n;
  int cplx;
  const double* ar[4];
  const double* ai[4];
  double* out[36];
};

namespace dd {
__device__ __forceinline__ DD sel(bool m, DD a, DD b) { return m ? a : b; }
__device__ __forceinline__ CD csel(bool m, CD a, CD b) { return m ? a : b; }
__device__ __forceinline__ CD cdiv_dd(CD a, DD s) { return {div(a.re, s), div(a.im, s)}; }
}  // namespace dd

__global__ void __launch_bounds__(128) k_oracle_svd2(const OracleArgs O) {
  using namespace dd;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < O.n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double re[4], im[4];
    double mags = 0.0, mi = 0.0;
    for (int t = 0; t < 4; t++) {
      re[t] = O.ar[t][i];
      im[t] = O.cplx ? O.ai[t][i] : 0.0;
      mags = fmax(mags, fabs(re[t]));
      mi = fmax(mi, fabs(im[t]));
    }
    mags = fmax(mags, mi);
    const double g = mags > 0.0 ? getexp_dev(mags) : 0.0;
    CD e[4];                                        // e11, e21, e12, e22
    for (int t = 0; t < 4; t++) e[t] = cfrom(scalef_dev(re[t], -g), scalef_dev(im[t], -g));
    const DD m11 = add(abs2(e[0]), abs2(e[1]));
    const DD m22 = add(abs2(e[2]), abs2(e[3]));
    const CD m12 = cadd(cmul(conj(e[0]), e[2]), cmul(conj(e[1]), e[3]));
    const DD trace = add(m11, m22);
    const DD diff = sub(m11, m22);
    const DD disc = sqrt(add(mul(diff, diff), scalb(abs2(m12), 2.0)));
    const DD lam_max = scalb(add(trace, disc), -1.0);
    DD smax = sqrt(lam_max);
    const CD det = csub(cmul(e[0], e[3]), cmul(e[2], e[1]));
    const DD absdet = sqrt(abs2(det));
    const bool zero_s = smax.hi == 0.0;
    const DD z = from(0.0), one = from(1.0);
    DD smin = sel(zero_s, z, div(absdet, smax));
    const bool big1 = m11.hi >= m22.hi;
    CD v11 = csel(big1, CD{sub(lam_max, m22), z}, m12);
    CD v21 = csel(big1, conj(m12), CD{sub(lam_max, m11), z});
    const DD nrm2 = add(abs2(v11), abs2(v21));
    const bool degen = nrm2.hi == 0.0;
    v11 = csel(degen, CD{one, z}, v11);
    v21 = csel(degen, CD{z, z}, v21);
    const DD nrm = sqrt(sel(degen, one, nrm2));
    v11 = cdiv_dd(v11, nrm);
    v21 = cdiv_dd(v21, nrm);
    const CD v12 = {neg(v21.re), v21.im};
    const CD v22 = conj(v11);
    const CD av1 = cadd(cmul(e[0], v11), cmul(e[2], v21));
    const CD av2 = cadd(cmul(e[1], v11), cmul(e[3], v21));
    const DD safe_smax = sel(zero_s, one, smax);
    const CD u11 = csel(zero_s, CD{one, z}, cdiv_dd(av1, safe_smax));
    const CD u21 = csel(zero_s, CD{z, z}, cdiv_dd(av2, safe_smax));
    const CD bv1 = cadd(cmul(e[0], v12), cmul(e[2], v22));
    const CD bv2 = cadd(cmul(e[1], v12), cmul(e[3], v22));
    const bool reliable = smin.hi > __dmul_rn(smax.hi, 1e-25);
    const DD safe_smin = sel(reliable, smin, one);
    const CD u12 = csel(reliable, cdiv_dd(bv1, safe_smin), CD{neg(u21.re), u21.im});
    const CD u22 = csel(reliable, cdiv_dd(bv2, safe_smin), conj(u11));
    smax = scalb(smax, g);
    smin = scalb(smin, g);
    double* const* o = O.out;
    o[0][i] = smax.hi; o[1][i] = smax.lo; o[2][i] = smin.hi; o[3][i] = smin.lo;
    const CD f[8] = {u11, u21, u12, u22, v11, v21, v12, v22};
    for (int k = 0; k < 8; k++) {
      o[4 + 4 * k][i] = f[k].re.hi;
      o[5 + 4 * k][i] = f[k].re.lo;
      o[6 + 4 * k][i] = f[k].im.hi;
      o[7 + 4 * k][i] = f[k].im.lo;
    }
  }
}

}  // namespace b2s

using namespace b2s;

extern "C" int b2s_oracle_svd2(int64_t n, const double* const a_re[4], const double* const a_im[4],
                               double* const out[36], void* stream) {
  if (n < 0) return fail(1, "negative batch size");
  if (!a_re || !out) return fail(5, "NULL argument");
  OracleArgs O{};
  O.n = n;
  O.cplx = a_im != nullptr;
  for (int t = 0; t < 4; t++) {
    if (!a_re[t] || (O.cplx && !a_im[t])) return fail(5, "NULL input train");
    O.ar[t] = a_re[t];
    if (O.cplx) O.ai[t] = a_im[t];
  }
  for (int k = 0; k < 36; k++) {
    if (!out[k]) return fail(5, "NULL output train");
    O.out[k] = out[k];
  }
  if (n == 0) return 0;
  int blocks = (int)((n + 127) / 128);
  if (blocks > 148 * 16) blocks = 148 * 16;
  k_oracle_svd2<<<blocks, 128, 0, (cudaStream_t)stream>>>(O);
  B2S_CUDA(cudaGetLastError());
  return 0;
}

extern "C" int b2s_metrics(int64_t n, const double* const a_re[4], const double* const a_im[4],
                           const double* const u_re[4], const double* const u_im[4],
                           const double* const v_re[4], const double* const v_im[4], const double* smax,
                           const double* smin, const double* shift, double* partial, int blocks,
                           double* lane_rho, double* lane_delta, double* lane_eta, void* stream) {
  if (n < 0) return fail(1, "negative batch size");
  if (blocks < 1) return fail(1, "blocks must be >= 1");
  if (!a_re || !u_re || !v_re || !smax || !smin || !shift || !partial) return fail(5, "NULL argument");
  const bool cplx = a_im != nullptr;
  if (cplx && (!u_im || !v_im)) return fail(5, "complex metrics need u_im and v_im");
  MetricArgs M{};
  M.n = n;
  M.cplx = cplx;
  for (int t = 0; t < 4; t++) {
    M.ar[t] = a_re[t]; M.ur[t] = u_re[t]; M.vr[t] = v_re[t];
    if (cplx) { M.ai[t] = a_im[t]; M.ui[t] = u_im[t]; M.vi[t] = v_im[t]; }
  }
  M.smax = smax; M.smin = smin; M.shift = shift; M.partial = partial;
  M.lane_rho = lane_rho; M.lane_delta = lane_delta; M.lane_eta = lane_eta;
  k_metrics<<<blocks, kMBlock, 0, (cudaStream_t)stream>>>(M);
  B2S_CUDA(cudaGetLastError());
  return 0;
}
