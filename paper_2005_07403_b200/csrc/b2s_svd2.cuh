// b2s_svd2.cuh -- the fused per-lane 2x2 SVD pipelines (real and complex).
//
// One lane = one matrix, held entirely in registers: scale (svd2.py:134-160)
// -> URV reduction (167-299) -> closed-form triangle SVD (306-343) -> U/V
// assembly (350-474) -> optional backscale (481-514).  Operation order and
// rounding match the reference exactly, so outputs are bit-identical to
// lanesvd.svd2.svd2_lanes + backscale for every finite input.
//
// Two arithmetic variants share the assembly code:
//  * Exact (svd2_real_x / svd2_complex_x): IEEE intrinsics for every
//    division / sqrt; valid for all inputs.  Runs as the cold fallback and
//    for the state-dump variant.
//  * Fast (svd2_real_f / svd2_complex_f, b2s_fast.cuh): inline
//    seed+Newton sequences specialised to the operand range of each call
//    site, with no library slow paths.  Any operand outside a site's proven
//    range sets the lane's `hard` flag and the caller recomputes the lane
//    with the exact variant, so results are identical either way.
#pragma once
#include "b2s_lane.cuh"

namespace b2s {

// Intermediate states exported by the optional state-dump variant, in the
// train order of driver.py:193-216.
struct LaneStates {
  double shift, swap_c, swap_r;
  double ph1r, ph1i, ph2r, ph2i, dtr, dti, dhr, dhi;
  double g_tan, g_cos, r11, r12, r22, l_tan, r_tan, smax, smin;
  // the rest of svd2_lanes' with_states tuple (B2S_FLAG_STATES_FULL)
  double l_sec2, l_cos, r_sec2, r_cos;
  double sp[8];                  // ScaleResult.parts, input component order
};

struct RealOut {
  double u[4], v[4];   // 11, 21, 12, 22
  double smax, smin, shift;
};

struct CplxOut {
  double ur[4], ui[4], vr[4], vi[4];
  double smax, smin, shift;
};

// svd2.py:306-343 triangular_svd outputs
struct Tri {
  double l_tan, l_sec2, l_cos, r_tan, r_sec2, r_cos, smax, smin;
};

__device__ __forceinline__ void swp(bool m, double& a, double& b) {
  double na = sel(m, a, b), nb = sel(m, b, a);
  a = na;
  b = nb;
}

// ---------------------------------------------------------------------------
// Phase 1, svd2.py:134-160.  The relaxed-min tree over the margins
// 1021 - getexp(p) reduces to an integer minimum: every margin is an exact
// integer (+inf for a zero component, absorbed by the DBL_MAX clamp).
// ---------------------------------------------------------------------------
template <int N>
__device__ __forceinline__ double scale_x(double (&p)[N]) {
  int s = 0x7FFFFFFF;
  #pragma unroll
  for (int i = 0; i < N; i++) {
    int m = (p[i] == 0.0) ? 0x7FFFFFFF : 1021 - ilogb_finite(p[i]);
    s = min(s, m);
  }
  if (s == 0x7FFFFFFF) return kDblMax();   // zero matrix: entries stay +-0
  #pragma unroll
  for (int i = 0; i < N; i++) p[i] = scale_up(p[i], s);
  return (double)s;
}

// Fast variant: every nonzero component normal and s >= 0 (always true for
// inputs with moderate exponent spread).  Margins come straight from the
// exponent fields, scaling is an exact exponent-field add; zero components
// stay untouched.  Subnormal components, s < 0 and the all-zero matrix set
// `hard`.
template <int N>
__device__ __forceinline__ double scale_f(double (&p)[N], bool& hard) {
  unsigned emax = 0, kmin = 0x7FF00000u;
  unsigned key[N];
  #pragma unroll
  for (int i = 0; i < N; i++) {
    const unsigned h = hi_(p[i]);
    emax = max(emax, (h >> 20) & 0x7FFu);
    key[i] = lop_and(h, 0x7FFFFFFFu) | lo_(p[i]);     // 0 <=> +-0
    const unsigned k = key[i] == 0u ? 0x7FF00000u : lop_and(h, 0x7FFFFFFFu);
    kmin = min(kmin, k);
  }
  const int s = 2044 - (int)emax;            // 1021 - (emax - 1023)
  hard |= (kmin < 0x00100000u) | (s < 0) | (emax == 0u);
  const unsigned add = (unsigned)s << 20;
  #pragma unroll
  for (int i = 0; i < N; i++) p[i] = mk_(key[i] == 0u ? hi_(p[i]) : hi_(p[i]) + add, lo_(p[i]));
  return (double)s;
}

// ---------------------------------------------------------------------------
// Phase 3, svd2.py:306-343 (exact arithmetic).
// ---------------------------------------------------------------------------
__device__ __forceinline__ Tri triangle_tail(double x, double y, double l_tan, double r11, double r22,
                                             double l_cos, double r_cos) {
  Tri T;
  T.l_tan = l_tan;
  T.l_sec2 = fma_(l_tan, l_tan, 1.0);
  T.l_cos = l_cos;
  T.r_tan = fma_(y, l_tan, -x);
  T.r_sec2 = fma_(T.r_tan, T.r_tan, 1.0);
  T.r_cos = r_cos;
  double cc = mul(T.l_cos, T.r_cos);
  T.smax = mul(mul(cc, T.r_sec2), r11);
  T.smin = mul(mul(cc, T.l_sec2), r22);
  return T;
}

__device__ __forceinline__ Tri triangle_x(double r11, double r12, double r22) {
  double x = rmax(div_x(r12, r11), 0.0);
  double y = rmax(div_x(r22, r11), 0.0);
  double num = mul(mul(rmin(x, y), 2.0), rmax(x, y));        // scalef(min, 1) * max
  double den = fma_(sub(x, y), add(x, y), 1.0);
  double tan2 = or_(rmin(rmax(div_x(num, den), 0.0), kSqrtDblMax()), kNegZero());
  double lt = div_x(tan2, add(1.0, sqrt_x(fma_(tan2, tan2, 1.0))));
  double ls2 = fma_(lt, lt, 1.0);
  double rt = fma_(y, lt, -x);
  return triangle_tail(x, y, lt, r11, r22, invsqrt_x(ls2), invsqrt_x(fma_(rt, rt, 1.0)));
}

// svd2.py:481-514 backscale; Mode 0 none, 1 safe, 2 unconditional.
template <int Mode>
__device__ __forceinline__ void backscale_lane(double& smax, double& smin, double& shift) {
  if (Mode == 0) return;
  double neg_s = neg_(shift);
  double bs_max = scalef_dev(smax, neg_s);
  double bs_min = scalef_dev(smin, neg_s);
  if (Mode == 2) { smax = bs_max; smin = bs_min; shift = kNegZero(); return; }
  double e_max = sub(getexp_dev(smax), shift);
  double e_min = sub(getexp_dev(smin), shift);
  bool ok = (e_max <= 1023.0) && ((smin == 0.0) || (e_min >= -1022.0));
  smax = sel(ok, smax, bs_max);
  smin = sel(ok, smin, bs_min);
  shift = sel(ok, shift, kNegZero());
}

// ---------------------------------------------------------------------------
// Phase 4, real lanes: assemble_uv / assemble_uv_sine (svd2.py:378-474).
// ---------------------------------------------------------------------------
struct RealUrv {
  bool C, R;
  double ph1, ph2;     // row phases (sign patterns)
  double mt, cg;       // -givens_tan, givens_cos
  double dt, dh;       // r12 / r22 phase sign patterns
};

template <bool Sine>
__device__ __forceinline__ void assemble_real(const RealUrv& U, const Tri& T, RealOut& o) {
  const double mt = U.mt, gt = neg_(U.mt), lt = T.l_tan, dh = U.dh;
  double p11, p12, p21, p22;
  if (!Sine) {
    // svd2.py:386-399
    double c = mul(U.cg, T.l_cos);
    double k11 = fma_(xor_(mt, dh), lt, 1.0);
    double k12 = add(lt, xor_(gt, dh));
    double k21 = add(gt, xor_(lt, dh));
    double k22 = fma_(mt, lt, xor_(1.0, dh));
    p11 = xor_(mul(c, k11), U.ph1);
    p12 = xor_(mul(c, k12), U.ph1);
    p21 = xor_(mul(c, k21), xor_(U.ph2, kNegZero()));
    p22 = xor_(mul(c, k22), U.ph2);
  } else {
    // svd2.py:436-455
    double sin_g = mul(U.cg, gt), sin_l = mul(T.l_cos, lt);
    double cc = mul(U.cg, T.l_cos), ss = mul(sin_g, sin_l);
    double cs = mul(U.cg, sin_l), sc = mul(sin_g, T.l_cos);
    double k11 = sub(cc, xor_(ss, dh));
    double k12 = add(cs, xor_(sc, dh));
    double k21 = add(sc, xor_(cs, dh));
    double k22 = sub(xor_(cc, dh), ss);
    p11 = xor_(k11, U.ph1);
    p12 = xor_(k12, U.ph1);
    p21 = xor_(k21, xor_(U.ph2, kNegZero()));
    p22 = xor_(k22, U.ph2);
  }
  // _finish_u, svd2.py:372-375
  o.u[0] = sel(U.R, p11, p21); o.u[1] = sel(U.R, p21, p11);
  o.u[2] = sel(U.R, p12, p22); o.u[3] = sel(U.R, p22, p12);
  // _assemble_v, svd2.py:350-369
  double cr = T.r_cos, sr = mul(cr, T.r_tan);
  double v11 = cr, v12 = sr, v21 = xor_(sr, xor_(U.dt, kNegZero())), v22 = xor_(cr, U.dt);
  o.v[0] = sel(U.C, v11, v21); o.v[1] = sel(U.C, v21, v11);
  o.v[2] = sel(U.C, v12, v22); o.v[3] = sel(U.C, v22, v12);
  o.smax = T.smax;
  o.smin = T.smin;
}

// ---------------------------------------------------------------------------
// Real lanes, exact arithmetic (svd2.py:521-570 with 4 trains).
// ---------------------------------------------------------------------------
template <bool Sine, bool States>
__device__ __forceinline__ void svd2_real_x(const double (&a)[4], RealOut& o, LaneStates* st) {
  double e[4] = {a[0], a[1], a[2], a[3]};            // e11 e21 e12 e22
  double shift = scale_x<4>(e);
  if (States) for (int t = 0; t < 4; t++) st->sp[t] = e[t];
  // column_norms, svd2.py:167-182
  double m11 = fabs_(e[0]), m21 = fabs_(e[1]), m12 = fabs_(e[2]), m22 = fabs_(e[3]);
  double n1 = hypot_x(m11, m21), n2 = hypot_x(m12, m22);
  // column_pivot, svd2.py:193-208
  RealUrv U;
  U.C = n1 < n2;
  swp(U.C, e[0], e[2]); swp(U.C, e[1], e[3]);
  swp(U.C, m11, m12); swp(U.C, m21, m22); swp(U.C, n1, n2);
  // row_sort, svd2.py:211-224
  U.R = m11 < m21;
  swp(U.R, e[0], e[1]); swp(U.R, e[2], e[3]);
  swp(U.R, m11, m21); swp(U.R, m12, m22);
  // left_phase_reduce, svd2.py:238-244
  U.ph1 = sgn_(e[0]); U.ph2 = sgn_(e[1]);
  double f12 = xor_(e[2], U.ph1), f22 = xor_(e[3], U.ph2);
  // givens_qr, svd2.py:253-276
  U.mt = rmax(div_x(m21, m11), 0.0);
  U.cg = invsqrt_x(fma_(U.mt, U.mt, 1.0));
  double r11 = n1;
  double g12 = mul(U.cg, fma_(U.mt, f22, f12));
  double g22 = mul(U.cg, fnma_(U.mt, f12, f22));
  // phase_fix_r, svd2.py:290-294
  U.dt = sgn_(g12);
  double w = xor_(g22, U.dt);
  double r12 = fabs_(g12), r22 = fabs_(w);
  U.dh = sgn_(w);
  Tri T = triangle_x(r11, r12, r22);
  assemble_real<Sine>(U, T, o);
  o.shift = shift;
  if (States) {
    st->shift = shift; st->swap_c = U.C ? 1.0 : 0.0; st->swap_r = U.R ? 1.0 : 0.0;
    st->ph1r = U.ph1; st->ph2r = U.ph2; st->dtr = U.dt; st->dhr = U.dh;
    st->g_tan = neg_(U.mt); st->g_cos = U.cg; st->r11 = r11; st->r12 = r12; st->r22 = r22;
    st->l_tan = T.l_tan; st->r_tan = T.r_tan; st->smax = T.smax; st->smin = T.smin;
    st->l_sec2 = T.l_sec2; st->l_cos = T.l_cos; st->r_sec2 = T.r_sec2; st->r_cos = T.r_cos;
  }
}

// ---------------------------------------------------------------------------
// Phase 4, complex lanes (svd2.py:404-418, 456-469, 360-366).
// ---------------------------------------------------------------------------
struct CplxUrv {
  bool C, R;
  double c1, s1, c2, s2;     // row phases
  double mt, cg;
  double dtr, dti, dhr, dhi;
};

template <bool Sine>
__device__ __forceinline__ void assemble_complex(const CplxUrv& U, const Tri& T, CplxOut& o) {
  const double mt = U.mt, gt = neg_(U.mt), lt = T.l_tan, dhr = U.dhr, dhi = U.dhi;
  double q[4][2];   // pre-swap U entries 11, 21, 12, 22
  if (!Sine) {
    double c = mul(U.cg, T.l_cos);
    double t = mul(mt, lt);
    double i11r = fma_(dhr, t, 1.0), i11i = mul(dhi, t);
    double i21r = fma_(dhr, lt, gt), i21i = mul(dhi, lt);
    double i12r = fma_(dhr, gt, lt), i12i = mul(dhi, gt);
    double i22r = fma_(mt, lt, dhr), i22i = dhi;
    double xr, xi;
    cmul(U.c1, U.s1, i11r, i11i, xr, xi); q[0][0] = mul(c, xr); q[0][1] = mul(c, xi);
    cmul(U.c2, U.s2, i21r, i21i, xr, xi); q[1][0] = neg_(mul(c, xr)); q[1][1] = neg_(mul(c, xi));
    cmul(U.c1, U.s1, i12r, i12i, xr, xi); q[2][0] = mul(c, xr); q[2][1] = mul(c, xi);
    cmul(U.c2, U.s2, i22r, i22i, xr, xi); q[3][0] = mul(c, xr); q[3][1] = mul(c, xi);
  } else {
    double sin_g = mul(U.cg, gt), sin_l = mul(T.l_cos, lt);
    double cc = mul(U.cg, T.l_cos), ss = mul(sin_g, sin_l);
    double cs = mul(U.cg, sin_l), sc = mul(sin_g, T.l_cos);
    double i11r = fnma_(dhr, ss, cc), i11i = neg_(mul(dhi, ss));
    double i12r = fma_(dhr, sc, cs), i12i = mul(dhi, sc);
    double i21r = fma_(dhr, cs, sc), i21i = mul(dhi, cs);
    double i22r = fma_(dhr, cc, -ss), i22i = mul(dhi, cc);
    double xr, xi;
    cmul(U.c1, U.s1, i11r, i11i, xr, xi); q[0][0] = xr; q[0][1] = xi;
    cmul(U.c2, U.s2, i21r, i21i, xr, xi); q[1][0] = neg_(xr); q[1][1] = neg_(xi);
    cmul(U.c1, U.s1, i12r, i12i, xr, xi); q[2][0] = xr; q[2][1] = xi;
    cmul(U.c2, U.s2, i22r, i22i, xr, xi); q[3][0] = xr; q[3][1] = xi;
  }
  // _finish_u
  o.ur[0] = sel(U.R, q[0][0], q[1][0]); o.ui[0] = sel(U.R, q[0][1], q[1][1]);
  o.ur[1] = sel(U.R, q[1][0], q[0][0]); o.ui[1] = sel(U.R, q[1][1], q[0][1]);
  o.ur[2] = sel(U.R, q[2][0], q[3][0]); o.ui[2] = sel(U.R, q[2][1], q[3][1]);
  o.ur[3] = sel(U.R, q[3][0], q[2][0]); o.ui[3] = sel(U.R, q[3][1], q[2][1]);
  // _assemble_v
  double cr = T.r_cos, sr = mul(cr, T.r_tan);
  double v11r = cr, v11i = 0.0, v12r = sr, v12i = 0.0;
  double v21r = neg_(mul(sr, U.dtr)), v21i = neg_(mul(sr, U.dti));
  double v22r = mul(cr, U.dtr), v22i = mul(cr, U.dti);
  o.vr[0] = sel(U.C, v11r, v21r); o.vi[0] = sel(U.C, v11i, v21i);
  o.vr[1] = sel(U.C, v21r, v11r); o.vi[1] = sel(U.C, v21i, v11i);
  o.vr[2] = sel(U.C, v12r, v22r); o.vi[2] = sel(U.C, v12i, v22i);
  o.vr[3] = sel(U.C, v22r, v12r); o.vi[3] = sel(U.C, v22i, v12i);
  o.smax = T.smax;
  o.smin = T.smin;
}

// ---------------------------------------------------------------------------
// Complex lanes, exact arithmetic: 8 trains, re/im per entry.
// ---------------------------------------------------------------------------
template <bool Sine, bool States>
__device__ __forceinline__ void svd2_complex_x(const double (&ar)[4], const double (&ai)[4], CplxOut& o,
                                               LaneStates* st) {
  // component order of svd2_lanes: e11r, e11i, e21r, e21i, e12r, ...
  double p[8] = {ar[0], ai[0], ar[1], ai[1], ar[2], ai[2], ar[3], ai[3]};
  double shift = scale_x<8>(p);
  if (States) for (int t = 0; t < 8; t++) st->sp[t] = p[t];
  double er[4] = {p[0], p[2], p[4], p[6]}, ei[4] = {p[1], p[3], p[5], p[7]};
  // column_norms, svd2.py:176-181
  double m11 = hypot_x(er[0], ei[0]), m21 = hypot_x(er[1], ei[1]);
  double m12 = hypot_x(er[2], ei[2]), m22 = hypot_x(er[3], ei[3]);
  double n1 = hypot_x(m11, m21), n2 = hypot_x(m12, m22);
  CplxUrv U;
  U.C = n1 < n2;
  swp(U.C, er[0], er[2]); swp(U.C, ei[0], ei[2]);
  swp(U.C, er[1], er[3]); swp(U.C, ei[1], ei[3]);
  swp(U.C, m11, m12); swp(U.C, m21, m22); swp(U.C, n1, n2);
  U.R = m11 < m21;
  swp(U.R, er[0], er[1]); swp(U.R, ei[0], ei[1]);
  swp(U.R, er[2], er[3]); swp(U.R, ei[2], ei[3]);
  swp(U.R, m11, m21); swp(U.R, m12, m22);
  // left_phase_reduce, svd2.py:245-250
  phase_x(er[0], ei[0], m11, U.c1, U.s1);
  phase_x(er[1], ei[1], m21, U.c2, U.s2);
  double f12r, f12i, f22r, f22i;
  cmul(U.c1, neg_(U.s1), er[2], ei[2], f12r, f12i);
  cmul(U.c2, neg_(U.s2), er[3], ei[3], f22r, f22i);
  // givens_qr, svd2.py:263-276
  U.mt = rmax(div_x(m21, m11), 0.0);
  U.cg = invsqrt_x(fma_(U.mt, U.mt, 1.0));
  double r11 = n1;
  double g12r = mul(U.cg, fma_(U.mt, f22r, f12r)), g12i = mul(U.cg, fma_(U.mt, f22i, f12i));
  double g22r = mul(U.cg, fnma_(U.mt, f12r, f22r)), g22i = mul(U.cg, fnma_(U.mt, f12i, f22i));
  // phase_fix_r, svd2.py:295-299
  double r12 = hypot_x(g12r, g12i);
  double c12, s12;
  phase_x(g12r, g12i, r12, c12, s12);
  double wr, wi;
  cmul(c12, neg_(s12), g22r, g22i, wr, wi);
  double r22 = hypot_x(wr, wi);
  phase_x(wr, wi, r22, U.dhr, U.dhi);
  U.dtr = c12;
  U.dti = neg_(s12);
  Tri T = triangle_x(r11, r12, r22);
  assemble_complex<Sine>(U, T, o);
  o.shift = shift;
  if (States) {
    st->shift = shift; st->swap_c = U.C ? 1.0 : 0.0; st->swap_r = U.R ? 1.0 : 0.0;
    st->ph1r = U.c1; st->ph1i = U.s1; st->ph2r = U.c2; st->ph2i = U.s2;
    st->dtr = U.dtr; st->dti = U.dti; st->dhr = U.dhr; st->dhi = U.dhi;
    st->g_tan = neg_(U.mt); st->g_cos = U.cg; st->r11 = r11; st->r12 = r12; st->r22 = r22;
    st->l_tan = T.l_tan; st->r_tan = T.r_tan; st->smax = T.smax; st->smin = T.smin;
    st->l_sec2 = T.l_sec2; st->l_cos = T.l_cos; st->r_sec2 = T.r_sec2; st->r_cos = T.r_cos;
  }
}

}  // namespace b2s
