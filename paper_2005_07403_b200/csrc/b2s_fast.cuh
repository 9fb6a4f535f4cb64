// b2s_fast.cuh -- fast per-lane pipelines with range-specialised arithmetic.
//
// Same operation sequence as the exact pipelines in b2s_svd2.cuh (and so as
// the reference, svd2.py:134-570); only the way each correctly rounded
// division / sqrt / reciprocal is evaluated differs.  The scaling phase pins
// the largest entry to [2^1021, 2^1022), which bounds the operands of every
// call site (derivations per site below).  Where an operand can leave the
// range in which the inline sequence is correctly rounded (tiny numerators,
// subnormal quotients, subnormal components), the lane's `hard` flag is set
// and the kernel recomputes that lane.
//
// Every site is templated on Fix.  Fix = false (the streaming kernel): a
// failed range check only sets `hard`.  Fix = true (the fix-up kernel that
// recomputes the marked lanes): the failing site itself is re-evaluated
// with the IEEE intrinsic on its original operands, so a hard lane costs one
// exact division, not a whole exact pipeline.
#pragma once
#include "b2s_svd2.cuh"

namespace b2s {

// Fix-mode repair of one failing division: the exponent-normalised division
// (exact for every normal operand pair, subnormal quotients included), or
// the IEEE intrinsic when an operand is subnormal.  Only called with a != 0.
__device__ __forceinline__ double div_fix(double a, double b) {
  bool h = false;
  const double q = div_den<true>(a, make_den(b), h);
  return h ? div_x(a, b) : q;
}

// (max, min) of two non-negative non-NaN magnitudes, one compare.  Equal
// magnitudes have identical bits, so this matches relaxed_max / relaxed_min
// (lanes.py:102-114) exactly on this domain.
__device__ __forceinline__ void maxmin(double a, double b, double& big, double& small) {
  const bool p = a > b;
  big = p ? a : b;
  small = p ? b : a;
}

// Subnormal operands at the exponent-normalised sites of the streaming
// kernels: normalised exactly on a cold per-lane branch (1) or declined to
// the fix-up kernel (0, the default: config 4 measured 3.99 ms per 2^26
// lanes with 0.3 % of lanes fixed up, 4.70 ms with mode 1 and none).
#ifndef B2S_WIDE_SUB
#define B2S_WIDE_SUB 0
#endif
constexpr bool kWideSub = B2S_WIDE_SUB != 0;

// Bnd (bounded) sites.  The streaming kernels run the fast variant only on
// warps whose every lane has its nonzero input components within
// kWideSpread binades of each other, all normal, with a nonnegative scale
// shift (the real kernel's `wide_or_sub` / the complex kernel's `wide_lane`
// dispatch).  After scaling, every nonzero component then lies in
// [2^121, 2^1022): entry moduli, column norms, the pivot modulus and the
// cos / sin quotients of the entry phases are all >= 2^-902 and the
// numerators >= 2^119, so those sites can never leave the range of the
// inline sequences and carry no checks at all.  (Sites fed by rotated,
// possibly cancelled intermediates -- r12, r22, their phases, the triangle
// -- keep theirs.)  A zero denominator comes with a zero numerator; its
// hi word is lifted to the smallest normal so the quotient is an exact +0.
__device__ __forceinline__ double lift_zero(double b) { return mk_(max(hi_(b), 0x00100000u), lo_(b)); }

// a / b for 0 <= a <= b (up to rounding), b < 2^1022; an exact +0 for a == 0
// (the reference gives 0/b = +0, or NaN for b == 0, which every caller
// absorbs into +0 through relaxed_max / the hypot identity).
template <bool Fix, bool Bnd = false>
__device__ __forceinline__ double div_pos_f(double a, double b, bool& hard) {
  if (Bnd) return quot_f(a, lift_zero(b), rcp_f(lift_zero(b)));
  const bool z = !nz_(a);
  const double d = z ? 1.0 : b;
  double q = quot_f(a, d, rcp_f(d));
  const bool h = !z & !(resid_ok(hi_(a)) & normal_q(hi_(q)));
  if (Fix) { if (h) q = div_fix(a, b); } else hard |= h;
  return q;
}

// Same for b < 2^1023: denominators >= 2^1022 are prescaled by 1/4 with the
// numerator (exact, since a resid_ok numerator is >= 2^-967).
template <bool Fix, bool Bnd = false>
__device__ __forceinline__ double div_pos_big_f(double a, double b, bool& hard) {
  const double sc = hi_(b) >= 0x7FD00000u ? 0.25 : 1.0;
  const double a2 = mul(a, sc);
  if (Bnd) {
    const double d = lift_zero(mul(b, sc));
    return quot_f(a2, d, rcp_f(d));
  }
  const bool z = !nz_(a);
  const double d = z ? 1.0 : mul(b, sc);
  double q = quot_f(a2, d, rcp_f(d));
  const bool h = !z & !(resid_ok(hi_(a2)) & normal_q(hi_(q)));
  if (Fix) { if (h) q = div_fix(a, b); } else hard |= h;
  return q;
}

// Inside hypot the quotient only enters through fma(q, q, 1): for
// q < 2^-28, q^2 < 2^-56 rounds away and the result is big * sqrt(1) = big
// whatever q's last bits are.  So a hypot whose quotient is that small never
// needs the exact path, even when q itself would be subnormal.  (A garbage
// fast quotient -- subnormal denominator -- comes out NaN or inf, not
// small.)  Since q = small / big <= 1, a quotient that matters (>= 2^-28) is
// normal whenever the numerator passes resid_ok, so that is the whole check.
__device__ __forceinline__ bool hypot_q_irrelevant(double q) { return hi_(q) < 0x3E300000u; }  // q < 2^-28

// lanes.py:213-227 for non-negative magnitudes m1, m2 < 2^1022.
template <bool Fix, bool Bnd = false>
__device__ __forceinline__ double hypot_f(double m1, double m2, bool& hard) {
  double big, small;
  maxmin(m1, m2, big, small);
  if (Bnd) {
    const double q = div_pos_f<false, true>(small, big, hard);
    return mul(big, sqrt_f(fma_(q, q, 1.0)));
  }
  const bool z = !nz_(small);
  const double d = z ? 1.0 : big;                   // small / max(big, TRUE_MIN), 0/0 -> 0
  double q = quot_f(small, d, rcp_f(d));
  const bool h = !resid_ok(hi_(small)) & !hypot_q_irrelevant(q);
  if (Fix) { if (h) q = div_fix(small, rmax(big, kTrueMin())); } else hard |= h;
  return mul(big, sqrt_f(fma_(q, q, 1.0)));
}

// lanes.py:213-227 for magnitudes < 2^1023 (complex column norms and the
// r12 / r22 moduli, which reach 2^1022.5).
template <bool Fix, bool Bnd = false>
__device__ __forceinline__ double hypot_big_f(double m1, double m2, bool& hard) {
  double big, small;
  maxmin(m1, m2, big, small);
  double q;
  if (Bnd) {
    q = div_pos_big_f<false, true>(small, big, hard);
  } else {
    const bool z = !nz_(small);
    const double sc = hi_(big) >= 0x7FD00000u ? 0.25 : 1.0;
    const double a2 = mul(small, sc);
    const double d = z ? 1.0 : mul(big, sc);
    q = quot_f(a2, d, rcp_f(d));
    const bool h = !resid_ok(hi_(a2)) & !hypot_q_irrelevant(q);
    if (Fix) { if (h) q = div_fix(small, rmax(big, kTrueMin())); } else hard |= h;
  }
  return mul(big, sqrt_f(fma_(q, q, 1.0)));
}

// lanes.py:248-259 unit phase of re + i*im with mag = hypot(re, im) < 2^1023.
// mag == 0 exactly when re == im == 0: then cos = +-1 (0/0 absorbed by the
// relaxed min) and sin = im / TRUE_MIN = +-0.
// Wide-exponent variant: quotients may be subnormal, so both use the
// exponent-normalised division (exact for all normal operands).
template <bool Fix>
__device__ __forceinline__ void phase_w(double re, double im, double mag, double& c, double& s, bool& hard) {
  const bool mz = !nz_(mag);
  const Den D = make_den<Fix || kWideSub>(mag);
  bool hc = false, hs = false;
  const double q1 = div_den<false, Fix || kWideSub, !Fix>(fabs_(re), D, hc);
  const double q2 = div_den<false, Fix || kWideSub, !Fix>(im, D, hs);
  c = or_(mz ? 1.0 : rmin(q1, 1.0), sgn_(re));
  s = q2;
  if (Fix) {
    if (hc) c = or_(rmin(div_x(fabs_(re), mag), 1.0), sgn_(re));
    if (hs) s = div_x(im, rmax(mag, kTrueMin()));
  } else {
    hard |= hc | hs;
  }
}

// (d_out, r_out: the prescaled denominator and its reciprocal, for a caller
// dividing something else by the same mag.)
template <bool Fix, bool Bnd = false>
__device__ __forceinline__ void phase_f(double re, double im, double mag, double& c, double& s, bool& hard,
                                        double* d_out = nullptr, double* r_out = nullptr) {
  const bool mz = !nz_(mag);
  const double sc = hi_(mag) >= 0x7FD00000u ? 0.25 : 1.0;
  const double d = mz ? 1.0 : mul(mag, sc);
  const double r = rcp_f(d);
  if (d_out) { *d_out = d; *r_out = r; }
  // A zero part gives an exactly zero quotient (0 / mag); it is selected
  // directly so that a garbage reciprocal (subnormal mag, flagged through
  // the other part) can never leak through it.
  // The streaming kernel (Fix = false) skips those selects: a garbage
  // reciprocal only arises for a subnormal mag, whose nonzero part is itself
  // subnormal and flags the lane below; with a usable reciprocal a zero part
  // already gives an exact zero quotient (signed through the OR).
  const double a1 = mul(fabs_(re), sc);
  const double q1 = quot_f(a1, d, r);
  const double cm = rmin(q1, 1.0);
  c = or_(mz ? 1.0 : (Fix ? (nz_(re) ? cm : 0.0) : cm), sgn_(re));
  const double a2 = mul(im, sc);
  const double q2 = quot_f(a2, d, r);
  const double sq = mk_(lop_or(lop_and(hi_(q2), 0x7FFFFFFFu), lop_and(hi_(im), 0x80000000u)), lo_(q2));
  s = Fix ? (nz_(im) ? sq : im) : sq;
  if (Bnd) return;                                 // entry phases of a bounded warp: in range
  const bool hc = nz_(a1) & !(resid_ok(hi_(a1)) & normal_q(hi_(q1)));
  const bool hs = nz_(im) & !(resid_ok(lop_and(hi_(a2), 0x7FFFFFFFu)) & normal_q(lop_and(hi_(q2), 0x7FFFFFFFu)));
  if (Fix) {
    if (hc) c = or_(rmin(div_fix(fabs_(re), mag), 1.0), sgn_(re));
    if (hs) s = div_fix(im, rmax(mag, kTrueMin()));
  } else {
    hard |= hc | hs;
  }
}

// svd2.py:306-343.  r11 = 0 or r11 in [2^1021, 2^1022.5] (the norm of the
// pivot column, which holds the scaled maximum entry); 0 <= r12, r22 <= r11.
template <bool Fix, bool Wide = false, bool Lean = !Fix>
__device__ __forceinline__ Tri triangle_f(double r11, double r12, double r22, bool& hard) {
  double qx, qy;
  bool hx = false, hy = false;
  if (Wide) {
    // exponent-normalised, exact for tiny ratios too (r11 = 0 only with
    // r12 = r22 = 0, giving +0 like the reference's absorbed 0/0)
    const Den D = make_den<Fix || kWideSub>(r11);
    qx = div_den<false, Fix || kWideSub, !Fix>(r12, D, hx);
    qy = div_den<false, Fix || kWideSub, !Fix>(r22, D, hy);
  } else {
    // one shared reciprocal of r11 / 4 (r11 = 0 gives NaN quotients,
    // absorbed to +0 exactly as the reference's 0/0 is)
    const double b = mul(r11, 0.25);
    const double r = rcp_f(b);
    const double a12 = mul(r12, 0.25), a22 = mul(r22, 0.25);
    qx = quot_f(a12, b, r);
    qy = quot_f(a22, b, r);
    hx = nz_(r12) & !(resid_ok(hi_(a12)) & normal_q(hi_(qx)));
    hy = nz_(r22) & !(resid_ok(hi_(a22)) & normal_q(hi_(qy)));
  }
  if (Fix) {
    if (hx) qx = div_fix(r12, r11);
    if (hy) qy = div_fix(r22, r11);
  } else {
    hard |= hx | hy;
  }
  // relaxed_max(q, 0) (svd2.py:324-325): q >= +0 whenever r11 > 0, which
  // holds on every lane the streaming kernel keeps (a zero matrix is flagged
  // hard by scale_f); r11 = 0 (0 / 0) only reaches the exact re-evaluation.
  const double x = Lean ? qx : rmax(qx, 0.0), y = Lean ? qy : rmax(qy, 0.0);
  double hi, lo;
  maxmin(x, y, hi, lo);
  const double num = mul(mul(lo, 2.0), hi);                  // scalef(min, 1) * max
  const double den = fma_(sub(x, y), add(x, y), 1.0);         // in [0, 2]
  // num / den: num == 0 gives +0 or NaN (den == 0), both absorbed to +0.
  double qn;
  bool hn = false;
  if (Wide) {
    qn = div_den<true, Fix || kWideSub, !Fix>(num, make_den<Fix || kWideSub>(den), hn);
  } else {
    qn = quot_f(num, den, rcp_f(den));
    hn = nz_(num) & !(resid_ok(hi_(num)) & normal_q(hi_(qn)));
  }
  if (Fix) { if (hn) qn = div_fix(num, den); } else hard |= hn;
  const double tan2 = or_(rmin(rmax(qn, 0.0), kSqrtDblMax()), kNegZero());
  // tan2 in [-sqrt(DBL_MAX), -0]; the denominator is in [2, 2^512].
  const double den2 = add(1.0, sqrt_f(fma_(tan2, tan2, 1.0)));
  double lt;
  bool hl = false;
  if (Wide) {
    lt = div_den<false, Fix || kWideSub, !Fix>(tan2, make_den<Fix || kWideSub>(den2), hl);
  } else {
    const double ql = quot_f(tan2, den2, rcp_f(den2));
    lt = mk_(lop_or(hi_(ql), 0x80000000u), lo_(ql));   // sign of -0 / den2
    hl = nz_(tan2) & !(resid_ok(lop_and(hi_(tan2), 0x7FFFFFFFu)) &
                        normal_q(lop_and(hi_(ql), 0x7FFFFFFFu)));
  }
  if (Fix) { if (hl) lt = div_fix(tan2, den2); } else hard |= hl;
  const double ls2 = fma_(lt, lt, 1.0);
  const double rt = fma_(y, lt, -x);
  return triangle_tail(x, y, lt, r11, r22, invsqrt_f(ls2), invsqrt_f(fma_(rt, rt, 1.0)));
}

// ---------------------------------------------------------------------------
// Real lanes.  Scaled entries are < 2^1022 in magnitude, so every column
// norm is < 2^1022.5 and the pivot magnitude m11 (>= n1 / sqrt 2) lies in
// [2^1020.5, 2^1022) unless the matrix is zero.
// ---------------------------------------------------------------------------
#ifndef B2S_REAL_LEAN
#define B2S_REAL_LEAN 1   // bench (power-capped): +1.2 % (43.9 vs 43.3 G SVD/s); cold 2^26: -0.5 %
#endif
template <bool Sine, bool Fix, bool Wide = false, bool Bnd = false>
__device__ __forceinline__ bool svd2_real_f(const double (&a)[4], RealOut& o) {
  bool hard = false;
  double e[4] = {a[0], a[1], a[2], a[3]};
  double shift = scale_f<4>(e, hard);
  if (Fix && hard) {
    e[0] = a[0]; e[1] = a[1]; e[2] = a[2]; e[3] = a[3];
    shift = scale_x<4>(e);
  }
  double m11 = fabs_(e[0]), m21 = fabs_(e[1]), m12 = fabs_(e[2]), m22 = fabs_(e[3]);
  double n1 = hypot_f<Fix, Bnd>(m11, m21, hard), n2 = hypot_f<Fix, Bnd>(m12, m22, hard);
  RealUrv U;
  U.C = n1 < n2;
  swp(U.C, e[0], e[2]); swp(U.C, e[1], e[3]);
  swp(U.C, m11, m12); swp(U.C, m21, m22);
  const double r11 = U.C ? n2 : n1;
  U.R = m11 < m21;
  swp(U.R, e[0], e[1]); swp(U.R, e[2], e[3]);
  swp(U.R, m11, m21);
  U.ph1 = sgn_(e[0]);
  U.ph2 = sgn_(e[1]);
  const double f12 = xor_(e[2], U.ph1), f22 = xor_(e[3], U.ph2);
  if (Wide) {
    bool h = false;
    U.mt = div_den<false, Fix || kWideSub, !Fix>(m21, make_den<Fix || kWideSub>(m11), h);   // relaxed_max(., 0) is the identity here
    if (Fix) { if (h) U.mt = div_fix(m21, m11); } else hard |= h;
  } else {
    U.mt = div_pos_f<Fix, Bnd>(m21, m11, hard);       // relaxed_max(., 0) is the identity here
  }
  U.cg = invsqrt_f(fma_(U.mt, U.mt, 1.0));
  const double g12 = mul(U.cg, fma_(U.mt, f22, f12));
  const double g22 = mul(U.cg, fnma_(U.mt, f12, f22));
  U.dt = sgn_(g12);
  const double w = xor_(g22, U.dt);
  U.dh = sgn_(w);
  const Tri T = triangle_f<Fix, Wide, B2S_REAL_LEAN && !Fix>(r11, fabs_(g12), fabs_(w), hard);
  assemble_real<Sine>(U, T, o);
  o.shift = shift;
  return hard;
}

// A lane whose nonzero components span more than kWideSpread binades can
// produce quotients below the normal range at the phase / rotation /
// triangle sites; a warp holding any such lane runs the exponent-normalised
// variant of those sites (warp-uniform, so no divergence).  The flag is only
// a cost heuristic: either variant is exact wherever it does not set `hard`.
constexpr int kWideSpread = 900;

template <int N>
__device__ __forceinline__ bool wide_lane(const double (&p)[N]) {
  int emax = 0, emin = 0x7FF;
  #pragma unroll
  for (int i = 0; i < N; i++) {
    const int e = (int)((hi_(p[i]) >> 20) & 0x7FFu);
    emax = max(emax, e);
    emin = min(emin, nz_(p[i]) ? e : 0x7FF);
  }
  return emax - emin > kWideSpread;
}

// Real lanes the fast pipeline may decline: components spanning more than
// kWideSpread binades (tiny quotients), a subnormal component, or a
// component within 2 binades of DBL_MAX (negative scale shift).
template <int N>
__device__ __forceinline__ bool wide_or_sub(const double (&p)[N]) {
  int emax = 0, emin = 0x7FF;
  #pragma unroll
  for (int i = 0; i < N; i++) {
    const int e = (int)((hi_(p[i]) >> 20) & 0x7FFu);
    emax = max(emax, e);
    emin = min(emin, nz_(p[i]) ? e : 0x7FF);
  }
  return (emax - emin > kWideSpread) | (emin == 0) | (emax >= 2045);
}

// ---------------------------------------------------------------------------
// Complex lanes.  Scaled components are < 2^1022, so entry moduli are
// < 2^1022.5; column norms, m11 and the rotated moduli r12, r22 stay below
// 2^1023 and use the prescaling variants.
// ---------------------------------------------------------------------------
template <bool Sine, bool Fix, bool Wide = false, bool Bnd = false>
__device__ __forceinline__ bool svd2_complex_f(const double (&ar)[4], const double (&ai)[4], CplxOut& o) {
  bool hard = false;
  double p[8] = {ar[0], ai[0], ar[1], ai[1], ar[2], ai[2], ar[3], ai[3]};
  double shift = scale_f<8>(p, hard);
  if (Fix && hard) {
    #pragma unroll
    for (int t = 0; t < 4; t++) { p[2 * t] = ar[t]; p[2 * t + 1] = ai[t]; }
    shift = scale_x<8>(p);
  }
  double er[4] = {p[0], p[2], p[4], p[6]}, ei[4] = {p[1], p[3], p[5], p[7]};
  double m11 = hypot_f<Fix, Bnd>(fabs_(er[0]), fabs_(ei[0]), hard);
  double m21 = hypot_f<Fix, Bnd>(fabs_(er[1]), fabs_(ei[1]), hard);
  double m12 = hypot_f<Fix, Bnd>(fabs_(er[2]), fabs_(ei[2]), hard);
  double m22 = hypot_f<Fix, Bnd>(fabs_(er[3]), fabs_(ei[3]), hard);
  double n1 = hypot_big_f<Fix, Bnd>(m11, m21, hard), n2 = hypot_big_f<Fix, Bnd>(m12, m22, hard);
  CplxUrv U;
  double d11 = 1.0, r11p = 1.0;             // e11's phase denominator m11 * sc and its reciprocal
  U.C = n1 < n2;
  swp(U.C, er[0], er[2]); swp(U.C, ei[0], ei[2]);
  swp(U.C, er[1], er[3]); swp(U.C, ei[1], ei[3]);
  swp(U.C, m11, m12); swp(U.C, m21, m22);
  const double r11 = U.C ? n2 : n1;
  U.R = m11 < m21;
  swp(U.R, er[0], er[1]); swp(U.R, ei[0], ei[1]);
  swp(U.R, er[2], er[3]); swp(U.R, ei[2], ei[3]);
  swp(U.R, m11, m21);
  if (Wide) {
    phase_w<Fix>(er[0], ei[0], m11, U.c1, U.s1, hard);
    phase_w<Fix>(er[1], ei[1], m21, U.c2, U.s2, hard);
  } else {
    phase_f<Fix, Bnd>(er[0], ei[0], m11, U.c1, U.s1, hard, &d11, &r11p);
    phase_f<Fix, Bnd>(er[1], ei[1], m21, U.c2, U.s2, hard);
  }
  double f12r, f12i, f22r, f22i;
  cmul(U.c1, neg_(U.s1), er[2], ei[2], f12r, f12i);
  cmul(U.c2, neg_(U.s2), er[3], ei[3], f22r, f22i);
  if (Wide) {
    bool h = false;
    U.mt = div_den<false, Fix || kWideSub, !Fix>(m21, make_den<Fix || kWideSub>(m11), h);   // m21 >= 0: relaxed_max is the identity
    if (Fix) { if (h) U.mt = div_fix(m21, m11); } else hard |= h;
  } else if (!Fix) {
    // m21 / m11 with the reciprocal e11's phase formed: on every lane the
    // streaming kernel keeps (m11 > 0) its denominator is m11 * sc, exactly
    // div_pos_big_f's.  m21 <= m11, so the quotient is <= 1.
    const double a2 = mul(m21, hi_(m11) >= 0x7FD00000u ? 0.25 : 1.0);
    U.mt = quot_f(a2, d11, r11p);
    if (!Bnd) hard |= nz_(m21) & !(resid_ok(hi_(a2)) & normal_q(hi_(U.mt)));
  } else {
    U.mt = div_pos_big_f<Fix, Bnd>(m21, m11, hard);
  }
  U.cg = invsqrt_f(fma_(U.mt, U.mt, 1.0));
  const double g12r = mul(U.cg, fma_(U.mt, f22r, f12r)), g12i = mul(U.cg, fma_(U.mt, f22i, f12i));
  const double g22r = mul(U.cg, fnma_(U.mt, f12r, f22r)), g22i = mul(U.cg, fnma_(U.mt, f12i, f22i));
  const double r12 = hypot_big_f<Fix>(fabs_(g12r), fabs_(g12i), hard);
  double c12, s12;
  if (Wide) phase_w<Fix>(g12r, g12i, r12, c12, s12, hard);
  else phase_f<Fix>(g12r, g12i, r12, c12, s12, hard);
  double wr, wi;
  cmul(c12, neg_(s12), g22r, g22i, wr, wi);
  const double r22 = hypot_big_f<Fix>(fabs_(wr), fabs_(wi), hard);
  if (Wide) phase_w<Fix>(wr, wi, r22, U.dhr, U.dhi, hard);
  else phase_f<Fix>(wr, wi, r22, U.dhr, U.dhi, hard);
  U.dtr = c12;
  U.dti = neg_(s12);
  const Tri T = triangle_f<Fix, Wide>(r11, r12, r22, hard);
  assemble_complex<Sine>(U, T, o);
  o.shift = shift;
  return hard;
}

// The same streaming pipeline as svd2_complex_f<Sine, false, Wide, !Wide>
// with the wide / bounded choice made at run time: `w` must be warp-uniform.
// Every phase the two variants share is compiled once and only the division
// sites branch (five warp-uniform branches), so warps of both kinds run one
// code body -- what a kernel mixing wide and narrow warps on one SM needs
// to keep its instructions in cache (B2S_CPLX_SORT4 variant).
template <bool Sine>
__device__ __forceinline__ bool svd2_complex_u(const double (&ar)[4], const double (&ai)[4], CplxOut& o,
                                               const bool w) {
  bool hard = false;
  double p[8] = {ar[0], ai[0], ar[1], ai[1], ar[2], ai[2], ar[3], ai[3]};
  const double shift = scale_f<8>(p, hard);
  double er[4] = {p[0], p[2], p[4], p[6]}, ei[4] = {p[1], p[3], p[5], p[7]};
  double m11, m21, m12, m22, n1, n2;
  if (w) {
    m11 = hypot_f<false, false>(fabs_(er[0]), fabs_(ei[0]), hard);
    m21 = hypot_f<false, false>(fabs_(er[1]), fabs_(ei[1]), hard);
    m12 = hypot_f<false, false>(fabs_(er[2]), fabs_(ei[2]), hard);
    m22 = hypot_f<false, false>(fabs_(er[3]), fabs_(ei[3]), hard);
    n1 = hypot_big_f<false, false>(m11, m21, hard);
    n2 = hypot_big_f<false, false>(m12, m22, hard);
  } else {
    m11 = hypot_f<false, true>(fabs_(er[0]), fabs_(ei[0]), hard);
    m21 = hypot_f<false, true>(fabs_(er[1]), fabs_(ei[1]), hard);
    m12 = hypot_f<false, true>(fabs_(er[2]), fabs_(ei[2]), hard);
    m22 = hypot_f<false, true>(fabs_(er[3]), fabs_(ei[3]), hard);
    n1 = hypot_big_f<false, true>(m11, m21, hard);
    n2 = hypot_big_f<false, true>(m12, m22, hard);
  }
  CplxUrv U;
  U.C = n1 < n2;
  swp(U.C, er[0], er[2]); swp(U.C, ei[0], ei[2]);
  swp(U.C, er[1], er[3]); swp(U.C, ei[1], ei[3]);
  swp(U.C, m11, m12); swp(U.C, m21, m22);
  const double r11 = U.C ? n2 : n1;
  U.R = m11 < m21;
  swp(U.R, er[0], er[1]); swp(U.R, ei[0], ei[1]);
  swp(U.R, er[2], er[3]); swp(U.R, ei[2], ei[3]);
  swp(U.R, m11, m21);
  if (w) {
    phase_w<false>(er[0], ei[0], m11, U.c1, U.s1, hard);
    phase_w<false>(er[1], ei[1], m21, U.c2, U.s2, hard);
    bool h = false;
    U.mt = div_den<false, kWideSub, true>(m21, make_den<kWideSub>(m11), h);
    hard |= h;
  } else {
    double d11 = 1.0, r11p = 1.0;
    phase_f<false, true>(er[0], ei[0], m11, U.c1, U.s1, hard, &d11, &r11p);
    phase_f<false, true>(er[1], ei[1], m21, U.c2, U.s2, hard);
    const double a2 = mul(m21, hi_(m11) >= 0x7FD00000u ? 0.25 : 1.0);
    U.mt = quot_f(a2, d11, r11p);
  }
  double f12r, f12i, f22r, f22i;
  cmul(U.c1, neg_(U.s1), er[2], ei[2], f12r, f12i);
  cmul(U.c2, neg_(U.s2), er[3], ei[3], f22r, f22i);
  U.cg = invsqrt_f(fma_(U.mt, U.mt, 1.0));
  const double g12r = mul(U.cg, fma_(U.mt, f22r, f12r)), g12i = mul(U.cg, fma_(U.mt, f22i, f12i));
  const double g22r = mul(U.cg, fnma_(U.mt, f12r, f22r)), g22i = mul(U.cg, fnma_(U.mt, f12i, f22i));
  const double r12 = hypot_big_f<false>(fabs_(g12r), fabs_(g12i), hard);
  double c12, s12;
  if (w) phase_w<false>(g12r, g12i, r12, c12, s12, hard);
  else phase_f<false>(g12r, g12i, r12, c12, s12, hard);
  double wr, wi;
  cmul(c12, neg_(s12), g22r, g22i, wr, wi);
  const double r22 = hypot_big_f<false>(fabs_(wr), fabs_(wi), hard);
  if (w) phase_w<false>(wr, wi, r22, U.dhr, U.dhi, hard);
  else phase_f<false>(wr, wi, r22, U.dhr, U.dhi, hard);
  U.dtr = c12;
  U.dti = neg_(s12);
  const Tri T = w ? triangle_f<false, true>(r11, r12, r22, hard) : triangle_f<false, false>(r11, r12, r22, hard);
  assemble_complex<Sine>(U, T, o);
  o.shift = shift;
  return hard;
}

}  // namespace b2s
