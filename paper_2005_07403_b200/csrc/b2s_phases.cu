// b2s_phases.cu -- the reference's pipeline phases as separate device
// entry points (`b2s_svd2_phase`): compute_scale, column_norms,
// column_pivot, row_sort, left_phase_reduce, givens_qr, phase_fix_r,
// triangular_svd and assemble_uv / assemble_uv_sine (svd2.py:134-474).
//
// The batch kernels fuse all phases in registers; these entry points expose
// each phase on its own, for callers of the reference's svd2 module API and
// for per-phase parity checks.  Each lane runs the exact (IEEE-intrinsic)
// arithmetic of the state-dump kernel (b2s_svd2.cuh), so a phase's outputs
// are bit-identical to the reference's for every finite input, whether or
// not the inputs came from the previous phase.
//
// `b2s_lane_op` does the same for the lane primitives of lanes.py:69-259
// (fma, relaxed min/max, select, getexp, scalef, sign algebra, hypot_lane,
// invsqrt_lane, complex_mul, phase_from_parts, polar).
//
// Train layout: K = 1 (real) or 2 (complex, re then im) trains per value;
// "entries" are e11, e21, e12, e22 in that order (4K trains).  Masks travel
// as 0.0 / 1.0 (any nonzero input is true).
#include "../../include/b2s.h"
#include "b2s_common.cuh"
#include "b2s_svd2.cuh"

namespace b2s {

struct PhaseArgs {
  int op, cplx, sine;
  int64_t n;
  const double* in[B2S_PHASE_MAX_TRAINS];
  double* out[B2S_PHASE_MAX_TRAINS];
};

// Number of input / output trains of each phase (K = 1 real, 2 complex).
__host__ __device__ inline void phase_arity(int op, int K, int* nin, int* nout) {
  switch (op) {
    case B2S_PHASE_COMPUTE_SCALE: *nin = 4 * K; *nout = 1 + 4 * K; break;
    case B2S_PHASE_COLUMN_NORMS: *nin = 4 * K; *nout = 6; break;
    case B2S_PHASE_COLUMN_PIVOT: *nin = 4 * K + 6; *nout = 4 * K + 7; break;
    case B2S_PHASE_ROW_SORT: *nin = 4 * K + 4; *nout = 4 * K + 5; break;
    case B2S_PHASE_LEFT_PHASE_REDUCE: *nin = 4 * K + 2; *nout = 2 + 4 * K; break;
    case B2S_PHASE_GIVENS_QR: *nin = 3 + 2 * K; *nout = 3 + 2 * K; break;
    case B2S_PHASE_PHASE_FIX_R: *nin = 2 * K; *nout = 2 + 2 * K; break;
    case B2S_PHASE_TRIANGULAR_SVD: *nin = 3; *nout = 8; break;
    case B2S_PHASE_ASSEMBLE_UV: *nin = 2 + 4 * K + 2 + 3 + 8 + 1; *nout = 8 * K + 3; break;
    default: *nin = *nout = -1;
  }
}

template <int K>
__device__ __forceinline__ void phase_lane(const PhaseArgs& A, int64_t i) {
  const double* const* in = A.in;
  double* const* out = A.out;
  auto I = [&](int k) { return in[k][i]; };
  auto O = [&](int k, double v) { out[k][i] = v; };
  switch (A.op) {
    case B2S_PHASE_COMPUTE_SCALE: {                          // svd2.py:134-160
      double p[4 * K];
      #pragma unroll
      for (int t = 0; t < 4 * K; t++) p[t] = I(t);
      O(0, scale_x<4 * K>(p));
      #pragma unroll
      for (int t = 0; t < 4 * K; t++) O(1 + t, p[t]);
    } break;
    case B2S_PHASE_COLUMN_NORMS: {                           // svd2.py:167-182
      double m[4];
      #pragma unroll
      for (int e = 0; e < 4; e++) m[e] = K == 1 ? fabs_(I(e)) : hypot_x(I(2 * e), I(2 * e + 1));
      #pragma unroll
      for (int e = 0; e < 4; e++) O(e, m[e]);
      O(4, hypot_x(m[0], m[1]));
      O(5, hypot_x(m[2], m[3]));
    } break;
    case B2S_PHASE_COLUMN_PIVOT: {                           // svd2.py:193-208
      double e[4][K], m[4];
      #pragma unroll
      for (int j = 0; j < 4; j++) {
        #pragma unroll
        for (int c = 0; c < K; c++) e[j][c] = I(K * j + c);
        m[j] = I(4 * K + j);
      }
      double n1 = I(4 * K + 4), n2 = I(4 * K + 5);
      const bool sw = n1 < n2;
      #pragma unroll
      for (int c = 0; c < K; c++) { swp(sw, e[0][c], e[2][c]); swp(sw, e[1][c], e[3][c]); }
      swp(sw, m[0], m[2]); swp(sw, m[1], m[3]); swp(sw, n1, n2);
      #pragma unroll
      for (int j = 0; j < 4; j++) {
        #pragma unroll
        for (int c = 0; c < K; c++) O(K * j + c, e[j][c]);
        O(4 * K + j, m[j]);
      }
      O(4 * K + 4, n1); O(4 * K + 5, n2); O(4 * K + 6, sw ? 1.0 : 0.0);
    } break;
    case B2S_PHASE_ROW_SORT: {                               // svd2.py:211-224
      double e[4][K], m[4];
      #pragma unroll
      for (int j = 0; j < 4; j++) {
        #pragma unroll
        for (int c = 0; c < K; c++) e[j][c] = I(K * j + c);
        m[j] = I(4 * K + j);
      }
      const bool sw = m[0] < m[1];
      #pragma unroll
      for (int c = 0; c < K; c++) { swp(sw, e[0][c], e[1][c]); swp(sw, e[2][c], e[3][c]); }
      swp(sw, m[0], m[1]); swp(sw, m[2], m[3]);
      #pragma unroll
      for (int j = 0; j < 4; j++) {
        #pragma unroll
        for (int c = 0; c < K; c++) O(K * j + c, e[j][c]);
        O(4 * K + j, m[j]);
      }
      O(4 * K + 4, sw ? 1.0 : 0.0);
    } break;
    case B2S_PHASE_LEFT_PHASE_REDUCE: {                      // svd2.py:227-250
      const double m11 = I(4 * K), m21 = I(4 * K + 1);
      O(0, m11);
      O(1, m21);
      if (K == 1) {
        const double ph1 = sgn_(I(0)), ph2 = sgn_(I(1));
        O(2, xor_(I(2), ph1)); O(3, xor_(I(3), ph2)); O(4, ph1); O(5, ph2);
      } else {
        double c1, s1, c2, s2, fr, fi;
        phase_x(I(0), I(1), m11, c1, s1);
        phase_x(I(2), I(3), m21, c2, s2);
        cmul(c1, neg_(s1), I(4), I(5), fr, fi); O(2, fr); O(3, fi);
        cmul(c2, neg_(s2), I(6), I(7), fr, fi); O(4, fr); O(5, fi);
        O(6, c1); O(7, s1); O(8, c2); O(9, s2);
      }
    } break;
    case B2S_PHASE_GIVENS_QR: {                              // svd2.py:253-276
      const double mt = rmax(div_x(I(1), I(0)), 0.0);
      const double cg = invsqrt_x(fma_(mt, mt, 1.0));
      O(0, neg_(mt)); O(1, cg); O(2, I(2 + 2 * K));
      #pragma unroll
      for (int c = 0; c < K; c++) {
        const double f12 = I(2 + c), f22 = I(2 + K + c);
        O(3 + c, mul(cg, fma_(mt, f22, f12)));
        O(3 + K + c, mul(cg, fnma_(mt, f12, f22)));
      }
    } break;
    case B2S_PHASE_PHASE_FIX_R: {                            // svd2.py:279-299
      if (K == 1) {
        const double dt = sgn_(I(0)), w = xor_(I(1), dt);
        O(0, fabs_(I(0))); O(1, fabs_(w)); O(2, dt); O(3, sgn_(w));
      } else {
        const double g12r = I(0), g12i = I(1), g22r = I(2), g22i = I(3);
        const double r12 = hypot_x(g12r, g12i);
        double c12, s12, wr, wi, c22, s22;
        phase_x(g12r, g12i, r12, c12, s12);
        cmul(c12, neg_(s12), g22r, g22i, wr, wi);
        const double r22 = hypot_x(wr, wi);
        phase_x(wr, wi, r22, c22, s22);
        O(0, r12); O(1, r22); O(2, c12); O(3, neg_(s12)); O(4, c22); O(5, s22);
      }
    } break;
    case B2S_PHASE_TRIANGULAR_SVD: {                         // svd2.py:306-343
      const Tri T = triangle_x(I(0), I(1), I(2));
      O(0, T.l_tan); O(1, T.l_sec2); O(2, T.l_cos); O(3, T.r_tan);
      O(4, T.r_sec2); O(5, T.r_cos); O(6, T.smax); O(7, T.smin);
    } break;
    case B2S_PHASE_ASSEMBLE_UV: {                            // svd2.py:350-474
      // in: swap_cols, swap_rows, row_phase1 (K), row_phase2 (K), givens_tan,
      //     givens_cos, r12_phase (K), r22_phase (K), r11, r12, r22,
      //     the 8 TriangleSvd trains, shift
      int k = 0;
      const bool C = I(k++) != 0.0, R = I(k++) != 0.0;
      double ph1[K], ph2[K], dt[K], dh[K];
      #pragma unroll
      for (int c = 0; c < K; c++) ph1[c] = I(k++);
      #pragma unroll
      for (int c = 0; c < K; c++) ph2[c] = I(k++);
      const double gt = I(k++), cg = I(k++);
      #pragma unroll
      for (int c = 0; c < K; c++) dt[c] = I(k++);
      #pragma unroll
      for (int c = 0; c < K; c++) dh[c] = I(k++);
      k += 3;                                                  // r11, r12, r22: not used by the assembly
      Tri T;
      T.l_tan = I(k++); T.l_sec2 = I(k++); T.l_cos = I(k++); T.r_tan = I(k++);
      T.r_sec2 = I(k++); T.r_cos = I(k++); T.smax = I(k++); T.smin = I(k++);
      const double shift = I(k++);
      if (K == 1) {
        RealUrv U;
        U.C = C; U.R = R; U.ph1 = ph1[0]; U.ph2 = ph2[0]; U.mt = neg_(gt); U.cg = cg;
        U.dt = dt[0]; U.dh = dh[0];
        RealOut o;
        if (A.sine) assemble_real<true>(U, T, o); else assemble_real<false>(U, T, o);
        for (int t = 0; t < 4; t++) { O(t, o.u[t]); O(4 + t, o.v[t]); }
        O(8, o.smax); O(9, o.smin); O(10, shift);
      } else {
        CplxUrv U;
        U.C = C; U.R = R; U.c1 = ph1[0]; U.s1 = ph1[K - 1]; U.c2 = ph2[0]; U.s2 = ph2[K - 1];
        U.mt = neg_(gt); U.cg = cg; U.dtr = dt[0]; U.dti = dt[K - 1]; U.dhr = dh[0]; U.dhi = dh[K - 1];
        CplxOut o;
        if (A.sine) assemble_complex<true>(U, T, o); else assemble_complex<false>(U, T, o);
        for (int t = 0; t < 4; t++) {
          O(2 * t, o.ur[t]); O(2 * t + 1, o.ui[t]);
          O(8 + 2 * t, o.vr[t]); O(8 + 2 * t + 1, o.vi[t]);
        }
        O(16, o.smax); O(17, o.smin); O(18, shift);
      }
    } break;
    default: break;
  }
}

// ---------------------------------------------------------------------------
// The lane primitives of lanes.py:69-259 as elementwise device ops
// (b2s_lane_op): the same device functions every kernel is built from, with
// the reference semantics for every input (NaN payload bits aside).
// ---------------------------------------------------------------------------
__device__ __forceinline__ double getexp_lane(double a) {       // lanes.py:126-140
  if (isnan(a)) return a;
  if (isinf(a)) return __longlong_as_double(0x7FF0000000000000ll);
  if (a == 0.0) return __longlong_as_double((long long)0xFFF0000000000000ull);
  return (double)ilogb_finite(a);
}

__device__ __forceinline__ double scalef_lane(double a, double e) {   // lanes.py:143-159
  const double ef = floor(e);
  if (!isfinite(ef)) return __dmul_rn(a, exp2(ef));            // 2^+-inf = inf / 0, NaN stays NaN
  const double sh = fmin(fmax(ef, -4500.0), 4500.0);
  return scalbn(a, (int)sh);                                     // one rounding, as ldexp
}

__device__ __forceinline__ double bits_op(double a, double b, int op) {
  const unsigned long long x = __double_as_longlong(a), y = __double_as_longlong(b);
  unsigned long long r;
  switch (op) {
    case B2S_LANE_BIT_AND: r = x & y; break;
    case B2S_LANE_BIT_OR: r = x | y; break;
    case B2S_LANE_BIT_XOR: r = x ^ y; break;
    default: r = ~x & y; break;                                  // bit_andnot
  }
  return __longlong_as_double((long long)r);
}

__host__ __device__ inline void lane_arity(int op, int* nin, int* nout) {
  switch (op) {
    case B2S_LANE_FMA: case B2S_LANE_FNMA: case B2S_LANE_SELECT: *nin = 3; *nout = 1; break;
    case B2S_LANE_RELAXED_MIN: case B2S_LANE_RELAXED_MAX: case B2S_LANE_SCALEF: case B2S_LANE_HYPOT:
    case B2S_LANE_BIT_AND: case B2S_LANE_BIT_OR: case B2S_LANE_BIT_XOR: case B2S_LANE_BIT_ANDNOT:
      *nin = 2; *nout = 1; break;
    case B2S_LANE_GETEXP: case B2S_LANE_INVSQRT: case B2S_LANE_FABS: case B2S_LANE_NEGATE:
    case B2S_LANE_SIGN_MASK: *nin = 1; *nout = 1; break;
    case B2S_LANE_COMPLEX_MUL: *nin = 4; *nout = 2; break;
    case B2S_LANE_PHASE_FROM_PARTS: *nin = 3; *nout = 2; break;
    case B2S_LANE_POLAR: *nin = 2; *nout = 3; break;
    default: *nin = *nout = -1;
  }
}

__global__ void __launch_bounds__(128) k_lane_op(const PhaseArgs A) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < A.n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double* const* in = A.in;
    double* const* out = A.out;
    auto I = [&](int k) { return in[k][i]; };
    switch (A.op) {
      case B2S_LANE_FMA: out[0][i] = fma_(I(0), I(1), I(2)); break;
      case B2S_LANE_FNMA: out[0][i] = fnma_(I(0), I(1), I(2)); break;
      case B2S_LANE_RELAXED_MIN: out[0][i] = rmin(I(0), I(1)); break;
      case B2S_LANE_RELAXED_MAX: out[0][i] = rmax(I(0), I(1)); break;
      case B2S_LANE_SELECT: out[0][i] = sel(I(0) != 0.0, I(1), I(2)); break;
      case B2S_LANE_GETEXP: out[0][i] = getexp_lane(I(0)); break;
      case B2S_LANE_SCALEF: out[0][i] = scalef_lane(I(0), I(1)); break;
      case B2S_LANE_HYPOT: out[0][i] = hypot_x(I(0), I(1)); break;
      case B2S_LANE_INVSQRT: out[0][i] = invsqrt_x(I(0)); break;
      case B2S_LANE_BIT_AND: case B2S_LANE_BIT_OR: case B2S_LANE_BIT_XOR: case B2S_LANE_BIT_ANDNOT:
        out[0][i] = bits_op(I(0), I(1), A.op); break;
      case B2S_LANE_FABS: out[0][i] = fabs_(I(0)); break;
      case B2S_LANE_NEGATE: out[0][i] = neg_(I(0)); break;
      case B2S_LANE_SIGN_MASK: out[0][i] = sgn_(I(0)); break;
      case B2S_LANE_COMPLEX_MUL: {
        double re, im;
        cmul(I(0), I(1), I(2), I(3), re, im);
        out[0][i] = re; out[1][i] = im;
      } break;
      case B2S_LANE_PHASE_FROM_PARTS: {
        double c, s;
        phase_x(I(0), I(1), I(2), c, s);
        out[0][i] = c; out[1][i] = s;
      } break;
      case B2S_LANE_POLAR: {
        const double mag = hypot_x(I(0), I(1));
        double c, s;
        phase_x(I(0), I(1), mag, c, s);
        out[0][i] = mag; out[1][i] = c; out[2][i] = s;
      } break;
      default: break;
    }
  }
}

template <int K>
__global__ void __launch_bounds__(128) k_phase(const PhaseArgs A) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < A.n; i += (int64_t)gridDim.x * blockDim.x)
    phase_lane<K>(A, i);
}

}  // namespace b2s

using namespace b2s;

extern "C" int b2s_svd2_phase(int op, int complex_field, int sine_form, int64_t n, int n_in,
                              const double* const* in, int n_out, double* const* out, void* stream) {
  if (n < 0) return fail(1, "negative batch size");
  const int K = complex_field ? 2 : 1;
  int want_in = 0, want_out = 0;
  phase_arity(op, K, &want_in, &want_out);
  if (want_in < 0) return fail(2, "unknown phase %d", op);
  if (n_in != want_in || n_out != want_out)
    return fail(2, "phase %d (%s) takes %d input and %d output trains, got %d and %d", op,
                complex_field ? "complex" : "real", want_in, want_out, n_in, n_out);
  if (!in || !out) return fail(5, "NULL train array");
  PhaseArgs A{};
  A.op = op;
  A.cplx = complex_field != 0;
  A.sine = sine_form != 0;
  A.n = n;
  for (int k = 0; k < n_in; k++) {
    if (!in[k]) return fail(5, "NULL input train %d", k);
    A.in[k] = in[k];
  }
  for (int k = 0; k < n_out; k++) {
    if (!out[k]) return fail(5, "NULL output train %d", k);
    A.out[k] = out[k];
  }
  if (n == 0) return 0;
  int blocks = (int)((n + 127) / 128);
  if (blocks > 148 * 16) blocks = 148 * 16;
  if (K == 1)
    k_phase<1><<<blocks, 128, 0, (cudaStream_t)stream>>>(A);
  else
    k_phase<2><<<blocks, 128, 0, (cudaStream_t)stream>>>(A);
  B2S_CUDA(cudaGetLastError());
  return 0;
}

extern "C" int b2s_lane_op(int op, int64_t n, int n_in, const double* const* in, int n_out, double* const* out,
                           void* stream) {
  if (n < 0) return fail(1, "negative batch size");
  int want_in = 0, want_out = 0;
  lane_arity(op, &want_in, &want_out);
  if (want_in < 0) return fail(2, "unknown lane op %d", op);
  if (n_in != want_in || n_out != want_out)
    return fail(2, "lane op %d takes %d input and %d output trains, got %d and %d", op, want_in, want_out, n_in,
                n_out);
  if (!in || !out) return fail(5, "NULL train array");
  PhaseArgs A{};
  A.op = op;
  A.n = n;
  for (int k = 0; k < n_in; k++) {
    if (!in[k]) return fail(5, "NULL input train %d", k);
    A.in[k] = in[k];
  }
  for (int k = 0; k < n_out; k++) {
    if (!out[k]) return fail(5, "NULL output train %d", k);
    A.out[k] = out[k];
  }
  if (n == 0) return 0;
  int blocks = (int)((n + 127) / 128);
  if (blocks > 148 * 16) blocks = 148 * 16;
  k_lane_op<<<blocks, 128, 0, (cudaStream_t)stream>>>(A);
  B2S_CUDA(cudaGetLastError());
  return 0;
}
