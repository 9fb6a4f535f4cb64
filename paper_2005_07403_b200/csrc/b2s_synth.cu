// b2s_synth.cu -- on-device generation of the BASELINE synthetic batches.
//
// Device twin of paper_2005_07403_b200/synth.py (the docstring there is the
// spec): every value is a pure function of (seed, config, stream, lane), so a
// GPU generates exactly its own contiguous shard, bit-identical to what NumPy
// produces for the same lane range.  All arithmetic is explicit-rounding
// (__d*_rn), matching NumPy's unfused evaluation.
#include "../../include/b2s.h"
#include "b2s_common.cuh"

namespace b2s {
namespace synth {

constexpr uint64_t M1 = 0xBF58476D1CE4E5B9ull, M2 = 0x94D049BB133111EBull;
constexpr uint64_t GOLD = 0x9E3779B97F4A7C15ull, KC = 0xC2B2AE3D27D4EB4Full, KS = 0x165667B19E3779F9ull;
constexpr uint64_t MANT = (1ull << 52) - 1;
constexpr int S_CLASS = 64, S_R1_SM = 70, S_R1_E = 71, S_PH = 80, S_C4_C = 90, S_WIDE = 100;

__host__ __device__ __forceinline__ uint64_t mix(uint64_t x) {
  x ^= x >> 30; x *= M1;
  x ^= x >> 27; x *= M2;
  return x ^ (x >> 31);
}

__host__ __device__ __forceinline__ uint64_t key(uint64_t seed, int config, int stream) {
  return mix(seed * GOLD + (uint64_t)config * KC + (uint64_t)stream * KS + 1ull);
}

struct Keys {
  uint64_t k[108];
};

__device__ __forceinline__ uint64_t draw(const Keys& K, int stream, uint64_t lane) {
  return mix(K.k[stream] + lane * GOLD);
}

__device__ __forceinline__ uint64_t mulhi_range(uint64_t r, uint64_t rng) {
  uint64_t h = r >> 32, lo = r & 0xFFFFFFFFull;
  return (h * rng + ((lo * rng) >> 32)) >> 32;
}

__device__ __forceinline__ double make_value(uint64_t sm, int64_t e) {
  uint64_t sign = sm & 0x8000000000000000ull, k = sm & MANT;
  if (e >= -1022) return __longlong_as_double((long long)(sign | ((uint64_t)(e + 1023) << 52) | k));
  uint64_t M = k | (1ull << 52);
  unsigned sh = (unsigned)(-1022 - e);
  uint64_t q = M >> sh, rem = M & ((1ull << sh) - 1), half = 1ull << (sh - 1);
  bool up = rem > half || (rem == half && (q & 1));
  return __longlong_as_double((long long)(sign | (q + (up ? 1 : 0))));
}

__device__ __forceinline__ double val(const Keys& K, int j, uint64_t lane, int lo, int hi, int estream = -1) {
  uint64_t sm = draw(K, 2 * j, lane);
  uint64_t er = draw(K, estream < 0 ? 2 * j + 1 : estream, lane);
  return make_value(sm, (int64_t)lo + (int64_t)mulhi_range(er, (uint64_t)(hi - lo + 1)));
}

__device__ __forceinline__ void cmulp(double ar, double ai, double br, double bi, double& r, double& i) {
  r = __dsub_rn(__dmul_rn(ar, br), __dmul_rn(ai, bi));
  i = __dadd_rn(__dmul_rn(ar, bi), __dmul_rn(ai, br));
}

__device__ __forceinline__ void phase(const Keys& K, int stream, uint64_t lane, double& c, double& s) {
  uint64_t r = draw(K, stream, lane);
  double t = __dmul_rn((double)((int64_t)(r >> 44) - (1ll << 19)), 0x1p-19);
  double tt = __dmul_rn(t, t);
  double den = __dadd_rn(1.0, tt);
  c = __ddiv_rn(__dsub_rn(1.0, tt), den);
  s = __ddiv_rn(__dadd_rn(t, t), den);
}

struct Args {
  int config;
  int64_t lane0, n;
  double* re[4];
  double* im[4];
};

__global__ void __launch_bounds__(256) k_synth(const Args A, const Keys K) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < A.n; i += stride) {
    const uint64_t lane = (uint64_t)(A.lane0 + i);
    const int cfg = A.config;
    if (cfg == 0 || cfg == 2 || cfg == 3) {
      int lo = cfg == 2 ? -1074 : (cfg == 3 ? -100 : -20);
      int hi = cfg == 2 ? 1023 : (cfg == 3 ? 100 : 20);
      double a[4];
      #pragma unroll
      for (int t = 0; t < 4; t++) a[t] = val(K, t, lane, lo, hi);
      if (cfg == 2) {
        uint64_t r = draw(K, S_CLASS, lane);
        int cls = (int)mulhi_range(r, 10);
        bool bit = r & 1;
        if (cls == 0) {
          if (!bit) { a[0] = 0.0; a[1] = 0.0; } else { a[2] = 0.0; a[3] = 0.0; }
        } else if (cls == 1) {
          int64_t e11 = -1074 + (int64_t)mulhi_range(draw(K, 1, lane), 2098);
          int64_t e21 = -1074 + (int64_t)mulhi_range(draw(K, 3, lane), 2098);
          int64_t hi_e = 1021 - (e11 > e21 ? e11 : e21);
          if (hi_e > 1023) hi_e = 1023;
          int64_t ep = -1074 + (int64_t)mulhi_range(draw(K, S_R1_E, lane), (uint64_t)(hi_e + 1075));
          double c = make_value(draw(K, S_R1_SM, lane), ep);
          a[2] = __dmul_rn(c, a[0]);
          a[3] = __dmul_rn(c, a[1]);
        } else if (cls == 2) {
          a[1] = 0.0; a[2] = 0.0;
        } else if (cls == 3) {
          a[1] = 0.0;
        }
      }
      #pragma unroll
      for (int t = 0; t < 4; t++) A.re[t][i] = a[t];
    } else {
      double r_[4], i_[4];
      #pragma unroll
      for (int t = 0; t < 4; t++) {
        r_[t] = val(K, 2 * t, lane, -20, 20);
        i_[t] = val(K, 2 * t + 1, lane, -20, 20);
      }
      if (cfg == 4) {
        int cls = (int)mulhi_range(draw(K, S_CLASS, lane), 10);
        if (cls == 6 || cls == 7) {
          double p1c, p1s, p2c, p2s, q1c, q1s, q2c, q2s, xr, xi;
          phase(K, S_PH + 0, lane, p1c, p1s);
          phase(K, S_PH + 1, lane, p2c, p2s);
          phase(K, S_PH + 2, lane, q1c, q1s);
          phase(K, S_PH + 3, lane, q2c, q2s);
          cmulp(p1c, p1s, r_[0], i_[0], xr, xi); cmulp(xr, xi, q1c, q1s, r_[0], i_[0]);
          cmulp(p1c, p1s, r_[2], i_[2], xr, xi); cmulp(xr, xi, q2c, q2s, r_[2], i_[2]);
          cmulp(p2c, p2s, r_[3], i_[3], xr, xi); cmulp(xr, xi, q2c, q2s, r_[3], i_[3]);
          r_[1] = 0.0; i_[1] = 0.0;
        } else if (cls == 8) {
          double cr = val(K, 45, lane, -20, 20, S_C4_C + 1);
          double ci = val(K, 46, lane, -20, 20, S_C4_C + 3);
          cmulp(cr, ci, r_[0], i_[0], r_[2], i_[2]);
          cmulp(cr, ci, r_[1], i_[1], r_[3], i_[3]);
        } else if (cls == 9) {
          #pragma unroll
          for (int t = 0; t < 4; t++) {
            r_[t] = val(K, 2 * t, lane, -1000, 1000, S_WIDE + 2 * t);
            i_[t] = val(K, 2 * t + 1, lane, -1000, 1000, S_WIDE + 2 * t + 1);
          }
        }
      }
      #pragma unroll
      for (int t = 0; t < 4; t++) { A.re[t][i] = r_[t]; A.im[t][i] = i_[t]; }
    }
  }
}

}  // namespace synth
}  // namespace b2s

using namespace b2s;

extern "C" int b2s_synth(int config, uint64_t seed, int64_t lane0, int64_t n, double* const re[4],
                         double* const im[4], void* stream) {
  if (config < 0 || config > 4) return fail(1, "config must be 0..4, got %d", config);
  if (n < 0 || lane0 < 0) return fail(1, "negative lane range");
  bool cplx = config == 1 || config == 4;
  if (!re) return fail(5, "re trains NULL");
  for (int t = 0; t < 4; t++) {
    if (!re[t]) return fail(5, "re train NULL");
    if (cplx && (!im || !im[t])) return fail(5, "complex config needs im trains");
  }
  if (n == 0) return 0;
  synth::Args A{};
  A.config = config;
  A.lane0 = lane0;
  A.n = n;
  for (int t = 0; t < 4; t++) { A.re[t] = re[t]; A.im[t] = cplx ? im[t] : nullptr; }
  synth::Keys K;
  for (int s = 0; s < 108; s++) K.k[s] = synth::key(seed, config, s);
  int err = 0;
  int grid = grid_for(synth::k_synth, 256, n, &err);
  synth::k_synth<<<grid, 256, 0, (cudaStream_t)stream>>>(A, K);
  B2S_CUDA(cudaGetLastError());
  return 0;
}
