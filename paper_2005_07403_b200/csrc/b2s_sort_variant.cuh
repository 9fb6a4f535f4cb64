// b2s_sort_variant.cuh -- the tile-sorted, warp-specialised complex
// streaming kernel (k_svd2_cplx_ws), measured and rejected in round 2
// (profiles/r2_sort_experiments/).  Included by
// b2s_kernels.cu only in variant builds (-DB2S_CPLX_SORT=128|256); the
// product library does not contain it.
#pragma once

namespace b2s {

#ifndef B2S_SORT_STAGES
#define B2S_SORT_STAGES 3
#endif
#ifndef B2S_SORT_MINB
#define B2S_SORT_MINB 5
#endif
constexpr int kOutCplx = 19;

template <int LT>
struct WsLayout {
  static constexpr int S = B2S_SORT_STAGES;
  static constexpr int W = LT / 32;
  static constexpr size_t kIn = (size_t)S * 8 * LT * sizeof(double);
  static constexpr size_t kOut = (size_t)kOutCplx * LT * sizeof(double);
  static constexpr size_t kBars = (size_t)(3 * S + 2) * sizeof(uint64_t);
  static constexpr size_t kSmem = kIn + kOut + kBars + S * sizeof(int) + W * sizeof(unsigned) +
                                  (size_t)S * LT * sizeof(unsigned short);
};

// Output train t of a complex launch: ur[0..3], ui[0..3], vr[0..3], vi[0..3],
// smax, smin, shift (the staging tile's row order).
__device__ __forceinline__ double* cplx_out_train(const CplxArgs& A, int t) {
  if (t < 4) return A.ur[t];
  if (t < 8) return A.ui[t - 4];
  if (t < 12) return A.vr[t - 8];
  if (t < 16) return A.vi[t - 12];
  return t == 16 ? A.smax : t == 17 ? A.smin : A.shift;
}

template <int Mode, bool Sine, int LT>
__global__ void __launch_bounds__(LT + 32, B2S_SORT_MINB) k_svd2_cplx_ws(const CplxArgs A) {
  extern __shared__ __align__(128) char smem[];
  using L = WsLayout<LT>;
  constexpr int S = L::S, W = L::W;
  double* in = reinterpret_cast<double*>(smem);                            // [S][8][LT]
  double* ob = reinterpret_cast<double*>(smem + L::kIn);                   // [19][LT]
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + L::kIn + L::kOut);   // [S] TMA landed
  uint64_t* empty = full + S;                                              // [S] gathered (W arrivals)
  uint64_t* plan = empty + S;                                              // [S] permutation ready
  uint64_t* ofull = plan + S;                                              // staged (W arrivals)
  uint64_t* oempty = ofull + 1;                                            // stores have read ob
  int* meta = reinterpret_cast<int*>(oempty + 1);                          // [S] wide count | rot << 16
  unsigned* hbits = reinterpret_cast<unsigned*>(meta + S);                 // [W] hard bits, tile order
  unsigned short* perm = reinterpret_cast<unsigned short*>(hbits + W);     // [S][LT] slot -> lane
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t tiles = A.n / LT;
  const int64_t mine = tiles > blockIdx.x ? (tiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  auto tile = [&](int64_t j) { return (int64_t)blockIdx.x + j * gridDim.x; };
  auto stage = [&](int s) { return in + (size_t)s * 8 * LT; };
  if (tid == 0) {
    for (int s = 0; s < S; s++) {
      tma::mbar_init(&full[s], 1);
      tma::mbar_init(&empty[s], W);
      tma::mbar_init(&plan[s], 1);
    }
    tma::mbar_init(ofull, W);
    tma::mbar_init(oempty, 1);
    tma::fence_init();
  }
  if (tid < W) hbits[tid] = 0;
  __syncthreads();

  if (warp == W) {
    // ------------------------------ producer ------------------------------
    const double* src[8];
    #pragma unroll
    for (int t = 0; t < 4; t++) { src[t] = A.ar[t]; src[4 + t] = A.ai[t]; }
    double* const my_dst = lane < kOutCplx ? cplx_out_train(A, lane) : nullptr;
    const uint64_t pol = tma::evict_first_policy();
    auto load = [&](int s, int64_t j) {
      tma::mbar_arrive_expect_tx(&full[s], 8 * LT * sizeof(double));
      #pragma unroll
      for (int t = 0; t < 8; t++)
        tma::bulk_load(stage(s) + t * LT, src[t] + tile(j) * LT, LT * sizeof(double), &full[s], pol);
    };
    if (lane == 0)
      for (int64_t j = 0; j < S && j < mine; j++) load((int)j, j);
    unsigned long long nh = 0;
    const unsigned lt_mask = (1u << lane) - 1u;
    auto store = [&](int64_t j) {                    // tile j's staged outputs -> HBM
      tma::mbar_wait_sleep(ofull, (uint32_t)(j & 1));
      if (lane < W) {
        const unsigned hb = hbits[lane];
        A.q.mask[((tile(j) * LT) >> 5) + lane] = hb;
        hbits[lane] = 0;
        nh += (unsigned)__popc(hb);
      }
      if (my_dst) {
        tma::bulk_store(my_dst + tile(j) * LT, ob + lane * LT, LT * sizeof(double));
        tma::bulk_commit();
        tma::bulk_wait_read<0>();
      }
      __syncwarp();
      if (lane == 0) tma::mbar_arrive(oempty);
    };
    for (int64_t j = 0; j < mine; j++) {
      const int s = (int)(j % S);
      tma::mbar_wait_sleep(&full[s], (uint32_t)((j / S) & 1));
      const double* st = stage(s);
      unsigned m[W];
      int wt = 0;
      #pragma unroll
      for (int q = 0; q < W; q++) {
        double p[8];
        #pragma unroll
        for (int t = 0; t < 8; t++) p[t] = st[t * LT + q * 32 + lane];
        m[q] = __ballot_sync(0xFFFFFFFFu, wide_lane<8>(p));
        wt += __popc(m[q]);
      }
      const int rot = (int)((blockIdx.x + (unsigned)j) % W);
      int pw = 0;
      unsigned short* pm = perm + (size_t)s * LT;
      #pragma unroll
      for (int q = 0; q < W; q++) {
        const bool w = (m[q] >> lane) & 1u;
        const int pn = q * 32 - pw;                  // narrow lanes before this group
        const int r = w ? pw + __popc(m[q] & lt_mask) : wt + pn + __popc(~m[q] & lt_mask);
        pm[(rot * 32 + r) & (LT - 1)] = (unsigned short)(q * 32 + lane);
        pw += __popc(m[q]);
      }
      if (lane == 0) meta[s] = wt | (rot << 16);
      __syncwarp();
      if (lane == 0) tma::mbar_arrive(&plan[s]);
      if (j > 0) {
        store(j - 1);
        // refill tile j-1's stage (its lanes were gathered before its outputs were staged)
        const int ps = (int)((j - 1) % S);
        if (lane == 0 && j - 1 + S < mine) {
          tma::mbar_wait_sleep(&empty[ps], (uint32_t)(((j - 1) / S) & 1));
          load(ps, j - 1 + S);
        }
        __syncwarp();
      }
    }
    if (mine > 0) {
      store(mine - 1);
      if (my_dst) tma::bulk_wait<0>();
    }
    if (nh) atomicAdd(A.q.cnt, nh);
    return;
  }

  // ------------------------------ compute warps ------------------------------
  for (int64_t k = 0; k < mine; k++) {
    const int s = (int)(k % S);
    const uint32_t par = (uint32_t)((k / S) & 1);
    tma::mbar_wait(&full[s], par);
    tma::mbar_wait(&plan[s], par);
    const int mt = meta[s];
    const int wt = mt & 0xFFFF, rot = (mt >> 16) * 32;
    const int sl = perm[(size_t)s * LT + tid];
    const double* st = stage(s);
    double ar[4], ai[4];
    #pragma unroll
    for (int t = 0; t < 4; t++) { ar[t] = st[t * LT + sl]; ai[t] = st[(4 + t) * LT + sl]; }
    consumed(ar);
    consumed(ai);
    __syncwarp();
    if (lane == 0) tma::mbar_arrive(&empty[s]);
    // slot tid holds a wide lane iff it lies in [rot, rot + wt) (mod LT)
    const bool wide_warp = __any_sync(0xFFFFFFFFu, ((tid - rot) & (LT - 1)) < wt);
    CplxOut o;
    bool hard;
    if (wide_warp)
      hard = svd2_complex_f<Sine, false, true>(ar, ai, o);
    else
      hard = svd2_complex_f<Sine, false, false, true>(ar, ai, o);
    backscale_lane<Mode>(o.smax, o.smin, o.shift);
    if (k > 0) tma::mbar_wait(oempty, (uint32_t)((k - 1) & 1));
    #pragma unroll
    for (int t = 0; t < 4; t++) {
      ob[t * LT + sl] = o.ur[t];
      ob[(4 + t) * LT + sl] = o.ui[t];
      ob[(8 + t) * LT + sl] = o.vr[t];
      ob[(12 + t) * LT + sl] = o.vi[t];
    }
    ob[16 * LT + sl] = o.smax;
    ob[17 * LT + sl] = o.smin;
    ob[18 * LT + sl] = o.shift;
    if (hard) atomicOr(&hbits[sl >> 5], 1u << (sl & 31));
    tma::fence_proxy_async();                 // staged writes -> the bulk stores
    __syncwarp();
    if (lane == 0) tma::mbar_arrive(ofull);
  }
}


}  // namespace b2s

// ---------------------------------------------------------------------------
// k_svd2_cplx_u4 (variant, -DB2S_CPLX_SORT4=1): the same producer-warp plan,
// but at sector granularity and with no output staging.  A tile of 256
// lanes is 64 units of 4 consecutive lanes (one 32-byte sector of every
// train); the producer sorts the units so the wide ones fill as few warps
// as possible, and each compute thread writes its lane's outputs straight
// to HBM -- four threads cover one whole sector, so no sector is ever split
// between writers and no warp waits for another's outputs.  Hard lanes
// are recorded with global atomics (the mask is cleared before launch).
// ---------------------------------------------------------------------------
namespace b2s {

#ifndef B2S_U4_STAGES
#define B2S_U4_STAGES 3
#endif
#ifndef B2S_U4_MINB
#define B2S_U4_MINB 2
#endif

struct U4Layout {
  static constexpr int LT = 256, S = B2S_U4_STAGES, W = LT / 32, U = LT / 4;
  static constexpr size_t kIn = (size_t)S * 8 * LT * sizeof(double);
  static constexpr size_t kBars = (size_t)(3 * S) * sizeof(uint64_t);
  static constexpr size_t kSmem = kIn + kBars + S * sizeof(int) + (size_t)S * U;
};

template <int Mode, bool Sine>
__global__ void __launch_bounds__(U4Layout::LT + 32, B2S_U4_MINB) k_svd2_cplx_u4(const CplxArgs A) {
  extern __shared__ __align__(128) char smem[];
  using L = U4Layout;
  constexpr int LT = L::LT, S = L::S, W = L::W, U = L::U;
  double* in = reinterpret_cast<double*>(smem);                            // [S][8][LT]
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + L::kIn);             // [S] TMA landed
  uint64_t* empty = full + S;                                              // [S] gathered (W arrivals)
  uint64_t* plan = empty + S;                                              // [S] unit order ready
  int* meta = reinterpret_cast<int*>(plan + S);                            // [S] wide units | rot << 16
  unsigned char* perm = reinterpret_cast<unsigned char*>(meta + S);        // [S][U] slot -> unit
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t tiles = A.n / LT;
  const int64_t mine = tiles > blockIdx.x ? (tiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  auto tile = [&](int64_t j) { return (int64_t)blockIdx.x + j * gridDim.x; };
  auto stage = [&](int s) { return in + (size_t)s * 8 * LT; };
  if (tid == 0) {
    for (int s = 0; s < S; s++) {
      tma::mbar_init(&full[s], 1);
      tma::mbar_init(&empty[s], W);
      tma::mbar_init(&plan[s], 1);
    }
    tma::fence_init();
  }
  __syncthreads();

  if (warp == W) {
    // ------------------------------ producer ------------------------------
    const double* src[8];
    #pragma unroll
    for (int t = 0; t < 4; t++) { src[t] = A.ar[t]; src[4 + t] = A.ai[t]; }
    const uint64_t pol = tma::evict_first_policy();
    auto load = [&](int s, int64_t j) {
      tma::mbar_arrive_expect_tx(&full[s], 8 * LT * sizeof(double));
      #pragma unroll
      for (int t = 0; t < 8; t++)
        tma::bulk_load(stage(s) + t * LT, src[t] + tile(j) * LT, LT * sizeof(double), &full[s], pol);
    };
    if (lane == 0)
      for (int64_t j = 0; j < S && j < mine; j++) load((int)j, j);
    for (int64_t j = 0; j < mine; j++) {
      const int s = (int)(j % S);
      tma::mbar_wait(&full[s], (uint32_t)((j / S) & 1));
      const double* st = stage(s);
      // unit flags: 8 units per 32-lane group, bit 4k of the nibble-ORed ballot
      unsigned uw[W];
      int wu = 0;
      #pragma unroll
      for (int q = 0; q < W; q++) {
        double p[8];
        #pragma unroll
        for (int t = 0; t < 8; t++) p[t] = st[t * LT + q * 32 + lane];
        const unsigned m = __ballot_sync(0xFFFFFFFFu, wide_lane<8>(p));
        uw[q] = (m | (m >> 1) | (m >> 2) | (m >> 3)) & 0x11111111u;
        wu += __popc(uw[q]);
      }
      const int rot = (int)((blockIdx.x + (unsigned)j) % W) * 8;      // first slot of the wide units
      if (lane < 8) {                                                  // lane k: units 8q + k of every group
        int pw = 0;
        unsigned char* pm = perm + (size_t)s * U;
        #pragma unroll
        for (int q = 0; q < W; q++) {
          const unsigned below = uw[q] & ((1u << (4 * lane)) - 1u);    // wide units before this one in group q
          const bool w = (uw[q] >> (4 * lane)) & 1u;
          const int pwi = pw + __popc(below);
          const int pni = 8 * q + lane - pwi;                          // narrow units before it
          const int r = w ? pwi : wu + pni;
          pm[(rot + r) & (U - 1)] = (unsigned char)(8 * q + lane);
          pw += __popc(uw[q]);
        }
      }
      if (lane == 0) meta[s] = wu | (rot << 16);
      __syncwarp();
      if (lane == 0) tma::mbar_arrive(&plan[s]);
      if (j > 0 && lane == 0 && j - 1 + S < mine) {
        const int ps = (int)((j - 1) % S);
        tma::mbar_wait_sleep(&empty[ps], (uint32_t)(((j - 1) / S) & 1));
        load(ps, j - 1 + S);
      }
      __syncwarp();
    }
    return;
  }

  // ------------------------------ compute warps ------------------------------
  const int slot = warp * 8 + (lane >> 2);
  for (int64_t k = 0; k < mine; k++) {
    const int s = (int)(k % S);
    const uint32_t par = (uint32_t)((k / S) & 1);
    tma::mbar_wait(&full[s], par);
    tma::mbar_wait(&plan[s], par);
    const int mt = meta[s];
    const int wu = mt & 0xFFFF, rot = mt >> 16;
    const int li = 4 * perm[(size_t)s * U + slot] + (lane & 3);       // lane within the tile
    const double* st = stage(s);
    double ar[4], ai[4];
    #pragma unroll
    for (int t = 0; t < 4; t++) { ar[t] = st[t * LT + li]; ai[t] = st[(4 + t) * LT + li]; }
    consumed(ar);
    consumed(ai);
    __syncwarp();
    if (lane == 0) tma::mbar_arrive(&empty[s]);
    const bool wide_warp = __any_sync(0xFFFFFFFFu, ((slot - rot) & (U - 1)) < wu);
    CplxOut o;
#if B2S_CPLX_UNIFIED
    const bool hard = svd2_complex_u<Sine>(ar, ai, o, wide_warp);
#else
    bool hard;
    if (wide_warp)
      hard = svd2_complex_f<Sine, false, true>(ar, ai, o);
    else
      hard = svd2_complex_f<Sine, false, false, true>(ar, ai, o);
#endif
    const int64_t gi = tile(k) * LT + li;
    store_cplx<Mode>(A, (uint32_t)gi, o);
    if (hard) {
      atomicOr(&A.q.mask[gi >> 5], 1u << (gi & 31));
      atomicAdd(A.q.cnt, 1ull);
    }
  }
}

}  // namespace b2s
