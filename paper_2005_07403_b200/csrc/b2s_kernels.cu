// b2s_kernels.cu -- sm_100a batched 2x2 SVD kernels and their C-ABI entry
// points (include/b2s.h).
//
// K1 real / K2 complex: one SVD per thread, the whole pipeline fused in
// registers; SoA trains streamed with coalesced evict-first stores.  The
// default kernels (k_svd2_*_tma) stage their inputs through a TMA ring in
// shared memory; the LDG kernels (k_svd2_real / k_svd2_complex: a resident
// grid-stride loop that prefetches the next lane's inputs into registers)
// serve misaligned trains, state dumps and the real kernel's sub-tile tail.
// K1f / K2f (k_fix_*) recompute the lanes a streaming kernel flagged.
#include "../../include/b2s.h"
#include "b2s_common.cuh"
#include "b2s_fast.cuh"
#include "b2s_tma.cuh"

#include <cstdlib>
#include <mutex>
#include <vector>

namespace b2s {

char* last_error_buf() {
  static thread_local char buf[512] = {0};
  return buf;
}

// Per-launch hard-lane mask: bit l of word w marks lane 32w + l as hard
// (its operands left a fast call site's proven range).  The fast kernel
// writes one ballot word per warp-iteration -- no atomics, 4 bytes per 32
// lanes of traffic -- and the fix-up kernel compacts the set bits and
// recomputes those lanes, packed, with exact arithmetic.
struct HardQueue {
  unsigned* mask;
  unsigned long long* cnt;   // hard lanes found by the fix-up (diagnostics)
};

struct RealArgs {
  HardQueue q;
  int aos;        // 1: a[0] points at AoSoA-8 records (cli.py:102-134 layout)
  int64_t n;
  const double* a[4];
  double* u[4];
  double* v[4];
  double *smax, *smin, *shift;
  double* st[B2S_STATES_COMPLEX_FULL];
  int full_states;      // B2S_FLAG_STATES_FULL
};

struct CplxArgs {
  HardQueue q;
  int aos;        // 1: ar[0] points at AoSoA-8 complex records
  int64_t n;
  const double* ar[4];
  const double* ai[4];
  double *ur[4], *ui[4], *vr[4], *vi[4];
  double *smax, *smin, *shift;
  double* st[B2S_STATES_COMPLEX_FULL];
  int full_states;
};

constexpr int kBlock = 256;

__device__ __forceinline__ double ld_stream(const double* p) { return __ldcs(p); }
// Output stores: evict-first streaming stores (default); B2S_STORE_MODE 1 =
// plain write-back stores, 2 = .cg (A/B variants: the config-3 bench moved
// by < 0.5 % either way, profiles/r2_store_ring_ab.log).
#ifndef B2S_STORE_MODE
#define B2S_STORE_MODE 0
#endif
__device__ __forceinline__ void st_stream(double* p, double v) {
#if B2S_STORE_MODE == 1
  *p = v;
#elif B2S_STORE_MODE == 2
  __stcg(p, v);
#else
  __stcs(p, v);
#endif
}

template <bool Cplx>
__device__ __forceinline__ void store_states(double* const* st, int64_t i, const LaneStates& s, bool full) {
  int k = 0;
  st_stream(st[k++] + i, s.shift);
  st_stream(st[k++] + i, s.swap_c);
  st_stream(st[k++] + i, s.swap_r);
  st_stream(st[k++] + i, s.ph1r); if (Cplx) st_stream(st[k++] + i, s.ph1i);
  st_stream(st[k++] + i, s.ph2r); if (Cplx) st_stream(st[k++] + i, s.ph2i);
  st_stream(st[k++] + i, s.dtr);  if (Cplx) st_stream(st[k++] + i, s.dti);
  st_stream(st[k++] + i, s.dhr);  if (Cplx) st_stream(st[k++] + i, s.dhi);
  st_stream(st[k++] + i, s.g_tan);
  st_stream(st[k++] + i, s.g_cos);
  st_stream(st[k++] + i, s.r11);
  st_stream(st[k++] + i, s.r12);
  st_stream(st[k++] + i, s.r22);
  st_stream(st[k++] + i, s.l_tan);
  st_stream(st[k++] + i, s.r_tan);
  st_stream(st[k++] + i, s.smax);
  st_stream(st[k++] + i, s.smin);
  if (full) {
    st_stream(st[k++] + i, s.l_sec2);
    st_stream(st[k++] + i, s.l_cos);
    st_stream(st[k++] + i, s.r_sec2);
    st_stream(st[k++] + i, s.r_cos);
    #pragma unroll
    for (int t = 0; t < (Cplx ? 8 : 4); t++) st_stream(st[k++] + i, s.sp[t]);
  }
}

template <int Mode>
// i < 2^31 (one sub-launch): 32-bit lane offsets let every address be a
// single IMAD.WIDE.U32 off the train base.
__device__ __forceinline__ void store_real(const RealArgs& A, uint32_t i, RealOut o) {
  backscale_lane<Mode>(o.smax, o.smin, o.shift);
  #pragma unroll
  for (int t = 0; t < 4; t++) st_stream(A.u[t] + i, o.u[t]);
  #pragma unroll
  for (int t = 0; t < 4; t++) st_stream(A.v[t] + i, o.v[t]);
  st_stream(A.smax + i, o.smax);
  st_stream(A.smin + i, o.smin);
  st_stream(A.shift + i, o.shift);
}

template <int Mode>
__device__ __forceinline__ void store_cplx(const CplxArgs& A, uint32_t i, CplxOut o) {
  backscale_lane<Mode>(o.smax, o.smin, o.shift);
  #pragma unroll
  for (int t = 0; t < 4; t++) { st_stream(A.ur[t] + i, o.ur[t]); st_stream(A.ui[t] + i, o.ui[t]); }
  #pragma unroll
  for (int t = 0; t < 4; t++) { st_stream(A.vr[t] + i, o.vr[t]); st_stream(A.vi[t] + i, o.vi[t]); }
  st_stream(A.smax + i, o.smax);
  st_stream(A.smin + i, o.smin);
  st_stream(A.shift + i, o.shift);
}

// Lane i's inputs from SoA trains, or from AoSoA-8 records: matrix i is lane
// i % 8 of record i / 8; a real record holds the 8-lane vectors e11, e21,
// e12, e22, a complex one e11re, e11im, e21re, ... (cli.py:102-134).
__device__ __forceinline__ void load_real(const RealArgs& A, int64_t i, double (&a)[4]) {
  if (A.aos) {
    const double* r = A.a[0] + (i >> 3) * 32 + (i & 7);
    #pragma unroll
    for (int t = 0; t < 4; t++) a[t] = r[8 * t];
  } else {
    #pragma unroll
    for (int t = 0; t < 4; t++) a[t] = A.a[t][i];
  }
}

__device__ __forceinline__ void load_cplx(const CplxArgs& A, int64_t i, double (&ar)[4], double (&ai)[4]) {
  if (A.aos) {
    const double* r = A.ar[0] + (i >> 3) * 64 + (i & 7);
    #pragma unroll
    for (int t = 0; t < 4; t++) { ar[t] = r[16 * t]; ai[t] = r[16 * t + 8]; }
  } else {
    #pragma unroll
    for (int t = 0; t < 4; t++) { ar[t] = A.ar[t][i]; ai[t] = A.ai[t][i]; }
  }
}

// The same with evict-first streaming loads (the LDG streaming kernels).
__device__ __forceinline__ void load_real_cs(const RealArgs& A, int64_t i, double (&a)[4]) {
  if (A.aos) {
    const double* r = A.a[0] + (i >> 3) * 32 + (i & 7);
    #pragma unroll
    for (int t = 0; t < 4; t++) a[t] = ld_stream(r + 8 * t);
  } else {
    #pragma unroll
    for (int t = 0; t < 4; t++) a[t] = ld_stream(A.a[t] + i);
  }
}

__device__ __forceinline__ void load_cplx_cs(const CplxArgs& A, int64_t i, double (&ar)[4], double (&ai)[4]) {
  if (A.aos) {
    const double* r = A.ar[0] + (i >> 3) * 64 + (i & 7);
    #pragma unroll
    for (int t = 0; t < 4; t++) { ar[t] = ld_stream(r + 16 * t); ai[t] = ld_stream(r + 16 * t + 8); }
  } else {
    #pragma unroll
    for (int t = 0; t < 4; t++) { ar[t] = ld_stream(A.ar[t] + i); ai[t] = ld_stream(A.ai[t] + i); }
  }
}

// A marked lane again, with every failing call site re-evaluated exactly.
template <int Mode, bool Sine>
__device__ __forceinline__ void redo_real(const RealArgs& A, int64_t i) {
  double a[4];
  load_real(A, i, a);
  RealOut o;
  svd2_real_f<Sine, true>(a, o);
  store_real<Mode>(A, i, o);
}

template <int Mode, bool Sine>
__device__ __forceinline__ void redo_cplx(const CplxArgs& A, int64_t i) {
  double ar[4], ai[4];
  load_cplx(A, i, ar, ai);
  CplxOut o;
  svd2_complex_f<Sine, true, true>(ar, ai, o);
  store_cplx<Mode>(A, i, o);
}

// Record this warp's hard lanes: one ballot word per 32 consecutive lanes.
// Lane 0 of the warp always holds the lowest (32-aligned) index.
// Returns the number of hard lanes in the word (meaningful on lane 0).
// Every caller reaches it with all 32 lanes of the warp (the loops are
// warp-uniform and out-of-range lanes pass hard = false), so the ballot
// uses the full mask -- it also forces warp 0 to reconverge after thread
// 0's producer work in the TMA kernels.
__device__ __forceinline__ unsigned mark_hard(const HardQueue& q, bool hard, int64_t i) {
  const unsigned m = __ballot_sync(0xFFFFFFFFu, hard);
  if ((threadIdx.x & 31) == 0) q.mask[i >> 5] = m;
  return (unsigned)__popc(m);
}

// One atomic per warp at kernel end: the launch's hard-lane total, which
// the fix-up kernel checks before scanning the mask.
__device__ __forceinline__ void count_hard(const HardQueue& q, unsigned long long n) {
  if ((threadIdx.x & 31) == 0 && n) atomicAdd(q.cnt, n);
}

template <int Mode, bool Sine, bool States>
__global__ void __launch_bounds__(kBlock, 3) k_svd2_real(const RealArgs A) {
  const int64_t stride = (int64_t)gridDim.x * kBlock;
  unsigned long long nh = 0;
  int64_t i = (int64_t)blockIdx.x * kBlock + threadIdx.x;
  // The loop is warp-uniform (lane 0 holds the warp's lowest index): every
  // lane of a warp iterates while any of its lanes is in range, so the
  // hard-lane ballot always runs with the full, converged mask.
  const int64_t lane = threadIdx.x & 31;
  if (i - lane >= A.n) return;
  double nx[4] = {0.0, 0.0, 0.0, 0.0};
  if (i < A.n) load_real_cs(A, i, nx);
  for (; i - lane < A.n; i += stride) {
    const bool in = i < A.n;
    double a[4] = {nx[0], nx[1], nx[2], nx[3]};
    const int64_t j = i + stride;
    if (j < A.n) load_real_cs(A, j, nx);
    RealOut o;
    bool hard = false;
    if (in) {
      if (States) {
        LaneStates s;
        svd2_real_x<Sine, true>(a, o, &s);
        store_real<Mode>(A, i, o);
        store_states<false>(A.st, i, s, A.full_states != 0);
      } else {
        hard = svd2_real_f<Sine, false>(a, o);
        store_real<Mode>(A, i, o);    // full sectors; hard lanes are rewritten by the fix-up
      }
    }
    if (!States) nh += mark_hard(A.q, hard, i);
  }
  count_hard(A.q, nh);
}

template <int Mode, bool Sine, bool States>
__global__ void __launch_bounds__(kBlock, 2) k_svd2_complex(const CplxArgs A) {
  const int64_t stride = (int64_t)gridDim.x * kBlock;
  unsigned long long nh = 0;
  int64_t i = (int64_t)blockIdx.x * kBlock + threadIdx.x;
  const int64_t lane = threadIdx.x & 31;     // warp-uniform loop, as k_svd2_real
  if (i - lane >= A.n) return;
  double nr[4] = {0.0, 0.0, 0.0, 0.0}, ni[4] = {0.0, 0.0, 0.0, 0.0};
  if (i < A.n) load_cplx_cs(A, i, nr, ni);
  for (; i - lane < A.n; i += stride) {
    const bool in = i < A.n;
    double ar[4] = {nr[0], nr[1], nr[2], nr[3]};
    double ai[4] = {ni[0], ni[1], ni[2], ni[3]};
    const int64_t j = i + stride;
    if (j < A.n) load_cplx_cs(A, j, nr, ni);
    CplxOut o;
    bool hard = false;
    if (in) {
      if (States) {
        LaneStates s;
        svd2_complex_x<Sine, true>(ar, ai, o, &s);
        store_cplx<Mode>(A, i, o);
        store_states<true>(A.st, i, s, A.full_states != 0);
      } else {
        hard = svd2_complex_f<Sine, false>(ar, ai, o);
        store_cplx<Mode>(A, i, o);    // full sectors; hard lanes are rewritten by the fix-up
      }
    }
    if (!States) nh += mark_hard(A.q, hard, i);
  }
  count_hard(A.q, nh);
}

// ---------------------------------------------------------------------------
// TMA-staged streaming kernels (the default when every train is 16-byte
// aligned).  A persistent grid; each CTA walks its tiles of kBlock lanes
// through a kStages-deep ring of shared-memory stages.  One thread arms the
// stage's mbarrier and issues one cp.async.bulk per input train; the loads
// of the next kStages-1 tiles are in flight while the CTA computes the
// current one.  Outputs go straight from registers with streaming stores
// (coalesced 256 B per warp per train).  The sub-tile tail (n mod 256
// lanes) is processed by CTA 0 with ordinary loads (complex) or by a
// one-CTA launch of the LDG kernel (real), see B2S_TMA_TAIL_*.
// ---------------------------------------------------------------------------
// Depth of the TMA input ring (3 and 6 measured within 0.7 % of 4 on the
// config-3 bench, profiles/r2_store_ring_ab.log).
#ifndef B2S_RING_STAGES
#define B2S_RING_STAGES 4
#endif
constexpr int kStages = B2S_RING_STAGES;
// The sub-tile tail (n mod 256 lanes): 1 = processed by CTA 0 of the TMA
// kernel with ordinary loads, 0 = a separate one-CTA launch of the LDG
// kernel (keeps another copy of the pipeline out of the TMA kernel).
// Measured per 2^26 lanes: real 0 is 3 % faster on config 2 and equal on
// config 3 (and in the bench); complex 0 is 0.3-0.6 % slower on configs 1
// and 4.  The LDG kernels read AoSoA-8 records too, for record tails.
#ifndef B2S_TMA_TAIL_REAL
#define B2S_TMA_TAIL_REAL 0
#endif
#ifndef B2S_TMA_TAIL_CPLX
#define B2S_TMA_TAIL_CPLX 1
#endif
// Bounded (check-free) entry sites for the real fast path, valid under the
// wide_or_sub dispatch.  Short cold-clock runs of 2^26 lanes measured it 3 %
// slower (1.50 vs 1.45 ms), but the bench workload (2^30 lanes, 20 steps,
// power-capped at ~700 W, SM clock ~1.78 GHz) is 2.4 % faster with it
// (43.1-43.2 vs 42.1-42.2 G SVD/s, two runs each): fewer instructions, less
// power, higher sustained clock.
#ifndef B2S_REAL_BND
#define B2S_REAL_BND 1
#endif
#ifndef B2S_REAL_WIDE
#define B2S_REAL_WIDE 2
#endif
constexpr int kWarps = kBlock / 32;

// Force the loaded values into registers (scoreboard wait) before what
// follows in program order.
__device__ __forceinline__ void consumed(const double (&v)[4]) {
  asm volatile("" ::"d"(v[0]), "d"(v[1]), "d"(v[2]), "d"(v[3]) : "memory");
}

// Producer/consumer ring without CTA barriers.  full[s] (an mbarrier)
// completes when the bulk copies of a tile land (one arrive.expect_tx plus
// the TMA transaction bytes).  Stage release is a shared counter: each warp,
// once its loads from the stage have landed (`consumed`), increments it, and
// the warp that brings it to kWarps -- the last reader -- resets it and
// issues the refill of that stage with the CTA's tile kStages ahead.  No
// warp ever waits for another except on data, and no thread polls.
template <int NT, int LANES = kBlock, int STAGES = kStages>
struct TmaRing {
  static constexpr uint32_t kTileBytes = LANES * sizeof(double);
  static constexpr size_t kBuf = (size_t)STAGES * NT * LANES * sizeof(double);
  static constexpr size_t kSmem = kBuf + STAGES * (sizeof(uint64_t) + sizeof(int));
  double* buf;      // [STAGES][NT][LANES]
  uint64_t* full;   // [STAGES]
  int* readers;     // [STAGES]
  const double* const* src;
  int64_t mine;
  int64_t tstride;    // elements between consecutive tiles of one source

  __device__ __forceinline__ double* stage(int s, int t) { return buf + ((size_t)s * NT + t) * LANES; }
  __device__ __forceinline__ int64_t tile(int64_t j) const { return blockIdx.x + j * gridDim.x; }

  __device__ __forceinline__ void init(char* smem, const double* const* src_, int64_t mine_,
                                      int64_t tstride_ = LANES) {
    buf = reinterpret_cast<double*>(smem);
    full = reinterpret_cast<uint64_t*>(smem + kBuf);
    readers = reinterpret_cast<int*>(full + STAGES);
    src = src_;
    mine = mine_;
    tstride = tstride_;
    if (threadIdx.x == 0) {
      for (int s = 0; s < STAGES; s++) {
        tma::mbar_init(&full[s], 1);
        readers[s] = 0;
      }
      tma::fence_init();
    }
    __syncthreads();
    if (threadIdx.x == 0)
      for (int64_t j = 0; j < STAGES && j < mine; j++) issue((int)j, tile(j));
  }

  __device__ __forceinline__ void issue(int s, int64_t t) {
    const uint64_t pol = tma::evict_first_policy();
    tma::mbar_arrive_expect_tx(&full[s], NT * kTileBytes);
    #pragma unroll
    for (int k = 0; k < NT; k++) tma::bulk_load(stage(s, k), src[k] + t * tstride, kTileBytes, &full[s], pol);
  }

  __device__ __forceinline__ void wait_full(int64_t j) {
    tma::mbar_wait(&full[(int)(j % STAGES)], (uint32_t)((j / STAGES) & 1));
  }

  __device__ __forceinline__ void release(int64_t j) {
    __syncwarp();
    if ((threadIdx.x & 31) == 0) {
      const int s = (int)(j % STAGES);
      __threadfence_block();                               // release this warp's reads
      if (atomicAdd(&readers[s], 1) == (LANES / 32) - 1) {
        __threadfence_block();                             // acquire the other warps' reads
        readers[s] = 0;
        if (j + STAGES < mine) {
          tma::fence_proxy_async();
          issue(s, tile(j + STAGES));
        }
      }
    }
  }
};

// AoS = true: the source is AoSoA-8 records; a 256-lane tile is one
// contiguous 8 KiB (real) / 16 KiB (complex) block of 32 records, fetched by
// the same NT 2 KiB bulk copies, and each thread picks its lane's components
// out of the record layout in shared memory (no separate repack pass).
template <int NT, bool AoS>
__device__ __forceinline__ double stage_val(double* st0, int v, int tid) {
  if (AoS) return st0[(tid >> 3) * (NT * 8) + v * 8 + (tid & 7)];
  return st0[v * kBlock + tid];
}

// Resident CTAs per SM for the real streaming kernel: 3 (80 registers) and 4
// (64 registers, 8 bytes of spills) measured equal in the bench (43.5 vs
// 43.6 G SVD/s, two runs each) and within 1 % on configs 2 / 3.
#ifndef B2S_REAL_MINB
#define B2S_REAL_MINB 3
#endif
template <int Mode, bool Sine, bool AoS>
__global__ void __launch_bounds__(kBlock, B2S_REAL_MINB) k_svd2_real_tma(const RealArgs A) {
  extern __shared__ __align__(128) char smem[];
  const double* src[4];
  #pragma unroll
  for (int t = 0; t < 4; t++) src[t] = AoS ? A.a[0] + t * kBlock : A.a[t];
  const int tid = threadIdx.x;
  unsigned long long nh = 0;
  const int64_t tiles = A.n / kBlock;
  const int64_t mine = tiles > blockIdx.x ? (tiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  TmaRing<4> R;
  R.init(smem, src, mine, AoS ? 4 * kBlock : kBlock);
  for (int64_t k = 0; k < mine; k++) {
    const int s = (int)(k % kStages);
    R.wait_full(k);
    double a[4];
    #pragma unroll
    for (int t = 0; t < 4; t++) a[t] = stage_val<4, AoS>(R.stage(s, 0), t, tid);
    consumed(a);
    R.release(k);
    const int64_t i = R.tile(k) * kBlock + tid;
    RealOut o;
    bool hard;
#if B2S_REAL_WIDE
    // A warp holding a full-range lane (BASELINE config 2) runs the
    // per-site-repairing pipeline in place, with the exponent-normalised
    // divisions at the rotation and triangle sites (B2S_REAL_WIDE 2; 1 =
    // repairs only): exact for every lane, so nothing is left for the fix-up
    // kernel.  Warp-uniform choice.  Config 2, 2^26 lanes: 4.85 ms with 58 %
    // of lanes fixed up afterwards -> 3.97 ms (mode 1) -> 2.83 ms (mode 2);
    // config 3 unchanged.
    if (__any_sync(0xFFFFFFFFu, wide_or_sub<4>(a))) {
      svd2_real_f<Sine, true, B2S_REAL_WIDE == 2>(a, o);
      hard = false;
    } else
#endif
    hard = svd2_real_f<Sine, false, false, B2S_REAL_WIDE != 0 && B2S_REAL_BND>(a, o);
    store_real<Mode>(A, i, o);
    nh += mark_hard(A.q, hard, i);
  }
  if (B2S_TMA_TAIL_REAL && blockIdx.x == 0) {
    const int64_t i = tiles * kBlock + tid;
    if (i - (tid & 31) < A.n) {             // warp-uniform: any lane of the warp in range
      bool hard = false;
      if (i < A.n) {
        double a[4];
        load_real(A, i, a);
        RealOut o;
        hard = svd2_real_f<Sine, false>(a, o);
        store_real<Mode>(A, i, o);
      }
      nh += mark_hard(A.q, hard, i);
    }
  }
  count_hard(A.q, nh);
}

template <int Mode, bool Sine, bool AoS>
#ifndef B2S_CPLX_MINB
#define B2S_CPLX_MINB 3
#endif
// 1: one code body for wide and bounded warps (svd2_complex_u) -- variant.
#ifndef B2S_CPLX_UNIFIED
#define B2S_CPLX_UNIFIED 0
#endif
#ifndef B2S_CPLX_STAGES
#define B2S_CPLX_STAGES kStages
#endif
__global__ void __launch_bounds__(kBlock, B2S_CPLX_MINB) k_svd2_cplx_tma(const CplxArgs A) {
  extern __shared__ __align__(128) char smem[];
  const double* src[8];
  #pragma unroll
  for (int t = 0; t < 4; t++) {
    src[t] = AoS ? A.ar[0] + t * kBlock : A.ar[t];
    src[4 + t] = AoS ? A.ar[0] + (4 + t) * kBlock : A.ai[t];
  }
  const int tid = threadIdx.x;
  unsigned long long nh = 0;
  const int64_t tiles = A.n / kBlock;
  const int64_t mine = tiles > blockIdx.x ? (tiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  TmaRing<8, kBlock, B2S_CPLX_STAGES> R;
  R.init(smem, src, mine, AoS ? 8 * kBlock : kBlock);
  for (int64_t k = 0; k < mine; k++) {
    const int s = (int)(k % B2S_CPLX_STAGES);
    R.wait_full(k);
    double ar[4], ai[4];
    #pragma unroll
    for (int t = 0; t < 4; t++) {
      // SoA stage order: re trains then im trains; record order: re/im per entry
      ar[t] = stage_val<8, AoS>(R.stage(s, 0), AoS ? 2 * t : t, tid);
      ai[t] = stage_val<8, AoS>(R.stage(s, 0), AoS ? 2 * t + 1 : 4 + t, tid);
    }
    consumed(ar);
    consumed(ai);
    R.release(k);
    const int64_t i = R.tile(k) * kBlock + tid;
    CplxOut o;
    bool hard;
    const double p[8] = {ar[0], ai[0], ar[1], ai[1], ar[2], ai[2], ar[3], ai[3]};
#if B2S_CPLX_UNIFIED
    hard = svd2_complex_u<Sine>(ar, ai, o, __any_sync(0xFFFFFFFFu, wide_lane<8>(p)));
#else
    if (__any_sync(0xFFFFFFFFu, wide_lane<8>(p)))
      hard = svd2_complex_f<Sine, false, true>(ar, ai, o);
    else
      hard = svd2_complex_f<Sine, false, false, true>(ar, ai, o);   // bounded warp
#endif
    store_cplx<Mode>(A, i, o);
    nh += mark_hard(A.q, hard, i);
  }
  if (B2S_TMA_TAIL_CPLX && blockIdx.x == 0) {
    const int64_t i = tiles * kBlock + tid;
    if (i - (tid & 31) < A.n) {             // warp-uniform: any lane of the warp in range
      bool hard = false;
      if (i < A.n) {
        double ar[4], ai[4];
        load_cplx(A, i, ar, ai);
        CplxOut o;
        hard = svd2_complex_f<Sine, false>(ar, ai, o);
        store_cplx<Mode>(A, i, o);
      }
      nh += mark_hard(A.q, hard, i);
    }
  }
  count_hard(A.q, nh);
}

// ---------------------------------------------------------------------------
// K2s -- tile-sorted, warp-specialised complex streaming kernel
// (`k_svd2_cplx_ws`).
//
// On BASELINE config 4, 10 % of lanes are "wide" (components spanning more
// than kWideSpread binades) and need the exponent-normalised divisions; in
// lane order 97 % of warps hold one, so almost every warp paid for them.
// Here each tile of LT lanes is sorted so the wide lanes fill as few warps
// as possible (about one of LT / 32), and the outputs go through a shared-
// memory staging tile written back with one bulk (TMA) store per output
// train -- whole rows, so regrouped lanes never split a DRAM sector between
// writers (why the register-store regroupings of round 1 lost, DESIGN.md
// section 3).
//
// Warp specialisation keeps the LT / 32 compute warps free of CTA barriers
// (a barrier-per-tile version of this kernel measured 21 % barrier stalls):
// one producer warp per CTA
//   * issues the TMA loads of a kSortStages-deep input ring,
//   * classifies each landed tile (8 components per lane), computes the
//     lane permutation (wide lanes first, from a rotating warp so the wide
//     warp moves across SM sub-partitions) and publishes it (mbarrier plan),
//   * once every compute warp has staged tile k's outputs (mbarrier ofull),
//     issues the tile's 19 bulk stores and hard-lane mask words, and frees
//     the staging tile when the stores have read it (mbarrier oempty).
// A compute warp waits only on data: the plan of its tile (ready a tile
// ahead) and, before staging, the read-out of the previous tile -- so warps
// drift up to one tile apart instead of meeting at a barrier every tile.
// ---------------------------------------------------------------------------
#ifndef B2S_CPLX_SORT
#define B2S_CPLX_SORT 0
#endif
#ifndef B2S_CPLX_SORT4
#define B2S_CPLX_SORT4 0
#endif
#if B2S_CPLX_SORT || B2S_CPLX_SORT4   // measured variants; variant builds only
}  // namespace b2s
#include "b2s_sort_variant.cuh"
namespace b2s {
#endif  // B2S_CPLX_SORT

#if B2S_DIAGNOSTICS
// Tools-only builds (`build.py --out PATH -DB2S_DIAGNOSTICS=1`); the
// product library exports exactly the functions include/b2s.h declares.
// Diagnostic: stream 4 trains through the TMA ring unchanged (tests the
// ring protocol in isolation; `spin` adds per-lane busy work so warps drift
// apart).
__global__ void __launch_bounds__(kBlock, 4) k_ring_probe(const RealArgs A, int spin) {
  extern __shared__ __align__(128) char smem[];
  const double* src[4] = {A.a[0], A.a[1], A.a[2], A.a[3]};
  const int tid = threadIdx.x;
  const int64_t tiles = A.n / kBlock;
  const int64_t mine = tiles > blockIdx.x ? (tiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  TmaRing<4> R;
  R.init(smem, src, mine);
  for (int64_t k = 0; k < mine; k++) {
    const int s = (int)(k % kStages);
    R.wait_full(k);
    double a[4];
    #pragma unroll
    for (int t = 0; t < 4; t++) a[t] = R.stage(s, t)[tid];
    consumed(a);
    R.release(k);
    const int64_t i = R.tile(k) * kBlock + tid;
    double x = a[0];
    const int w = tid >> 5;
    const int reps = spin >= 0 ? spin * (w + 1) : -spin * (kWarps - w) * (1 + (int)((i * 2654435761u) >> 28 & 3));
    for (int r = 0; r < reps; r++) x = __fma_rn(x, 1.0, 0.0);
    A.u[0][i] = x;
    A.u[1][i] = a[1];
    A.u[2][i] = a[2];
    A.u[3][i] = a[3];
    if (A.v[0]) {                          // traffic probe: the SVD kernel's 11 output trains
      #pragma unroll
      for (int t = 0; t < 4; t++) st_stream(A.v[t] + i, a[t]);
      st_stream(A.smax + i, a[0]);
      st_stream(A.smin + i, a[1]);
      st_stream(A.shift + i, a[2]);
    }
  }
}

// Diagnostic: the same traffic shape with the output side staged through
// shared memory and written by bulk (TMA) stores, 11 x 2 KiB per 256-lane
// tile, double-buffered, one CTA barrier per tile.
__global__ void __launch_bounds__(kBlock, 2) k_traffic_bulk(const RealArgs A) {
  extern __shared__ __align__(128) char smem[];
  const double* src[4] = {A.a[0], A.a[1], A.a[2], A.a[3]};
  double* dst[11] = {A.u[0], A.u[1], A.u[2], A.u[3], A.v[0], A.v[1], A.v[2], A.v[3], A.smax, A.smin, A.shift};
  const int tid = threadIdx.x;
  const int64_t tiles = A.n / kBlock;
  const int64_t mine = tiles > blockIdx.x ? (tiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  TmaRing<4> R;
  R.init(smem, src, mine);
  double* stagebuf = reinterpret_cast<double*>(smem + (TmaRing<4>::kSmem + 127) / 128 * 128);
  for (int64_t k = 0; k < mine; k++) {
    const int s = (int)(k % kStages);
    R.wait_full(k);
    double a[4];
    #pragma unroll
    for (int t = 0; t < 4; t++) a[t] = R.stage(s, t)[tid];
    consumed(a);
    R.release(k);
    double* ob = stagebuf + (size_t)(k & 1) * 11 * kBlock;
    #pragma unroll
    for (int t = 0; t < 11; t++) ob[t * kBlock + tid] = a[t & 3];
    tma::fence_proxy_async();
    if (tid == 0) tma::bulk_wait_read<0>();
    __syncthreads();
    if (tid == 0) {
      const int64_t base = R.tile(k) * kBlock;
      #pragma unroll
      for (int t = 0; t < 11; t++) tma::bulk_store(dst[t] + base, ob + t * kBlock, kBlock * 8);
      tma::bulk_commit();
    }
  }
  if (tid == 0) tma::bulk_wait<0>();
}
#endif  // B2S_DIAGNOSTICS

// Exact fix-up of the marked hard lanes.  Each warp scans 32 mask words
// (1024 lanes) at a time and appends their set bits to its shared-memory
// list with a warp prefix sum; whenever 32 lanes are pending it recomputes
// them as one full warp, and the remainder (< 32) at the end.  Hard lanes
// are sparse (0.3 % on BASELINE config 4, ~3 per 1024), so pooling them
// across the warp's chunks keeps its lanes busy: recomputing each chunk's
// few lanes on its own ran the exact pipeline at ~10 % SIMT efficiency.
constexpr int kFixWarps = kBlock / 32;

template <typename Redo>
__device__ __forceinline__ void fix_lanes(const HardQueue& q, int64_t n, Redo redo) {
  __shared__ unsigned list[kFixWarps][1024 + 32];
  if (*q.cnt == 0ull) return;               // the streaming kernel found no hard lane
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t words = (n + 31) >> 5;
  const int64_t nwarps = (int64_t)gridDim.x * kFixWarps;
  int pending = 0;                          // warp-uniform: listed, not yet recomputed (< 32 between chunks)
  for (int64_t base = ((int64_t)blockIdx.x * kFixWarps + warp) * 32; base < words; base += nwarps * 32) {
    const unsigned w = (base + lane < words) ? q.mask[base + lane] : 0u;
    const int c = __popc(w);
    int incl = c;
    #pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const int v = __shfl_up_sync(0xFFFFFFFFu, incl, d);
      if (lane >= d) incl += v;
    }
    const int total = __shfl_sync(0xFFFFFFFFu, incl, 31);
    if (total == 0) continue;
    int pos = pending + incl - c;
    unsigned bitsleft = w;
    while (bitsleft) {
      const int b = __ffs(bitsleft) - 1;
      bitsleft &= bitsleft - 1;
      list[warp][pos++] = (unsigned)(((base + lane) << 5) + b);
    }
    pending += total;
    __syncwarp();
    while (pending >= 32) {                 // full warps from the top of the list
      pending -= 32;
      redo((int64_t)list[warp][pending + lane]);
      __syncwarp();
    }
  }
  if (lane < pending) redo((int64_t)list[warp][lane]);
}

template <int Mode, bool Sine>
__global__ void __launch_bounds__(kBlock) k_fix_real(const RealArgs A) {
  fix_lanes(A.q, A.n, [&](int64_t i) { redo_real<Mode, Sine>(A, i); });
}

template <int Mode, bool Sine>
#ifndef B2S_FIX_MINB
#define B2S_FIX_MINB 1
#endif
__global__ void __launch_bounds__(kBlock, B2S_FIX_MINB) k_fix_cplx(const CplxArgs A) {
  fix_lanes(A.q, A.n, [&](int64_t i) { redo_cplx<Mode, Sine>(A, i); });
}

template <int Mode>
__global__ void __launch_bounds__(kBlock) k_backscale(int64_t n, const double* smax, const double* smin,
                                                     const double* shift, double* omax, double* omin,
                                                     double* oshift) {
  const int64_t stride = (int64_t)gridDim.x * kBlock;
  for (int64_t i = (int64_t)blockIdx.x * kBlock + threadIdx.x; i < n; i += stride) {
    double a = smax[i], b = smin[i], s = shift[i];
    backscale_lane<Mode>(a, b, s);
    omax[i] = a;
    omin[i] = b;
    oshift[i] = s;
  }
}

// Element-wise probe of the engine's inline arithmetic (tests only).  Ops
// with a range-check flag write kHardMarker where the fast path declines.
__device__ __forceinline__ double hard_marker() { return dbl(0x7FF4DEADBEEF0000ull); }

__global__ void __launch_bounds__(kBlock) k_math_probe(int op, int64_t n, const double* a, const double* b,
                                                      double* o) {
  const int64_t stride = (int64_t)gridDim.x * kBlock;
  for (int64_t i = (int64_t)blockIdx.x * kBlock + threadIdx.x; i < n; i += stride) {
    double x = a[i], y = b ? b[i] : 0.0, r;
    bool hard = false;
    switch (op) {
      case 0: r = quot_f(x, y, rcp_f(y)); break;
      case 1: r = sqrt_f(x); break;
      case 2: r = rcp_f(x); break;
      case 3: r = invsqrt_f(x); break;
      case 4: r = hypot_big_f<false>(fabs_(x), fabs_(y), hard); break;
      case 5: r = scale_up(x, (int)y); break;
      case 6: r = div_den<true>(x, make_den(y), hard); break;
      case 9: r = div_pos_big_f<false>(x, y, hard); break;
      case 10: r = div_den<true, false, true, 0>(x, make_den<false>(y), hard); break;
      case 11: r = div_den<true, false, true, 1>(x, make_den<false>(y), hard); break;
      case 12: r = div_den<true, false, true, 2>(x, make_den<false>(y), hard); break;
      case 13: r = div_den<true, false, true, 3>(x, make_den<false>(y), hard); break;
      default: { double c, s; phase_f<false>(x, y, hypot_x(x, y), c, s, hard); r = (op == 7) ? c : s; } break;
    }
    o[i] = hard ? hard_marker() : r;
  }
}

// lanes.py:274-302 assert_fp_env, evaluated by the device's own FP64 units.
__global__ void k_fp_env(const double* in, int* out) {
  double one = in[0], eps = in[1];
  int ok = 1;
  // round to nearest even
  if (!(__dadd_rn(one, eps) == one && __dadd_rn(one, __dmul_rn(2.0, eps)) > one)) ok = 0;
  if (__dadd_rn(one, __dmul_rn(3.0, __dmul_rn(eps, 0.5))) != __dadd_rn(one, __dmul_rn(2.0, eps))) ok = 0;
  // gradual underflow
  double tiny = in[2];
  if (!(tiny > 0.0 && __dmul_rn(tiny, 0.5) == 0.0 && __dmul_rn(__dmul_rn(tiny, 2.0), 0.5) == tiny)) ok = 0;
  // fused multiply-add canary: (1+2^-52)^2 - (1+2^-51) == 2^-104
  double x = __dadd_rn(one, __dmul_rn(eps, 2.0));
  double y = __dadd_rn(one, __dmul_rn(eps, 4.0));
  if (__fma_rn(x, x, -y) != in[3]) ok = 0;
  out[0] = ok;
}

// ---------------------------------------------------------------------------
// launch plumbing
// ---------------------------------------------------------------------------

template <typename K>
static int resident_grid(K kernel, int64_t n) {
  int err = 0;
  return grid_for(kernel, kBlock, n, &err);
}

// Hard-lane mask storage (4 bytes per 32 lanes of one sub-launch) plus the
// launch's counter, one set per (device, stream): launches on different
// streams may run concurrently, so they must not share it.  A launch
// enqueues its counter reset, streaming kernel and fix-up while holding the
// device's workspace lock, so two host threads sharing one stream cannot
// interleave those three either.  Allocated on first use of a stream and
// grown on demand; b2s_reserve_workspace pre-allocates (before CUDA-graph
// capture, where allocation is not allowed).
struct LaneQueue {
  cudaStream_t stream;
  unsigned* mask = nullptr;
  unsigned long long* cnt = nullptr;
  size_t words = 0;
};

struct Workspace {
  std::mutex mu;
  std::vector<LaneQueue> queues;
  int last = -1;                       // queue of the most recent launch
};

static Workspace& workspace(int dev) {
  static Workspace ws[64];
  return ws[dev & 63];
}

constexpr int64_t kMaxLaunch = int64_t(1) << 31;     // lanes per sub-launch

// Lanes per sub-launch: kMaxLaunch, or B2S_MAX_LAUNCH (a multiple of 256,
// read once) so tests can cross sub-launch boundaries with small batches.
static int64_t max_launch() {
  static const int64_t v = [] {
    const char* e = getenv("B2S_MAX_LAUNCH");
    const long long x = e ? atoll(e) : 0;
    return (x >= 256 && x % 256 == 0 && x <= kMaxLaunch) ? (int64_t)x : kMaxLaunch;
  }();
  return v;
}

// Debug / A-B switches read once from the environment (e.g. B2S_NO_TMA=1
// selects the register-prefetch streaming kernels).
static bool getenv_flag(const char* name) {
  const char* v = getenv(name);
  return v && *v && *v != '0';
}

// The queue of stream `s` on the current device, large enough for n lanes.
// Caller holds the device workspace lock.
static int get_queue(Workspace& w, cudaStream_t s, int64_t n, HardQueue* q) {
  int k = -1;
  for (size_t j = 0; j < w.queues.size(); j++)
    if (w.queues[j].stream == s) k = (int)j;
  if (k < 0) {
    w.queues.push_back(LaneQueue{s});
    k = (int)w.queues.size() - 1;
  }
  LaneQueue& Q = w.queues[k];
  size_t want = (size_t)((n + 31) / 32);
  if (want < 4096) want = 4096;
  if (!Q.cnt) B2S_CUDA(cudaMalloc(&Q.cnt, sizeof(unsigned long long)));
  if (Q.words < want) {
    if (Q.mask) {
      B2S_CUDA(cudaStreamSynchronize(s));          // earlier launches on s may still read it
      cudaFree(Q.mask);
    }
    Q.mask = nullptr;
    Q.words = 0;
    B2S_CUDA(cudaMalloc(&Q.mask, want * sizeof(unsigned)));
    Q.words = want;
  }
  q->mask = Q.mask;
  q->cnt = Q.cnt;
  w.last = k;
  return 0;
}

static Workspace& current_workspace() {
  int dev = 0;
  cudaGetDevice(&dev);
  return workspace(dev);
}

static inline bool a16(const void* p) { return ((uintptr_t)p & 15u) == 0; }

static bool tma_ok_real(const RealArgs& A) {
  if (getenv_flag("B2S_NO_TMA")) return false;
  for (int t = 0; t < 4; t++) if (!a16(A.a[t])) return false;
  return true;
}

static bool tma_ok_cplx(const CplxArgs& A) {
  if (getenv_flag("B2S_NO_TMA")) return false;
  for (int t = 0; t < 4; t++) if (!a16(A.ar[t]) || !a16(A.ai[t])) return false;
  return true;
}

// Persistent grid: SMs x resident CTAs (registers and shared memory).
template <typename K>
static int tma_grid(K kernel, size_t smem, int64_t n) {
  int dev = 0, sms = 148, per_sm = 1;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, kBlock, smem);
  if (per_sm < 1) per_sm = 1;
  int64_t tiles = n / kBlock;
  int64_t g = (int64_t)sms * per_sm;
  if (tiles < g) g = tiles;
  return g < 1 ? 1 : (int)g;
}

template <int Mode, bool Sine, bool States>
static int launch_real(RealArgs A, cudaStream_t s) {
  const int64_t total = A.n;
  Workspace& W = current_workspace();
  std::unique_lock<std::mutex> lock(W.mu, std::defer_lock);
  if (!States) lock.lock();                       // see LaneQueue
  const RealArgs base = A;
  const int64_t step = max_launch();
  for (int64_t lo = 0; lo < total; lo += step) {
    A = base;
    A.n = (total - lo) < step ? (total - lo) : step;
    for (int t = 0; t < 4; t++) { A.u[t] += lo; A.v[t] += lo; }
    if (A.aos) A.a[0] += lo * 4;                 // 32 doubles per 8 lanes
    else for (int t = 0; t < 4; t++) A.a[t] += lo;
    A.smax += lo; A.smin += lo; A.shift += lo;
    if (States) for (int k = 0; k < (A.full_states ? B2S_STATES_REAL_FULL : B2S_STATES_REAL); k++) A.st[k] += lo;
    if (!States) {
      int rc = get_queue(W, s, A.n, &A.q);
      if (rc) return rc;
      B2S_CUDA(cudaMemsetAsync(A.q.cnt, 0, sizeof(unsigned long long), s));
    }
    if (!States && (A.aos || tma_ok_real(A))) {
      auto k = A.aos ? k_svd2_real_tma<Mode, Sine, true> : k_svd2_real_tma<Mode, Sine, false>;
      const size_t sm = TmaRing<4>::kSmem;
      B2S_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
      k<<<tma_grid(k, sm, A.n), kBlock, sm, s>>>(A);
      const int64_t head = A.n / kBlock * kBlock;
      if (!B2S_TMA_TAIL_REAL && head < A.n) {
        RealArgs T = A;
        T.n = A.n - head;
        for (int t = 0; t < 4; t++) { T.u[t] += head; T.v[t] += head; }
        if (T.aos) T.a[0] += head * 4;
        else for (int t = 0; t < 4; t++) T.a[t] += head;
        T.smax += head; T.smin += head; T.shift += head;
        T.q.mask += head >> 5;
        k_svd2_real<Mode, Sine, false><<<1, kBlock, 0, s>>>(T);
      }
    } else {
      auto k = k_svd2_real<Mode, Sine, States>;
      k<<<resident_grid(k, A.n), kBlock, 0, s>>>(A);
    }
    B2S_CUDA(cudaGetLastError());
    if (!States) {
      auto f = k_fix_real<Mode, Sine>;
      f<<<resident_grid(f, (int64_t)kBlock * 148 * 4), kBlock, 0, s>>>(A);
      B2S_CUDA(cudaGetLastError());
    }
  }
  return 0;
}

template <int Mode, bool Sine, bool States>
static int launch_cplx(CplxArgs A, cudaStream_t s) {
  const int64_t total = A.n;
  Workspace& W = current_workspace();
  std::unique_lock<std::mutex> lock(W.mu, std::defer_lock);
  if (!States) lock.lock();                       // see LaneQueue
  const CplxArgs base = A;
  const int64_t step = max_launch();
  for (int64_t lo = 0; lo < total; lo += step) {
    A = base;
    A.n = (total - lo) < step ? (total - lo) : step;
    for (int t = 0; t < 4; t++) { A.ur[t] += lo; A.ui[t] += lo; A.vr[t] += lo; A.vi[t] += lo; }
    if (A.aos) A.ar[0] += lo * 8;                // 64 doubles per 8 lanes
    else for (int t = 0; t < 4; t++) { A.ar[t] += lo; A.ai[t] += lo; }
    A.smax += lo; A.smin += lo; A.shift += lo;
    if (States) for (int k = 0; k < (A.full_states ? B2S_STATES_COMPLEX_FULL : B2S_STATES_COMPLEX); k++) A.st[k] += lo;
    if (!States) {
      int rc = get_queue(W, s, A.n, &A.q);
      if (rc) return rc;
      B2S_CUDA(cudaMemsetAsync(A.q.cnt, 0, sizeof(unsigned long long), s));
    }
#if B2S_CPLX_SORT4
    if (!States && !A.aos && tma_ok_cplx(A) && !getenv_flag("B2S_NO_SORT")) {
      auto k = k_svd2_cplx_u4<Mode, Sine>;
      const size_t sm = U4Layout::kSmem;
      B2S_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
      int dev = 0, sms = 148, per_sm = 1;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, U4Layout::LT + 32, sm);
      const int64_t tiles = A.n / U4Layout::LT;
      int64_t g = (int64_t)sms * (per_sm < 1 ? 1 : per_sm);
      if (tiles < g) g = tiles;
      const int64_t head = tiles * U4Layout::LT;
      B2S_CUDA(cudaMemsetAsync(A.q.mask, 0, (size_t)(head >> 5) * sizeof(unsigned), s));
      if (g > 0) k<<<(int)g, U4Layout::LT + 32, sm, s>>>(A);
      if (head < A.n) {
        CplxArgs T = A;
        T.n = A.n - head;
        for (int t = 0; t < 4; t++) { T.ur[t] += head; T.ui[t] += head; T.vr[t] += head; T.vi[t] += head; }
        for (int t = 0; t < 4; t++) { T.ar[t] += head; T.ai[t] += head; }
        T.smax += head; T.smin += head; T.shift += head;
        T.q.mask += head >> 5;
        k_svd2_complex<Mode, Sine, false><<<1, kBlock, 0, s>>>(T);
      }
    } else
#endif
#if B2S_CPLX_SORT
    if (!States && !A.aos && tma_ok_cplx(A) && !getenv_flag("B2S_NO_SORT")) {
      constexpr int LT = B2S_CPLX_SORT > 0 ? B2S_CPLX_SORT : 128;
      auto k = k_svd2_cplx_ws<Mode, Sine, LT>;
      const size_t sm = WsLayout<LT>::kSmem;
      B2S_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
      int dev = 0, sms = 148, per_sm = 1;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, LT + 32, sm);
      const int64_t tiles = A.n / LT;
      int64_t g = (int64_t)sms * (per_sm < 1 ? 1 : per_sm);
      if (tiles < g) g = tiles;
      if (g > 0) k<<<(int)g, LT + 32, sm, s>>>(A);
      const int64_t head = tiles * LT;
      if (head < A.n) {                           // sub-tile tail: one CTA of the LDG kernel
        CplxArgs T = A;
        T.n = A.n - head;
        for (int t = 0; t < 4; t++) { T.ur[t] += head; T.ui[t] += head; T.vr[t] += head; T.vi[t] += head; }
        for (int t = 0; t < 4; t++) { T.ar[t] += head; T.ai[t] += head; }
        T.smax += head; T.smin += head; T.shift += head;
        T.q.mask += head >> 5;
        k_svd2_complex<Mode, Sine, false><<<1, kBlock, 0, s>>>(T);
      }
    } else
#endif
    if (!States && (A.aos || tma_ok_cplx(A))) {
      auto k = A.aos ? k_svd2_cplx_tma<Mode, Sine, true> : k_svd2_cplx_tma<Mode, Sine, false>;
      const size_t sm = TmaRing<8, kBlock, B2S_CPLX_STAGES>::kSmem;
      B2S_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
      k<<<tma_grid(k, sm, A.n), kBlock, sm, s>>>(A);
      const int64_t head = A.n / kBlock * kBlock;
      if (!B2S_TMA_TAIL_CPLX && head < A.n) {
        CplxArgs T = A;
        T.n = A.n - head;
        for (int t = 0; t < 4; t++) { T.ur[t] += head; T.ui[t] += head; T.vr[t] += head; T.vi[t] += head; }
        if (T.aos) T.ar[0] += head * 8;
        else for (int t = 0; t < 4; t++) { T.ar[t] += head; T.ai[t] += head; }
        T.smax += head; T.smin += head; T.shift += head;
        T.q.mask += head >> 5;
        k_svd2_complex<Mode, Sine, false><<<1, kBlock, 0, s>>>(T);
      }
    } else {
      auto k = k_svd2_complex<Mode, Sine, States>;
      k<<<resident_grid(k, A.n), kBlock, 0, s>>>(A);
    }
    B2S_CUDA(cudaGetLastError());
    if (!States) {
      auto f = k_fix_cplx<Mode, Sine>;
      f<<<resident_grid(f, (int64_t)kBlock * 148 * 4), kBlock, 0, s>>>(A);
      B2S_CUDA(cudaGetLastError());
    }
  }
  return 0;
}

#define B2S_DISPATCH(LAUNCH, A, mode, sine, states, s)                                   \
  do {                                                                                   \
    if (states) {                                                                        \
      if (sine) {                                                                        \
        if (mode == 0) return LAUNCH<0, true, true>(A, s);                               \
        if (mode == 1) return LAUNCH<1, true, true>(A, s);                               \
        return LAUNCH<2, true, true>(A, s);                                              \
      }                                                                                  \
      if (mode == 0) return LAUNCH<0, false, true>(A, s);                                \
      if (mode == 1) return LAUNCH<1, false, true>(A, s);                                \
      return LAUNCH<2, false, true>(A, s);                                               \
    }                                                                                    \
    if (sine) {                                                                          \
      if (mode == 0) return LAUNCH<0, true, false>(A, s);                                \
      if (mode == 1) return LAUNCH<1, true, false>(A, s);                                \
      return LAUNCH<2, true, false>(A, s);                                               \
    }                                                                                    \
    if (mode == 0) return LAUNCH<0, false, false>(A, s);                                 \
    if (mode == 1) return LAUNCH<1, false, false>(A, s);                                 \
    return LAUNCH<2, false, false>(A, s);                                                \
  } while (0)

int check_common(int64_t n, int mode, int flags, double* const* states) {
  if (n < 0) return fail(1, "negative batch size %lld", (long long)n);
  if (mode < 0 || mode > 2) return fail(2, "backscale_mode must be 0 (none), 1 (safe) or 2 (unconditional), got %d", mode);
  if (flags & ~(B2S_FLAG_SINE_FORM | B2S_FLAG_STATES | B2S_FLAG_STATES_FULL))
    return fail(3, "unknown flag bits 0x%x", flags);
  if ((flags & B2S_FLAG_STATES) && !states) return fail(4, "B2S_FLAG_STATES needs a states train array");
  if ((flags & B2S_FLAG_STATES_FULL) && !(flags & B2S_FLAG_STATES))
    return fail(3, "B2S_FLAG_STATES_FULL needs B2S_FLAG_STATES");
  return 0;
}

#define B2S_CHECK_PTR(p, what)                                                \
  do {                                                                        \
    if (!(p)) return fail(5, "%s is NULL", what);                              \
    if (!aligned8(p)) return fail(6, "%s is not 8-byte aligned", what);     \
  } while (0)

int real_entry(int64_t n, const double* const a[4], double* const u[4], double* const v[4], double* smax,
               double* smin, double* shift, int mode, int flags, double* const* states, cudaStream_t s,
               int aos = 0) {
  int rc = check_common(n, mode, flags, states);
  if (rc) return rc;
  if (!a || !u || !v) return fail(5, "train pointer array is NULL");
  RealArgs A{};
  A.n = n;
  A.aos = aos;
  for (int t = 0; t < 4; t++) {
    B2S_CHECK_PTR(a[t], "input train");
    B2S_CHECK_PTR(u[t], "u train");
    B2S_CHECK_PTR(v[t], "v train");
    A.a[t] = a[t]; A.u[t] = u[t]; A.v[t] = v[t];
  }
  B2S_CHECK_PTR(smax, "smax"); B2S_CHECK_PTR(smin, "smin"); B2S_CHECK_PTR(shift, "shift");
  A.smax = smax; A.smin = smin; A.shift = shift;
  bool st = flags & B2S_FLAG_STATES;
  if (st) {
    A.full_states = (flags & B2S_FLAG_STATES_FULL) != 0;
    for (int k = 0; k < (A.full_states ? B2S_STATES_REAL_FULL : B2S_STATES_REAL); k++) {
      B2S_CHECK_PTR(states[k], "state train");
      A.st[k] = states[k];
    }
  }
  if (n == 0) return 0;
  bool sine = flags & B2S_FLAG_SINE_FORM;
  B2S_DISPATCH(launch_real, A, mode, sine, st, s);
}

int cplx_entry(int64_t n, const double* const ar[4], const double* const ai[4], double* const ur[4],
               double* const ui[4], double* const vr[4], double* const vi[4], double* smax, double* smin,
               double* shift, int mode, int flags, double* const* states, cudaStream_t s, int aos = 0) {
  int rc = check_common(n, mode, flags, states);
  if (rc) return rc;
  if (!ar || !ai || !ur || !ui || !vr || !vi) return fail(5, "train pointer array is NULL");
  CplxArgs A{};
  A.n = n;
  A.aos = aos;
  for (int t = 0; t < 4; t++) {
    B2S_CHECK_PTR(ar[t], "input re train"); B2S_CHECK_PTR(ai[t], "input im train");
    B2S_CHECK_PTR(ur[t], "u_re train"); B2S_CHECK_PTR(ui[t], "u_im train");
    B2S_CHECK_PTR(vr[t], "v_re train"); B2S_CHECK_PTR(vi[t], "v_im train");
    A.ar[t] = ar[t]; A.ai[t] = ai[t]; A.ur[t] = ur[t]; A.ui[t] = ui[t]; A.vr[t] = vr[t]; A.vi[t] = vi[t];
  }
  B2S_CHECK_PTR(smax, "smax"); B2S_CHECK_PTR(smin, "smin"); B2S_CHECK_PTR(shift, "shift");
  A.smax = smax; A.smin = smin; A.shift = shift;
  bool st = flags & B2S_FLAG_STATES;
  if (st) {
    A.full_states = (flags & B2S_FLAG_STATES_FULL) != 0;
    for (int k = 0; k < (A.full_states ? B2S_STATES_COMPLEX_FULL : B2S_STATES_COMPLEX); k++) {
      B2S_CHECK_PTR(states[k], "state train");
      A.st[k] = states[k];
    }
  }
  if (n == 0) return 0;
  bool sine = flags & B2S_FLAG_SINE_FORM;
  B2S_DISPATCH(launch_cplx, A, mode, sine, st, s);
}

}  // namespace b2s

using namespace b2s;

extern "C" {

int b2s_version(void) { return 100; }

const char* b2s_last_error(void) { return last_error_buf(); }

int b2s_svd2_real(int64_t n, const double* const a[4], double* const u[4], double* const v[4], double* smax,
                  double* smin, double* shift, int backscale_mode, int flags, double* const* states,
                  void* stream) {
  return real_entry(n, a, u, v, smax, smin, shift, backscale_mode, flags, states, (cudaStream_t)stream);
}

int b2s_svd2_complex(int64_t n, const double* const a_re[4], const double* const a_im[4], double* const u_re[4],
                     double* const u_im[4], double* const v_re[4], double* const v_im[4], double* smax,
                     double* smin, double* shift, int backscale_mode, int flags, double* const* states,
                     void* stream) {
  return cplx_entry(n, a_re, a_im, u_re, u_im, v_re, v_im, smax, smin, shift, backscale_mode, flags, states,
                    (cudaStream_t)stream);
}

int b2s_svd2_real_records(int64_t n, const double* records, double* const u[4], double* const v[4],
                          double* smax, double* smin, double* shift, int backscale_mode, int flags,
                          void* stream) {
  if (flags & B2S_FLAG_STATES) return fail(3, "state dumps need SoA trains (b2s_svd2_real)");
  if (!records) return fail(5, "records is NULL");
  if (((uintptr_t)records & 15u) != 0) return fail(6, "records must be 16-byte aligned");
  const double* a[4] = {records, records, records, records};
  return real_entry(n, a, u, v, smax, smin, shift, backscale_mode, flags, nullptr, (cudaStream_t)stream, 1);
}

int b2s_svd2_complex_records(int64_t n, const double* records, double* const u_re[4], double* const u_im[4],
                             double* const v_re[4], double* const v_im[4], double* smax, double* smin,
                             double* shift, int backscale_mode, int flags, void* stream) {
  if (flags & B2S_FLAG_STATES) return fail(3, "state dumps need SoA trains (b2s_svd2_complex)");
  if (!records) return fail(5, "records is NULL");
  if (((uintptr_t)records & 15u) != 0) return fail(6, "records must be 16-byte aligned");
  const double* a[4] = {records, records, records, records};
  return cplx_entry(n, a, a, u_re, u_im, v_re, v_im, smax, smin, shift, backscale_mode, flags, nullptr,
                    (cudaStream_t)stream, 1);
}

int b2s_backscale(int64_t n, const double* smax, const double* smin, const double* shift, int backscale_mode,
                  double* out_smax, double* out_smin, double* out_shift, void* stream) {
  if (n < 0) return fail(1, "negative batch size");
  if (backscale_mode < 0 || backscale_mode > 2) return fail(2, "unknown backscale mode %d", backscale_mode);
  if (!smax || !smin || !shift || !out_smax || !out_smin || !out_shift) return fail(5, "NULL train");
  if (n == 0) return 0;
  cudaStream_t s = (cudaStream_t)stream;
  int err = 0;
  if (backscale_mode == 0) {
    int g = grid_for(k_backscale<0>, kBlock, n, &err);
    k_backscale<0><<<g, kBlock, 0, s>>>(n, smax, smin, shift, out_smax, out_smin, out_shift);
  } else if (backscale_mode == 1) {
    int g = grid_for(k_backscale<1>, kBlock, n, &err);
    k_backscale<1><<<g, kBlock, 0, s>>>(n, smax, smin, shift, out_smax, out_smin, out_shift);
  } else {
    int g = grid_for(k_backscale<2>, kBlock, n, &err);
    k_backscale<2><<<g, kBlock, 0, s>>>(n, smax, smin, shift, out_smax, out_smin, out_shift);
  }
  B2S_CUDA(cudaGetLastError());
  return 0;
}

int b2s_math_probe(int op, int64_t n, const double* a, const double* b, double* out, void* stream) {
  if (op < 0 || op > 13) return fail(1, "unknown probe op %d", op);
  if (n < 0) return fail(1, "negative n");
  if (!a || !out || ((op == 0 || op >= 4) && !b)) return fail(5, "NULL operand");
  if (n == 0) return 0;
  int err = 0;
  int g = grid_for(k_math_probe, kBlock, n, &err);
  k_math_probe<<<g, kBlock, 0, (cudaStream_t)stream>>>(op, n, a, b, out);
  B2S_CUDA(cudaGetLastError());
  return 0;
}

int b2s_reserve_workspace(int device, int64_t lanes, void* stream) {
  if (lanes < 0) return fail(1, "negative lane count");
  if (lanes > kMaxLaunch) lanes = kMaxLaunch;
  int prev = 0;
  B2S_CUDA(cudaGetDevice(&prev));
  B2S_CUDA(cudaSetDevice(device));
  Workspace& w = workspace(device);
  HardQueue q;
  int rc;
  {
    std::lock_guard<std::mutex> lock(w.mu);
    rc = get_queue(w, (cudaStream_t)stream, lanes, &q);
  }
  cudaSetDevice(prev);
  return rc;
}

long long b2s_hard_lane_count(int device) {
  int prev = 0;
  if (cudaGetDevice(&prev) != cudaSuccess) return -1;
  if (cudaSetDevice(device) != cudaSuccess) return -1;
  Workspace& w = workspace(device);
  unsigned long long c = 0;
  long long out = 0;
  unsigned long long* cnt = nullptr;
  {
    std::lock_guard<std::mutex> lock(w.mu);
    if (w.last >= 0) cnt = w.queues[w.last].cnt;
  }
  if (cnt) {
    if (cudaDeviceSynchronize() != cudaSuccess ||
        cudaMemcpy(&c, cnt, sizeof c, cudaMemcpyDeviceToHost) != cudaSuccess)
      out = -1;
    else
      out = (long long)c;
  }
  cudaSetDevice(prev);
  return out;
}

#if B2S_DIAGNOSTICS
int b2s_traffic_bulk(int64_t n, const double* const a[4], double* const out[11], void* stream) {
  RealArgs A{};
  A.n = n;
  for (int t = 0; t < 4; t++) { A.a[t] = a[t]; A.u[t] = out[t]; A.v[t] = out[4 + t]; }
  A.smax = out[8]; A.smin = out[9]; A.shift = out[10];
  const size_t sm = (TmaRing<4>::kSmem + 127) / 128 * 128 + 2 * 11 * kBlock * sizeof(double);
  B2S_CUDA(cudaFuncSetAttribute(k_traffic_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
  k_traffic_bulk<<<tma_grid(k_traffic_bulk, sm, n), kBlock, sm, (cudaStream_t)stream>>>(A);
  B2S_CUDA(cudaGetLastError());
  return 0;
}

// Diagnostic (tests / tools): spin == 1000000 selects the 11-output traffic
// probe (out[0..10]), otherwise the 4-train ring copy with busy work.
int b2s_ring_probe(int64_t n, const double* const a[4], double* const out[11], int spin, void* stream) {
  RealArgs A{};
  A.n = n;
  for (int t = 0; t < 4; t++) { A.a[t] = a[t]; A.u[t] = out[t]; A.v[t] = spin == 1000000 ? out[4 + t] : nullptr; }
  if (spin == 1000000) { A.smax = out[8]; A.smin = out[9]; A.shift = out[10]; spin = 0; }
  const size_t sm = TmaRing<4>::kSmem;
  B2S_CUDA(cudaFuncSetAttribute(k_ring_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
  k_ring_probe<<<tma_grid(k_ring_probe, sm, n), kBlock, sm, (cudaStream_t)stream>>>(A, spin);
  B2S_CUDA(cudaGetLastError());
  return 0;
}
#endif  // B2S_DIAGNOSTICS

int b2s_check_fp_env(int device) {
  int prev = 0;
  B2S_CUDA(cudaGetDevice(&prev));
  B2S_CUDA(cudaSetDevice(device));
  const double h_in[4] = {1.0, 0x1p-53, 0x1p-1074, 0x1p-104};
  double* d_in = nullptr;
  int* d_out = nullptr;
  int ok = 0;
  cudaError_t e = cudaMalloc(&d_in, sizeof h_in);
  if (e == cudaSuccess) e = cudaMalloc(&d_out, sizeof(int));
  if (e == cudaSuccess) e = cudaMemcpy(d_in, h_in, sizeof h_in, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) {
    k_fp_env<<<1, 1>>>(d_in, d_out);
    e = cudaGetLastError();
  }
  if (e == cudaSuccess) e = cudaMemcpy(&ok, d_out, sizeof(int), cudaMemcpyDeviceToHost);
  cudaFree(d_in);
  cudaFree(d_out);
  cudaSetDevice(prev);
  if (e != cudaSuccess) return cuda_fail(e, "b2s_check_fp_env");
  return ok ? 0 : fail(7, "device FP environment check failed (rounding, gradual underflow or fma)");
}

}  // extern "C"
