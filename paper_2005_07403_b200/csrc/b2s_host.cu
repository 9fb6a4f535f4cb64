// b2s_host.cu -- host-buffer entry points: the reference-facing call path.
//
// b2s_svd2_{real,complex}_host take HOST trains (what a ctypes binding of
// lanesvd.driver.run_batch, driver.py:149-190, holds) and stream the batch
// through one GPU: per chunk, copy-in of the input trains, the fused SVD
// kernel, copy-out of the output trains, round-robin over three streams so
// the H2D of chunk c+1, the kernel of chunk c and the D2H of chunk c-1
// overlap.  Device staging buffers are cached per device between calls.
//
// Pageable host trains (a lanesvd caller's aligned_zeros arrays,
// layout.py:42-51) cannot be copied asynchronously: cudaMemcpyAsync from
// pageable memory is staged synchronously by the driver and the copy /
// compute / copy overlap collapses.  When any train is pageable the
// pipeline bounces every chunk through per-stage pinned host buffers
// instead, filled and drained by the host cores in parallel (OpenMP) while
// the GPU streams other stages -- no page pinning of the caller's memory.
#include <emmintrin.h>
#include <omp.h>

#include <cstdlib>

#include <mutex>
#include <vector>

#include "../../include/b2s.h"
#include "b2s_common.cuh"

namespace b2s {

constexpr int kStages = 3;

struct DeviceCtx {
  std::mutex mu;
  bool init = false;
  cudaStream_t streams[kStages];
  cudaEvent_t done[kStages];
  double* buf[kStages] = {nullptr, nullptr, nullptr};
  size_t buf_bytes = 0;
  double* hbuf[kStages] = {nullptr, nullptr, nullptr};   // pinned bounce buffers (pageable callers)
  size_t hbuf_bytes = 0;
};

static bool pageable(const void* p) {
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return true;
  }
  return at.type == cudaMemoryTypeUnregistered;
}

static int ensure_host(DeviceCtx& c, size_t bytes) {
  if (c.hbuf_bytes >= bytes) return 0;
  for (int s = 0; s < kStages; s++) {
    if (c.hbuf[s]) cudaFreeHost(c.hbuf[s]);
    c.hbuf[s] = nullptr;
  }
  c.hbuf_bytes = 0;
  for (int s = 0; s < kStages; s++) B2S_CUDA(cudaMallocHost(&c.hbuf[s], bytes));
  c.hbuf_bytes = bytes;
  return 0;
}

// Copy with non-temporal (streaming) stores: the destination lines are not
// read for ownership first, so a copy moves 2x its size through host DRAM
// instead of 3x -- the bounce pipeline is bound by exactly this traffic.
static void stream_copy(double* dst, const double* src, int64_t n) {
  int64_t i = 0;
  for (; i < n && ((uintptr_t)(dst + i) & 15u); i++) dst[i] = src[i];    // align the destination
  const int64_t body = i + ((n - i) & ~(int64_t)7);
  for (; i < body; i += 8) {
    const __m128d a = _mm_loadu_pd(src + i), b = _mm_loadu_pd(src + i + 2);
    const __m128d c = _mm_loadu_pd(src + i + 4), d = _mm_loadu_pd(src + i + 6);
    _mm_stream_pd(dst + i, a);
    _mm_stream_pd(dst + i + 2, b);
    _mm_stream_pd(dst + i + 4, c);
    _mm_stream_pd(dst + i + 6, d);
  }
  for (; i < n; i++) dst[i] = src[i];
  _mm_sfence();                                     // this thread's streaming stores, before the barrier
}

// Host threads for the bounce copies: B2S_COPY_THREADS if set, else the
// host's cores shared among the processes of one node (LOCAL_WORLD_SIZE,
// set by torchrun -- which also sets OMP_NUM_THREADS=1, so the OpenMP
// default would leave every rank with one copy thread).
static int copy_threads() {
  static int n = 0;
  if (n == 0) {
    const char* e = std::getenv("B2S_COPY_THREADS");
    int t = e ? std::atoi(e) : 0;
    if (t <= 0) {
      const char* l = std::getenv("LOCAL_WORLD_SIZE");
      const int ranks = l ? std::atoi(l) : 1;
      t = omp_get_num_procs() / (ranks > 0 ? ranks : 1);
    }
    n = t > 0 ? t : 1;
  }
  return n;
}

// Parallel copy of `ntr` trains' chunks (host cores; each train split into
// 1 MiB pieces so every thread has work).
static void par_copy(int ntr, double* const* dst, const double* const* src, int64_t m) {
  const int64_t piece = 1 << 17;                     // doubles
  const int64_t per = (m + piece - 1) / piece;
  const int64_t total = per * ntr;
  const int nt = copy_threads();
  #pragma omp parallel for schedule(static) num_threads(nt)
  for (int64_t w = 0; w < total; w++) {
    const int t = (int)(w / per);
    const int64_t lo = (w % per) * piece;
    const int64_t len = (m - lo) < piece ? (m - lo) : piece;
    stream_copy(dst[t] + lo, src[t] + lo, len);
  }
}

static DeviceCtx& ctx_for(int dev) {
  static DeviceCtx ctxs[64];
  return ctxs[dev & 63];
}

static int ensure(DeviceCtx& c, size_t bytes) {
  if (!c.init) {
    for (int s = 0; s < kStages; s++) {
      B2S_CUDA(cudaStreamCreateWithFlags(&c.streams[s], cudaStreamNonBlocking));
      B2S_CUDA(cudaEventCreateWithFlags(&c.done[s], cudaEventDisableTiming));
    }
    c.init = true;
  }
  if (c.buf_bytes < bytes) {
    for (int s = 0; s < kStages; s++) {
      if (c.buf[s]) cudaFree(c.buf[s]);
      c.buf[s] = nullptr;
    }
    c.buf_bytes = 0;
    for (int s = 0; s < kStages; s++) B2S_CUDA(cudaMalloc(&c.buf[s], bytes));
    c.buf_bytes = bytes;
  }
  return 0;
}

// Chunked pipeline through pinned bounce buffers: chunk k's inputs are
// copied into stage k % 3's pinned buffer by the host cores, streamed in,
// decomposed and streamed back into the same stage's pinned buffer; its
// outputs are copied to the caller when the stage comes round again (or at
// the end), so host copies of one stage overlap the GPU work of the others.
template <typename Launch>
static int bounce_pipeline(DeviceCtx& c, int64_t n, int64_t chunk, int n_in, const double* const* in,
                           int n_out, double* const* out, Launch launch) {
  const int64_t nchunks = (n + chunk - 1) / chunk;
  std::vector<const double*> src(n_in > n_out ? n_in : n_out);
  std::vector<double*> dst(n_in > n_out ? n_in : n_out);
  auto drain = [&](int64_t k) -> int {                 // chunk k's outputs -> caller
    const int s = (int)(k % kStages);
    B2S_CUDA(cudaEventSynchronize(c.done[s]));
    const int64_t lo = k * chunk;
    const int64_t m = (n - lo) < chunk ? (n - lo) : chunk;
    for (int t = 0; t < n_out; t++) {
      src[t] = c.hbuf[s] + (size_t)(n_in + t) * chunk;
      dst[t] = out[t] + lo;
    }
    par_copy(n_out, dst.data(), src.data(), m);
    return 0;
  };
  for (int64_t k = 0; k < nchunks; k++) {
    const int s = (int)(k % kStages);
    cudaStream_t st = c.streams[s];
    if (k >= kStages) {
      int rc = drain(k - kStages);
      if (rc) return rc;
    }
    const int64_t lo = k * chunk;
    const int64_t m = (n - lo) < chunk ? (n - lo) : chunk;
    const size_t mb = (size_t)m * sizeof(double);
    for (int t = 0; t < n_in; t++) {
      src[t] = in[t] + lo;
      dst[t] = c.hbuf[s] + (size_t)t * chunk;
    }
    par_copy(n_in, dst.data(), src.data(), m);
    std::vector<const double*> din(n_in);
    std::vector<double*> dout(n_out);
    for (int t = 0; t < n_in; t++) {
      double* d = c.buf[s] + (size_t)t * chunk;
      B2S_CUDA(cudaMemcpyAsync(d, c.hbuf[s] + (size_t)t * chunk, mb, cudaMemcpyHostToDevice, st));
      din[t] = d;
    }
    for (int t = 0; t < n_out; t++) dout[t] = c.buf[s] + (size_t)(n_in + t) * chunk;
    int rc = launch(m, din.data(), dout.data(), st);
    if (rc) return rc;
    for (int t = 0; t < n_out; t++)
      B2S_CUDA(cudaMemcpyAsync(c.hbuf[s] + (size_t)(n_in + t) * chunk, dout[t], mb, cudaMemcpyDeviceToHost,
                               st));
    B2S_CUDA(cudaEventRecord(c.done[s], st));
  }
  for (int64_t k = nchunks > kStages ? nchunks - kStages : 0; k < nchunks; k++) {
    int rc = drain(k);
    if (rc) return rc;
  }
  return 0;
}

// Generic chunked pipeline. n_in input trains, n_out output trains; `launch`
// runs the device entry on the staged chunk.
template <typename Launch>
static int pipeline(int64_t n, int device, int64_t chunk, int n_in, const double* const* in, int n_out,
                    double* const* out, Launch launch) {
  if (n < 0) return fail(1, "negative batch size");
  if (n == 0) return 0;
  int ndev = 0;
  B2S_CUDA(cudaGetDeviceCount(&ndev));
  if (device < 0 || device >= ndev) return fail(8, "device %d out of range (have %d)", device, ndev);
  int prev = 0;
  B2S_CUDA(cudaGetDevice(&prev));
  struct Restore {
    int dev;
    ~Restore() { cudaSetDevice(dev); }
  } restore{prev};                                  // the caller's current device survives the call
  B2S_CUDA(cudaSetDevice(device));
  if (chunk <= 0) chunk = 1 << 22;
  chunk = (chunk + 255) / 256 * 256;
  if (chunk > n) chunk = (n + 1) / 2 * 2;
  const int trains = n_in + n_out;
  const size_t tbytes = (size_t)chunk * sizeof(double);
  DeviceCtx& c = ctx_for(device);
  std::lock_guard<std::mutex> lock(c.mu);
  int rc = ensure(c, tbytes * trains);
  if (rc) return rc;
  const int64_t nchunks = (n + chunk - 1) / chunk;
  bool bounce = false;
  for (int t = 0; t < n_in; t++) bounce |= pageable(in[t]);
  for (int t = 0; t < n_out; t++) bounce |= pageable(out[t]);
  if (bounce) {
    rc = ensure_host(c, tbytes * trains);
    if (rc) return rc;
    return bounce_pipeline(c, n, chunk, n_in, in, n_out, out, launch);
  }
  for (int64_t k = 0; k < nchunks; k++) {
    const int s = (int)(k % kStages);
    cudaStream_t st = c.streams[s];
    const int64_t lo = k * chunk;
    const int64_t m = (n - lo) < chunk ? (n - lo) : chunk;
    const size_t mb = (size_t)m * sizeof(double);
    std::vector<const double*> din(n_in);
    std::vector<double*> dout(n_out);
    for (int t = 0; t < n_in; t++) {
      double* d = c.buf[s] + (size_t)t * chunk;
      B2S_CUDA(cudaMemcpyAsync(d, in[t] + lo, mb, cudaMemcpyHostToDevice, st));
      din[t] = d;
    }
    for (int t = 0; t < n_out; t++) dout[t] = c.buf[s] + (size_t)(n_in + t) * chunk;
    rc = launch(m, din.data(), dout.data(), st);
    if (rc) return rc;
    for (int t = 0; t < n_out; t++)
      B2S_CUDA(cudaMemcpyAsync(out[t] + lo, dout[t], mb, cudaMemcpyDeviceToHost, st));
  }
  for (int s = 0; s < kStages; s++) B2S_CUDA(cudaStreamSynchronize(c.streams[s]));
  return 0;
}

}  // namespace b2s

using namespace b2s;

extern "C" {

int b2s_svd2_real_host(int64_t n, const double* const a[4], double* const u[4], double* const v[4],
                       double* smax, double* smin, double* shift, int backscale_mode, int flags, int device,
                       int64_t chunk) {
  if (!a || !u || !v || !smax || !smin || !shift) return fail(5, "NULL host train");
  if (flags & B2S_FLAG_STATES) return fail(3, "state dumps are device-only (use b2s_svd2_real)");
  if (int rc = check_common(n, backscale_mode, flags, nullptr)) return rc;    // before any CUDA call
  const double* in[4] = {a[0], a[1], a[2], a[3]};
  double* out[11] = {u[0], u[1], u[2], u[3], v[0], v[1], v[2], v[3], smax, smin, shift};
  for (int t = 0; t < 4; t++) if (!in[t]) return fail(5, "NULL host train");
  for (int t = 0; t < 11; t++) if (!out[t]) return fail(5, "NULL host train");
  return pipeline(n, device, chunk, 4, in, 11, out,
                  [&](int64_t m, const double* const* di, double* const* d, cudaStream_t st) {
                    return b2s_svd2_real(m, di, d, d + 4, d[8], d[9], d[10], backscale_mode, flags, nullptr,
                                         (void*)st);
                  });
}

int b2s_svd2_complex_host(int64_t n, const double* const a_re[4], const double* const a_im[4],
                          double* const u_re[4], double* const u_im[4], double* const v_re[4],
                          double* const v_im[4], double* smax, double* smin, double* shift, int backscale_mode,
                          int flags, int device, int64_t chunk) {
  if (!a_re || !a_im || !u_re || !u_im || !v_re || !v_im || !smax || !smin || !shift)
    return fail(5, "NULL host train");
  if (flags & B2S_FLAG_STATES) return fail(3, "state dumps are device-only (use b2s_svd2_complex)");
  if (int rc = check_common(n, backscale_mode, flags, nullptr)) return rc;    // before any CUDA call
  const double* in[8] = {a_re[0], a_re[1], a_re[2], a_re[3], a_im[0], a_im[1], a_im[2], a_im[3]};
  double* out[19] = {u_re[0], u_re[1], u_re[2], u_re[3], u_im[0], u_im[1], u_im[2], u_im[3],
                     v_re[0], v_re[1], v_re[2], v_re[3], v_im[0], v_im[1], v_im[2], v_im[3],
                     smax, smin, shift};
  for (int t = 0; t < 8; t++) if (!in[t]) return fail(5, "NULL host train");
  for (int t = 0; t < 19; t++) if (!out[t]) return fail(5, "NULL host train");
  return pipeline(n, device, chunk, 8, in, 19, out,
                  [&](int64_t m, const double* const* di, double* const* d, cudaStream_t st) {
                    return b2s_svd2_complex(m, di, di + 4, d, d + 4, d + 8, d + 12, d[16], d[17], d[18],
                                            backscale_mode, flags, nullptr, (void*)st);
                  });
}

}  // extern "C"
