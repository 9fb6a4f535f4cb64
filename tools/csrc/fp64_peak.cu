// fp64_peak.cu -- FP64 pipe throughput microbenchmark (tools only).
//
// SURVEY 7.1.6 / north_star: the roofline's FP64 term needs a measured FP64
// peak (MEASURED_PEAKS.json has none).  Every thread runs kChains
// independent dependency chains of DFMA (op 0), DMUL (op 1) or DADD (op 2)
// so the FP64 pipe, not latency, is the limit; a resident grid of
// SMs x 8 CTAs x 256 threads.  Timed with CUDA events around one launch.
#include <cuda_runtime.h>
#include <cstdint>

namespace {
constexpr int kChains = 8;

__global__ void __launch_bounds__(256) k_fp64(int op, int64_t iters, double seed, double* sink) {
  double x[kChains];
  #pragma unroll
  for (int c = 0; c < kChains; c++) x[c] = seed + threadIdx.x * 1e-9 + c * 1e-7;
  const double a = 0.999999999, b = 1e-12;
  if (op == 0) {
    for (int64_t i = 0; i < iters; i++) {
      #pragma unroll
      for (int c = 0; c < kChains; c++) x[c] = __fma_rn(x[c], a, b);
    }
  } else if (op == 1) {
    for (int64_t i = 0; i < iters; i++) {
      #pragma unroll
      for (int c = 0; c < kChains; c++) x[c] = __dmul_rn(x[c], a);
    }
  } else {
    for (int64_t i = 0; i < iters; i++) {
      #pragma unroll
      for (int c = 0; c < kChains; c++) x[c] = __dadd_rn(x[c], b);
    }
  }
  double s = 0.0;
  #pragma unroll
  for (int c = 0; c < kChains; c++) s += x[c];
  if (s == 12345.678) sink[threadIdx.x] = s;     // keeps the chains live
}
}  // namespace

extern "C" int fp64_peak(int op, long long iters, int ctas_per_sm, double* out_ops_per_s,
                         float* out_ms) {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  double* sink = nullptr;
  if (cudaMalloc(&sink, 256 * sizeof(double)) != cudaSuccess) return -1;
  const int grid = sms * ctas_per_sm;
  k_fp64<<<grid, 256>>>(op, 1000, 1.0, sink);      // warm-up
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k_fp64<<<grid, 256>>>(op, iters, 1.0, sink);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(sink);
  if (cudaGetLastError() != cudaSuccess) return -2;
  *out_ms = ms;
  *out_ops_per_s = (double)grid * 256 * kChains * (double)iters / (ms * 1e-3);
  return 0;
}
