// b2s_common.cuh -- error plumbing and launch helpers shared by the C-ABI files.
#pragma once
#include <cuda_runtime.h>
#include <cstdarg>
#include <cstdint>
#include <cstdio>

namespace b2s {

// Thread-local last-error message behind b2s_last_error().
char* last_error_buf();

inline int fail(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(last_error_buf(), 512, fmt, ap);
  va_end(ap);
  return code;
}

inline int cuda_fail(cudaError_t e, const char* what) {
  return fail(-(int)e, "%s: %s (%s)", what, cudaGetErrorName(e), cudaGetErrorString(e));
}

#define B2S_CUDA(call)                                   \
  do {                                                   \
    cudaError_t e_ = (call);                             \
    if (e_ != cudaSuccess) return ::b2s::cuda_fail(e_, #call); \
  } while (0)

inline bool aligned8(const void* p) { return ((uintptr_t)p & 7u) == 0; }

// Resident-grid size for a grid-stride kernel: SMs x resident CTAs per SM,
// capped by the work available.
template <typename K>
inline int grid_for(K kernel, int block, int64_t work_items, int* err) {
  int dev = 0, sms = 148, per_sm = 1;
  *err = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) { *err = 1; return 1; }
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, block, 0);
  if (per_sm < 1) per_sm = 1;
  int64_t full = (int64_t)sms * per_sm;
  int64_t need = (work_items + block - 1) / block;
  if (need < 1) need = 1;
  return (int)(need < full ? need : full);
}

// Argument checks shared by the device and host-buffer entry points
// (b2s_kernels.cu): batch size, backscale mode, flag bits, states array.
int check_common(int64_t n, int mode, int flags, double* const* states);

}  // namespace b2s
