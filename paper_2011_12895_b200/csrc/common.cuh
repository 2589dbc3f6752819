// Shared device/host helpers for the B200 (sm_100a) learner path.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <stdexcept>
#include <string>

namespace tlg {

struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

#define TLG_CUDA(expr)                                                                    \
  do {                                                                                    \
    cudaError_t _e = (expr);                                                              \
    if (_e != cudaSuccess)                                                                \
      throw ::tlg::CudaError(std::string(#expr) + ": " + cudaGetErrorString(_e) + " at " + \
                             __FILE__ + ":" + std::to_string(__LINE__));                  \
  } while (0)

#define TLG_CHECK_LAUNCH() TLG_CUDA(cudaGetLastError())

inline int ceil_div(long a, long b) { return int((a + b - 1) / b); }

// Function attributes are per device: raise a kernel's dynamic shared-memory limit once
// on every device it is launched on (one bit per device in `done`).
template <typename Kernel>
inline void ensure_smem_attr(Kernel kern, int bytes, std::atomic<unsigned long long>& done) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) throw CudaError("cudaGetDevice failed");
  const unsigned long long bit = 1ull << (dev & 63);
  if (done.load(std::memory_order_acquire) & bit) return;
  const cudaError_t e =
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e != cudaSuccess)
    throw CudaError(std::string("cudaFuncSetAttribute: ") + cudaGetErrorString(e));
  done.fetch_or(bit, std::memory_order_acq_rel);
}

// ---------------------------------------------------------------------------
// TF32 hi/lo split.  hi keeps the 10 explicit mantissa bits a tcgen05 kind::tf32
// MMA consumes; lo = x - hi is exact in fp32.  hi*b_hi + hi*b_lo + lo*b_hi
// (3xTF32) reproduces the fp32 product to ~2^-21 relative.
__device__ __forceinline__ float tf32_hi(float x) {
  return __uint_as_float(__float_as_uint(x) & 0xFFFFE000u);
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

}  // namespace tlg
