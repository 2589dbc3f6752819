// Shared device/host helpers for the B200 (sm_100a) learner path.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <cstdlib>
#include <utility>
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

// ---------------------------------------------------------------------------
// Programmatic dependent launch (PDL).  Every kernel of this library is launched with
// cudaLaunchAttributeProgrammaticStreamSerialization, so it may be scheduled while its
// predecessor on the stream drains (launch latency and the prologue -- barrier init,
// TMEM allocation, tensor-map prefetch -- overlap the predecessor's tail, also inside
// captured CUDA graphs).  Each kernel therefore calls pdl_wait() before it touches memory
// a predecessor wrote (griddepcontrol.wait returns once the preceding grid has completed
// and its writes are visible; it is a no-op without a programmatic dependency) and then
// pdl_trigger() to let its own successor launch early.  Because every kernel waits, the
// completion order along a stream is transitive as with ordinary launches.
// TLG_NO_PDL=1 launches without the attribute (A/B runs).
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
#define TLG_PDL_ENTRY()     \
  do {                      \
    ::tlg::pdl_wait();      \
    ::tlg::pdl_trigger();   \
  } while (0)

inline bool pdl_enabled() {
  static const bool on = std::getenv("TLG_NO_PDL") == nullptr;
  return on;
}

// Append the PDL attribute to a launch configuration whose attribute array has room.
inline void add_pdl(cudaLaunchConfig_t& cfg, cudaLaunchAttribute* at) {
  if (!pdl_enabled()) return;
  at[cfg.numAttrs].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[cfg.numAttrs].val.programmaticStreamSerializationAllowed = 1;
  cfg.numAttrs += 1;
}

// cudaLaunchKernelEx with the PDL attribute.
template <typename... KArgs, typename... Args>
inline void launch_k(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                     cudaStream_t stream, Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute at[1];
  int na = 0;
  if (pdl_enabled()) {
    at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  cfg.attrs = at;
  cfg.numAttrs = na;
  TLG_CUDA(cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...));
}

// The same with a thread-block cluster of `cluster_x` CTAs.
template <typename... KArgs, typename... Args>
inline void launch_k_cluster(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                             cudaStream_t stream, int cluster_x, Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute at[2];
  int na = 0;
  at[na].id = cudaLaunchAttributeClusterDimension;
  at[na].val.clusterDim.x = unsigned(cluster_x);
  at[na].val.clusterDim.y = 1;
  at[na].val.clusterDim.z = 1;
  ++na;
  if (pdl_enabled()) {
    at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  cfg.attrs = at;
  cfg.numAttrs = na;
  TLG_CUDA(cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...));
}

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

// tanh within ~3 ulp of the correctly rounded value (measured max 0.77 ulp on the
// polynomial branch, 3.2 ulp on the exponential one, fp32 emulation in
// tools/tanh_fast_check.py) in about a third of libm tanhf's instructions: an odd
// least-squares polynomial x + x^3 q(x^2) on |x| < 0.625, else 1 - 2 / (e^{2|x|} + 1)
// with the SFU exp2 and a fast reciprocal.  The GEMM epilogues that apply the trunk's
// tanh are bound by this instruction count (fwd2 / InfServer at C3, C4).
__device__ __forceinline__ float tanh_fast(float x) {
  const float t = fabsf(x);
  if (t < 0.625f) {
    const float x2 = x * x;
    float q = -0.0057981000281870365f;
    q = fmaf(q, x2, 0.020720280706882477f);
    q = fmaf(q, x2, -0.053763799369335175f);
    q = fmaf(q, x2, 0.13331718742847443f);
    q = fmaf(q, x2, -0.33333292603492737f);
    return fmaf(x * x2, q, x);
  }
  float e;  // e^{2t} = 2^{2t log2(e)}
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(t * 2.8853900817779268f));
  return copysignf(1.f - __fdividef(2.f, e + 1.f), x);
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
