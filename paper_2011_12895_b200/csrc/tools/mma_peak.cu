// Instruction-level tensor-core ceilings on this B200 (test tool; not part of the product
// library): every CTA pair of a persistent grid issues back-to-back tcgen05.mma
// (cta_group::2, M = 256, N = 256) from operand tiles already in shared memory into a
// TMEM accumulator -- no loads, no epilogue -- for each instruction kind the learner uses:
//
//   kind::f16  (bf16 x bf16 -> f32, K = 16 per MMA)   calibrates against the cuBLAS bf16
//                                                     peak of MEASURED_PEAKS.json
//   kind::tf32 (K = 8)                                 the 3xTF32 GEMMs' instruction
//   kind::i8   (u8 x s8 -> s32, K = 32)                the int8 layer-1 GEMMs' instruction
//
// Prints one JSON line with the achieved rate per kind (dense ops/s, CUDA events over the
// kernel, best of 5) so each GEMM's roofline fraction can be stated against its own
// instruction kind.  nvcc -gencode arch=compute_100a,code=sm_100a -O2 mma_peak.cu
#include <cstdio>
#include <cstdlib>

#include "../gemm_i8.cuh"

using namespace tlg;
using namespace tlg::gemm;

namespace {

enum Kind { kBf16 = 0, kTf32 = 1, kI8 = 2 };

template <int KIND, int N = 256>
__device__ __forceinline__ constexpr uint32_t idesc_for() {
  // D format f32 (1) / s32 (2); A/B formats: f16 kind: bf16 = 1; tf32 kind: tf32 = 2;
  // i8 kind: u8 = 0, s8 = 1.  Both K-major, N = 256, M = 256 (pair).
  constexpr uint32_t d = KIND == kI8 ? 2u : 1u;
  constexpr uint32_t a = KIND == kBf16 ? 1u : KIND == kTf32 ? 2u : 0u;
  constexpr uint32_t b = KIND == kBf16 ? 1u : KIND == kTf32 ? 2u : 1u;
  return (d << 4) | (a << 7) | (b << 10) | (uint32_t(N >> 3) << 17) | (uint32_t(256 >> 4) << 24);
}

template <int KIND>
__device__ __forceinline__ void mma_pair(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc,
                                         uint32_t acc) {
  if constexpr (KIND == kBf16)
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc));
  else if constexpr (KIND == kTf32)
    mma_tf32_pair(tmem_d, a, b, idesc, acc);
  else
    mma_i8<2>(tmem_d, a, b, idesc, acc);
}

// Per CTA: a 128-row A tile and a 128-row B tile of one 128-B swizzle row per row (16 KB
// each); the pair's MMA reads both CTAs' halves.
template <int KIND, int N = 256>
__global__ void __launch_bounds__(128, 1) mma_peak_kernel(int iters) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const uint32_t sbase = smem_u32(smem);
  const uint32_t a_tile = sbase, b_tile = sbase + 16384;
  const uint32_t bar = sbase + 32768;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + 32768 + 64);
  for (int i = threadIdx.x; i < 32768 / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
  const uint32_t rank = cluster_rank();
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  fence_async_smem();
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "n"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  if (threadIdx.x == 0 && rank == 0) {
    constexpr uint32_t idesc = idesc_for<KIND, N>();
    const uint64_t da = make_sdesc<false>(a_tile, 16, 1024);
    const uint64_t db = make_sdesc<false>(b_tile, 16, 1024);
    // one 128-B row holds 64 bf16, 32 tf32 or 128 int8 elements: 4 K-steps per row
    for (int i = 0; i < iters; ++i) {
#pragma unroll
      for (int k = 0; k < 4; ++k) mma_pair<KIND>(tmem, da + 2 * k, db + 2 * k, idesc, 1u);
    }
    mma_commit_pair(bar);
  }
  if (threadIdx.x == 0) mbar_wait(bar, 0);
  __syncthreads();
  tc_fence_before();
  cluster_sync_all();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(256));
  }
}

// The int8 layer-1 forward's MMA pattern with everything else removed: per 32-element K
// step, (x<<7)·q0 and x·q1 into accumulator a, x·q2 into accumulator b, N = 128, the
// operand tiles at their own smem addresses (x, x<<7: 16 KB; q0..q2: 8 KB per CTA).
__global__ void __launch_bounds__(128, 1) i8_pattern_kernel(int iters) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const uint32_t sbase = smem_u32(smem);
  const uint32_t x = sbase, x7 = sbase + 16384, q = sbase + 32768;  // q0, q1, q2: 8 KB each
  const uint32_t bar = sbase + 57344;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + 57344 + 64);
  for (int i = threadIdx.x; i < 57344 / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
  const uint32_t rank = cluster_rank();
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  fence_async_smem();
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "n"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  if (threadIdx.x == 0 && rank == 0) {
    constexpr uint32_t idesc = idesc_for<kI8, 128>();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const uint64_t dx = make_sdesc<false>(x + k * 32, 16, 1024);
        const uint64_t dx7 = make_sdesc<false>(x7 + k * 32, 16, 1024);
        const uint64_t d0 = make_sdesc<false>(q + k * 32, 16, 1024);
        const uint64_t d1 = make_sdesc<false>(q + 8192 + k * 32, 16, 1024);
        const uint64_t d2 = make_sdesc<false>(q + 16384 + k * 32, 16, 1024);
        mma_i8<2>(tmem, dx7, d0, idesc, 1u);
        mma_i8<2>(tmem, dx, d1, idesc, 1u);
        mma_i8<2>(tmem + 128, dx, d2, idesc, 1u);
      }
    }
    mma_commit_pair(bar);
  }
  if (threadIdx.x == 0) mbar_wait(bar, 0);
  __syncthreads();
  tc_fence_before();
  cluster_sync_all();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(256));
  }
}

double run_pattern(int iters) {
  auto kern = i8_pattern_kernel;
  const int bytes = 57344 + 1024 + 1024;
  TLG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
  int sms = 0;
  TLG_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const int pairs = sms / 2;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int rep = 0; rep < 6; ++rep) {
    cudaEventRecord(e0);
    launch_k_cluster(kern, dim3(2 * pairs), dim3(128), size_t(bytes), cudaStream_t(0), 2, iters);
    cudaEventRecord(e1);
    TLG_CUDA(cudaEventSynchronize(e1));
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    if (rep > 0 && ms < best) best = ms;
  }
  // 12 MMAs of M=256 N=128 K=32 per iteration
  return double(pairs) * iters * 12 * 2.0 * 256 * 128 * 32 / (best * 1e-3);
}

template <int KIND, int N = 256>
double run(int iters) {
  auto kern = mma_peak_kernel<KIND, N>;
  const int bytes = 32768 + 1024 + 1024;
  TLG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
  int sms = 0;
  TLG_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const int pairs = sms / 2;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int rep = 0; rep < 6; ++rep) {
    cudaEventRecord(e0);
    launch_k_cluster(kern, dim3(2 * pairs), dim3(128), size_t(bytes), cudaStream_t(0), 2, iters);
    cudaEventRecord(e1);
    TLG_CUDA(cudaEventSynchronize(e1));
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    if (rep > 0 && ms < best) best = ms;  // rep 0 warms up
  }
  // ops per MMA: 2 * M * N * K with K = 16 (bf16), 8 (tf32), 32 (i8)
  const double k = KIND == kBf16 ? 16 : KIND == kTf32 ? 8 : 32;
  const double ops = double(pairs) * iters * 4 * 2.0 * 256 * N * k;
  return ops / (best * 1e-3);
}

}  // namespace

int main(int argc, char** argv) {
  const int iters = argc > 1 ? std::atoi(argv[1]) : 20000;
  try {
    const double bf16 = run<kBf16>(iters), tf32 = run<kTf32>(iters), i8 = run<kI8>(iters);
    std::printf(
        "{\"tool\": \"mma_peak\", \"what\": \"tcgen05.mma cta_group::2 M=256 N=256 back to back "
        "from smem, all SM pairs, best of 5\", \"iters\": %d, \"bf16_tflops\": %.1f, "
        "\"tf32_tflops\": %.1f, \"i8_tops\": %.1f}\n",
        iters, bf16 / 1e12, tf32 / 1e12, i8 / 1e12);
    // narrower tiles (the N of the learner's 128-column GEMM tiles)
    const double bf16_128 = run<kBf16, 128>(iters), tf32_128 = run<kTf32, 128>(iters),
                 i8_128 = run<kI8, 128>(iters), i8_64 = run<kI8, 64>(iters);
    std::printf(
        "{\"tool\": \"mma_peak\", \"what\": \"same, N=128 (and i8 N=64)\", \"bf16_n128_tflops\": "
        "%.1f, \"tf32_n128_tflops\": %.1f, \"i8_n128_tops\": %.1f, \"i8_n64_tops\": %.1f}\n",
        bf16_128 / 1e12, tf32_128 / 1e12, i8_128 / 1e12, i8_64 / 1e12);
    std::printf("{\"tool\": \"mma_peak\", \"what\": \"int8 layer-1 forward MMA pattern "
                "(x<<7.q0 + x.q1 -> a, x.q2 -> b, N=128)\", \"i8_pattern_tops\": %.1f}\n",
                run_pattern(iters) / 1e12);
  } catch (const std::exception& e) {
    std::printf("EXCEPTION: %s\n", e.what());
    return 2;
  }
  return 0;
}
