// tcgen05 / TMA / TMEM GEMM for sm_100a with a 3xTF32 split ("fp32-exact" mode).
//
//   C[M x N] = A[M x K] . B[N x K]^T        (fp32 accumulate in TMEM)
//
// Each fp32 operand arrives as two planes written by its producer: the full
// fp32 value (which the tensor core truncates to tf32 -- verified on B200, see
// tools/gemm_selftest.cu FULLHI cases) and lo = x - trunc_tf32(x), exact in fp32.  Per K step the MMA
// warp issues hi.hi + hi.lo + lo.hi (the lo.lo term, ~2^-22, is dropped); an
// operand known to be exact in tf32 (binary observation planes) has no lo
// plane and saves its pass.  Either operand may be K-major or MN-major in
// global memory: the smem tiles are TMA-loaded with the 128-byte swizzle and
// described to the tensor core with the matching canonical layout, so no
// transposes are ever materialised (the backward dW = dZ^T . H and
// dX = dZ . W GEMMs read the forward's buffers in place).
//
// Warp roles (192 threads, one output tile of 128 x BN per CTA):
//   warp 0      TMA producer (one elected lane), smem ring of STAGES stages
//   warp 1      TMEM allocator + single-thread tcgen05.mma issuer
//   warps 2..5  epilogue: tcgen05.ld TMEM -> registers -> fused op -> global
// Pipelines: full[s] (TMA -> MMA, tx-count), empty[s] (tcgen05.commit -> TMA),
// tmem_full (final commit -> epilogue).
#pragma once

#include "common.cuh"

namespace tlg::gemm {

enum Epi : int {
  kEpiFwdTanh = 0,   // out = tanh(acc + bias[n])          -> out (full) / out_lo planes
  kEpiBwdTanh = 1,   // out = acc * (1 - h[m][n]^2)         -> out (full) / out_lo planes
  kEpiStore = 2,     // ws[split][m][n] = acc               (split-K partials, fp32)
};

constexpr int kBM = 128;
constexpr int kBK = 32;  // fp32 elements per 128-byte swizzle row
constexpr int kThreads = 192;

struct Params {
  int M, N, K;
  int kb_per_split;  // K blocks (of kBK) per blockIdx.z
  // epilogue
  float* out_hi;
  float* out_lo;
  long ldo;
  const float* bias;
  const float* act_hi;  // full fp32 activation plane (bwd tanh)
  long ld_act;
  float* ws;
  long ws_split_stride;
};

// ---------------------------------------------------------------------------
// PTX wrappers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "LAB_WAIT:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@P1 bra DONE;\n"
      "bra LAB_WAIT;\n"
      "DONE:\n"
      "}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, int x, int y,
                                            uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(bar)
      : "memory");
}

__device__ __forceinline__ void prefetch_tmap(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}

// UMMA shared-memory descriptor (sm_100: version 1 at bit 46, layout type at 61..63).
// K-major fp32 tiles use SWIZZLE_128B (2); MN-major fp32 (tf32) tiles must use
// SWIZZLE_128B_BASE32B (1), matching TMA's CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B.
template <bool MN>
__device__ __forceinline__ uint64_t make_sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= uint64_t((saddr >> 4) & 0x3FFFu);
  d |= uint64_t((lbo >> 4) & 0x3FFFu) << 16;
  d |= uint64_t((sbo >> 4) & 0x3FFFu) << 32;
  d |= uint64_t(1) << 46;  // descriptor version (Blackwell)
  d |= uint64_t(MN ? 1 : 2) << 61;
  return d;
}

// Instruction descriptor for kind::tf32, fp32 accumulate, M=128.
template <int BN, bool A_MN, bool B_MN>
__device__ __forceinline__ constexpr uint32_t make_idesc() {
  return (1u << 4)                        // D format: f32
         | (2u << 7)                      // A format: tf32
         | (2u << 10)                     // B format: tf32
         | (uint32_t(A_MN) << 15)         // A major (0 = K, 1 = MN)
         | (uint32_t(B_MN) << 16)         // B major
         | (uint32_t(BN >> 3) << 17)      // N >> 3
         | (uint32_t(kBM >> 4) << 24);    // M >> 4
}

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void mma_commit(uint32_t bar) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar)
      : "memory");
}

__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

#define TLG_R32(i) "=r"(r[i])
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : TLG_R32(0), TLG_R32(1), TLG_R32(2), TLG_R32(3), TLG_R32(4), TLG_R32(5), TLG_R32(6),
        TLG_R32(7), TLG_R32(8), TLG_R32(9), TLG_R32(10), TLG_R32(11), TLG_R32(12), TLG_R32(13),
        TLG_R32(14), TLG_R32(15), TLG_R32(16), TLG_R32(17), TLG_R32(18), TLG_R32(19),
        TLG_R32(20), TLG_R32(21), TLG_R32(22), TLG_R32(23), TLG_R32(24), TLG_R32(25),
        TLG_R32(26), TLG_R32(27), TLG_R32(28), TLG_R32(29), TLG_R32(30), TLG_R32(31)
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
#undef TLG_R32

// ---------------------------------------------------------------------------
template <int BN, bool A_LO, bool B_LO>
struct Smem {
  static constexpr int kA = kBM * kBK * 4;  // 16 KB
  static constexpr int kB = BN * kBK * 4;
  static constexpr int kStage = kA * (A_LO ? 2 : 1) + kB * (B_LO ? 2 : 1);
  static constexpr int kStages = (200 * 1024 / kStage) < 2 ? 2
                                 : (200 * 1024 / kStage) > 6 ? 6
                                                             : (200 * 1024 / kStage);
  static constexpr int kBarOff = kStages * kStage;
  static constexpr int kBytes = kBarOff + (2 * kStages + 2) * 8 + 16 + 1024;  // + align slack
  static constexpr int kTmemCols = BN <= 32 ? 32 : BN <= 64 ? 64 : BN <= 128 ? 128 : 256;
};

template <int BN, bool A_MN, bool B_MN, bool A_LO, bool B_LO, int EPI>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_tf32x3_kernel(const __grid_constant__ CUtensorMap tmA_hi,
                       const __grid_constant__ CUtensorMap tmA_lo,
                       const __grid_constant__ CUtensorMap tmB_hi,
                       const __grid_constant__ CUtensorMap tmB_lo, const Params p) {
  using S = Smem<BN, A_LO, B_LO>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  const uint32_t sbase = smem_u32(smem);
  const uint32_t bar_full = sbase + S::kBarOff;
  const uint32_t bar_empty = bar_full + S::kStages * 8;
  const uint32_t bar_tmem = bar_empty + S::kStages * 8;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + S::kBarOff + (2 * S::kStages + 2) * 8);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int m0 = blockIdx.x * kBM;
  const int n0 = blockIdx.y * BN;
  const int kb_total = (p.K + kBK - 1) / kBK;
  const int kb_begin = blockIdx.z * p.kb_per_split;
  const int kb_end = min(kb_total, kb_begin + p.kb_per_split);

  if (warp == 0 && lane == 0) {
    prefetch_tmap(&tmA_hi);
    prefetch_tmap(&tmB_hi);
    if (A_LO) prefetch_tmap(&tmA_lo);
    if (B_LO) prefetch_tmap(&tmB_lo);
    for (int s = 0; s < S::kStages; ++s) {
      mbar_init(bar_full + 8 * s, 1);
      mbar_init(bar_empty + 8 * s, 1);
    }
    mbar_init(bar_tmem, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "n"(S::kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      // ===== TMA producer =====
      int stage = 0;
      uint32_t phase = 0;
      for (int kb = kb_begin; kb < kb_end; ++kb) {
        mbar_wait(bar_empty + 8 * stage, phase ^ 1);
        const uint32_t st = sbase + stage * S::kStage;
        const uint32_t full = bar_full + 8 * stage;
        mbar_expect_tx(full, S::kStage);
        const int k0 = kb * kBK;
        uint32_t off = st;
        // A tile: 128 rows (M) x 32 (K)
        if (!A_MN) {
          tma_load_2d(off, &tmA_hi, k0, m0, full);
          if (A_LO) tma_load_2d(off + S::kA, &tmA_lo, k0, m0, full);
        } else {
#pragma unroll
          for (int j = 0; j < kBM / 32; ++j) {
            tma_load_2d(off + j * 4096, &tmA_hi, m0 + 32 * j, k0, full);
            if (A_LO) tma_load_2d(off + S::kA + j * 4096, &tmA_lo, m0 + 32 * j, k0, full);
          }
        }
        off += S::kA * (A_LO ? 2 : 1);
        // B tile: BN rows (N) x 32 (K)
        if (!B_MN) {
          tma_load_2d(off, &tmB_hi, k0, n0, full);
          if (B_LO) tma_load_2d(off + S::kB, &tmB_lo, k0, n0, full);
        } else {
#pragma unroll
          for (int j = 0; j < BN / 32; ++j) {
            tma_load_2d(off + j * 4096, &tmB_hi, n0 + 32 * j, k0, full);
            if (B_LO) tma_load_2d(off + S::kB + j * 4096, &tmB_lo, n0 + 32 * j, k0, full);
          }
        }
        if (++stage == S::kStages) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ===== MMA issuer =====
      constexpr uint32_t idesc = make_idesc<BN, A_MN, B_MN>();
      int stage = 0;
      uint32_t phase = 0;
      for (int kb = kb_begin; kb < kb_end; ++kb) {
        mbar_wait(bar_full + 8 * stage, phase);
        tc_fence_after();
        const uint32_t a_hi = sbase + stage * S::kStage;
        const uint32_t a_lo = a_hi + S::kA;
        const uint32_t b_hi = a_hi + S::kA * (A_LO ? 2 : 1);
        const uint32_t b_lo = b_hi + S::kB;
#pragma unroll
        for (int k = 0; k < kBK / 8; ++k) {
          // K-major: +32 B per 8-element K step inside the 128-B swizzle row;
          //   SBO = 1 KB between 8-row (MN) atoms.
          // MN-major: +1 KB per 8 K rows (128 B each); SBO = 512 B between the
          //   4-row swizzle atoms along K, LBO = 4 KB between 32-element MN chunks.
          const uint32_t ao = A_MN ? k * 1024 : k * 32;
          const uint32_t bo = B_MN ? k * 1024 : k * 32;
          const uint32_t albo = A_MN ? 4096 : 16, asbo = A_MN ? 512 : 1024;
          const uint32_t blbo = B_MN ? 4096 : 16, bsbo = B_MN ? 512 : 1024;
          const uint64_t dah = make_sdesc<A_MN>(a_hi + ao, albo, asbo);
          const uint64_t dbh = make_sdesc<B_MN>(b_hi + bo, blbo, bsbo);
          const uint32_t acc = (kb > kb_begin || k > 0) ? 1u : 0u;
          if (B_LO) mma_tf32(tmem_base, dah, make_sdesc<B_MN>(b_lo + bo, blbo, bsbo), idesc, acc);
          if (A_LO)
            mma_tf32(tmem_base, make_sdesc<A_MN>(a_lo + ao, albo, asbo), dbh, idesc,
                     (B_LO || acc) ? 1u : 0u);
          mma_tf32(tmem_base, dah, dbh, idesc, (A_LO || B_LO || acc) ? 1u : 0u);
        }
        mma_commit(bar_empty + 8 * stage);
        if (++stage == S::kStages) {
          stage = 0;
          phase ^= 1;
        }
      }
      mma_commit(bar_tmem);
    }
  } else {
    // ===== Epilogue: warps 2..5 cover TMEM lane quadrants (warp % 4) =====
    const int q = warp & 3;
    const int row = m0 + q * 32 + lane;
    mbar_wait(bar_tmem, 0);
    tc_fence_after();
    const bool row_ok = row < p.M;
#pragma unroll 1
    for (int c = 0; c < BN; c += 32) {
      uint32_t r[32];
      tmem_ld32(tmem_base + (uint32_t(q * 32) << 16) + uint32_t(c), r);
      const int nb = n0 + c;
      if (!row_ok || nb >= p.N) continue;
      const int ncols = min(32, p.N - nb);
      if (EPI == kEpiStore) {
        float* dst = p.ws + long(blockIdx.z) * p.ws_split_stride + long(row) * p.N + nb;
        if (ncols == 32 && (p.N & 3) == 0) {
#pragma unroll
          for (int j = 0; j < 32; j += 4)
            *reinterpret_cast<float4*>(dst + j) =
                make_float4(__uint_as_float(r[j]), __uint_as_float(r[j + 1]),
                            __uint_as_float(r[j + 2]), __uint_as_float(r[j + 3]));
        } else {
          for (int j = 0; j < ncols; ++j) dst[j] = __uint_as_float(r[j]);
        }
      } else {
        // out = full fp32 value (the tensor core truncates it to tf32 itself when it is
        // consumed as the next GEMM's "hi" operand); out_lo = exact residual.
        float* dhi = p.out_hi + long(row) * p.ldo + nb;
        float* dlo = p.out_lo + long(row) * p.ldo + nb;
        float o[32];
        if (EPI == kEpiFwdTanh) {
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const float b = (j < ncols) ? __ldg(p.bias + nb + j) : 0.f;
            o[j] = tanhf(__uint_as_float(r[j]) + b);
          }
        } else {
          const float* ah = p.act_hi + long(row) * p.ld_act + nb;
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const float h = (j < ncols) ? __ldg(ah + j) : 0.f;
            o[j] = __uint_as_float(r[j]) * (1.f - h * h);
          }
        }
        if (ncols == 32 && (p.ldo & 3) == 0) {
#pragma unroll
          for (int j = 0; j < 32; j += 4) {
            *reinterpret_cast<float4*>(dhi + j) = make_float4(o[j], o[j + 1], o[j + 2], o[j + 3]);
            *reinterpret_cast<float4*>(dlo + j) =
                make_float4(o[j] - tf32_hi(o[j]), o[j + 1] - tf32_hi(o[j + 1]),
                            o[j + 2] - tf32_hi(o[j + 2]), o[j + 3] - tf32_hi(o[j + 3]));
          }
        } else {
          for (int j = 0; j < ncols; ++j) {
            dhi[j] = o[j];
            dlo[j] = o[j] - tf32_hi(o[j]);
          }
        }
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "n"(S::kTmemCols));
  }
}

// ---------------------------------------------------------------------------
// Host side
struct Operand {
  const float* hi = nullptr;
  const float* lo = nullptr;  // null: exact in tf32, the lo pass is skipped
  long ld = 0;                // row pitch (elements) of the stored matrix
  bool mn_major = false;      // false: stored [MN rows][K cols]; true: stored [K rows][MN cols]
};

// Launch C = A . B^T with the given epilogue on `stream`.  splits > 1 only for
// kEpiStore (partials into p.ws).  Throws tlg::CudaError on misuse.
void launch(const Operand& A, const Operand& B, int M, int N, int K, int epi, Params p,
            int splits, cudaStream_t stream);

// Number of K splits that fills the GPU for a (M, N, K) problem, given a cap.
int pick_splits(int M, int N, int K, int max_splits);

}  // namespace tlg::gemm
