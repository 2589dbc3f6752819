// Exact-integer tcgen05 GEMM for binary observation planes (kind::i8, sm_100a).
//
// The first trunk layer of the Pommerman-shaped configs multiplies {0,1} observation
// planes by fp32 weights.  The planes are exact integers, so the product can run on the
// int8 tensor cores (4x the tf32 rate) without losing the fp32-exact contract of the
// 3xTF32 path, once the weights are written as fixed-point pieces:
//
//   W[n][k] = s_n (q0 + q1 / 2^7 + q2 / 2^14) + e,   q_i int8,   |e| <= s_n 2^-15,
//   s_n = max_k |W[n][k]| / 127                         (quantize_rows_kernel)
//
// and the planes arrive LSB-first bit-packed (TLG_OBS_BITS: 1 bit per plane element,
// 8x fewer bytes than uint8 in HBM and over PCIe).  Per 128-element k-block the
// converter warps expand the 16-byte bit rows into two int8 operand tiles in the MMA's
// 128-B swizzled layout: x (0/1) and x << 7 (0/128).  Two int32 TMEM accumulators
//
//   acc_a = sum_k (x<<7) q0 + x q1 = 2^7 sum x q0 + sum x q1,     acc_b = sum_k x q2
//
// are exact; the epilogue forms s_n (acc_a 2^-7 + acc_b 2^-14) in fp32 (one rounding)
// and applies the fused bias + tanh.  Error vs the fp32 product: <= s_n 2^-15 per weight
// (2.4e-7 of the row's largest weight), the same order as the 3xTF32 split's 2^-22.
//
// Layout, per CTA (pair mode: cta_group::2, 256-row tiles, each CTA holds half of the
// piece rows; one elected thread of rank 0 issues the MMAs for both):
//   warp 0      TMA producer: bit rows (local barrier), 3 piece tiles (leader barrier)
//   warp 1      TMEM allocator + MMA issuer
//   warps 2..5  epilogue: TMEM -> registers -> s (a/128 + b/16384) + bias -> tanh ->
//               hi / tf32-residual planes -> swizzled smem -> TMA store
//   warps 6..9  converters: bits -> x, x<<7 tiles
// (gemm_i8_bits_fwd_dec_kernel below keeps the same roles with separate operand rings and
// up to three epilogue warp groups; it is the default for CTA pairs.)
#pragma once

#include "gemm_sm100.cuh"

namespace tlg::gemm {

constexpr int kBKi = 128;  // int8 K elements per k-block (one 128-B swizzle row)
constexpr int kConvWarps = 4;
constexpr int kThreadsI8 = 32 * (2 + kEpiWarps + kConvWarps);

struct I8Params {
  int M, N, K;
  const float* scale;  // [N] piece scale per output column
  const float* bias;   // [N]
  long q_rows;         // rows per piece in the stacked [3][q_rows][Kp] piece array
  int8_t* out_q;       // optional: tanh outputs as int8 pieces [3][M][N] (scale 1/127)
  int write_lo;        // store the tf32 residual plane (0: the consumers derive it)
};

template <int BN, int CG>
struct SmemI8 {
  static constexpr int kX = kBM * kBKi;         // 16 KB operand tile (x, x<<7)
  static constexpr int kBits = kBM * kBKi / 8;  // 2 KB packed source rows
  static constexpr int kBN = BN / CG;           // piece rows held by this CTA
  static constexpr int kQ = kBN * kBKi;         // bytes per piece tile
  static constexpr int kStage = 2 * kX + 3 * kQ;
  // the bit rows stream through their own ring, kRing k-blocks ahead of the stages
  // (they come from HBM; the pieces are L2-resident)
  static constexpr int kRing = 8;
  static constexpr int kEpi = kEpiWarps * 2 * 4096;
  static constexpr int kStagesRaw = (225 * 1024 - kEpi - kRing * kBits - 2048) / kStage;
  static constexpr int kStages = kStagesRaw > 6 ? 6 : kStagesRaw;
  static constexpr int kRingOff = kStages * kStage;
  static constexpr int kBarOff = kRingOff + kRing * kBits;
  // full (pieces, leader), conv (leader), empty per stage; ufull/uempty per ring slot;
  // tfull[2], tempty[2]
  static constexpr int kNumBars = 3 * kStages + 2 * kRing + 4;
  static constexpr int kEpiOff = (kBarOff + kNumBars * 8 + 16 + 1023) / 1024 * 1024;
  static constexpr int kBytes = kEpiOff + kEpi + 1024;
  // 2 accumulators, double-buffered while they fit TMEM's 512 columns (BN <= 128); a
  // 256-wide tile keeps one buffer (the epilogue then drains before the next tile's MMAs)
  static constexpr int kBufs = 4 * BN <= 512 ? 2 : 1;
  static constexpr int kTmemCols = 2 * BN * kBufs;
  static_assert(kStage % 1024 == 0, "stages must keep the 1 KB swizzle alignment");
  static_assert(kStages >= 2, "pipeline needs two stages");
  static_assert(kTmemCols <= 512, "TMEM has 512 columns");
};

// kind::i8 instruction descriptor: s32 accumulate, A u8 (x planes), B s8 (pieces), both
// K-major, M = 128 * CG.
template <int BN, int CG>
__device__ __forceinline__ constexpr uint32_t make_idesc_i8() {
  return (2u << 4)                          // D format: s32
         | (0u << 7)                        // A format: unsigned 8-bit
         | (1u << 10)                       // B format: signed 8-bit
         | (uint32_t(BN >> 3) << 17)        // N >> 3
         | (uint32_t((kBM * CG) >> 4) << 24);  // M >> 4
}

template <int CG>
__device__ __forceinline__ void mma_i8(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc,
                                       uint32_t accumulate) {
  if (CG == 2)
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
        "l"(a), "l"(b), "r"(idesc), "r"(accumulate));
  else
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
        "l"(a), "l"(b), "r"(idesc), "r"(accumulate));
}

// shared::cluster address of the same smem offset in CTA `r` of the cluster
__device__ __forceinline__ uint32_t map_rank(uint32_t addr, uint32_t r) {
  uint32_t out;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(out) : "r"(addr), "r"(r));
  return out;
}
// TMA into this smem offset of every CTA in `mask`, each completion counted on the
// destination pair leader's mbarrier (cta_group::2)
__device__ __forceinline__ void tma_load_2d_pair_mc(uint32_t dst, const CUtensorMap* map, int x,
                                                    int y, uint32_t leader_bar, uint16_t mask) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      ".multicast::cluster [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(leader_bar), "h"(mask)
      : "memory");
}
__device__ __forceinline__ void mma_commit_pair_mask(uint32_t bar, uint16_t mask) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], %1;" ::"r"(bar),
      "h"(mask)
      : "memory");
}

// 4 bits (LSB first) -> 4 bytes of 0/1
__device__ __forceinline__ uint32_t spread4(uint32_t nib) { return (nib * 0x00204081u) & 0x01010101u; }

// One 16-byte bit row (128 elements) -> row r of the x tile (0/1) and of the x<<7 tile
// (0/128), 128 bytes each, 16-B chunk c stored at chunk c ^ (r & 7) (the 128-B swizzle;
// the same byte layout serves a K-major row and an MN-major row).
__device__ __forceinline__ void expand_bit_row(const uint8_t* src, uint8_t* x_tile,
                                               uint8_t* x7_tile, int r) {
  const uint4 b = *reinterpret_cast<const uint4*>(src);
  const uint32_t bw[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    // chunk c: elements 16c..16c+15 = bytes 2c, 2c+1 of the bit row
    const uint32_t two = (bw[c >> 1] >> ((c & 1) * 16)) & 0xFFFFu;
    const uint4 x = make_uint4(spread4(two & 15u), spread4((two >> 4) & 15u),
                               spread4((two >> 8) & 15u), spread4(two >> 12));
    const uint32_t off = uint32_t(r * 128 + ((c ^ (r & 7)) << 4));
    *reinterpret_cast<uint4*>(x_tile + off) = x;
    *reinterpret_cast<uint4*>(x7_tile + off) = make_uint4(x.x << 7, x.y << 7, x.z << 7, x.w << 7);
  }
}

// Epilogue of the bit-plane forward (warps 2..5; warp % 4 = TMEM lane quadrant): per
// 32-column chunk TMEM -> registers (thread = row) -> s (acc_a 2^-7 + acc_b 2^-14) + bias
// -> tanh -> [int8 activation pieces] -> swizzled smem block -> TMA store of the full
// plane (+ the tf32 residual plane through a second block when `lo_block`).
// row_off: this CTA's first row inside a kRowsT-row tile; leader: the CTA of the cluster
// whose tempty barrier counts the drain; MS: 128-row M subtiles per CTA and tile (their
// accumulator pairs side by side in TMEM, rows row_off + 128 s).
template <int BN, int CG, int KBUFS, int MS = 1, int EG = 1>
__device__ __forceinline__ void i8_fwd_epilogue(const I8Params& p, const TileMap& tm,
                                                const CUtensorMap* tmOut,
                                                const CUtensorMap* tmOutLo, uint32_t tmem_base,
                                                uint32_t bar_tfull, uint32_t bar_tempty,
                                                uint32_t leader, uint32_t row_off, int kRowsT,
                                                int cl_id, int n_cl, uint32_t blk,
                                                uint8_t* blk_ptr, bool lo_block) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int q = warp & 3;
  // EG > 1: further groups of 4 epilogue warps (warps 10..13, 14..17) take every EG-th
  // chunk
  const int grp = warp < 2 + kEpiWarps ? 0 : (warp - 2 - kEpiWarps - kConvWarps) / kEpiWarps + 1;
  const int num_tiles = tm.m_tiles * tm.n_tiles;
  const bool write_lo = lo_block && p.write_lo;
  int it = 0;
  for (int t = cl_id; t < num_tiles; t += n_cl, ++it) {
    const int nt = t % tm.n_tiles, mt = t / tm.n_tiles;
    const int n0 = nt * BN;
    const int acc_buf = it % KBUFS;
    mbar_wait(bar_tfull + 8 * acc_buf, (it / KBUFS) & 1);
    tc_fence_after();
#pragma unroll 1
    for (int sub = 0; sub < MS; ++sub) {
    const int rbase = mt * kRowsT + int(row_off) + sub * kBM + q * 32;
    const uint32_t ta = tmem_base + uint32_t((acc_buf * MS + sub) * 2 * BN) + (uint32_t(q * 32) << 16);
    const uint32_t tb = ta + uint32_t(BN);
#pragma unroll 1
    for (int c = 32 * grp; c < BN; c += 32 * EG) {
      const int nb = n0 + c;
      uint32_t ra[32], rb[32];
      tmem_ld32(ta + uint32_t(c), ra);
      tmem_ld32(tb + uint32_t(c), rb);
      const bool colok = nb + lane < p.N;
      const float sc = colok ? __ldg(p.scale + nb + lane) : 0.f;
      const float bi = colok ? __ldg(p.bias + nb + lane) : 0.f;
      float o[32];
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const float s = __shfl_sync(0xffffffffu, sc, j);
        const float bj = __shfl_sync(0xffffffffu, bi, j);
        const float z = fmaf(float(int(ra[j])), s * 0.0078125f,
                             float(int(rb[j])) * (s * 6.103515625e-05f));
        o[j] = tanh_fast(z + bj);
      }
      // the same activations as int8 pieces for the next layer's int8 GEMM
      if (p.out_q != nullptr && nb < p.N && rbase + lane < p.M)
        write_act_pieces(o, p.out_q, long(p.M) * p.N, long(rbase + lane) * p.N + nb);
      if (lane == 0) bulk_wait_read();
      __syncwarp();
#pragma unroll
      for (int j4 = 0; j4 < 8; ++j4) {
        *reinterpret_cast<float4*>(blk_ptr + swz(lane, j4)) =
            make_float4(o[4 * j4], o[4 * j4 + 1], o[4 * j4 + 2], o[4 * j4 + 3]);
        if (write_lo)
          *reinterpret_cast<float4*>(blk_ptr + 4096 + swz(lane, j4)) = make_float4(
              o[4 * j4] - tf32_hi(o[4 * j4]), o[4 * j4 + 1] - tf32_hi(o[4 * j4 + 1]),
              o[4 * j4 + 2] - tf32_hi(o[4 * j4 + 2]), o[4 * j4 + 3] - tf32_hi(o[4 * j4 + 3]));
      }
      fence_async_smem();
      __syncwarp();
      if (lane == 0) {
        tma_store_2d(tmOut, nb, rbase, blk);
        if (write_lo) tma_store_2d(tmOutLo, nb, rbase, blk + 4096);
        bulk_commit();
      }
    }
    }
    tc_fence_before();
    __syncwarp();
    if (lane == 0) {
      if (CG == 2) mbar_arrive_cluster(map_rank(bar_tempty + 8 * acc_buf, leader));
      else mbar_arrive(bar_tempty + 8 * acc_buf);
    }
  }
}

// MC == 2 (CG == 2 only): clusters of two CTA pairs stacked along M (512-row tiles)
// sharing each weight-piece tile: pair 0 TMA-multicasts it into both pairs' smem, halving
// the L2->SM piece traffic that bounds this kernel.
template <int BN, int CG, int MC = 1>
__global__ void __launch_bounds__(kThreadsI8, 1)
    gemm_i8_bits_fwd_kernel(const __grid_constant__ CUtensorMap tmBits,
                            const __grid_constant__ CUtensorMap tmQ,
                            const __grid_constant__ CUtensorMap tmOut,
                            const __grid_constant__ CUtensorMap tmOutLo, const I8Params p,
                            const TileMap tm) {
  using S = SmemI8<BN, CG>;
  static_assert(MC == 1 || CG == 2, "multicast pairs need CTA pairs");
  constexpr int kCl = CG * MC;                      // CTAs per cluster
  const uint32_t crank = CG == 2 ? cluster_rank() : 0u;
  const uint32_t rank = crank & 1u;                 // rank within the pair
  const uint32_t pair = crank >> 1;                 // pair within the cluster (MC == 2)
  const uint32_t leader = crank & ~1u;              // this pair's leader CTA
  const int cl_id = int(blockIdx.x) / kCl;
  const int n_cl = int(gridDim.x) / kCl;
  constexpr int kRowsT = kBM * CG * MC;             // rows per tile
  auto to_leader = [&](uint32_t a) { return MC == 2 ? map_rank(a, leader) : map_rank0(a); };
  extern __shared__ uint8_t smem_raw[];
  // 1 KB-aligned base by pointer arithmetic on the __shared__ array (an integer round
  // trip would turn every staging access into a generic LD/ST)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const uint32_t sbase = smem_u32(smem);
  const uint32_t bar_full = sbase + S::kBarOff;
  const uint32_t bar_conv = bar_full + 8 * S::kStages;
  const uint32_t bar_empty = bar_conv + 8 * S::kStages;
  const uint32_t bar_ufull = bar_empty + 8 * S::kStages;   // [ring]
  const uint32_t bar_uempty = bar_ufull + 8 * S::kRing;    // [ring]
  const uint32_t bar_tfull = bar_uempty + 8 * S::kRing;    // [2]
  const uint32_t bar_tempty = bar_tfull + 16;              // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + S::kBarOff + S::kNumBars * 8);
  constexpr int kOffX128 = S::kX, kOffQ = 2 * S::kX;

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int num_tiles = tm.m_tiles * tm.n_tiles;
  const int kb_total = (p.K + kBKi - 1) / kBKi;

  if (warp == 0 && lane == 0) {
    prefetch_tmap(&tmBits);
    prefetch_tmap(&tmQ);
    for (int s = 0; s < S::kStages; ++s) {
      mbar_init(bar_full + 8 * s, 1);
      mbar_init(bar_conv + 8 * s, kConvWarps * CG);
      mbar_init(bar_empty + 8 * s, MC);  // every pair whose MMAs read the shared pieces
    }
    for (int u = 0; u < S::kRing; ++u) {
      mbar_init(bar_ufull + 8 * u, 1);
      mbar_init(bar_uempty + 8 * u, kConvWarps);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(bar_tfull + 8 * a, 1);
      mbar_init(bar_tempty + 8 * a, kEpiWarps * CG);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    if (CG == 2) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                       smem_u32(tmem_slot)),
                   "n"(S::kTmemCols));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                       smem_u32(tmem_slot)),
                   "n"(S::kTmemCols));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
  }
  tc_fence_before();
  if (CG == 2) cluster_sync_all();
  else __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  // prologue done (barriers, TMEM, tensor maps): wait for the predecessor's writes
  pdl_wait();
  pdl_trigger();

  if (warp == 0) {
    if (lane == 0) {
      // ===== TMA producer =====
      int stage = 0;
      uint32_t phase = 0;
      // bit-row ring cursor, running up to kRing k-blocks ahead of the stages
      int bt = cl_id, bkb = 0, ui = 0;
      uint32_t uph = 0;
      long issued = 0, done = 0;
      for (int t = cl_id; t < num_tiles; t += n_cl) {
        const int nt = t % tm.n_tiles;
        const int n0 = nt * BN + int(rank) * S::kBN;
        for (int kb = 0; kb < kb_total; ++kb, ++done) {
          while (bt < num_tiles && issued < done + S::kRing) {
            mbar_wait(bar_uempty + 8 * ui, uph ^ 1);
            mbar_expect_tx(bar_ufull + 8 * ui, S::kBits);
            const int bm0 = (bt / tm.n_tiles) * kRowsT + int(pair) * kBM * CG + int(rank) * kBM;
            tma_load_2d(sbase + S::kRingOff + ui * S::kBits, &tmBits, bkb * (kBKi / 8), bm0,
                        bar_ufull + 8 * ui);
            ++issued;
            if (++bkb == kb_total) {
              bkb = 0;
              bt += n_cl;
            }
            if (++ui == S::kRing) {
              ui = 0;
              uph ^= 1;
            }
          }
          mbar_wait(bar_empty + 8 * stage, phase ^ 1);
          const uint32_t st = sbase + stage * S::kStage;
          const uint32_t full = CG == 2 ? to_leader(bar_full + 8 * stage) : bar_full + 8 * stage;
          if (rank == 0) mbar_expect_tx(bar_full + 8 * stage, 3 * S::kQ * CG);
          if (MC == 1 || pair == 0) {
#pragma unroll
            for (int pc = 0; pc < 3; ++pc) {
              const int row = pc * int(p.q_rows) + n0;
              if (MC == 2)
                tma_load_2d_pair_mc(st + kOffQ + pc * S::kQ, &tmQ, kb * kBKi, row, full,
                                    uint16_t((1u << rank) | (1u << (rank + 2))));
              else if (CG == 2)
                tma_load_2d_pair(st + kOffQ + pc * S::kQ, &tmQ, kb * kBKi, row, full);
              else
                tma_load_2d(st + kOffQ + pc * S::kQ, &tmQ, kb * kBKi, row, full);
            }
          }
          if (++stage == S::kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && rank == 0) {
      // ===== MMA issuer =====
      constexpr uint32_t idesc = make_idesc_i8<BN, CG>();
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (int t = cl_id; t < num_tiles; t += n_cl, ++it) {
        const int acc_buf = it % S::kBufs;
        mbar_wait(bar_tempty + 8 * acc_buf, ((it / S::kBufs) & 1) ^ 1);
        tc_fence_after();
        const uint32_t tacc_a = tmem_base + uint32_t(acc_buf * 2 * BN);
        const uint32_t tacc_b = tacc_a + uint32_t(BN);
        for (int kb = 0; kb < kb_total; ++kb) {
          mbar_wait(bar_full + 8 * stage, phase);
          mbar_wait(bar_conv + 8 * stage, phase);
          tc_fence_after();
          const uint32_t st = sbase + stage * S::kStage;
#pragma unroll
          for (int k = 0; k < kBKi / 32; ++k) {
            // K-major SW128: +32 B per 32-element K step; SBO = 1 KB between 8-row atoms
            const uint64_t dx = make_sdesc<false>(st + k * 32, 16, 1024);
            const uint64_t dx7 = make_sdesc<false>(st + kOffX128 + k * 32, 16, 1024);
            const uint64_t dq0 = make_sdesc<false>(st + kOffQ + k * 32, 16, 1024);
            const uint64_t dq1 = make_sdesc<false>(st + kOffQ + S::kQ + k * 32, 16, 1024);
            const uint64_t dq2 = make_sdesc<false>(st + kOffQ + 2 * S::kQ + k * 32, 16, 1024);
            const uint32_t acc = (kb > 0 || k > 0) ? 1u : 0u;
            mma_i8<CG>(tacc_a, dx7, dq0, idesc, acc);
            mma_i8<CG>(tacc_a, dx, dq1, idesc, 1u);
            mma_i8<CG>(tacc_b, dx, dq2, idesc, acc);
          }
          if (MC == 2) mma_commit_pair_mask(bar_empty + 8 * stage, uint16_t(0xF));
          else if (CG == 2) mma_commit_pair(bar_empty + 8 * stage);
          else mma_commit(bar_empty + 8 * stage);
          if (++stage == S::kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
        if (MC == 2) mma_commit_pair_mask(bar_tfull + 8 * acc_buf, uint16_t(3u << leader));
        else if (CG == 2) mma_commit_pair(bar_tfull + 8 * acc_buf);
        else mma_commit(bar_tfull + 8 * acc_buf);
      }
    }
  } else if (warp >= 2 + kEpiWarps) {
    // ===== converters: 16-B bit row -> 128-B x row and x<<7 row (SW128 K-major) =====
    const int r = threadIdx.x - (2 + kEpiWarps) * 32;  // tile row 0..127
    int stage = 0;
    uint32_t phase = 0;
    int ui = 0;
    uint32_t uph = 0;
    for (int t = cl_id; t < num_tiles; t += n_cl) {
      for (int kb = 0; kb < kb_total; ++kb) {
        mbar_wait(bar_ufull + 8 * ui, uph);           // bit rows arrived
        mbar_wait(bar_empty + 8 * stage, phase ^ 1);  // the MMA released this stage
        uint8_t* st = smem + stage * S::kStage;
        expand_bit_row(smem + S::kRingOff + ui * S::kBits + r * 16, st, st + kOffX128, r);
        fence_async_smem();
        __syncwarp();
        if (lane == 0) {
          if (CG == 2) mbar_arrive_cluster(to_leader(bar_conv + 8 * stage));
          else mbar_arrive(bar_conv + 8 * stage);
          mbar_arrive(bar_uempty + 8 * ui);
        }
        if (++ui == S::kRing) {
          ui = 0;
          uph ^= 1;
        }
        if (++stage == S::kStages) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else {
    // ===== epilogue: warps 2..5 own TMEM lane quadrants (warp % 4) =====
    const int ew = warp - 2;
    i8_fwd_epilogue<BN, CG, S::kBufs>(p, tm, &tmOut, &tmOutLo, tmem_base, bar_tfull, bar_tempty,
                                      leader, pair * kBM * CG + rank * kBM, kRowsT, cl_id, n_cl,
                                      sbase + S::kEpiOff + uint32_t(ew * 2 * 4096),
                                      smem + S::kEpiOff + ew * 2 * 4096, true);
    if (lane == 0) bulk_wait_all();
  }

  tc_fence_before();
  if (CG == 2) cluster_sync_all();
  else __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    if (CG == 2)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                   "n"(S::kTmemCols));
    else
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                   "n"(S::kTmemCols));
  }
}

// ---------------------------------------------------------------------------
// Decoupled-ring variant of the bit-plane forward.  In gemm_i8_bits_fwd_kernel one stage
// holds both operands of a k-block (x, x<<7 from the converters, the three weight-piece
// tiles by TMA from L2), so a released stage waits for the slower of the two refills and
// only three 56 KB stages fit.  Here the two operands have their own rings, sized by
// their refill latency:
//   Q ring  NQ x 24 KB  weight pieces (TMA, L2 latency), refilled NQ k-blocks ahead
//   X ring  NX x 32 KB  expanded planes (converter warps, a few hundred cycles)
//   bit rows 4 x 2 KB   (TMA from HBM, feeding the converters)
// The MMA of k-block kb waits for Q slot kb % NQ and X slot kb % NX and releases both
// with one commit each.  The epilogue stages through one 4 KB block per warp (the
// residual plane is not written: write_lo must be 0).  MS: 128-row M subtiles per CTA
// sharing each piece tile; EG: epilogue warp groups (warps 2..5, 10..13, 14..17) on
// alternate 32-column chunks.  The default (launch_i8_bits_fwd) is <256, 2, 2, 2, 1, 3>:
// 256-column tiles, single-buffered accumulators drained by twelve epilogue warps.
template <int BN, int CG, int NQ, int NX, int MS = 1, int EG = 1>
struct SmemI8Dec {
  static constexpr int kX = kBM * kBKi;           // 16 KB operand tile (x, x<<7)
  static constexpr int kBits = MS * kBM * kBKi / 8;  // packed source rows of the CTA's rows
  static constexpr int kBN = BN / CG;
  static constexpr int kQ = kBN * kBKi;           // one piece tile
  static constexpr int kQSlot = 3 * kQ;
  static constexpr int kXSlot = MS * 2 * kX;      // per M subtile: x, x<<7
  static constexpr int kRing = MS == 1 ? 4 : 2;
  static constexpr int kXOff = NQ * kQSlot;
  static constexpr int kRingOff = kXOff + NX * kXSlot;
  static constexpr int kBarOff = kRingOff + kRing * kBits;
  // q_full, q_empty [NQ]; x_full, x_empty [NX]; u_full, u_empty [ring]; tfull, tempty [2]
  static constexpr int kNumBars = 2 * NQ + 2 * NX + 2 * kRing + 4;
  static constexpr int kEpiOff = (kBarOff + kNumBars * 8 + 16 + 1023) / 1024 * 1024;
  static constexpr int kBytes = kEpiOff + EG * kEpiWarps * 4096 + 1024;
  static constexpr int kBufs = 4 * BN * MS <= 512 ? 2 : 1;
  static constexpr int kTmemCols = 2 * BN * MS * kBufs;
  static_assert(kQSlot % 1024 == 0 && kXSlot % 1024 == 0, "1 KB swizzle alignment");
  static_assert(NQ >= 2 && NX >= 2, "rings need two slots");
  static_assert(kBytes <= 227 * 1024, "shared memory budget");
};

// ring cursor: slot and phase of the n-th use
struct RingPos {
  int slot = 0;
  uint32_t phase = 0;
  __device__ __forceinline__ void next(int n) {
    if (++slot == n) {
      slot = 0;
      phase ^= 1u;
    }
  }
};

template <int BN, int CG, int NQ, int NX, int MS = 1, int EG = 1>
__global__ void __launch_bounds__(kThreadsI8 + 32 * kEpiWarps * (EG - 1), 1)
    gemm_i8_bits_fwd_dec_kernel(const __grid_constant__ CUtensorMap tmBits,
                                const __grid_constant__ CUtensorMap tmQ,
                                const __grid_constant__ CUtensorMap tmOut,
                                const __grid_constant__ CUtensorMap tmOutLo, const I8Params p,
                                const TileMap tm) {
  using S = SmemI8Dec<BN, CG, NQ, NX, MS, EG>;
  const uint32_t rank = CG == 2 ? cluster_rank() : 0u;
  const int cl_id = CG == 2 ? int(blockIdx.x >> 1) : int(blockIdx.x);
  const int n_cl = CG == 2 ? int(gridDim.x >> 1) : int(gridDim.x);
  // rows per tile; CTA `rank` holds rows [rank * 128 MS, (rank + 1) * 128 MS) of it, and
  // M subtile s of the pair MMA is rows 128 s of each CTA's block
  constexpr int kRowsT = kBM * CG * MS;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const uint32_t sbase = smem_u32(smem);
  const uint32_t q_full = sbase + S::kBarOff;
  const uint32_t q_empty = q_full + 8 * NQ;
  const uint32_t x_full = q_empty + 8 * NQ;
  const uint32_t x_empty = x_full + 8 * NX;
  const uint32_t u_full = x_empty + 8 * NX;
  const uint32_t u_empty = u_full + 8 * S::kRing;
  const uint32_t bar_tfull = u_empty + 8 * S::kRing;  // [2]
  const uint32_t bar_tempty = bar_tfull + 16;         // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + S::kBarOff + S::kNumBars * 8);
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int num_tiles = tm.m_tiles * tm.n_tiles;
  const int kb_total = (p.K + kBKi - 1) / kBKi;
  auto leader_bar = [&](uint32_t a) { return CG == 2 ? map_rank0(a) : a; };

  if (warp == 0 && lane == 0) {
    prefetch_tmap(&tmBits);
    prefetch_tmap(&tmQ);
    for (int i = 0; i < NQ; ++i) {
      mbar_init(q_full + 8 * i, 1);
      mbar_init(q_empty + 8 * i, 1);
    }
    for (int i = 0; i < NX; ++i) {
      mbar_init(x_full + 8 * i, kConvWarps * CG);
      mbar_init(x_empty + 8 * i, 1);
    }
    for (int u = 0; u < S::kRing; ++u) {
      mbar_init(u_full + 8 * u, 1);
      mbar_init(u_empty + 8 * u, kConvWarps);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(bar_tfull + 8 * a, 1);
      mbar_init(bar_tempty + 8 * a, kEpiWarps * EG * CG);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    if (CG == 2) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                       smem_u32(tmem_slot)),
                   "n"(S::kTmemCols));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                       smem_u32(tmem_slot)),
                   "n"(S::kTmemCols));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
  }
  tc_fence_before();
  if (CG == 2) cluster_sync_all();
  else __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  pdl_wait();
  pdl_trigger();

  if (warp == 0) {
    if (lane == 0) {
      // ===== TMA producer: weight pieces NQ k-blocks ahead of the MMA; bit rows up to
      // kRing k-blocks ahead of the pieces (the converters consume them in order) =====
      RingPos qp, up;
      int bt = cl_id, bkb = 0;
      long issued_bits = 0, issued_q = 0;
      for (int t = cl_id; t < num_tiles; t += n_cl) {
        const int n0 = (t % tm.n_tiles) * BN + int(rank) * S::kBN;
        for (int kb = 0; kb < kb_total; ++kb, ++issued_q) {
          while (bt < num_tiles && issued_bits < issued_q + S::kRing) {
            mbar_wait(u_empty + 8 * up.slot, up.phase ^ 1);
            mbar_expect_tx(u_full + 8 * up.slot, S::kBits);
            const int bm0 = (bt / tm.n_tiles) * kRowsT + int(rank) * kBM * MS;
            tma_load_2d(sbase + S::kRingOff + up.slot * S::kBits, &tmBits, bkb * (kBKi / 8),
                        bm0, u_full + 8 * up.slot);
            ++issued_bits;
            if (++bkb == kb_total) {
              bkb = 0;
              bt += n_cl;
            }
            up.next(S::kRing);
          }
          mbar_wait(q_empty + 8 * qp.slot, qp.phase ^ 1);
          const uint32_t dst = sbase + qp.slot * S::kQSlot;
          const uint32_t full = leader_bar(q_full + 8 * qp.slot);
          if (rank == 0) mbar_expect_tx(q_full + 8 * qp.slot, S::kQSlot * CG);
#pragma unroll
          for (int pc = 0; pc < 3; ++pc) {
            const int row = pc * int(p.q_rows) + n0;
            if (CG == 2) tma_load_2d_pair(dst + pc * S::kQ, &tmQ, kb * kBKi, row, full);
            else tma_load_2d(dst + pc * S::kQ, &tmQ, kb * kBKi, row, full);
          }
          qp.next(NQ);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && rank == 0) {
      // ===== MMA issuer =====
      constexpr uint32_t idesc = make_idesc_i8<BN, CG>();
      RingPos qp, xp;
      int it = 0;
      for (int t = cl_id; t < num_tiles; t += n_cl, ++it) {
        const int acc_buf = it % S::kBufs;
        mbar_wait(bar_tempty + 8 * acc_buf, ((it / S::kBufs) & 1) ^ 1);
        tc_fence_after();
        for (int kb = 0; kb < kb_total; ++kb) {
          mbar_wait(q_full + 8 * qp.slot, qp.phase);
          mbar_wait(x_full + 8 * xp.slot, xp.phase);
          tc_fence_after();
          const uint32_t qs = sbase + qp.slot * S::kQSlot;
#pragma unroll
          for (int sub = 0; sub < MS; ++sub) {
          // the M subtiles share this k-block's weight-piece tiles
          const uint32_t tacc_a = tmem_base + uint32_t((acc_buf * MS + sub) * 2 * BN);
          const uint32_t tacc_b = tacc_a + uint32_t(BN);
          const uint32_t xs = sbase + S::kXOff + xp.slot * S::kXSlot + sub * 2 * S::kX;
#pragma unroll
          for (int k = 0; k < kBKi / 32; ++k) {
            const uint64_t dx = make_sdesc<false>(xs + k * 32, 16, 1024);
            const uint64_t dx7 = make_sdesc<false>(xs + S::kX + k * 32, 16, 1024);
            const uint64_t dq0 = make_sdesc<false>(qs + k * 32, 16, 1024);
            const uint64_t dq1 = make_sdesc<false>(qs + S::kQ + k * 32, 16, 1024);
            const uint64_t dq2 = make_sdesc<false>(qs + 2 * S::kQ + k * 32, 16, 1024);
            const uint32_t acc = (kb > 0 || k > 0) ? 1u : 0u;
            mma_i8<CG>(tacc_a, dx7, dq0, idesc, acc);
            mma_i8<CG>(tacc_a, dx, dq1, idesc, 1u);
            mma_i8<CG>(tacc_b, dx, dq2, idesc, acc);
          }
          }
          if (CG == 2) {
            mma_commit_pair(q_empty + 8 * qp.slot);
            mma_commit_pair(x_empty + 8 * xp.slot);
          } else {
            mma_commit(q_empty + 8 * qp.slot);
            mma_commit(x_empty + 8 * xp.slot);
          }
          qp.next(NQ);
          xp.next(NX);
        }
        if (CG == 2) mma_commit_pair(bar_tfull + 8 * acc_buf);
        else mma_commit(bar_tfull + 8 * acc_buf);
      }
    }
  } else if (warp >= 2 + kEpiWarps && warp < 2 + kEpiWarps + kConvWarps) {
    // ===== converters: 16-B bit row -> 128-B x row and x<<7 row (SW128 K-major) =====
    const int r = threadIdx.x - (2 + kEpiWarps) * 32;  // tile row 0..127
    RingPos xp, up;
    for (int t = cl_id; t < num_tiles; t += n_cl) {
      for (int kb = 0; kb < kb_total; ++kb) {
        mbar_wait(u_full + 8 * up.slot, up.phase);           // bit rows arrived
        mbar_wait(x_empty + 8 * xp.slot, xp.phase ^ 1);      // the MMA released the slot
        uint8_t* xs = smem + S::kXOff + xp.slot * S::kXSlot;
#pragma unroll
        for (int sub = 0; sub < MS; ++sub)
          expand_bit_row(smem + S::kRingOff + up.slot * S::kBits + (sub * kBM + r) * 16,
                         xs + sub * 2 * S::kX, xs + sub * 2 * S::kX + S::kX, r);
        fence_async_smem();
        __syncwarp();
        if (lane == 0) {
          if (CG == 2) mbar_arrive_cluster(map_rank0(x_full + 8 * xp.slot));
          else mbar_arrive(x_full + 8 * xp.slot);
          mbar_arrive(u_empty + 8 * up.slot);
        }
        up.next(S::kRing);
        xp.next(NX);
      }
    }
  } else {
    // ===== epilogue (warps 2..5, + 10..13 when EG >= 2, + 14..17 when EG == 3) =====
    const int ew = warp < 2 + kEpiWarps ? warp - 2 : warp - 2 - kConvWarps;
    i8_fwd_epilogue<BN, CG, S::kBufs, MS, EG>(p, tm, &tmOut, &tmOutLo, tmem_base, bar_tfull,
                                          bar_tempty, 0u, rank * kBM * MS, kRowsT, cl_id, n_cl,
                                      sbase + S::kEpiOff + uint32_t(ew * 4096),
                                      smem + S::kEpiOff + ew * 4096, false);
    if (lane == 0) bulk_wait_all();
  }

  tc_fence_before();
  if (CG == 2) cluster_sync_all();
  else __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    if (CG == 2)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                   "n"(S::kTmemCols));
    else
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                   "n"(S::kTmemCols));
  }
}

// ---------------------------------------------------------------------------
// Forward of a layer whose input activations are int8 pieces (fixed scale 1/127, from the
// int8 layer-1 epilogue) and whose weights are int8 row pieces (scale s_n):
//   A = a0 + a1/2^7 + a2/2^14 (x 1/127),  B = s_n (b0 + b1/2^7 + b2/2^14)
//   sum_k A B = s_n/127 [acc0 + acc1/2^7 + acc2/2^14],
//   acc0 = a0.b0,  acc1 = a0.b1 + a1.b0,  acc2 = a0.b2 + a1.b1 + a2.b0  (six int8 MMAs;
// the dropped a1.b2 + a2.b1 + a2.b2 terms are < 2^-21 of a0.b0's scale).
// Three int32 TMEM accumulators (single-buffered); epilogue as the tf32 forward: bias +
// tanh, optional fused policy/value heads, full fp32 plane (+ optional residual plane).
struct I8x2Params {
  int M, N, K;
  const float* scale;  // [N] weight piece scales
  const float* bias;   // [N]
  long a_rows;         // rows per piece of the stacked activation pieces [3][a_rows][K]
  long q_rows;         // rows per piece of the stacked weight pieces [3][q_rows][Kp]
  const float* head_w;   // fused heads as in Params (gemm_sm100.cuh)
  const float* head_wv;
  int head_k;
  float* head_part;
  int has_lo;
  int8_t* out_q;  // optional: tanh outputs as int8 pieces [3][M][N] for the next int8 layer
  int has_out;    // 0: no fp32 plane (the pieces or the fused heads are what is read)
};

template <int BN_, int CG>
struct SmemI8x2 {
  static constexpr int BN = BN_;
  // three accumulators; double-buffered when they fit TMEM twice (BN = 64)
  static constexpr int kBufs = 6 * BN <= 512 ? 2 : 1;
  static constexpr int kA = kBM * kBKi;          // 16 KB per activation piece tile
  static constexpr int kBN = BN / CG;
  static constexpr int kQ = kBN * kBKi;          // per weight piece tile
  static constexpr int kStage = 3 * kA + 3 * kQ;
  static constexpr int kEpi = kEpiWarps * (2 * 4096 + 1024);
  static constexpr int kStagesRaw = (225 * 1024 - kEpi - 2048) / kStage;
  static constexpr int kStages = kStagesRaw > 4 ? 4 : kStagesRaw;
  static constexpr int kBarOff = kStages * kStage;
  static constexpr int kNumBars = 2 * kStages + 4;  // full, empty; tfull[2], tempty[2]
  static constexpr int kEpiOff = (kBarOff + kNumBars * 8 + 16 + 1023) / 1024 * 1024;
  static constexpr int kBytes = kEpiOff + kEpi + 1024;
  static constexpr int kTmemCols = 512;  // 3 x 128 accumulator columns
  static_assert(kStage % 1024 == 0, "stages must keep the 1 KB swizzle alignment");
  static_assert(kStages >= 2, "pipeline needs two stages");
};

template <int BN, int CG>
__device__ __forceinline__ constexpr uint32_t make_idesc_i8x2() {
  return (2u << 4) | (1u << 7) | (1u << 10)  // s32 <- s8 x s8, both K-major
         | (uint32_t(BN >> 3) << 17) | (uint32_t((kBM * CG) >> 4) << 24);
}

template <int BN_, int CG>
__global__ void __launch_bounds__(32 * (2 + kEpiWarps), 1)
    gemm_i8x2_fwd_kernel(const __grid_constant__ CUtensorMap tmA,
                         const __grid_constant__ CUtensorMap tmQ,
                         const __grid_constant__ CUtensorMap tmOut,
                         const __grid_constant__ CUtensorMap tmOutLo, const I8x2Params p,
                         const TileMap tm) {
  using S = SmemI8x2<BN_, CG>;
  constexpr int BN = S::BN;
  const uint32_t rank = CG == 2 ? cluster_rank() : 0u;
  const int cl_id = CG == 2 ? int(blockIdx.x >> 1) : int(blockIdx.x);
  const int n_cl = CG == 2 ? int(gridDim.x >> 1) : int(gridDim.x);
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const uint32_t sbase = smem_u32(smem);
  const uint32_t bar_full = sbase + S::kBarOff;
  const uint32_t bar_empty = bar_full + 8 * S::kStages;
  const uint32_t bar_tfull = bar_empty + 8 * S::kStages;  // [2]
  const uint32_t bar_tempty = bar_tfull + 16;              // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + S::kBarOff + S::kNumBars * 8);
  constexpr int kOffQ = 3 * S::kA;

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int num_tiles = tm.m_tiles * tm.n_tiles;
  const int kb_total = (p.K + kBKi - 1) / kBKi;

  if (warp == 0 && lane == 0) {
    prefetch_tmap(&tmA);
    prefetch_tmap(&tmQ);
    for (int s = 0; s < S::kStages; ++s) {
      mbar_init(bar_full + 8 * s, 1);
      mbar_init(bar_empty + 8 * s, 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(bar_tfull + 8 * b, 1);
      mbar_init(bar_tempty + 8 * b, kEpiWarps * CG);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    if (CG == 2) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                       smem_u32(tmem_slot)),
                   "n"(S::kTmemCols));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                       smem_u32(tmem_slot)),
                   "n"(S::kTmemCols));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
  }
  tc_fence_before();
  if (CG == 2) cluster_sync_all();
  else __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  // prologue done (barriers, TMEM, tensor maps): wait for the predecessor's writes
  pdl_wait();
  pdl_trigger();

  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int t = cl_id; t < num_tiles; t += n_cl) {
        const int nt = t % tm.n_tiles, mt = t / tm.n_tiles;
        const int m0 = mt * kBM * CG + int(rank) * kBM;
        const int n0 = nt * BN + int(rank) * S::kBN;
        for (int kb = 0; kb < kb_total; ++kb) {
          mbar_wait(bar_empty + 8 * stage, phase ^ 1);
          const uint32_t st = sbase + stage * S::kStage;
          const uint32_t full = CG == 2 ? map_rank0(bar_full + 8 * stage) : bar_full + 8 * stage;
          if (rank == 0) mbar_expect_tx(bar_full + 8 * stage, (3 * S::kA + 3 * S::kQ) * CG);
#pragma unroll
          for (int pc = 0; pc < 3; ++pc) {
            const int arow = int(pc * p.a_rows) + m0, qrow = int(pc * p.q_rows) + n0;
            if (CG == 2) {
              tma_load_2d_pair(st + pc * S::kA, &tmA, kb * kBKi, arow, full);
              tma_load_2d_pair(st + kOffQ + pc * S::kQ, &tmQ, kb * kBKi, qrow, full);
            } else {
              tma_load_2d(st + pc * S::kA, &tmA, kb * kBKi, arow, full);
              tma_load_2d(st + kOffQ + pc * S::kQ, &tmQ, kb * kBKi, qrow, full);
            }
          }
          if (++stage == S::kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && rank == 0) {
      constexpr uint32_t idesc = make_idesc_i8x2<BN, CG>();
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (int t = cl_id; t < num_tiles; t += n_cl, ++it) {
        const int buf = S::kBufs == 2 ? (it & 1) : 0;
        const uint32_t tph = S::kBufs == 2 ? ((it >> 1) & 1) : (it & 1);
        mbar_wait(bar_tempty + 8 * buf, tph ^ 1);
        tc_fence_after();
        const uint32_t t0 = tmem_base + uint32_t(buf * 3 * BN), t1 = t0 + uint32_t(BN),
                       t2 = t0 + uint32_t(2 * BN);
        for (int kb = 0; kb < kb_total; ++kb) {
          mbar_wait(bar_full + 8 * stage, phase);
          tc_fence_after();
          const uint32_t st = sbase + stage * S::kStage;
#pragma unroll
          for (int k = 0; k < kBKi / 32; ++k) {
            uint64_t da[3], dq[3];
#pragma unroll
            for (int pc = 0; pc < 3; ++pc) {
              da[pc] = make_sdesc<false>(st + pc * S::kA + k * 32, 16, 1024);
              dq[pc] = make_sdesc<false>(st + kOffQ + pc * S::kQ + k * 32, 16, 1024);
            }
            const uint32_t acc = (kb > 0 || k > 0) ? 1u : 0u;
            mma_i8<CG>(t0, da[0], dq[0], idesc, acc);
            mma_i8<CG>(t1, da[0], dq[1], idesc, acc);
            mma_i8<CG>(t1, da[1], dq[0], idesc, 1u);
            mma_i8<CG>(t2, da[0], dq[2], idesc, acc);
            mma_i8<CG>(t2, da[1], dq[1], idesc, 1u);
            mma_i8<CG>(t2, da[2], dq[0], idesc, 1u);
          }
          if (CG == 2) mma_commit_pair(bar_empty + 8 * stage);
          else mma_commit(bar_empty + 8 * stage);
          if (++stage == S::kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
        if (CG == 2) mma_commit_pair(bar_tfull + 8 * buf);
        else mma_commit(bar_tfull + 8 * buf);
      }
    }
  } else {
    const int q = warp & 3;
    const int ew = warp - 2;
    const uint32_t blk = sbase + S::kEpiOff + uint32_t(ew * (2 * 4096 + 1024));
    uint8_t* blk_ptr = smem + S::kEpiOff + ew * (2 * 4096 + 1024);
    float* wsm = reinterpret_cast<float*>(blk_ptr + 2 * 4096);  // head weights [8][32]
    constexpr int kHK = 8;
    const bool do_head = p.head_k > 0;
    int it = 0;
    for (int t = cl_id; t < num_tiles; t += n_cl, ++it) {
      const int nt = t % tm.n_tiles, mt = t / tm.n_tiles;
      const int m0 = mt * kBM * CG + int(rank) * kBM, n0 = nt * BN;
      const int rbase = m0 + q * 32;
      const int buf = S::kBufs == 2 ? (it & 1) : 0;
      mbar_wait(bar_tfull + 8 * buf, S::kBufs == 2 ? ((it >> 1) & 1) : (it & 1));
      tc_fence_after();
      const uint32_t ta = tmem_base + uint32_t(buf * 3 * BN) + (uint32_t(q * 32) << 16);
      float zacc[kHK];
#pragma unroll
      for (int k = 0; k < kHK; ++k) zacc[k] = 0.f;
#pragma unroll 1
      for (int c = 0; c < BN; c += 32) {
        const int nb = n0 + c;
        uint32_t r0[32], r1[32], r2[32];
        tmem_ld32(ta + uint32_t(c), r0);
        tmem_ld32(ta + uint32_t(BN + c), r1);
        tmem_ld32(ta + uint32_t(2 * BN + c), r2);
        const bool colok = nb + lane < p.N;
        const float sc = colok ? __ldg(p.scale + nb + lane) * (1.f / 127.f) : 0.f;
        const float bi = colok ? __ldg(p.bias + nb + lane) : 0.f;
        float o[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const float s = __shfl_sync(0xffffffffu, sc, j);
          const float bj = __shfl_sync(0xffffffffu, bi, j);
          const float v = fmaf(float(int(r2[j])), 6.103515625e-05f,
                               fmaf(float(int(r1[j])), 0.0078125f, float(int(r0[j]))));
          o[j] = tanh_fast(fmaf(v, s, bj));
        }
        if (p.out_q != nullptr && nb < p.N && rbase + lane < p.M)
          write_act_pieces(o, p.out_q, long(p.M) * p.N, long(rbase + lane) * p.N + nb);
        if (do_head) {
#pragma unroll
          for (int k = 0; k < kHK; ++k) {
            float wk = 0.f;
            if (k < p.head_k && colok) {
              const float* wrow = k < p.head_k - 1 ? p.head_w + long(k) * p.N : p.head_wv;
              wk = __ldg(wrow + nb + lane);
            }
            wsm[k * 32 + lane] = wk;
          }
          __syncwarp();
          // j-outer / k-inner: the head_k dot products advance together (independent
          // FMA chains hide the latency; per k the summation order is unchanged)
#pragma unroll
          for (int j4 = 0; j4 < 8; ++j4) {
#pragma unroll
            for (int k = 0; k < kHK; ++k) {
              if (k < p.head_k) {
                const float4 w4 = *reinterpret_cast<const float4*>(wsm + k * 32 + 4 * j4);
                zacc[k] = fmaf(w4.x, o[4 * j4], zacc[k]);
                zacc[k] = fmaf(w4.y, o[4 * j4 + 1], zacc[k]);
                zacc[k] = fmaf(w4.z, o[4 * j4 + 2], zacc[k]);
                zacc[k] = fmaf(w4.w, o[4 * j4 + 3], zacc[k]);
              }
            }
          }
          __syncwarp();
        }
        if (!p.has_out) continue;
        if (lane == 0) bulk_wait_read();
        __syncwarp();
#pragma unroll
        for (int j4 = 0; j4 < 8; ++j4) {
          *reinterpret_cast<float4*>(blk_ptr + swz(lane, j4)) =
              make_float4(o[4 * j4], o[4 * j4 + 1], o[4 * j4 + 2], o[4 * j4 + 3]);
          if (p.has_lo)
            *reinterpret_cast<float4*>(blk_ptr + 4096 + swz(lane, j4)) =
                make_float4(o[4 * j4] - tf32_hi(o[4 * j4]), o[4 * j4 + 1] - tf32_hi(o[4 * j4 + 1]),
                            o[4 * j4 + 2] - tf32_hi(o[4 * j4 + 2]),
                            o[4 * j4 + 3] - tf32_hi(o[4 * j4 + 3]));
        }
        fence_async_smem();
        __syncwarp();
        if (lane == 0) {
          tma_store_2d(&tmOut, nb, rbase, blk);
          if (p.has_lo) tma_store_2d(&tmOutLo, nb, rbase, blk + 4096);
          bulk_commit();
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if (CG == 2) mbar_arrive_cluster(map_rank0(bar_tempty + 8 * buf));
        else mbar_arrive(bar_tempty + 8 * buf);
      }
      if (do_head && rbase + lane < p.M) {
        float* hp = p.head_part + (long(nt) * p.M + rbase + lane) * p.head_k;
#pragma unroll
        for (int k = 0; k < kHK; ++k)
          if (k < p.head_k) hp[k] = zacc[k];
      }
    }
    if (lane == 0) bulk_wait_all();
  }

  tc_fence_before();
  if (CG == 2) cluster_sync_all();
  else __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    if (CG == 2)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                   "n"(S::kTmemCols));
    else
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                   "n"(S::kTmemCols));
  }
}

// ---------------------------------------------------------------------------
// Weight gradient of a binary-plane layer:  dW[m][n] = sum_f dZ[f][m] X[f][n]
//   A = dZ as fixed-point int8 pieces, MN-major [3][F][M] (quantize_cols_kernel, one
//       scale per (K split, m): s = colmax / 127, colmax from the dX epilogue);
//   B = X bit rows [F][pitch] (MN-major after expansion);  K = frames, split-K.
// Each CTA holds 128 rows of M (a pair: 256) and 128 columns of N; per split the int32
// accumulators are exact (|acc| < 2^31 for <= 131072 frames per split) and the epilogue
// writes s_m (acc_a / 2^7 + acc_b / 2^14) into the fp32 split-K workspace.
template <int CG>
struct SmemI8Dw {
  static constexpr int kPiece = kBM * kBKi;     // 16 KB: 128 k rows x 128 m bytes
  static constexpr int kX = kBKi * 128;         // 16 KB: 128 k rows x 128 n
  static constexpr int kBits = kBKi * 16;       // 2 KB
  static constexpr int kStage = 3 * kPiece + 2 * kX + kBits;
  static constexpr int kEpi = kEpiWarps * 4096;
  static constexpr int kStagesRaw = (225 * 1024 - kEpi - 2048) / kStage;
  static constexpr int kStages = kStagesRaw > 4 ? 4 : kStagesRaw;
  static constexpr int kBarOff = kStages * kStage;
  static constexpr int kNumBars = 4 * kStages + 2;  // full, xfull, conv, empty; tfull, tempty
  static constexpr int kEpiOff = (kBarOff + kNumBars * 8 + 16 + 1023) / 1024 * 1024;
  static constexpr int kBytes = kEpiOff + kEpi + 1024;
  static constexpr int BN = 128 * CG;
  static constexpr int kTmemCols = 2 * BN;  // 2 accumulators, single-buffered
  static_assert(kStage % 1024 == 0, "stages must keep the 1 KB swizzle alignment");
  static_assert(kStages >= 2, "pipeline needs two stages");
};

struct I8DwParams {
  int M, N, K;          // M = out features (dZ columns), N = in features (planes), K = frames
  int kb_per_split;     // 128-frame k-blocks per split (colmax group = kb_per_split * 128 rows)
  long f_rows;          // rows per piece in the stacked [3][f_rows][M] piece array
  const unsigned* colmax;  // [splits][M] float bits
};

template <int CG>
__device__ __forceinline__ constexpr uint32_t make_idesc_i8_dw() {
  return (2u << 4)       // D: s32
         | (1u << 7)     // A: signed 8-bit (dZ pieces)
         | (0u << 10)    // B: unsigned 8-bit (planes)
         | (1u << 15)    // A MN-major
         | (1u << 16)    // B MN-major
         | (uint32_t((128 * CG) >> 3) << 17)  // N = 128 * CG
         | (uint32_t((kBM * CG) >> 4) << 24);
}

template <int CG>
__global__ void __launch_bounds__(kThreadsI8, 1)
    gemm_i8_bits_dw_kernel(const __grid_constant__ CUtensorMap tmP,
                           const __grid_constant__ CUtensorMap tmBits,
                           const __grid_constant__ CUtensorMap tmWs, const I8DwParams p,
                           const TileMap tm) {
  using S = SmemI8Dw<CG>;
  constexpr int BN = S::BN;
  const uint32_t rank = CG == 2 ? cluster_rank() : 0u;
  const int cl_id = CG == 2 ? int(blockIdx.x >> 1) : int(blockIdx.x);
  const int n_cl = CG == 2 ? int(gridDim.x >> 1) : int(gridDim.x);
  extern __shared__ uint8_t smem_raw[];
  // 1 KB-aligned base by pointer arithmetic on the __shared__ array (an integer round
  // trip would turn every staging access into a generic LD/ST)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const uint32_t sbase = smem_u32(smem);
  const uint32_t bar_full = sbase + S::kBarOff;
  const uint32_t bar_xfull = bar_full + 8 * S::kStages;
  const uint32_t bar_conv = bar_xfull + 8 * S::kStages;
  const uint32_t bar_empty = bar_conv + 8 * S::kStages;
  const uint32_t bar_tfull = bar_empty + 8 * S::kStages;
  const uint32_t bar_tempty = bar_tfull + 8;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + S::kBarOff + S::kNumBars * 8);
  constexpr int kOffX = 3 * S::kPiece, kOffX128 = kOffX + S::kX, kOffBits = kOffX + 2 * S::kX;

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int num_tiles = tm.m_tiles * tm.n_tiles * tm.splits;
  const int kb_total = (p.K + kBKi - 1) / kBKi;

  if (warp == 0 && lane == 0) {
    prefetch_tmap(&tmP);
    prefetch_tmap(&tmBits);
    for (int s = 0; s < S::kStages; ++s) {
      mbar_init(bar_full + 8 * s, 1);
      mbar_init(bar_xfull + 8 * s, 1);
      mbar_init(bar_conv + 8 * s, kConvWarps * CG);
      mbar_init(bar_empty + 8 * s, 1);
    }
    mbar_init(bar_tfull, 1);
    mbar_init(bar_tempty, kEpiWarps * CG);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    if (CG == 2) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                       smem_u32(tmem_slot)),
                   "n"(S::kTmemCols));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                       smem_u32(tmem_slot)),
                   "n"(S::kTmemCols));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
  }
  tc_fence_before();
  if (CG == 2) cluster_sync_all();
  else __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  // prologue done (barriers, TMEM, tensor maps): wait for the predecessor's writes
  pdl_wait();
  pdl_trigger();

  auto decode = [&](int t, int& mt, int& nt, int& sp) {
    nt = t % tm.n_tiles;
    const int r = t / tm.n_tiles;
    mt = r % tm.m_tiles;
    sp = r / tm.m_tiles;
  };

  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int t = cl_id; t < num_tiles; t += n_cl) {
        int mt, nt, sp;
        decode(t, mt, nt, sp);
        const int m0 = mt * kBM * CG + int(rank) * kBM;
        const int n0 = nt * BN + int(rank) * 128;
        const int kb0 = sp * p.kb_per_split, kb1 = min(kb_total, kb0 + p.kb_per_split);
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(bar_empty + 8 * stage, phase ^ 1);
          const uint32_t st = sbase + stage * S::kStage;
          mbar_expect_tx(bar_xfull + 8 * stage, S::kBits);
          tma_load_2d(st + kOffBits, &tmBits, n0 / 8, kb * kBKi, bar_xfull + 8 * stage);
          const uint32_t full = CG == 2 ? map_rank0(bar_full + 8 * stage) : bar_full + 8 * stage;
          if (rank == 0) mbar_expect_tx(bar_full + 8 * stage, 3 * S::kPiece * CG);
#pragma unroll
          for (int pc = 0; pc < 3; ++pc) {
            const int row = int(pc * p.f_rows) + kb * kBKi;
            if (CG == 2) tma_load_2d_pair(st + pc * S::kPiece, &tmP, m0, row, full);
            else tma_load_2d(st + pc * S::kPiece, &tmP, m0, row, full);
          }
          if (++stage == S::kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && rank == 0) {
      constexpr uint32_t idesc = make_idesc_i8_dw<CG>();
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (int t = cl_id; t < num_tiles; t += n_cl, ++it) {
        int mt, nt, sp;
        decode(t, mt, nt, sp);
        const int kb0 = sp * p.kb_per_split, kb1 = min(kb_total, kb0 + p.kb_per_split);
        mbar_wait(bar_tempty, (it & 1) ^ 1);
        tc_fence_after();
        const uint32_t tacc_a = tmem_base, tacc_b = tmem_base + uint32_t(BN);
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(bar_full + 8 * stage, phase);
          mbar_wait(bar_conv + 8 * stage, phase);
          tc_fence_after();
          const uint32_t st = sbase + stage * S::kStage;
#pragma unroll
          for (int k = 0; k < kBKi / 32; ++k) {
            // MN-major int8 SW128 (layout type 2 as K-major; the major-ness is in the
            // instruction descriptor): 32 k rows of 128 B per K=32 step, SBO = 1 KB per
            // 8 rows; one 128-element MN chunk per CTA, so LBO is never used
            const uint32_t ko = uint32_t(k) * 4096u;
            const uint64_t dp0 = make_sdesc<false>(st + ko, 16384, 1024);
            const uint64_t dp1 = make_sdesc<false>(st + S::kPiece + ko, 16384, 1024);
            const uint64_t dp2 = make_sdesc<false>(st + 2 * S::kPiece + ko, 16384, 1024);
            const uint64_t dx = make_sdesc<false>(st + kOffX + ko, 16384, 1024);
            const uint64_t dx7 = make_sdesc<false>(st + kOffX128 + ko, 16384, 1024);
            const uint32_t acc = (kb > kb0 || k > 0) ? 1u : 0u;
            mma_i8<CG>(tacc_a, dp0, dx7, idesc, acc);
            mma_i8<CG>(tacc_a, dp1, dx, idesc, 1u);
            mma_i8<CG>(tacc_b, dp2, dx, idesc, acc);
          }
          if (CG == 2) mma_commit_pair(bar_empty + 8 * stage);
          else mma_commit(bar_empty + 8 * stage);
          if (++stage == S::kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
        if (CG == 2) mma_commit_pair(bar_tfull);
        else mma_commit(bar_tfull);
      }
    }
  } else if (warp >= 2 + kEpiWarps) {
    const int r = threadIdx.x - (2 + kEpiWarps) * 32;  // k row 0..127
    int stage = 0;
    uint32_t phase = 0;
    for (int t = cl_id; t < num_tiles; t += n_cl) {
      int mt, nt, sp;
      decode(t, mt, nt, sp);
      const int kb0 = sp * p.kb_per_split, kb1 = min(kb_total, kb0 + p.kb_per_split);
      for (int kb = kb0; kb < kb1; ++kb) {
        mbar_wait(bar_xfull + 8 * stage, phase);
        uint8_t* st = smem + stage * S::kStage;
        expand_bit_row(st + kOffBits + r * 16, st + kOffX, st + kOffX128, r);
        fence_async_smem();
        __syncwarp();
        if (lane == 0) {
          if (CG == 2) mbar_arrive_cluster(map_rank0(bar_conv + 8 * stage));
          else mbar_arrive(bar_conv + 8 * stage);
        }
        if (++stage == S::kStages) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else {
    const int q = warp & 3;
    const int ew = warp - 2;
    const uint32_t blk = sbase + S::kEpiOff + uint32_t(ew * 4096);
    uint8_t* blk_ptr = smem + S::kEpiOff + ew * 4096;
    int it = 0;
    for (int t = cl_id; t < num_tiles; t += n_cl, ++it) {
      int mt, nt, sp;
      decode(t, mt, nt, sp);
      const int m0 = mt * kBM * CG + int(rank) * kBM, n0 = nt * BN;
      const int rbase = m0 + q * 32;
      const int m = rbase + lane;
      float sc = 0.f;
      if (m < p.M) {
        const float mx = __uint_as_float(p.colmax[long(sp) * p.M + m]);
        sc = mx > 0.f ? mx / 127.f : 1.f;
      }
      const float sa = sc * 0.0078125f, sb = sc * 6.103515625e-05f;
      mbar_wait(bar_tfull, it & 1);
      tc_fence_after();
      const uint32_t ta = tmem_base + (uint32_t(q * 32) << 16);
      const uint32_t tb = ta + uint32_t(BN);
#pragma unroll 1
      for (int c = 0; c < BN; c += 32) {
        uint32_t ra[32], rb[32];
        tmem_ld32(ta + uint32_t(c), ra);
        tmem_ld32(tb + uint32_t(c), rb);
        float o[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) o[j] = fmaf(float(int(ra[j])), sa, float(int(rb[j])) * sb);
        if (lane == 0) bulk_wait_read();
        __syncwarp();
#pragma unroll
        for (int j4 = 0; j4 < 8; ++j4)
          *reinterpret_cast<float4*>(blk_ptr + swz(lane, j4)) =
              make_float4(o[4 * j4], o[4 * j4 + 1], o[4 * j4 + 2], o[4 * j4 + 3]);
        fence_async_smem();
        __syncwarp();
        if (lane == 0) {
          tma_store_3d(&tmWs, n0 + c, rbase, sp, blk);
          bulk_commit();
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if (CG == 2) mbar_arrive_cluster(map_rank0(bar_tempty));
        else mbar_arrive(bar_tempty);
      }
    }
    if (lane == 0) bulk_wait_all();
  }

  tc_fence_before();
  if (CG == 2) cluster_sync_all();
  else __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    if (CG == 2)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                   "n"(S::kTmemCols));
    else
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                   "n"(S::kTmemCols));
  }
}

// ---------------------------------------------------------------------------
// Host side

// W [N][K] (row pitch ldw floats) -> pieces q [3][N][Kp] (int8, zero past K) and per-row
// scales s [N] (see the header comment).  Kp % 16 == 0.
void launch_quantize_rows(const float* W, int N, int K, long ldw, int8_t* q, long Kp, float* s,
                          cudaStream_t stream);

// out = tanh(X . W^T + b) with X binary planes bit-packed LSB first ([M] rows of `rowb`
// bytes, rowb % 16 == 0, bits past K ignored) and W given as launch_quantize_rows pieces.
// Writes the full fp32 plane and the tf32 residual plane (row pitch ldo).
LaunchInfo launch_i8_bits_fwd(const uint8_t* bits, long rowb, const int8_t* q, long Kp,
                              const float* scale, const float* bias, int M, int N, int K,
                              float* out, float* out_lo, int ldo, cudaStream_t stream,
                              int8_t* out_q = nullptr);

// out = tanh(A . W^T + b) with A given as int8 pieces [3][M][K] (scale 1/127, e.g. the
// out_q of launch_i8_bits_fwd) and W as launch_quantize_rows pieces.  Optional fused
// heads (Params::head_* semantics) and residual plane (out_lo may be null).  K % 16 == 0.
// out may be null (out_lo then null too) when out_q or the fused heads carry the result.
LaunchInfo launch_i8x2_fwd(const int8_t* a, const int8_t* q, long Kp, const float* scale,
                           const float* bias, int M, int N, int K, float* out, float* out_lo,
                           int ldo, const float* head_w, const float* head_wv, int head_k,
                           float* head_part, cudaStream_t stream, int8_t* out_q = nullptr);

// dZ [F][M] (row pitch ldz floats) -> pieces P [3][F][M] int8 with one scale per
// (split, column): s = colmax[f / rows_per_split][m] / 127.  M % 4 == 0.
void launch_quantize_cols(const float* Z, long F, int M, long ldz, const unsigned* colmax,
                          long rows_per_split, int8_t* P, cudaStream_t stream);

// ws[split][m][n] = sum over the split's frames of dZ[f][m] X[f][n]  (X bit rows, pitch
// `rowb` bytes; dZ as launch_quantize_cols pieces).  M % 128 == 0, N % 128 == 0 not
// required (TMA clips), rows_per_split = kb_per_split * 128 and <= 131072.
void launch_i8_bits_dw(const int8_t* P, const uint8_t* bits, long rowb, const unsigned* colmax,
                       int M, int N, int K, int kb_per_split, float* ws, cudaStream_t stream);

}  // namespace tlg::gemm
