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
// Persistent CTAs (one per SM), 192 threads, 128 x BN output tiles:
//   warp 0      TMA producer (one elected lane), smem ring of STAGES stages
//   warp 1      TMEM allocator + single-thread tcgen05.mma issuer
//   warps 2..5  epilogue: tcgen05.ld TMEM -> registers -> fused op -> smem transpose ->
//               coalesced 128-B row stores (+ fused per-tile column sums for dZ)
// Pipelines: full[s] (TMA -> MMA, tx-count), empty[s] (tcgen05.commit -> TMA),
// tmem_full[2] / tmem_empty[2] (double-buffered accumulators: the epilogue of tile i
// overlaps the MMAs of tile i+1).
#pragma once

#include <cudaTypedefs.h>

#include "common.cuh"

namespace tlg::gemm {

enum Epi : int {
  kEpiFwdTanh = 0,   // out = tanh(acc + bias[n])          -> out (full) / out_lo planes
  kEpiBwdTanh = 1,   // out = acc * (1 - h[m][n]^2)         -> out (full) / out_lo planes
  kEpiStore = 2,     // ws[split][m][n] = acc               (split-K partials, fp32)
  kEpiFwdLoss = 3,   // last trunk layer + heads + PPO loss: writes dZ_L, not h_L (below)
};

// kEpiFwdLoss: the top trunk layer's forward fused with the policy/value heads, the PPO
// loss (rlmath.cpp:116-185) and dZ_L = (dlogits . W_head) * (1 - h^2), per row of the
// tile (BN = N: the whole row is in TMEM).  Pass 1 over the row's chunks: h = tanh(acc+b)
// and the head dot products; the per-row loss math; pass 2: h again, dZ_L (full + tf32
// residual planes, TMA-stored), and per-CTA partial sums of the head weight gradient
// sum_f d_k h_j, of the top bias gradient sum_f dZ_L and of the head bias gradient and
// loss statistics -- fixed order, one partial row per CTA.  h_L never reaches HBM.
struct LossEpi {
  const int* action;
  const float* blogp;
  const int* valid;
  int T;
  const float* adv;
  const float* target;
  const double* stats;  // StepStatsDev: mean [2], sd [3], inv_n [4]
  float clip_eps, vf_coef, ent_coef;
  long bpi, bv;          // head bias offsets in `params` (-1: none)
  const float* params;
  float* hg_partial;     // [ctas][A1][N]
  float* db_partial;     // [ctas][N]
  double* loss_partial;  // [ctas][5]
  float* bias_partial;   // [ctas][A1]
  int* err;
};

constexpr int kBM = 128;
constexpr int kBK = 32;  // fp32 elements per 128-byte swizzle row
constexpr int kThreads = 192;
constexpr int kThreadsU8 = 320;  // + 4 converter warps for uint8 operands

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
  float* colsum;  // kEpiBwdTanh: optional column sums of the output, one row per CTA:
                  // colsum[cta][n] (N <= kColMax); the caller sums the rows in order
  // kEpiBwdTanh: optional column max |out| per group of colmax_rows rows (rows of a
  // group never straddle a 256-row tile): colmax[m / colmax_rows][n], as float bits
  // (atomicMax on non-negative floats); zeroed by the caller.  Feeds the fixed-point
  // scales of the int8 weight-gradient GEMM (gemm_i8.cuh).
  unsigned* colmax;
  int colmax_rows;
  // kEpiFwdTanh on the last trunk layer: fused policy/value head partial dot products
  //   head_part[n_tile][m][k] = sum_{n in tile} Whead[k][n] * out[m][n], k < head_k
  const float* head_w;   // W_pi [head_k - 1][N] row-major
  const float* head_wv;  // w_v [N]
  int head_k;            // n_actions + 1 (<= 8), 0 = no fused head
  float* head_part;
  // U8 == 1: also write the expanded fp32 A operand (exact) to this [M][K] buffer
  // (tmAct map) from the n_tile == 0 CTAs, so a later GEMM can read it as plain fp32
  float* a_expand;
  // kEpiFwdTanh: also write the tanh outputs as fixed-scale int8 pieces [3][M][N] (scale
  // 1/127) for a following int8 x int8 layer (gemm_i8x2_fwd_kernel); N % 32 == 0
  int8_t* out_q;
  LossEpi loss;  // kEpiFwdLoss only
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

// Instruction descriptor for kind::tf32, fp32 accumulate, M = 128 * CG.
template <int BN, bool A_MN, bool B_MN, int CG = 1>
__device__ __forceinline__ constexpr uint32_t make_idesc() {
  return (1u << 4)                        // D format: f32
         | (2u << 7)                      // A format: tf32
         | (2u << 10)                     // B format: tf32
         | (uint32_t(A_MN) << 15)         // A major (0 = K, 1 = MN)
         | (uint32_t(B_MN) << 16)         // B major
         | (uint32_t(BN >> 3) << 17)      // N >> 3
         | (uint32_t((kBM * CG) >> 4) << 24);  // M >> 4
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

// ---- CTA-pair (cta_group::2) helpers
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
// shared::cluster address of the same smem offset in CTA rank 0 of the pair
__device__ __forceinline__ uint32_t map_rank0(uint32_t addr) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(r) : "r"(addr));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::
                   : "memory");
}
// (default .release.cta semantics, as CUTLASS's ClusterBarrier::arrive: the explicit
// .release.cluster form compiles to MEMBAR.ALL.GPU + ERRBAR, ~1 us per arrive)
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
// TMA into this CTA's smem, completion counted on the pair leader's mbarrier
__device__ __forceinline__ void tma_load_2d_pair(uint32_t dst, const CUtensorMap* map, int x, int y,
                                                 uint32_t leader_bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(leader_bar)
      : "memory");
}
__device__ __forceinline__ void mma_tf32_pair(uint32_t tmem_d, uint64_t a, uint64_t b,
                                              uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(accumulate));
}
// arrive on the barrier at this smem offset in both CTAs of the pair
__device__ __forceinline__ void mma_commit_pair(uint32_t bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], %1;" ::"r"(bar),
      "h"(uint16_t(3))
      : "memory");
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
constexpr int kEpiWarps = 4;
// Epilogue warp groups: the tanh forward on a derived-residual operand (short K: the
// per-element tanh + fused head dot products are the critical path) runs two groups of 4
// epilogue warps (warps 2..5 and 10..13) that take alternate 32-column chunks, so every
// scheduler holds two epilogue warps.  Selected by launch() through lod bit 3 (kLodEg2):
// 128-column tiles, and 256-column tiles of short K loops (a long K loop hides the
// epilogue, and its pipeline would lose a stage to the extra staging); each group's head
// partials cover BN / 2 columns (LaunchInfo::bn).
constexpr int kLodEg2 = 8, kLodEg3 = 16;  // (kLodEg3: three groups, warps 14..17 too)
__host__ __device__ constexpr int epi_groups(int bn, int epi, int u8, int lod) {
  // (the dX epilogue is written for any count; measured no faster with two groups)
  return epi == 0 /* kEpiFwdTanh */ && (lod & (kLodEg2 | kLodEg3)) && (lod & 3) && u8 == 0 &&
                 bn >= 128
             ? ((lod & kLodEg3) ? 3 : 2)
             : 1;
}
constexpr int kColMax = 2048;  // widest N with fused column sums
constexpr int kStageBuf = 32 * 33;  // per-warp 32x32 transpose buffer (+1 pad: no bank conflicts)

// U8: 0 = fp32 operands; 1 = A arrives as uint8 planes (K-major); 2 = B arrives as uint8
// planes (MN-major).  A uint8 operand is TMA-loaded into a byte staging tile and expanded
// to fp32 in the MMA's swizzled layout by 4 converter warps (exact: 0..255).
// Shared-memory plan of one instantiation, constexpr so the host launcher picks tiles
// with exactly the arithmetic the kernel is compiled with.
struct SmemPlan {
  int stage, tma_bytes, u8_slot, u8_ring, epi_blocks, warp_epi, extra, stages;
  bool share_lo;
  int ring_off, bar_off, num_bars, epi_off, bytes;
};
constexpr int plan_stages(int stage, int epi_bytes, int ring_bytes) {
  const int b = (225 * 1024 - epi_bytes - ring_bytes - 1024 - 256) / stage;
  return b < 2 ? 2 : b > 8 ? 8 : b;
}
// lod: bit 0 / bit 1 = the lo plane of A / B is derived in shared memory from the hi tile
// (lo = x - trunc_tf32(x), elementwise, so any swizzled layout) by the converter warps
// instead of being TMA-loaded from a residual plane in HBM.
constexpr SmemPlan smem_plan(int BN, bool a_lo, bool b_lo, int epi, int u8, int cg, int lod = 0) {
  SmemPlan q{};
  const int kA = kBM * kBK * 4;          // 16 KB
  const int kB = (BN / cg) * kBK * 4;    // B rows held by this CTA (a pair splits N)
  q.stage = kA * (a_lo ? 2 : 1) + kB * (b_lo ? 2 : 1);
  q.tma_bytes = q.stage - (u8 == 1 ? kA : u8 == 2 ? kB : 0) - ((lod & 1) ? kA : 0) -
                ((lod & 2) ? kB : 0);
  // a uint8 operand's byte tiles stream through their own ring (u8_ring slots), filled
  // by the producer up to u8_ring k-blocks ahead of the fp32 stages, so only the
  // conversion itself sits on the MMA's critical path.
  q.u8_slot = u8 == 1 ? kBM * kBK : u8 == 2 ? (BN / cg) * kBK : 0;
  q.u8_ring = u8 == 0 ? 0 : (16384 / q.u8_slot) < 2 ? 2 : (16384 / q.u8_slot) > 8 ? 8
                                                                                 : (16384 / q.u8_slot);
  // per epilogue warp: 4 KB TMA-store staging for out, another for out_lo, + a 4 KB
  // TMA-prefetched activation block (bwd), + 1 KB of head weights (fwd).  out and out_lo
  // share one block (stores serialised) when that buys the pipeline a third stage: the
  // uint8-input forward and the wide 3-pass tiles, whose long K loops hide it.
  q.extra = epi == kEpiBwdTanh   ? kEpiWarps * BN * 4 + kColMax * 4
            : epi == kEpiFwdLoss ? kEpiWarps * (8 * BN + BN) * 4  // per-warp hg [8][BN], db [BN]
                                 : 0;
  const int head = epi == kEpiFwdTanh ? 1024 : epi == kEpiFwdLoss ? 2048 : 0;
  const int ring = q.u8_ring * q.u8_slot;
  const int ew = kEpiWarps * epi_groups(BN, epi, u8, lod);
  auto epi_bytes = [&](int blocks) { return ew * (blocks * 4096 + head) + q.extra; };
  // blocks: out (+ out_lo) (+ act for bwd, + h staging for the fused loss)
  const int sep_blocks = epi == kEpiStore ? 1 : 2 + (epi == kEpiBwdTanh || epi == kEpiFwdLoss ? 1 : 0);
  const int sep = plan_stages(q.stage, epi_bytes(sep_blocks), ring);
  const int shr = plan_stages(q.stage, epi_bytes(sep_blocks - 1), ring);
  // The tanh forward shares whenever that buys a stage: its consumers derive the tf32
  // residual in their own shared memory, so out_lo is normally null (TLG_LO_HBM only).
  q.share_lo = epi != kEpiStore && epi != kEpiFwdLoss &&
               (u8 == 1 || (sep < 3 && shr > sep) || (epi == kEpiFwdTanh && shr > sep) ||
                (lod & kLodEg3));  // (three groups fit only with one block per warp)
  q.epi_blocks = q.share_lo ? sep_blocks - 1 : sep_blocks;
  q.warp_epi = q.epi_blocks * 4096 + head;
  q.stages = q.share_lo ? shr : sep;
  q.ring_off = q.stages * q.stage;
  q.bar_off = q.ring_off + ring;
  // full/empty per stage, tmem full/empty x2, act-block full x4, converted per stage,
  // u8 ring full/empty per slot
  q.num_bars = 2 * q.stages + 4 + ew + (u8 ? q.stages + 2 * q.u8_ring : 0) +
               (lod ? 2 * q.stages : 0);  // lod: converted + local hi-landed per stage
  q.epi_off = (q.bar_off + q.num_bars * 8 + 16 + 1023) / 1024 * 1024;
  q.bytes = q.epi_off + ew * q.warp_epi + q.extra + 1024;  // + 1 KB alignment slack
  return q;
}

// U8: 0 = fp32 operands; 1 = A arrives as uint8 planes (K-major); 2 = B arrives as uint8
// planes (MN-major).  A uint8 operand is TMA-loaded into a byte staging tile and expanded
// to fp32 in the MMA's swizzled layout by 4 converter warps (exact: 0..255).
template <int BN, bool A_LO, bool B_LO, int EPI, int U8 = 0, int CG = 1, int LOD = 0>
struct Smem {
  static constexpr SmemPlan P = smem_plan(BN, A_LO, B_LO, EPI, U8, CG, LOD);
  static constexpr int kA = kBM * kBK * 4;
  static constexpr int kBN = BN / CG;
  static constexpr int kB = kBN * kBK * 4;
  static constexpr int kU8 = P.u8_slot;
  static constexpr int kU8Ring = P.u8_ring;
  static constexpr int kStage = P.stage;
  static constexpr int kTmaBytes = P.tma_bytes;
  static constexpr bool kShareLo = P.share_lo;
  static constexpr int kExtra = P.extra;
  static constexpr int kEpiBlocks = P.epi_blocks;
  static constexpr int kWarpEpi = P.warp_epi;
  static constexpr int kStages = P.stages;
  static constexpr int kRingOff = P.ring_off;
  static constexpr int kBarOff = P.bar_off;
  static constexpr int kNumBars = P.num_bars;
  static constexpr int kEpiOff = P.epi_off;
  static constexpr int kBytes = P.bytes;
  static constexpr bool kFits = kBytes <= 227 * 1024;
  static constexpr int kAccCols = BN <= 32 ? 32 : BN <= 64 ? 64 : BN <= 128 ? 128 : 256;
  static constexpr int kTmemCols = 2 * kAccCols;  // double-buffered accumulators
};

struct TileMap {
  int m_tiles, n_tiles, splits;
  __device__ __forceinline__ void decode(int t, int& m, int& n, int& s) const {
    n = t % n_tiles;  // n fastest: the N-tiles of one M row run together (A re-read hits L2)
    const int r = t / n_tiles;
    m = r % m_tiles;
    s = r / m_tiles;
  }
};

// (tile, k-block) walk of one CTA (or CTA pair) through its persistent work list.
struct KCursor {
  int t, kb, kb1, mt, nt, sp;
  __device__ __forceinline__ void load(const TileMap& tm, int kb_per_split, int kb_total) {
    tm.decode(t, mt, nt, sp);
    kb = sp * kb_per_split;
    kb1 = min(kb_total, kb + kb_per_split);
  }
  __device__ __forceinline__ void init(int t0, int, int num_tiles, const TileMap& tm,
                                       int kb_per_split, int kb_total) {
    t = t0;
    if (t < num_tiles) load(tm, kb_per_split, kb_total);
  }
  __device__ __forceinline__ bool valid(int num_tiles) const { return t < num_tiles; }
  __device__ __forceinline__ void next(int n_cl, int num_tiles, const TileMap& tm,
                                       int kb_per_split, int kb_total) {
    if (++kb >= kb1) {
      t += n_cl;
      if (t < num_tiles) load(tm, kb_per_split, kb_total);
    }
  }
};

__device__ __forceinline__ void named_bar(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}

// Persistent, warp-specialised: CTA b processes tiles b, b + grid, ...  The MMA warp
// accumulates tile i into TMEM buffer (i & 1) while the epilogue drains tile i-1.
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, int x, int y, uint32_t src) {
  asm volatile(
      "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
          reinterpret_cast<uint64_t>(map)),
      "r"(x), "r"(y), "r"(src)
      : "memory");
}
__device__ __forceinline__ void tma_store_3d(const CUtensorMap* map, int x, int y, int z,
                                             uint32_t src) {
  asm volatile(
      "cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];" ::"l"(
          reinterpret_cast<uint64_t>(map)),
      "r"(x), "r"(y), "r"(z), "r"(src)
      : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
template <int N>
__device__ __forceinline__ void bulk_wait_read_n() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
// Four uint8 -> four exact fp32 without I2F: byte b placed in the mantissa of 2^23 gives
// 2^23 + b; subtracting 2^23 is exact (PRMT + FADD at full ALU rate).
__device__ __forceinline__ float4 u8x4_to_f32(uint32_t v) {
  const float k = 8388608.f;
  return make_float4(__uint_as_float(__byte_perm(v, 0x4B000000u, 0x7440)) - k,
                     __uint_as_float(__byte_perm(v, 0x4B000000u, 0x7441)) - k,
                     __uint_as_float(__byte_perm(v, 0x4B000000u, 0x7442)) - k,
                     __uint_as_float(__byte_perm(v, 0x4B000000u, 0x7443)) - k);
}

// byte offset of element (row r, col c) in a 32x32 fp32 block with the 128-B TMA swizzle
__device__ __forceinline__ uint32_t swz(int r, int c4) { return uint32_t(r * 128 + ((c4 ^ (r & 7)) << 4)); }

// tanh output o in (-1, 1) -> three int8 pieces of o * 127 (fixed scale 1/127), packed
// four columns per word; magic-constant rounding (exact residual steps)
__device__ __forceinline__ void act_pieces4(const float* o, uint32_t& w0, uint32_t& w1,
                                            uint32_t& w2) {
  constexpr float kMagic = 12582912.f;
  w0 = w1 = w2 = 0u;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const float x = o[j] * 127.f;
    const float m0 = x + kMagic;
    const float x1 = (x - (m0 - kMagic)) * 128.f;
    const float m1 = x1 + kMagic;
    const float m2 = (x1 - (m1 - kMagic)) * 128.f + kMagic;
    w0 |= (__float_as_uint(m0) & 0xFFu) << (8 * j);
    w1 |= (__float_as_uint(m1) & 0xFFu) << (8 * j);
    w2 |= (__float_as_uint(m2) & 0xFFu) << (8 * j);
  }
}

// One thread's 32 consecutive columns of one row (starting at element `at` of a [M][N]
// plane, 16-B aligned) -> the three piece planes (plane stride `plane`).
__device__ __forceinline__ void write_act_pieces(const float* o, int8_t* q, long plane, long at) {
  q += at;
#pragma unroll
  for (int j16 = 0; j16 < 2; ++j16) {
    uint32_t a[4], b[4], c4[4];
#pragma unroll
    for (int w = 0; w < 4; ++w) act_pieces4(o + 16 * j16 + 4 * w, a[w], b[w], c4[w]);
    *reinterpret_cast<uint4*>(q + 16 * j16) = make_uint4(a[0], a[1], a[2], a[3]);
    *reinterpret_cast<uint4*>(q + plane + 16 * j16) = make_uint4(b[0], b[1], b[2], b[3]);
    *reinterpret_cast<uint4*>(q + 2 * plane + 16 * j16) = make_uint4(c4[0], c4[1], c4[2], c4[3]);
  }
}

__host__ __device__ constexpr int kernel_threads(int bn, int epi, int u8, int lod) {
  return ((u8 || lod) ? kThreadsU8 : kThreads) + 32 * kEpiWarps * (epi_groups(bn, epi, u8, lod) - 1);
}

template <int BN, bool A_MN, bool B_MN, bool A_LO, bool B_LO, int EPI, int U8, int CG, int LOD>
__global__ void __launch_bounds__(kernel_threads(BN, EPI, U8, LOD), 1)
    gemm_tf32x3_kernel(const __grid_constant__ CUtensorMap tmA_hi,
                       const __grid_constant__ CUtensorMap tmA_lo,
                       const __grid_constant__ CUtensorMap tmB_hi,
                       const __grid_constant__ CUtensorMap tmB_lo,
                       const __grid_constant__ CUtensorMap tmOut,
                       const __grid_constant__ CUtensorMap tmOutLo,
                       const __grid_constant__ CUtensorMap tmAct, const Params p,
                       const TileMap tm) {
  using S = Smem<BN, A_LO, B_LO, EPI, U8, CG, LOD>;
  static_assert(!(U8 && LOD), "derived lo planes and uint8 operands do not mix");
  static_assert(!(LOD & 1) || A_LO, "A lo derived needs the A lo slot");
  static_assert(!(LOD & 2) || B_LO, "B lo derived needs the B lo slot");
  constexpr int kEG = epi_groups(BN, EPI, U8, LOD);
  // CG == 2: a cluster of two CTAs shares each (256 x BN) tile; rank r owns rows
  // [128 r, 128 r + 128) of A / D and B rows [r BN/2, (r+1) BN/2).  Only rank 0 issues
  // the MMAs (cta_group::2), reading both CTAs' smem and writing both CTAs' TMEM.
  const uint32_t rank = CG == 2 ? cluster_rank() : 0u;
  const int cl_id = CG == 2 ? int(blockIdx.x >> 1) : int(blockIdx.x);
  const int n_cl = CG == 2 ? int(gridDim.x >> 1) : int(gridDim.x);
  extern __shared__ uint8_t smem_raw[];
  // 1 KB-aligned base by pointer arithmetic on the __shared__ array (an integer round
  // trip would turn every staging access into a generic LD/ST)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const uint32_t sbase = smem_u32(smem);
  const uint32_t bar_full = sbase + S::kBarOff;
  const uint32_t bar_empty = bar_full + S::kStages * 8;
  const uint32_t bar_tfull = bar_empty + S::kStages * 8;  // [2]
  const uint32_t bar_tempty = bar_tfull + 16;               // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + S::kBarOff + S::kNumBars * 8);
  const uint32_t bar_act = bar_tempty + 16;                 // [epilogue warps]
  const uint32_t bar_conv = bar_act + 8 * kEpiWarps * kEG;  // [stages] (U8)
  const uint32_t bar_ufull = bar_conv + 8 * S::kStages;     // [ring] (U8)
  const uint32_t bar_uempty = bar_ufull + 8 * S::kU8Ring;   // [ring] (U8)
  const uint32_t bar_hfull = bar_uempty + 8 * S::kU8Ring;   // [stages] (LOD): local tiles landed
  float* colpart = reinterpret_cast<float*>(smem + S::kEpiOff + kEpiWarps * kEG * S::kWarpEpi);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int num_tiles = tm.m_tiles * tm.n_tiles * tm.splits;
  const int kb_total = (p.K + kBK - 1) / kBK;

  if (warp == 0 && lane == 0) {
    prefetch_tmap(&tmA_hi);
    prefetch_tmap(&tmB_hi);
    if (A_LO && !(LOD & 1)) prefetch_tmap(&tmA_lo);
    if (B_LO && !(LOD & 2)) prefetch_tmap(&tmB_lo);
    for (int s = 0; s < S::kStages; ++s) {
      mbar_init(bar_full + 8 * s, 1);
      mbar_init(bar_empty + 8 * s, 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(bar_tfull + 8 * a, 1);
      mbar_init(bar_tempty + 8 * a, kEpiWarps * kEG * CG);  // both CTAs' epilogues drain
    }
    for (int w = 0; w < kEpiWarps * kEG; ++w) mbar_init(bar_act + 8 * w, 1);
    if (LOD) {
      for (int st = 0; st < S::kStages; ++st) {
        mbar_init(bar_conv + 8 * st, 4 * CG);  // one arrive per converter warp (x CTAs)
        mbar_init(bar_hfull + 8 * st, 1);      // this CTA's tiles (local tx count)
      }
    }
    if (U8) {
      for (int st = 0; st < S::kStages; ++st)
        mbar_init(bar_conv + 8 * st, 4 * CG);  // one arrive per converter warp (x CTAs)
      for (int u = 0; u < S::kU8Ring; ++u) {
        mbar_init(bar_ufull + 8 * u, 1);
        mbar_init(bar_uempty + 8 * u, 4);  // the 4 local converter warps
      }
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
  if (CG == 2) cluster_sync_all();  // the peer's barriers exist before any remote arrive
  else __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  // prologue done (barriers, TMEM, tensor maps): wait for the predecessor's writes
  pdl_wait();
  pdl_trigger();

  if (warp == 0) {
    if (lane == 0) {
      // ===== TMA producer =====
#define TMA_FP32(dst, map, x, y, bar)                                   \
  do {                                                                 \
    if (CG == 2 && !LOD) tma_load_2d_pair(dst, map, x, y, bar);        \
    else tma_load_2d(dst, map, x, y, bar);                             \
  } while (0)
      int stage = 0;
      uint32_t phase = 0;
      // u8 ring cursor, running up to kU8Ring k-blocks ahead of the fp32 stages
      KCursor cu;
      cu.init(cl_id, n_cl, num_tiles, tm, p.kb_per_split, kb_total);
      int ui = 0;
      uint32_t uph = 0;
      long issued_u8 = 0, done_fp32 = 0;
      KCursor cf;
      cf.init(cl_id, n_cl, num_tiles, tm, p.kb_per_split, kb_total);
      for (; cf.valid(num_tiles); cf.next(n_cl, num_tiles, tm, p.kb_per_split, kb_total), ++done_fp32) {
        if (U8) {
          while (cu.valid(num_tiles) && issued_u8 < done_fp32 + S::kU8Ring) {
            mbar_wait(bar_uempty + 8 * ui, uph ^ 1);
            mbar_expect_tx(bar_ufull + 8 * ui, S::kU8);
            const uint32_t dst = sbase + S::kRingOff + ui * S::kU8;
            if (U8 == 1)  // u8 box {32 k, 128 m}
              tma_load_2d(dst, &tmA_hi, cu.kb * kBK, cu.mt * kBM * CG + int(rank) * kBM,
                          bar_ufull + 8 * ui);
            else          // u8 box {BN/CG n, 32 k}
              tma_load_2d(dst, &tmB_hi, cu.nt * BN + int(rank) * S::kBN, cu.kb * kBK,
                          bar_ufull + 8 * ui);
            cu.next(n_cl, num_tiles, tm, p.kb_per_split, kb_total);
            ++issued_u8;
            if (++ui == S::kU8Ring) {
              ui = 0;
              uph ^= 1;
            }
          }
        }
        const int m0 = cf.mt * kBM * CG + int(rank) * kBM;
        const int n0 = cf.nt * BN + int(rank) * S::kBN;
        const int kb = cf.kb;
        {
          mbar_wait(bar_empty + 8 * stage, phase ^ 1);
          const uint32_t st = sbase + stage * S::kStage;
          // CG == 2: both CTAs' fp32 tiles complete on the leader's full barrier; with
          // derived lo planes each CTA's tiles complete locally (its converters go next)
          const uint32_t full = LOD        ? bar_hfull + 8 * stage
                                : CG == 2 ? map_rank0(bar_full + 8 * stage)
                                          : bar_full + 8 * stage;
          if (LOD) mbar_expect_tx(bar_hfull + 8 * stage, S::kTmaBytes);
          else if (rank == 0) mbar_expect_tx(bar_full + 8 * stage, S::kTmaBytes * CG);
          const int k0 = kb * kBK;
          uint32_t off = st;
          if (U8 == 1) {
            // converted by the converter warps
          } else if (!A_MN) {
            TMA_FP32(off, &tmA_hi, k0, m0, full);
            if (A_LO && !(LOD & 1)) TMA_FP32(off + S::kA, &tmA_lo, k0, m0, full);
          } else {
#pragma unroll
            for (int j = 0; j < kBM / 32; ++j) {
              TMA_FP32(off + j * 4096, &tmA_hi, m0 + 32 * j, k0, full);
              if (A_LO && !(LOD & 1))
                TMA_FP32(off + S::kA + j * 4096, &tmA_lo, m0 + 32 * j, k0, full);
            }
          }
          off += S::kA * (A_LO ? 2 : 1);
          if (U8 == 2) {
            // converted by the converter warps
          } else if (!B_MN) {
            TMA_FP32(off, &tmB_hi, k0, n0, full);
            if (B_LO && !(LOD & 2)) TMA_FP32(off + S::kB, &tmB_lo, k0, n0, full);
          } else {
#pragma unroll
            for (int j = 0; j < S::kBN / 32; ++j) {
              TMA_FP32(off + j * 4096, &tmB_hi, n0 + 32 * j, k0, full);
              if (B_LO && !(LOD & 2))
                TMA_FP32(off + S::kB + j * 4096, &tmB_lo, n0 + 32 * j, k0, full);
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
#undef TMA_FP32
    if (lane == 0 && rank == 0) {
      // ===== MMA issuer (pair leader) =====
      constexpr uint32_t idesc = make_idesc<BN, A_MN, B_MN, CG>();
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (int t = cl_id; t < num_tiles; t += n_cl, ++it) {
        int mt, nt, sp;
        tm.decode(t, mt, nt, sp);
        const int kb0 = sp * p.kb_per_split, kb1 = min(kb_total, kb0 + p.kb_per_split);
        const int acc_buf = it & 1;
        const uint32_t acc_phase = (it >> 1) & 1;
        mbar_wait(bar_tempty + 8 * acc_buf, acc_phase ^ 1);  // epilogue drained this buffer
        tc_fence_after();
        const uint32_t tmem_d = tmem_base + uint32_t(acc_buf * S::kAccCols);
        for (int kb = kb0; kb < kb1; ++kb) {
          if (!LOD) mbar_wait(bar_full + 8 * stage, phase);
          if (U8 || LOD) mbar_wait(bar_conv + 8 * stage, phase);
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
            const uint32_t acc = (kb > kb0 || k > 0) ? 1u : 0u;
            auto mma = [&](uint64_t da, uint64_t db, uint32_t ac) {
              if (CG == 2) mma_tf32_pair(tmem_d, da, db, idesc, ac);
              else mma_tf32(tmem_d, da, db, idesc, ac);
            };
            if (B_LO) mma(dah, make_sdesc<B_MN>(b_lo + bo, blbo, bsbo), acc);
            if (A_LO) mma(make_sdesc<A_MN>(a_lo + ao, albo, asbo), dbh, (B_LO || acc) ? 1u : 0u);
            mma(dah, dbh, (A_LO || B_LO || acc) ? 1u : 0u);
          }
          if (CG == 2) mma_commit_pair(bar_empty + 8 * stage);
          else mma_commit(bar_empty + 8 * stage);
          if (++stage == S::kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
        if (CG == 2) mma_commit_pair(bar_tfull + 8 * acc_buf);
        else mma_commit(bar_tfull + 8 * acc_buf);
      }
    }
  } else if (LOD && warp >= 2 + kEpiWarps && warp < 2 + 2 * kEpiWarps) {
    // ===== Converter warps 6..9: lo = x - trunc_tf32(x) of the landed hi tiles =====
    // Elementwise over the tile bytes, so the swizzled K- or MN-major layout is kept.
    const int ct = threadIdx.x - (2 + kEpiWarps) * 32;  // 0..127
    int stage = 0;
    uint32_t phase = 0;
    KCursor cc;
    cc.init(cl_id, n_cl, num_tiles, tm, p.kb_per_split, kb_total);
    auto derive = [&](uint8_t* hi, int bytes) {
      for (int o = ct * 16; o < bytes; o += 128 * 16) {
        const float4 x = *reinterpret_cast<const float4*>(hi + o);
        *reinterpret_cast<float4*>(hi + bytes + o) =
            make_float4(x.x - tf32_hi(x.x), x.y - tf32_hi(x.y), x.z - tf32_hi(x.z),
                        x.w - tf32_hi(x.w));
      }
    };
    for (; cc.valid(num_tiles); cc.next(n_cl, num_tiles, tm, p.kb_per_split, kb_total)) {
      mbar_wait(bar_hfull + 8 * stage, phase);  // this CTA's tiles landed
      uint8_t* st = smem + stage * S::kStage;
      if (LOD & 1) derive(st, S::kA);
      if (LOD & 2) derive(st + S::kA * (A_LO ? 2 : 1), S::kB);
      fence_async_smem();  // generic-proxy writes -> visible to the tensor core
      __syncwarp();
      if ((threadIdx.x & 31) == 0) {
        if (CG == 2) mbar_arrive_cluster(map_rank0(bar_conv + 8 * stage));
        else mbar_arrive(bar_conv + 8 * stage);
      }
      if (++stage == S::kStages) {
        stage = 0;
        phase ^= 1;
      }
    }
  } else if (U8 && warp >= 2 + kEpiWarps) {
    // ===== Converter warps 6..9: uint8 staging -> fp32 operand tile (MMA layout) =====
    const int ct = threadIdx.x - (2 + kEpiWarps) * 32;  // 0..127
    const bool expand = U8 == 1 && p.a_expand != nullptr;
    int stage = 0;
    uint32_t phase = 0;
    int ui = 0;
    uint32_t uph = 0;
    KCursor cc;
    cc.init(cl_id, n_cl, num_tiles, tm, p.kb_per_split, kb_total);
    for (; cc.valid(num_tiles); cc.next(n_cl, num_tiles, tm, p.kb_per_split, kb_total)) {
      const int mt = cc.mt, nt = cc.nt, kb = cc.kb;
      {
        if (expand) {  // the bulk store issued from this stage's tile last round must be done
          // (a tile that issues no stores must not rely on the count: wait for all)
          if (ct == 0) {
            if (nt == 0) bulk_wait_read_n<S::kStages - 1>();
            else bulk_wait_read();
          }
          named_bar(2, 128);
        }
        mbar_wait(bar_ufull + 8 * ui, uph);
        mbar_wait(bar_empty + 8 * stage, phase ^ 1);  // the MMA released this stage's tile
        uint8_t* st = smem + stage * S::kStage;
        const uint8_t* us = smem + S::kRingOff + ui * S::kU8;
        if (U8 == 1) {
          // K-major SW128: row r (128 B) holds k = 0..31; 16-B chunk c stored at c ^ (r & 7)
          const int r = ct;
          const uint4 u0 = *reinterpret_cast<const uint4*>(us + r * 32);
          const uint4 u1 = *reinterpret_cast<const uint4*>(us + r * 32 + 16);
          const uint32_t w[8] = {u0.x, u0.y, u0.z, u0.w, u1.x, u1.y, u1.z, u1.w};
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            const uint32_t v = w[c];
            *reinterpret_cast<float4*>(st + r * 128 + ((c ^ (r & 7)) << 4)) = u8x4_to_f32(v);
          }
        } else {
          // MN-major SW128_BASE32B: 32-element n chunk j at j*4 KB, k row at k*128 B,
          // 32-B atom a = (n & 31) >> 3 stored at a ^ (k & 3)
          uint8_t* bt = st + S::kA * (A_LO ? 2 : 1);
          // lane -> (row k within a group of 4, 16-B slot c of the 128-B row): the 8 lanes
          // of a row cover all 8 slots, so each float4 store is one conflict-free wavefront
          // per row.  Warp w converts k rows [8w, 8w + 8).
          const int lane = threadIdx.x & 31, w = ct >> 5;
          const int c = lane & 7;
          const int a = c >> 1;  // 32-B atom of n_local = 4c
#pragma unroll
          for (int kk = 0; kk < 2; ++kk) {
            const int k = 8 * w + 4 * kk + (lane >> 3);
            const uint32_t row_off = uint32_t(k * 128 + ((a ^ (k & 3)) << 5) + (c & 1) * 16);
#pragma unroll
            for (int j = 0; j < S::kBN / 32; ++j) {
              const uint32_t v = *reinterpret_cast<const uint32_t*>(us + k * S::kBN + j * 32 + c * 4);
              *reinterpret_cast<float4*>(bt + j * 4096 + row_off) = u8x4_to_f32(v);
            }
          }
        }
        fence_async_smem();  // generic-proxy writes -> visible to the tensor core
        __syncwarp();
        if ((threadIdx.x & 31) == 0) {
          if (CG == 2) mbar_arrive_cluster(map_rank0(bar_conv + 8 * stage));
          else mbar_arrive(bar_conv + 8 * stage);
        }
        if (expand && nt == 0) {
          named_bar(2, 128);
          if (ct == 0) {
            tma_store_2d(&tmAct, kb * kBK, mt * kBM * CG + int(rank) * kBM, sbase + stage * S::kStage);
            bulk_commit();
          }
        }
        if ((threadIdx.x & 31) == 0) mbar_arrive(bar_uempty + 8 * ui);  // byte slot consumed
        if (++ui == S::kU8Ring) {
          ui = 0;
          uph ^= 1;
        }
        if (++stage == S::kStages) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
    if (expand && ct == 0) bulk_wait_all();
  } else if (EPI == kEpiFwdLoss) {
    // ===== fused forward + heads + PPO loss + dZ_L epilogue (see LossEpi) =====
    const int q = warp & 3;
    const int ew = warp - 2;
    const uint32_t blk = sbase + S::kEpiOff + uint32_t(ew * S::kWarpEpi);
    uint8_t* bp = smem + S::kEpiOff + ew * S::kWarpEpi;  // [out][lo][h][wsm 1K][dsm 1K]
    float* wsm = reinterpret_cast<float*>(bp + 3 * 4096);         // head weights [8][32]
    float* dsm = reinterpret_cast<float*>(bp + 3 * 4096 + 1024);  // d [32 rows][8]
    float* hgw = reinterpret_cast<float*>(smem + S::kEpiOff + kEpiWarps * S::kWarpEpi) +
                 long(ew) * 9 * BN;  // this warp's head-grad [8][BN] then db [BN]
    float* dbw = hgw + 8 * BN;
    const LossEpi& L = p.loss;
    const int A1 = p.head_k, A = A1 - 1;
    for (int i = lane; i < 9 * BN; i += 32) hgw[i] = 0.f;
    const double mean = L.stats[2], sd = L.stats[3];
    const float inv_n = float(L.stats[4]);
    double sl[5] = {0, 0, 0, 0, 0};  // loss, ratio, entropy, value loss, clipped (this warp)
    float sb[8];                      // head bias gradient partials (this warp, lane 0)
#pragma unroll
    for (int k = 0; k < 8; ++k) sb[k] = 0.f;
    auto load_w = [&](int nb) {       // head weights of one 32-column chunk -> wsm
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        float wk = 0.f;
        if (k < A1 && nb + lane < p.N) {
          const float* wrow = k < A ? p.head_w + long(k) * p.N : p.head_wv;
          wk = __ldg(wrow + nb + lane);
        }
        wsm[k * 32 + lane] = wk;
      }
      __syncwarp();
    };
    int it = 0;
    for (int t = cl_id; t < num_tiles; t += n_cl, ++it) {
      int mt, nt, sp;
      tm.decode(t, mt, nt, sp);
      const int m0 = mt * kBM * CG + int(rank) * kBM;
      const int rbase = m0 + q * 32;
      const long f = rbase + lane;  // this thread's frame (row)
      const int acc_buf = it & 1;
      mbar_wait(bar_tfull + 8 * acc_buf, (it >> 1) & 1);
      tc_fence_after();
      const uint32_t tbase = tmem_base + uint32_t(acc_buf * S::kAccCols) + (uint32_t(q * 32) << 16);
      // ---- pass 1: h and the head dot products
      float z[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) z[k] = 0.f;
#pragma unroll 1
      for (int c = 0; c < BN; c += 32) {
        uint32_t r[32];
        tmem_ld32(tbase + uint32_t(c), r);
        const float bl = (c + lane < p.N) ? __ldg(p.bias + c + lane) : 0.f;
        float h[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) h[j] = tanh_fast(__uint_as_float(r[j]) + __shfl_sync(0xffffffffu, bl, j));
        load_w(c);
#pragma unroll
        for (int j4 = 0; j4 < 8; ++j4) {
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            if (k < A1) {
              const float4 w4 = *reinterpret_cast<const float4*>(wsm + k * 32 + 4 * j4);
              z[k] = fmaf(w4.x, h[4 * j4], z[k]);
              z[k] = fmaf(w4.y, h[4 * j4 + 1], z[k]);
              z[k] = fmaf(w4.z, h[4 * j4 + 2], z[k]);
              z[k] = fmaf(w4.w, h[4 * j4 + 3], z[k]);
            }
          }
        }
        __syncwarp();
      }
      // ---- the per-row PPO loss (rlmath.cpp:129-182), as loss_math_kernel
      float d[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) d[k] = 0.f;
      bool valid = false;
      if (f < p.M) {
        const int sg = int(f / L.T), tt = int(f % L.T);
        valid = tt < L.valid[sg];
      }
      if (valid) {
#pragma unroll
        for (int k = 0; k < 8; ++k)
          if (k < A1) {
            const long boff = k < A ? (L.bpi >= 0 ? L.bpi + k : -1) : L.bv;
            if (boff >= 0) z[k] += L.params[boff];
          }
        float mx = -INFINITY;
#pragma unroll
        for (int k = 0; k < 8; ++k)
          if (k < A) mx = fmaxf(mx, z[k]);
        float se = 0.f;
#pragma unroll
        for (int k = 0; k < 8; ++k)
          if (k < A) se += expf(z[k] - mx);
        const float lse = mx + logf(se);
        float pk[8], lpk[8], ent = 0.f;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          lpk[k] = z[k] - lse;
          pk[k] = k < A ? expf(lpk[k]) : 0.f;
          if (k < A && pk[k] > 0.f) ent -= pk[k] * lpk[k];
        }
        const int ar = L.action[f];
        if (ar < 0 || ar >= A) atomicOr(L.err, 2 /* kErrActionRange */);
        const int a = min(max(ar, 0), A - 1);
        float logp = 0.f, V = 0.f;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          if (k == a) logp = lpk[k];
          if (k == A) V = z[k];
        }
        const float verr = V - L.target[f];
        const float ad = float((double(L.adv[f]) - mean) / sd);
        const float ratio = expf(logp - L.blogp[f]);
        const float clipped = fminf(fmaxf(ratio, 1.f - L.clip_eps), 1.f + L.clip_eps);
        const float t1 = ratio * ad, t2 = clipped * ad;
        const float loss_i = -fminf(t1, t2) + L.vf_coef * verr * verr - L.ent_coef * ent;
        const bool surr = t1 <= t2;
#pragma unroll
        for (int k = 0; k < 8; ++k)
          if (k < A) {
            float g = L.ent_coef * pk[k] * ((pk[k] > 0.f ? lpk[k] : 0.f) + ent);
            if (surr) g += -ad * ratio * ((k == a ? 1.f : 0.f) - pk[k]);
            d[k] = g * inv_n;
          }
#pragma unroll
        for (int k = 0; k < 8; ++k)
          if (k == A) d[k] = 2.f * L.vf_coef * verr * inv_n;
        sl[0] += loss_i;
        sl[1] += ratio;
        sl[2] += ent;
        sl[3] += double(verr) * double(verr);
        if (t2 < t1) sl[4] += 1.0;
      }
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        dsm[lane * 8 + k] = d[k];
        const float t = warp_sum(d[k]);
        if (lane == 0) sb[k] += t;
      }
      __syncwarp();
      // ---- pass 2: dZ_L and the gradient partials
#pragma unroll 1
      for (int c = 0; c < BN; c += 32) {
        const int nb = c;
        uint32_t r[32];
        tmem_ld32(tbase + uint32_t(c), r);
        const float bl = (c + lane < p.N) ? __ldg(p.bias + c + lane) : 0.f;
        float h[32], o[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) h[j] = tanh_fast(__uint_as_float(r[j]) + __shfl_sync(0xffffffffu, bl, j));
        load_w(c);
#pragma unroll
        for (int j4 = 0; j4 < 8; ++j4) {
          float dh[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            if (k < A1) {
              const float4 w4 = *reinterpret_cast<const float4*>(wsm + k * 32 + 4 * j4);
              dh[0] = fmaf(d[k], w4.x, dh[0]);
              dh[1] = fmaf(d[k], w4.y, dh[1]);
              dh[2] = fmaf(d[k], w4.z, dh[2]);
              dh[3] = fmaf(d[k], w4.w, dh[3]);
            }
          }
#pragma unroll
          for (int e = 0; e < 4; ++e) o[4 * j4 + e] = dh[e] * (1.f - h[4 * j4 + e] * h[4 * j4 + e]);
        }
        // staging: dZ (full, residual) for the TMA store, h for the head-gradient sums
        if (lane == 0) bulk_wait_read();
        __syncwarp();
#pragma unroll
        for (int j4 = 0; j4 < 8; ++j4) {
          *reinterpret_cast<float4*>(bp + swz(lane, j4)) =
              make_float4(o[4 * j4], o[4 * j4 + 1], o[4 * j4 + 2], o[4 * j4 + 3]);
          if (p.out_lo != nullptr)
            *reinterpret_cast<float4*>(bp + 4096 + swz(lane, j4)) = make_float4(
                o[4 * j4] - tf32_hi(o[4 * j4]), o[4 * j4 + 1] - tf32_hi(o[4 * j4 + 1]),
                o[4 * j4 + 2] - tf32_hi(o[4 * j4 + 2]), o[4 * j4 + 3] - tf32_hi(o[4 * j4 + 3]));
          *reinterpret_cast<float4*>(bp + 8192 + swz(lane, j4)) =
              make_float4(h[4 * j4], h[4 * j4 + 1], h[4 * j4 + 2], h[4 * j4 + 3]);
        }
        fence_async_smem();
        __syncwarp();
        if (lane == 0) {
          tma_store_2d(&tmOut, nb, rbase, blk);
          if (p.out_lo != nullptr) tma_store_2d(&tmOutLo, nb, rbase, blk + 4096);
          bulk_commit();
        }
        // lane = column j: sum over this warp's 32 rows (rows past M carry d = 0, and
        // their dZ is 0 since d = 0)
        float hgs[8], dbs = 0.f;
#pragma unroll
        for (int k = 0; k < 8; ++k) hgs[k] = 0.f;
#pragma unroll 4
        for (int rr = 0; rr < 32; ++rr) {
          const float hv = *reinterpret_cast<const float*>(bp + 8192 + swz(rr, lane >> 2) + (lane & 3) * 4);
          const float ov = *reinterpret_cast<const float*>(bp + swz(rr, lane >> 2) + (lane & 3) * 4);
          dbs += ov;
#pragma unroll
          for (int k = 0; k < 8; ++k)
            if (k < A1) hgs[k] = fmaf(dsm[rr * 8 + k], hv, hgs[k]);
        }
#pragma unroll
        for (int k = 0; k < 8; ++k)
          if (k < A1) hgw[k * BN + c + lane] += hgs[k];
        dbw[c + lane] += dbs;
        __syncwarp();
      }
      // TMEM buffer drained
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if (CG == 2) mbar_arrive_cluster(map_rank0(bar_tempty + 8 * acc_buf));
        else mbar_arrive(bar_tempty + 8 * acc_buf);
      }
    }
    if (lane == 0) bulk_wait_all();
    // ---- this CTA's partial rows: the 4 warps in order (deterministic)
    double* sld = reinterpret_cast<double*>(wsm);  // 5 doubles + 8 floats per warp
#pragma unroll
    for (int i = 0; i < 5; ++i) {
      const double v = warp_sum(sl[i]);
      if (lane == 0) sld[i] = v;
    }
    if (lane == 0) {
#pragma unroll
      for (int k = 0; k < 8; ++k) wsm[10 + k] = sb[k];
    }
    named_bar(1, kEpiWarps * 32);
    const int tid = threadIdx.x - 64;
    const float* hg0 = reinterpret_cast<float*>(smem + S::kEpiOff + kEpiWarps * S::kWarpEpi);
    for (int i = tid; i < A1 * p.N; i += kEpiWarps * 32) {
      const int k = i / p.N, j = i % p.N;
      float v = 0.f;
      for (int w = 0; w < kEpiWarps; ++w) v += hg0[long(w) * 9 * BN + k * BN + j];
      L.hg_partial[long(blockIdx.x) * A1 * p.N + i] = v;
    }
    for (int j = tid; j < p.N; j += kEpiWarps * 32) {
      float v = 0.f;
      for (int w = 0; w < kEpiWarps; ++w) v += hg0[long(w) * 9 * BN + 8 * BN + j];
      L.db_partial[long(blockIdx.x) * p.N + j] = v;
    }
    if (tid < 5 + A1) {
      auto wbase = [&](int w) {
        return reinterpret_cast<const uint8_t*>(smem + S::kEpiOff + w * S::kWarpEpi + 3 * 4096);
      };
      if (tid < 5) {
        double v = 0.0;
        for (int w = 0; w < kEpiWarps; ++w) v += reinterpret_cast<const double*>(wbase(w))[tid];
        L.loss_partial[long(blockIdx.x) * 5 + tid] = v;
      } else {
        const int k = tid - 5;
        float v = 0.f;
        for (int w = 0; w < kEpiWarps; ++w) v += reinterpret_cast<const float*>(wbase(w))[10 + k];
        L.bias_partial[long(blockIdx.x) * A1 + k] = v;
      }
    }
  } else {
    // ===== Epilogue: warps 2..5 own TMEM lane quadrants (warp % 4) =====
    // Per 32-column chunk each warp handles a 32x32 block: TMEM -> registers (thread =
    // row) -> fused op -> 128-B-swizzled smem staging -> TMA bulk store.  The bwd
    // activation block is TMA-prefetched one chunk ahead into its own swizzled buffer.
    const int q = warp & 3;
    // epilogue group: warps 2..5 -> 0, (converters 6..9), 10..13 -> 1, 14..17 -> 2
    const int grp = warp < 2 + kEpiWarps ? 0 : (warp - 2 - 2 * kEpiWarps) / kEpiWarps + 1;
    const int ew = grp ? warp - 2 - kEpiWarps : warp - 2;
    const uint32_t blk = sbase + S::kEpiOff + uint32_t(ew * S::kWarpEpi);
    const uint32_t st_out = blk, st_lo = S::kShareLo ? blk : blk + 4096;
    const uint32_t st_act = blk + (S::kEpiBlocks - 1) * 4096;
    const int act_off = (S::kEpiBlocks - 1) * 4096;
    uint8_t* blk_ptr = smem + S::kEpiOff + ew * S::kWarpEpi;
    float* wsm = reinterpret_cast<float*>(blk_ptr + S::kEpiBlocks * 4096);  // fwd head W [8][32]
    float* cpart = colpart + q * BN;
    const uint32_t abar = bar_act + 8 * ew;
    uint32_t act_phase = 0;
    // the (tile, chunk) sequence this warp walks, for the act prefetch
    auto act_issue = [&](int t, int c) {
      if (EPI != kEpiBwdTanh || t >= num_tiles) return;
      int mt2, nt2, sp2;
      tm.decode(t, mt2, nt2, sp2);
      if (lane == 0) {
        mbar_expect_tx(abar, 4096);
        tma_load_2d(st_act, &tmAct, nt2 * BN + c, mt2 * kBM * CG + int(rank) * kBM + q * 32, abar);
      }
    };
    act_issue(cl_id, 32 * grp);
    // column partials: slot q (the groups write disjoint chunks of the same slots)
    float* csacc = colpart + kEpiWarps * BN;  // [kColMax] CTA-level column sums
    const int etid = ew * 32 + lane;          // 0 .. 32 * kEpiWarps * kEG - 1
    constexpr int kEpiThreads = 32 * kEpiWarps * kEG;
    if (EPI == kEpiBwdTanh && p.colsum != nullptr) {
      for (int i = etid; i < p.N; i += kEpiThreads) csacc[i] = 0.f;
    }
    constexpr int kHK = 8;  // fused head width limit (n_actions + 1)
    const bool do_head = EPI == kEpiFwdTanh && p.head_k > 0;
    // kEpiFwdTanh with fused heads: the bias and head weights of the next 32-column chunk
    // are loaded one chunk ahead (registers), so their latency overlaps this chunk's math
    float bnext = 0.f, wnext[kHK];
    auto fetch = [&](int t_next, int c_next) {
      if (EPI != kEpiFwdTanh || t_next >= num_tiles) return;
      int mt_, nt_, sp_;
      tm.decode(t_next, mt_, nt_, sp_);
      const int col = nt_ * BN + c_next + lane;
      const bool ok = col < p.N;
      bnext = ok ? __ldg(p.bias + col) : 0.f;
#pragma unroll
      for (int k = 0; k < kHK; ++k) {
        wnext[k] = 0.f;
        if (do_head && k < p.head_k && ok)
          wnext[k] = __ldg((k < p.head_k - 1 ? p.head_w + long(k) * p.N : p.head_wv) + col);
      }
    };
    if (do_head) fetch(cl_id, 32 * grp);
    int it = 0;
    for (int t = cl_id; t < num_tiles; t += n_cl, ++it) {
      int mt, nt, sp;
      tm.decode(t, mt, nt, sp);
      const int m0 = mt * kBM * CG + int(rank) * kBM, n0 = nt * BN;
      const int rbase = m0 + q * 32;  // first row of this warp's 32-row slab
      const int acc_buf = it & 1;
      mbar_wait(bar_tfull + 8 * acc_buf, (it >> 1) & 1);
      tc_fence_after();
      const uint32_t tbase = tmem_base + uint32_t(acc_buf * S::kAccCols) + (uint32_t(q * 32) << 16);
      float zacc[kHK];
#pragma unroll
      for (int k = 0; k < kHK; ++k) zacc[k] = 0.f;
#pragma unroll 1
      for (int c = 32 * grp; c < BN; c += 32 * kEG) {
        const int nb = n0 + c;
        float h[32];
        if (EPI == kEpiBwdTanh) {
          mbar_wait(abar, act_phase);
          act_phase ^= 1;
#pragma unroll
          for (int j4 = 0; j4 < 8; ++j4) {
            const float4 v = *reinterpret_cast<const float4*>(blk_ptr + act_off + swz(lane, j4));
            h[4 * j4] = v.x; h[4 * j4 + 1] = v.y; h[4 * j4 + 2] = v.z; h[4 * j4 + 3] = v.w;
          }
          // the generic-proxy reads of this block are ordered before the TMA (async
          // proxy) refill below: without the proxy fence the refill can overtake loads
          // still in flight (a rare write-after-read race on the act block)
          fence_async_smem();
          __syncwarp();
          if (c + 32 * kEG < BN) act_issue(t, c + 32 * kEG);
          else act_issue(t + n_cl, 32 * grp);
        }
        uint32_t r[32];
        tmem_ld32(tbase + uint32_t(c), r);
        float o[32];
        if (EPI == kEpiFwdTanh) {
          float bl;
          if (do_head) {
            bl = bnext;
            // this chunk's head weights -> smem (read back as broadcast LDS.128 below)
#pragma unroll
            for (int k = 0; k < kHK; ++k) wsm[k * 32 + lane] = wnext[k];
            if (c + 32 * kEG < BN) fetch(t, c + 32 * kEG);
            else fetch(t + n_cl, 32 * grp);
          } else {
            // (measured: the one-chunk-ahead loads slow the head-less, epilogue-bound
            // short-K forward, e.g. C4 layer 1, by 15 %)
            bl = (nb + lane < p.N) ? __ldg(p.bias + nb + lane) : 0.f;
          }
#pragma unroll
          for (int j = 0; j < 32; ++j)
            o[j] = tanh_fast(__uint_as_float(r[j]) + __shfl_sync(0xffffffffu, bl, j));
          if (p.out_q != nullptr && nb < p.N && rbase + lane < p.M)
            write_act_pieces(o, p.out_q, long(p.M) * p.N, long(rbase + lane) * p.N + nb);
          if (do_head) {
            __syncwarp();  // the chunk's head weights are in wsm
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
        } else if (EPI == kEpiBwdTanh) {
#pragma unroll
          for (int j = 0; j < 32; ++j) o[j] = __uint_as_float(r[j]) * (1.f - h[j] * h[j]);
        } else {
#pragma unroll
          for (int j = 0; j < 32; ++j) o[j] = __uint_as_float(r[j]);
        }
        // kEpiFwdTanh with out_hi null: the int8 pieces are the only output
        if (EPI != kEpiFwdTanh || p.out_hi != nullptr) {
        // staging buffers are free once the previous chunk's bulk store has read them
        if (lane == 0) bulk_wait_read();
        __syncwarp();
#pragma unroll
        for (int j4 = 0; j4 < 8; ++j4) {
          *reinterpret_cast<float4*>(blk_ptr + swz(lane, j4)) =
              make_float4(o[4 * j4], o[4 * j4 + 1], o[4 * j4 + 2], o[4 * j4 + 3]);
          if (EPI != kEpiStore && !S::kShareLo && p.out_lo != nullptr)
            *reinterpret_cast<float4*>(blk_ptr + 4096 + swz(lane, j4)) =
                make_float4(o[4 * j4] - tf32_hi(o[4 * j4]), o[4 * j4 + 1] - tf32_hi(o[4 * j4 + 1]),
                            o[4 * j4 + 2] - tf32_hi(o[4 * j4 + 2]),
                            o[4 * j4 + 3] - tf32_hi(o[4 * j4 + 3]));
        }
        fence_async_smem();
        __syncwarp();
        if (lane == 0) {
          if (EPI == kEpiStore) {
            tma_store_3d(&tmOut, nb, rbase, sp, st_out);
          } else {
            tma_store_2d(&tmOut, nb, rbase, st_out);
            if (!S::kShareLo && p.out_lo != nullptr) tma_store_2d(&tmOutLo, nb, rbase, st_lo);
          }
          bulk_commit();
        }
        }
        if (EPI == kEpiBwdTanh) {
          // column sums of this warp's 32 rows (rows past M are exact zeros)
          float csum = 0.f, cmax = 0.f;
#pragma unroll 8
          for (int rr = 0; rr < 32; ++rr) {
            const float v = *reinterpret_cast<const float*>(blk_ptr + swz(rr, lane >> 2) + (lane & 3) * 4);
            csum += v;
            cmax = fmaxf(cmax, fabsf(v));
          }
          cpart[c + lane] = csum;
          if (p.colmax != nullptr && nb + lane < p.N)
            atomicMax(p.colmax + long(rbase / p.colmax_rows) * p.N + nb + lane, __float_as_uint(cmax));
        }
        if (EPI != kEpiStore && S::kShareLo && p.out_lo != nullptr) {
          // residual plane through the same block once the full-value store has read it
          if (lane == 0) bulk_wait_read();
          __syncwarp();
#pragma unroll
          for (int j4 = 0; j4 < 8; ++j4)
            *reinterpret_cast<float4*>(blk_ptr + swz(lane, j4)) =
                make_float4(o[4 * j4] - tf32_hi(o[4 * j4]), o[4 * j4 + 1] - tf32_hi(o[4 * j4 + 1]),
                            o[4 * j4 + 2] - tf32_hi(o[4 * j4 + 2]),
                            o[4 * j4 + 3] - tf32_hi(o[4 * j4 + 3]));
          fence_async_smem();
          __syncwarp();
          if (lane == 0) {
            tma_store_2d(&tmOutLo, nb, rbase, st_lo);
            bulk_commit();
          }
        }
      }
      // TMEM buffer drained: hand it back to the MMA warp
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if (CG == 2) mbar_arrive_cluster(map_rank0(bar_tempty + 8 * acc_buf));
        else mbar_arrive(bar_tempty + 8 * acc_buf);
      }
      if (do_head && rbase + lane < p.M) {
        // kEG groups: one partial slice per group (BN / kEG columns, LaunchInfo::bn)
        float* hp = p.head_part + (long(nt * kEG + grp) * p.M + rbase + lane) * p.head_k;
#pragma unroll
        for (int k = 0; k < kHK; ++k)
          if (k < p.head_k) hp[k] = zacc[k];
      }
      if (EPI == kEpiBwdTanh && p.colsum != nullptr) {
        // fixed-order sum of the 4 warps' column partials into the CTA accumulator
        named_bar(1, kEpiThreads);
        for (int cidx = etid; cidx < BN; cidx += kEpiThreads) {
          const int n = n0 + cidx;
          if (n < p.N)
            csacc[n] += colpart[cidx] + colpart[BN + cidx] + colpart[2 * BN + cidx] +
                        colpart[3 * BN + cidx];
        }
        named_bar(1, kEpiThreads);
      }
    }
    if (EPI == kEpiBwdTanh && p.colsum != nullptr) {
      for (int i = etid; i < p.N; i += kEpiThreads)
        p.colsum[long(blockIdx.x) * p.N + i] = csacc[i];
    }
    if (lane == 0) bulk_wait_all();
  }

  tc_fence_before();
  if (CG == 2) cluster_sync_all();  // no CTA leaves while its pair may still touch its smem/TMEM
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
struct Operand {
  const float* hi = nullptr;
  const float* lo = nullptr;  // null: exact in tf32, the lo pass is skipped
  long ld = 0;                // row pitch (elements) of the stored matrix
  bool mn_major = false;      // false: stored [MN rows][K cols]; true: stored [K rows][MN cols]
  const uint8_t* u8 = nullptr;  // set: the operand is uint8 planes (exact), hi/lo unused;
                                // A must be K-major, B must be MN-major; ld % 16 == 0
  bool lo_smem = false;         // the lo pass runs, on lo = hi - trunc_tf32(hi) derived in
                                // shared memory from the hi tile (lo ignored): no residual
                                // plane in HBM (fp32 operands only)
};

struct LaunchInfo {
  int bn;           // N tile width / epilogue groups
  int ctas;         // persistent CTAs (the fused column sums write this many rows)
  int head_slices;  // fused heads: partial slices written per row (N tiles x epilogue
                    // groups) -- the n_tiles of launch_head_finalize
};

// Launch C = A . B^T with the given epilogue on `stream`.  splits > 1 only for
// kEpiStore (partials into p.ws).  Throws tlg::CudaError on misuse.
LaunchInfo launch(const Operand& A, const Operand& B, int M, int N, int K, int epi, Params p,
            int splits, cudaStream_t stream);

// Number of K splits that fills the GPU for a (M, N, K) problem, given a cap.
int pick_splits(int M, int N, int K, int max_splits);

int num_sms();
// cuTensorMapEncodeTiled through the runtime's driver entry point
PFN_cuTensorMapEncodeTiled_v12000 encode_fn();

}  // namespace tlg::gemm
