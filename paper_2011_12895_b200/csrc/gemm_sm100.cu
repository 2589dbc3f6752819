// Host launcher for the tcgen05 3xTF32 GEMM (see gemm_sm100.cuh).
#include <cudaTypedefs.h>

#include <cstdlib>
#include <cstring>
#include <mutex>

#include "gemm_sm100.cuh"

namespace tlg::gemm {

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    TLG_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    if (q != cudaDriverEntryPointSuccess || p == nullptr)
      throw CudaError("cuTensorMapEncodeTiled unavailable");
    fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

int num_sms() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    TLG_CUDA(cudaGetDevice(&dev));
    TLG_CUDA(cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev));
  }
  return n;
}

namespace {

// 2D fp32 tensor map, 128-byte swizzle, box {32 (inner), box_rows}.
// uint8 2D map, no swizzle (the converter warps lay the tile out for the MMA).
CUtensorMap make_u8_map(const uint8_t* base, long inner, long outer, long ld, int box_inner,
                        int box_outer) {
  CUtensorMap m;
  if ((reinterpret_cast<uintptr_t>(base) & 15) != 0 || ld % 16 != 0)
    throw CudaError("uint8 operand must be 16-byte aligned with a row pitch multiple of 16");
  cuuint64_t dims[2] = {cuuint64_t(inner), cuuint64_t(outer)};
  cuuint64_t strides[1] = {cuuint64_t(ld)};
  cuuint32_t box[2] = {cuuint32_t(box_inner), cuuint32_t(box_outer)};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<uint8_t*>(base), dims,
                           strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                           CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw CudaError("cuTensorMapEncodeTiled(u8) failed: " + std::to_string(r));
  return m;
}

// 3D map for the split-K workspace [splits][M][N], box {32, 32, 1}.
CUtensorMap make_map3(const float* base, long n, long m, long splits) {
  CUtensorMap t;
  cuuint64_t dims[3] = {cuuint64_t(n), cuuint64_t(m), cuuint64_t(splits)};
  cuuint64_t strides[2] = {cuuint64_t(n) * 4, cuuint64_t(n) * m * 4};
  cuuint32_t box[3] = {32, 32, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  if ((reinterpret_cast<uintptr_t>(base) & 15) != 0 || (n * 4) % 16 != 0)
    throw CudaError("gemm workspace must be 16-byte aligned with N a multiple of 4");
  CUresult r = encode_fn()(&t, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(base), dims,
                           strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                           CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw CudaError("cuTensorMapEncodeTiled(3d) failed: " + std::to_string(r));
  return t;
}

CUtensorMap make_map(const float* base, long inner, long outer, long ld, int box_rows,
                     CUtensorMapSwizzle swz) {
  CUtensorMap m;
  if (base == nullptr) {
    std::memset(&m, 0, sizeof(m));
    return m;
  }
  if ((reinterpret_cast<uintptr_t>(base) & 15) != 0 || (ld * 4) % 16 != 0)
    throw CudaError("gemm operand must be 16-byte aligned with a row pitch multiple of 4 floats");
  cuuint64_t dims[2] = {cuuint64_t(inner), cuuint64_t(outer)};
  cuuint64_t strides[1] = {cuuint64_t(ld) * 4};
  cuuint32_t box[2] = {32, cuuint32_t(box_rows)};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims,
                           strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                           swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw CudaError("cuTensorMapEncodeTiled failed: " + std::to_string(r));
  return m;
}

CUtensorMap operand_map(const float* ptr, const Operand& op, long mn, long k, int box_mn) {
  if (!op.mn_major)  // [mn][k]
    return make_map(ptr, k, mn, op.ld, box_mn, CU_TENSOR_MAP_SWIZZLE_128B);
  // [k][mn]: 32-byte swizzle atoms, the layout tcgen05 expects for MN-major tf32
  return make_map(ptr, mn, k, op.ld, 32, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B);
}

thread_local int g_cg = 1;  // CTA-pair mode chosen by launch() for the current call

struct EpiMaps {
  CUtensorMap out, out_lo, act;
};

template <int BN, bool A_MN, bool B_MN, bool A_LO, bool B_LO, int EPI, int U8 = 0, int CG = 1,
          int LOD = 0>
void run(const CUtensorMap& ah, const CUtensorMap& al, const CUtensorMap& bh,
         const CUtensorMap& bl, const EpiMaps& em, const Params& p, dim3 grid,
         cudaStream_t stream) {
  auto kern = gemm_tf32x3_kernel<BN, A_MN, B_MN, A_LO, B_LO, EPI, U8, CG, LOD>;
  constexpr int bytes = Smem<BN, A_LO, B_LO, EPI, U8, CG, LOD>::kBytes;
  constexpr int threads = kernel_threads(BN, EPI, U8, LOD);
  static_assert(bytes <= 227 * 1024, "shared memory budget");
  static std::atomic<unsigned long long> attr{0};  // per device
  ensure_smem_attr(kern, bytes, attr);
  const TileMap tm{int(grid.x), int(grid.y), int(grid.z)};  // grid.x counts (128*CG)-row tiles
  const int tiles = tm.m_tiles * tm.n_tiles * tm.splits;
  if (CG == 1) {
    ::tlg::launch_k(kern, dim3(std::min(tiles, num_sms())), dim3(threads), size_t(bytes), stream, 
        ah, al, bh, bl, em.out, em.out_lo, em.act, p, tm);
  } else {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(2 * std::min(tiles, num_sms() / 2));
    cfg.blockDim = dim3(threads);
    cfg.dynamicSmemBytes = bytes;
    cfg.stream = stream;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    add_pdl(cfg, cfg.attrs);
    TLG_CUDA(cudaLaunchKernelEx(&cfg, kern, ah, al, bh, bl, em.out, em.out_lo, em.act, p, tm));
  }
  TLG_CHECK_LAUNCH();
}

template <int BN, bool A_MN, bool B_MN, bool A_LO, bool B_LO, int EPI, int U8 = 0, int LOD = 0>
void run_if_fits(const CUtensorMap& ah, const CUtensorMap& al, const CUtensorMap& bh,
                 const CUtensorMap& bl, const EpiMaps& em, const Params& p, dim3 grid,
                 cudaStream_t s) {
  if (g_cg == 2) {
    if constexpr (Smem<BN, A_LO, B_LO, EPI, U8, 2, LOD>::kFits && BN >= 128)
      return run<BN, A_MN, B_MN, A_LO, B_LO, EPI, U8, 2, LOD>(ah, al, bh, bl, em, p, grid, s);
    throw CudaError("gemm: pair tile does not fit shared memory");
  }
  if constexpr (Smem<BN, A_LO, B_LO, EPI, U8, 1, LOD>::kFits)
    run<BN, A_MN, B_MN, A_LO, B_LO, EPI, U8, 1, LOD>(ah, al, bh, bl, em, p, grid, s);
  else
    throw CudaError("gemm: tile does not fit shared memory");
}

template <int BN>
void dispatch_bn(bool a_mn, bool b_mn, bool a_lo, bool b_lo, int epi, int u8, int lod,
                 const CUtensorMap& ah, const CUtensorMap& al, const CUtensorMap& bh,
                 const CUtensorMap& bl, const EpiMaps& em, const Params& p, dim3 grid,
                 cudaStream_t s) {
  // derived lo planes (Operand::lo_smem): the learner's activations / dZ / observations
  if (lod) {
    if (u8) throw CudaError("gemm: derived lo planes need fp32 operands");
    if (!a_mn && !b_mn && a_lo && b_lo && epi == kEpiFwdTanh && lod == 1)
      return run_if_fits<BN, false, false, true, true, kEpiFwdTanh, 0, 1>(ah, al, bh, bl, em, p, grid, s);
    if (!a_mn && !b_mn && a_lo && b_lo && epi == kEpiFwdTanh && lod == (1 | kLodEg2))
      return run_if_fits<BN, false, false, true, true, kEpiFwdTanh, 0, 1 | kLodEg2>(ah, al, bh, bl, em, p, grid, s);
    if (!a_mn && !b_mn && a_lo && b_lo && epi == kEpiFwdTanh && lod == (1 | kLodEg3))
      return run_if_fits<BN, false, false, true, true, kEpiFwdTanh, 0, 1 | kLodEg3>(ah, al, bh, bl, em, p, grid, s);
    if (!a_mn && !b_mn && a_lo && b_lo && epi == kEpiFwdLoss && lod == 1)
      return run_if_fits<BN, false, false, true, true, kEpiFwdLoss, 0, 1>(ah, al, bh, bl, em, p, grid, s);
    if (!a_mn && b_mn && a_lo && b_lo && epi == kEpiBwdTanh && lod == 1)
      return run_if_fits<BN, false, true, true, true, kEpiBwdTanh, 0, 1>(ah, al, bh, bl, em, p, grid, s);
    if (a_mn && b_mn && a_lo && b_lo && epi == kEpiStore && lod == 3)
      return run_if_fits<BN, true, true, true, true, kEpiStore, 0, 3>(ah, al, bh, bl, em, p, grid, s);
    if (a_mn && b_mn && a_lo && !b_lo && epi == kEpiStore && lod == 1)
      return run_if_fits<BN, true, true, true, false, kEpiStore, 0, 1>(ah, al, bh, bl, em, p, grid, s);
    throw CudaError("gemm: unsupported derived-lo operand combination");
  }
  // uint8 observation planes: forward (A = obs) and dW of layer 1 (B = obs)
  if (u8 == 1 && !a_mn && !b_mn && b_lo && epi == kEpiFwdTanh)
    return run_if_fits<BN, false, false, false, true, kEpiFwdTanh, 1>(ah, al, bh, bl, em, p, grid, s);
  if (u8 == 2 && a_mn && b_mn && a_lo && epi == kEpiStore)
    return run_if_fits<BN, true, true, true, false, kEpiStore, 2>(ah, al, bh, bl, em, p, grid, s);
  if (u8) throw CudaError("gemm: unsupported uint8 operand combination");
  // forward: A = activations (K-major), B = W (K-major)
  if (!a_mn && !b_mn && b_lo && epi == kEpiFwdTanh) {
    if (a_lo) return run_if_fits<BN, false, false, true, true, kEpiFwdTanh>(ah, al, bh, bl, em, p, grid, s);
    return run_if_fits<BN, false, false, false, true, kEpiFwdTanh>(ah, al, bh, bl, em, p, grid, s);
  }
  // fused top layer + heads + PPO loss + dZ_L (A = activations, B = W, both 3-pass)
  if (epi == kEpiFwdLoss && !a_mn && !b_mn && a_lo && b_lo)
    return run_if_fits<BN, false, false, true, true, kEpiFwdLoss>(ah, al, bh, bl, em, p, grid, s);
  // dX: A = dZ (K-major), B = W (MN-major)
  if (!a_mn && b_mn && a_lo && b_lo && epi == kEpiBwdTanh)
    return run_if_fits<BN, false, true, true, true, kEpiBwdTanh>(ah, al, bh, bl, em, p, grid, s);
  // dX with a transposed copy of W (B K-major)
  if (!a_mn && !b_mn && a_lo && b_lo && epi == kEpiBwdTanh)
    return run_if_fits<BN, false, false, true, true, kEpiBwdTanh>(ah, al, bh, bl, em, p, grid, s);
  // dW: A = dZ^T (MN-major), B = H (MN-major), split-K partials
  if (a_mn && b_mn && a_lo && epi == kEpiStore) {
    if (b_lo) return run_if_fits<BN, true, true, true, true, kEpiStore>(ah, al, bh, bl, em, p, grid, s);
    return run_if_fits<BN, true, true, true, false, kEpiStore>(ah, al, bh, bl, em, p, grid, s);
  }
  // generic K-major store (used by the testkit)
  if (!a_mn && !b_mn && a_lo && b_lo && epi == kEpiStore)
    return run_if_fits<BN, false, false, true, true, kEpiStore>(ah, al, bh, bl, em, p, grid, s);
  throw CudaError("gemm: unsupported operand/epilogue combination");
}

}  // namespace

int pick_splits(int M, int N, int K, int max_splits) {
  // Split-K count for the dW GEMMs (K = frames): minimise a simple cost model of
  //   waves(s) x K-blocks per split  (+ the workspace round trip of the fixed-order reduce),
  // with the launcher's own tile plan (256-wide tiles; CTA pairs once there are enough
  // 256-row tiles to occupy every pair).  Without the pair term a 2048x2048 dW picked one
  // split and ran 128 single-CTA tiles on 148 SMs (C5: 4.8 ms vs 3.6 ms at 8 splits).
  const int BN = N > 128 ? 256 : N > 64 ? 128 : 64;
  const int kb = ceil_div(K, kBK);
  const int units2 = num_sms() / 2;
  const int s_max = std::max(1, std::min(max_splits, kb / 4));  // keep >= 4 K blocks per split
  const double kblock_us = 1.33 * BN / 256.0;  // one 128xBN x 32 3xTF32 K block per SM
  const double ws_us_per_elem = 2.0 * 4.0 / 6.0e6;  // write + read back at ~6 TB/s
  double best = 0;
  int best_s = 1;
  for (int s = 1; s <= s_max; ++s) {
    const int per = ceil_div(kb, s);
    const int se = ceil_div(kb, per);  // launch() drops empty splits the same way
    if (se != s) continue;
    const long t2 = long(ceil_div(M, 2 * kBM)) * ceil_div(N, BN) * s;
    long waves;
    if (BN >= 128 && M >= 2 * kBM && t2 >= units2 && per >= 8)
      waves = (t2 + units2 - 1) / units2;
    else
      waves = (long(ceil_div(M, kBM)) * ceil_div(N, BN) * s + num_sms() - 1) / num_sms();
    const double t = double(waves) * per * kblock_us + ws_us_per_elem * s * double(M) * N +
                     (s > 1 ? 3.0 : 0.0);
    if (s == 1 || t < 0.98 * best) {
      best = t;
      best_s = s;
    }
  }
  return best_s;
}

LaunchInfo launch(const Operand& A, const Operand& B, int M, int N, int K, int epi, Params p,
                  int splits, cudaStream_t stream) {
  if (M <= 0 || N <= 0 || K <= 0) throw CudaError("gemm: empty problem");
  const bool a_lo0 = (A.lo != nullptr || A.lo_smem) && !A.u8,
             b_lo0 = (B.lo != nullptr || B.lo_smem) && !B.u8;
  const int lod = (A.lo_smem && !A.u8 ? 1 : 0) | (B.lo_smem && !B.u8 ? 2 : 0);
  const int u8_0 = A.u8 ? 1 : B.u8 ? 2 : 0;
  // the tanh forward may drop its fp32 plane when the int8 pieces or the fused heads are
  // what the caller reads
  if (p.out_hi == nullptr && epi != kEpiStore &&
      !(epi == kEpiFwdTanh && p.out_lo == nullptr && (p.out_q != nullptr || p.head_k > 0)))
    throw CudaError("gemm: missing output plane");
  if (p.out_q != nullptr &&
      (epi != kEpiFwdTanh || N % 32 != 0 || (reinterpret_cast<uintptr_t>(p.out_q) & 15) != 0))
    throw CudaError("gemm: int8 activation pieces need the tanh forward, N % 32 == 0, 16-B alignment");
  if (epi == kEpiBwdTanh && p.colsum != nullptr && N > kColMax)
    throw CudaError("gemm: fused column sums need N <= 2048");
  const int kb_total = ceil_div(K, kBK);
  if (splits < 1) splits = 1;
  if (epi != kEpiStore) splits = 1;
  p.kb_per_split = ceil_div(kb_total, splits);
  splits = ceil_div(kb_total, p.kb_per_split);
  p.M = M;
  p.N = N;
  p.K = K;
  // Tile width: 256 columns when the K loop is long enough to hide the wider epilogue,
  // else 128 (short-K fused epilogues are the critical path; narrower tiles balance) --
  // except with derived residuals, where 256-column tiles halve the A-operand traffic
  // per product: the tanh forward then drains through two epilogue warp groups, the dX
  // epilogue keeps up as it is (C3: layer-2 forward 119 -> 103 us, dX 102 -> 99 us).
  int BN = N > 128 ? 256 : N > 64 ? 128 : 64;
  const int kb_tile = p.kb_per_split;  // K blocks per tile
  // two epilogue warp groups (kLodEg2) for the derived-residual tanh forward on 128-column
  // tiles and on short-K 256-column tiles
  auto lod_k = [&](int bn) {
    if (epi != kEpiFwdTanh || lod == 0 || u8_0 != 0) return lod;
    // three groups where the K loop is nearly empty (K <= 64: the epilogue is the kernel)
    if (bn == 256 && kb_tile <= 2 && !std::getenv("TLG_GEMM_EG2")) return lod | kLodEg3;
    if (bn == 256 && kb_tile < 16) return lod | kLodEg2;
    return bn == 128 ? lod | kLodEg2 : lod;
  };
  const bool wide_lod = (lod & 1) && (epi == kEpiFwdTanh || epi == kEpiBwdTanh) &&
                        !std::getenv("TLG_GEMM_NARROW");
  if (BN == 256 && epi != kEpiStore && epi != kEpiFwdLoss && kb_tile < 16 && !wide_lod &&
      !std::getenv("TLG_GEMM_WIDE"))
    BN = 128;
  if (epi == kEpiFwdLoss) {  // whole rows per tile, CTA pairs (the only plan that fits)
    if (N > 256 || M < 2 * kBM || p.head_k < 2 || p.head_k > 8)
      throw CudaError("gemm: fused loss epilogue needs N <= 256, M >= 256, 2 <= A+1 <= 8");
    BN = 256;
  }
  if (const char* e = std::getenv("TLG_GEMM_MAX_BN")) {  // tuning experiments only
    const int cap = std::atoi(e);
    while (BN > 64 && BN > cap) BN /= 2;
  }
  // CTA pairs (cta_group::2) when there are enough 256-row tiles to fill the GPU; then
  // the widest tile whose pipeline (>= 2 stages) + epilogue staging fits 227 KB.
  int cg = 1;
  for (;;) {
    cg = 1;
    const long tiles2 = long(ceil_div(M, 2 * kBM)) * ceil_div(N, BN) * splits;
    // (short K loops too when the residual is derived: C4 layer 1, K = 64, 108 -> 98 us)
    if (BN >= 128 && M >= 2 * kBM && tiles2 >= num_sms() / 2 && (kb_tile >= 8 || wide_lod))
      cg = 2;
    if (const char* e = std::getenv("TLG_GEMM_CG")) cg = std::atoi(e) == 2 && BN >= 128 ? 2 : 1;
    if (epi == kEpiFwdLoss) cg = 2;
    if (const char* e = std::getenv("TLG_GEMM_CG_U8"))  // tuning experiments only
      if ((A.u8 || B.u8) && std::atoi(e) == 2 && BN >= 128) cg = 2;
    if (BN == 64 || epi == kEpiFwdLoss ||
        smem_plan(BN, a_lo0, b_lo0, epi, u8_0, cg, lod_k(BN)).bytes <= 227 * 1024)
      break;
    BN /= 2;
  }
  const int u8 = A.u8 ? 1 : B.u8 ? 2 : 0;
  if (A.u8 && (A.mn_major || A.ld % 16)) throw CudaError("gemm: uint8 A must be K-major, ld % 16 == 0");
  if (B.u8 && (!B.mn_major || B.ld % 16)) throw CudaError("gemm: uint8 B must be MN-major, ld % 16 == 0");
  const CUtensorMap ah = A.u8 ? make_u8_map(A.u8, K, M, A.ld, 32, kBM) : operand_map(A.hi, A, M, K, kBM);
  const CUtensorMap al = operand_map(A.lo_smem ? nullptr : A.lo, A, M, K, kBM);
  const CUtensorMap bh = B.u8 ? make_u8_map(B.u8, N, K, B.ld, BN / cg, 32)
                              : operand_map(B.hi, B, N, K, BN / cg);
  const CUtensorMap bl = operand_map(B.lo_smem ? nullptr : B.lo, B, N, K, BN / cg);
  dim3 grid(ceil_div(M, kBM * cg), ceil_div(N, BN), splits);
  g_cg = cg;
  const bool a_lo = a_lo0, b_lo = b_lo0;
  // epilogue maps: 32x32 fp32 blocks with the 128-B swizzle
  EpiMaps em;
  std::memset(&em, 0, sizeof(em));
  if (epi == kEpiStore) {
    em.out = make_map3(p.ws, N, M, splits);
  } else {
    em.out = make_map(p.out_hi, N, M, p.ldo, 32, CU_TENSOR_MAP_SWIZZLE_128B);
    em.out_lo = make_map(p.out_lo, N, M, p.ldo, 32, CU_TENSOR_MAP_SWIZZLE_128B);
    if (epi == kEpiBwdTanh) em.act = make_map(p.act_hi, N, M, p.ld_act, 32, CU_TENSOR_MAP_SWIZZLE_128B);
    if (A.u8 && p.a_expand) em.act = make_map(p.a_expand, K, M, A.ld, kBM, CU_TENSOR_MAP_SWIZZLE_128B);
  }
  const int lodk = lod_k(BN);
  switch (BN) {
    case 256: dispatch_bn<256>(A.mn_major, B.mn_major, a_lo, b_lo, epi, u8, lodk, ah, al, bh, bl, em, p, grid, stream); break;
    case 128: dispatch_bn<128>(A.mn_major, B.mn_major, a_lo, b_lo, epi, u8, lodk, ah, al, bh, bl, em, p, grid, stream); break;
    default: dispatch_bn<64>(A.mn_major, B.mn_major, a_lo, b_lo, epi, u8, lodk, ah, al, bh, bl, em, p, grid, stream); break;
  }
  const int tiles = int(grid.x * grid.y * grid.z);
  const int eg = epi_groups(BN, epi, u8, lodk);
  return {BN / eg, cg == 2 ? 2 * std::min(tiles, num_sms() / 2) : std::min(tiles, num_sms()),
          ceil_div(N, BN) * eg};
}

}  // namespace tlg::gemm
