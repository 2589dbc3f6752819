// Host side of the exact-integer binary-plane GEMM (gemm_i8.cuh) + the weight quantizer.
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "gemm_i8.cuh"

namespace tlg::gemm {

namespace {

CUtensorMap make_bytes_map(const void* base, long inner, long outer, long ld, int box_inner,
                           int box_outer, CUtensorMapSwizzle swz) {
  CUtensorMap m;
  if ((reinterpret_cast<uintptr_t>(base) & 15) != 0 || ld % 16 != 0)
    throw CudaError("int8 operand must be 16-byte aligned with a row pitch multiple of 16");
  cuuint64_t dims[2] = {cuuint64_t(inner), cuuint64_t(outer)};
  cuuint64_t strides[1] = {cuuint64_t(ld)};
  cuuint32_t box[2] = {cuuint32_t(box_inner), cuuint32_t(box_outer)};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(base), dims,
                           strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw CudaError("cuTensorMapEncodeTiled(i8) failed: " + std::to_string(r));
  return m;
}

CUtensorMap make_f32_out_map(float* base, long n, long m, long ld) {
  CUtensorMap t;
  if ((reinterpret_cast<uintptr_t>(base) & 15) != 0 || (ld * 4) % 16 != 0)
    throw CudaError("gemm output must be 16-byte aligned with a row pitch multiple of 4 floats");
  cuuint64_t dims[2] = {cuuint64_t(n), cuuint64_t(m)};
  cuuint64_t strides[1] = {cuuint64_t(ld) * 4};
  cuuint32_t box[2] = {32, 32};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = encode_fn()(&t, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, base, dims, strides, box,
                           estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw CudaError("cuTensorMapEncodeTiled(out) failed: " + std::to_string(r));
  return t;
}

template <int BN, int CG, int MC = 1>
void run_i8_fwd(const CUtensorMap& tb, const CUtensorMap& tq, const CUtensorMap& to,
                const CUtensorMap& tl, const I8Params& p, const TileMap& tm, cudaStream_t stream) {
  auto kern = gemm_i8_bits_fwd_kernel<BN, CG, MC>;
  constexpr int bytes = SmemI8<BN, CG>::kBytes;
  static_assert(bytes <= 227 * 1024, "shared memory budget");
  static std::atomic<unsigned long long> attr{0};  // per device
  ensure_smem_attr(kern, bytes, attr);
  const int tiles = tm.m_tiles * tm.n_tiles;
  if (CG == 1) {
    ::tlg::launch_k(kern, dim3(std::min(tiles, num_sms())), dim3(kThreadsI8), size_t(bytes), stream, tb, tq, to, tl, p, tm);
  } else {
    cudaLaunchConfig_t cfg{};
    constexpr int kCl = CG * MC;
    cfg.blockDim = dim3(kThreadsI8);
    cfg.dynamicSmemBytes = bytes;
    cfg.stream = stream;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = kCl;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    // persistent grid = the clusters that are co-resident (GPCs need not hold a multiple of
    // kCl SMs; a second partial wave of persistent clusters would double the time)
    // (pairs: every GPC holds an even number of SMs, and the occupancy query under-reports
    // them — 74 pairs measured faster than the queried count)
    static std::atomic<int> max_cl{0};
    if (max_cl.load() == 0) {
      int n = num_sms() / kCl;
      if (MC == 2) {
        cfg.gridDim = dim3(kCl * n);
        TLG_CUDA(cudaOccupancyMaxActiveClusters(&n, kern, &cfg));
      }
      if (std::getenv("TLG_DEBUG_CLUSTERS")) {
        int q = 0;
        cfg.gridDim = dim3(kCl * (num_sms() / kCl));
        cudaOccupancyMaxActiveClusters(&q, kern, &cfg);
        fprintf(stderr, "i8 fwd: cluster %d, persistent clusters %d, occupancy query %d\n",
                kCl, n, q);
      }
      max_cl.store(std::max(1, std::min(n, num_sms() / kCl)));
    }
    cfg.gridDim = dim3(kCl * std::min(tiles, max_cl.load()));
    add_pdl(cfg, cfg.attrs);
    TLG_CUDA(cudaLaunchKernelEx(&cfg, kern, tb, tq, to, tl, p, tm));
  }
  TLG_CHECK_LAUNCH();
}

template <int BN, int CG, int NQ, int NX, int MS = 1, int EG = 1>
void run_i8_fwd_dec(const CUtensorMap& tb, const CUtensorMap& tq, const CUtensorMap& to,
                    const CUtensorMap& tl, const I8Params& p, const TileMap& tm,
                    cudaStream_t stream) {
  auto kern = gemm_i8_bits_fwd_dec_kernel<BN, CG, NQ, NX, MS, EG>;
  constexpr int bytes = SmemI8Dec<BN, CG, NQ, NX, MS, EG>::kBytes;
  constexpr int kThreads = kThreadsI8 + 32 * kEpiWarps * (EG - 1);
  static std::atomic<unsigned long long> attr{0};  // per device
  ensure_smem_attr(kern, bytes, attr);
  const int tiles = tm.m_tiles * tm.n_tiles;
  if (CG == 1) {
    ::tlg::launch_k(kern, dim3(std::min(tiles, num_sms())), dim3(kThreads), size_t(bytes),
                    stream, tb, tq, to, tl, p, tm);
  } else {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(2 * std::min(tiles, num_sms() / 2));
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = bytes;
    cfg.stream = stream;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    add_pdl(cfg, cfg.attrs);
    TLG_CUDA(cudaLaunchKernelEx(&cfg, kern, tb, tq, to, tl, p, tm));
  }
  TLG_CHECK_LAUNCH();
}

// one block per row: max |W[n][:]| (fixed-order tree), then the three pieces
__global__ void __launch_bounds__(256) quantize_rows_kernel(const float* __restrict__ W, int K,
                                                            long ldw, int8_t* __restrict__ q,
                                                            long Kp, long plane,
                                                            float* __restrict__ scale) {
  TLG_PDL_ENTRY();
  __shared__ float red[8];
  const int n = blockIdx.x;
  const float* w = W + long(n) * ldw;
  float mx = 0.f;
  for (int k = threadIdx.x; k < K; k += blockDim.x) mx = fmaxf(mx, fabsf(w[k]));
  mx = warp_max(mx);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
  __syncthreads();
  if (threadIdx.x < 32) {
    float v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.f;
    v = warp_max(v);
    if (threadIdx.x == 0) red[0] = v;
  }
  __syncthreads();
  const float s = red[0] > 0.f ? red[0] / 127.f : 1.f;
  const float inv = red[0] > 0.f ? 127.f / red[0] : 1.f;  // the epilogue multiplies by s
  if (threadIdx.x == 0) scale[n] = s;
  int8_t* q0 = q + long(n) * Kp;
  constexpr float kMagic = 12582912.f;  // round-to-nearest-even via 1.5 * 2^23
  for (long k = threadIdx.x; k < Kp; k += blockDim.x) {
    uint32_t a = 0, b = 0, c = 0;
    if (k < K) {
      // x = w * 127 / max rounds once; the residual steps are exact
      const float x = fminf(fmaxf(w[k] * inv, -127.f), 127.f);
      const float m0 = x + kMagic;
      const float x1 = (x - (m0 - kMagic)) * 128.f;  // |x1| <= 64
      const float m1 = x1 + kMagic;
      const float m2 = (x1 - (m1 - kMagic)) * 128.f + kMagic;
      a = __float_as_uint(m0);
      b = __float_as_uint(m1);
      c = __float_as_uint(m2);
    }
    q0[k] = int8_t(a & 0xFFu);
    q0[plane + k] = int8_t(b & 0xFFu);
    q0[2 * plane + k] = int8_t(c & 0xFFu);
  }
}

template <int CG>
void run_i8_dw(const CUtensorMap& tp, const CUtensorMap& tb, const CUtensorMap& tw,
               const I8DwParams& p, const TileMap& tm, cudaStream_t stream) {
  auto kern = gemm_i8_bits_dw_kernel<CG>;
  constexpr int bytes = SmemI8Dw<CG>::kBytes;
  static_assert(bytes <= 227 * 1024, "shared memory budget");
  static std::atomic<unsigned long long> attr{0};  // per device
  ensure_smem_attr(kern, bytes, attr);
  const int tiles = tm.m_tiles * tm.n_tiles * tm.splits;
  if (CG == 1) {
    ::tlg::launch_k(kern, dim3(std::min(tiles, num_sms())), dim3(kThreadsI8), size_t(bytes), stream, tp, tb, tw, p, tm);
  } else {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(2 * std::min(tiles, num_sms() / 2));
    cfg.blockDim = dim3(kThreadsI8);
    cfg.dynamicSmemBytes = bytes;
    cfg.stream = stream;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    add_pdl(cfg, cfg.attrs);
    TLG_CUDA(cudaLaunchKernelEx(&cfg, kern, tp, tb, tw, p, tm));
  }
  TLG_CHECK_LAUNCH();
}

// dZ -> three int8 pieces per element, scale per (split, column) from the dX epilogue's
// column maxima.  A block covers kQRows frames (never straddling a split) x all columns:
// thread = (4-column quad, frame lane), scale inverses computed once per thread.
constexpr int kQRows = 64;
__global__ void __launch_bounds__(256) quantize_cols_kernel(const float* __restrict__ Z, long F,
                                                            int M, long ldz,
                                                            const unsigned* __restrict__ colmax,
                                                            long rows_per_split,
                                                            int8_t* __restrict__ P) {
  TLG_PDL_ENTRY();
  const int quads = M / 4;
  const int lanes = max(1, 256 / quads);
  const int per_pass = (256 / quads) > 0 ? quads : 256;  // quads handled per pass
  const long plane = F * M;
  const long f0 = long(blockIdx.x) * kQRows;
  const long g = f0 / rows_per_split;
  for (int q0 = 0; q0 < quads; q0 += per_pass) {
    const int qi = q0 + int(threadIdx.x) % per_pass;
    const int lane = int(threadIdx.x) / per_pass;
    if (qi >= quads || lane >= lanes) continue;
    const int m = qi * 4;
    float inv[4], lim[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float mx = __uint_as_float(colmax[g * M + m + j]);
      inv[j] = mx > 0.f ? 127.f / mx : 1.f;  // the GEMM epilogue multiplies by mx / 127
      lim[j] = 127.f;
    }
    const long fend = min(F, f0 + kQRows);
    // four rows per round: their loads are in flight together
    for (long fb = f0 + lane; fb < fend; fb += 4L * lanes) {
      float4 zr[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const long f = fb + long(u) * lanes;
        zr[u] = f < fend ? *reinterpret_cast<const float4*>(Z + f * ldz + m)
                         : make_float4(0.f, 0.f, 0.f, 0.f);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const long f = fb + long(u) * lanes;
        if (f >= fend) break;
        const float zv[4] = {zr[u].x, zr[u].y, zr[u].z, zr[u].w};
        uint32_t w0 = 0, w1 = 0, w2 = 0;
        // round-to-nearest-even via the 1.5 * 2^23 magic constant: the sum's low mantissa
        // bits are the integer in two's complement (no F2I / FRND on the quarter-rate pipe)
        constexpr float kMagic = 12582912.f;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          // x = z * (127 / max) rounds once (|x| <= 127 (1 + 2^-23)); the residual steps
          // are exact (Sterbenz, power-of-two scaling)
          const float x = fminf(fmaxf(zv[j] * inv[j], -lim[j]), lim[j]);
          const float m0 = x + kMagic;
          const float x1 = (x - (m0 - kMagic)) * 128.f;
          const float m1 = x1 + kMagic;
          const float x2 = (x1 - (m1 - kMagic)) * 128.f;
          const float m2 = x2 + kMagic;
          w0 |= (__float_as_uint(m0) & 0xFFu) << (8 * j);
          w1 |= (__float_as_uint(m1) & 0xFFu) << (8 * j);
          w2 |= (__float_as_uint(m2) & 0xFFu) << (8 * j);
        }
        const long o = f * M + m;
        *reinterpret_cast<uint32_t*>(P + o) = w0;
        *reinterpret_cast<uint32_t*>(P + plane + o) = w1;
        *reinterpret_cast<uint32_t*>(P + 2 * plane + o) = w2;
      }
    }
  }
}

CUtensorMap make_ws_map(float* base, long n, long m, long splits) {
  CUtensorMap t;
  cuuint64_t dims[3] = {cuuint64_t(n), cuuint64_t(m), cuuint64_t(splits)};
  cuuint64_t strides[2] = {cuuint64_t(n) * 4, cuuint64_t(n) * m * 4};
  cuuint32_t box[3] = {32, 32, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  if ((reinterpret_cast<uintptr_t>(base) & 15) != 0 || (n * 4) % 16 != 0)
    throw CudaError("gemm workspace must be 16-byte aligned with N a multiple of 4");
  CUresult r = encode_fn()(&t, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, base, dims, strides, box, estr,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw CudaError("cuTensorMapEncodeTiled(ws) failed: " + std::to_string(r));
  return t;
}

}  // namespace

void launch_quantize_cols(const float* Z, long F, int M, long ldz, const unsigned* colmax,
                          long rows_per_split, int8_t* P, cudaStream_t stream) {
  if (M % 4 != 0 || ldz % 4 != 0) throw CudaError("quantize_cols: M and ldz must be multiples of 4");
  if (rows_per_split % kQRows != 0) throw CudaError("quantize_cols: split rows % 64 != 0");
  ::tlg::launch_k(quantize_cols_kernel, dim3(ceil_div(F, kQRows)), dim3(256), size_t(0), stream, Z, F, M, ldz, colmax,
                                                                rows_per_split, P);
  TLG_CHECK_LAUNCH();
}

void launch_i8_bits_dw(const int8_t* P, const uint8_t* bits, long rowb, const unsigned* colmax,
                       int M, int N, int K, int kb_per_split, float* ws, cudaStream_t stream) {
  if (M <= 0 || N <= 0 || K <= 0) throw CudaError("gemm_i8_dw: empty problem");
  if (long(kb_per_split) * kBKi > 131072) throw CudaError("gemm_i8_dw: split too long for int32");
  if (M % 16 != 0) throw CudaError("gemm_i8_dw: M must be a multiple of 16");
  int cg = M >= 2 * kBM ? 2 : 1;
  if (const char* e = std::getenv("TLG_I8_CG")) cg = std::atoi(e) == 2 ? 2 : 1;
  const int kb_total = ceil_div(K, kBKi);
  const int splits = ceil_div(kb_total, kb_per_split);
  const TileMap tm{ceil_div(M, kBM * cg), ceil_div(N, 128 * cg), splits};
  I8DwParams p{M, N, K, kb_per_split, long(K), colmax};
  const CUtensorMap tp = make_bytes_map(P, M, 3L * K, M, kBM, kBKi, CU_TENSOR_MAP_SWIZZLE_128B);
  const CUtensorMap tb = make_bytes_map(bits, rowb, K, rowb, 16, kBKi, CU_TENSOR_MAP_SWIZZLE_NONE);
  const CUtensorMap tw = make_ws_map(ws, N, M, splits);
  if (cg == 2) run_i8_dw<2>(tp, tb, tw, p, tm, stream);
  else run_i8_dw<1>(tp, tb, tw, p, tm, stream);
}

template <int BN, int CG>
void run_i8x2_fwd(const CUtensorMap& ta, const CUtensorMap& tq, const CUtensorMap& to,
                  const CUtensorMap& tl, const I8x2Params& p, const TileMap& tm,
                  cudaStream_t stream) {
  auto kern = gemm_i8x2_fwd_kernel<BN, CG>;
  constexpr int bytes = SmemI8x2<BN, CG>::kBytes;
  static_assert(bytes <= 227 * 1024, "shared memory budget");
  static std::atomic<unsigned long long> attr{0};  // per device
  ensure_smem_attr(kern, bytes, attr);
  const int tiles = tm.m_tiles * tm.n_tiles;
  constexpr int threads = 32 * (2 + kEpiWarps);
  if (CG == 1) {
    ::tlg::launch_k(kern, dim3(std::min(tiles, num_sms())), dim3(threads), size_t(bytes), stream, ta, tq, to, tl, p, tm);
  } else {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(2 * std::min(tiles, num_sms() / 2));
    cfg.blockDim = dim3(threads);
    cfg.dynamicSmemBytes = bytes;
    cfg.stream = stream;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    add_pdl(cfg, cfg.attrs);
    TLG_CUDA(cudaLaunchKernelEx(&cfg, kern, ta, tq, to, tl, p, tm));
  }
  TLG_CHECK_LAUNCH();
}

LaunchInfo launch_i8x2_fwd(const int8_t* a, const int8_t* q, long Kp, const float* scale,
                           const float* bias, int M, int N, int K, float* out, float* out_lo,
                           int ldo, const float* head_w, const float* head_wv, int head_k,
                           float* head_part, cudaStream_t stream, int8_t* out_q) {
  if (M <= 0 || N <= 0 || K <= 0) throw CudaError("gemm_i8x2: empty problem");
  if (out_q != nullptr && (N % 32 != 0 || (reinterpret_cast<uintptr_t>(out_q) & 15) != 0))
    throw CudaError("gemm_i8x2: int8 activation pieces need N % 32 == 0 and 16-B alignment");
  if (K % 16 != 0 || Kp < K) throw CudaError("gemm_i8x2: K must be a multiple of 16");
  if (head_k > 8) throw CudaError("gemm_i8x2: fused heads need n_actions + 1 <= 8");
  // 64-column tiles: three accumulators double-buffered in TMEM (the epilogue of one tile
  // overlaps the MMAs of the next).  CTA pairs only (a single CTA's six piece tiles
  // would leave one pipeline stage)
  int BN = 64;
  if (const char* e = std::getenv("TLG_I8X2_BN")) BN = std::atoi(e) == 128 ? 128 : 64;
  if (M < 2 * kBM) throw CudaError("gemm_i8x2: needs M >= 256");
  constexpr int cg = 2;
  I8x2Params p{M, N, K, scale, bias, long(M), long(N), head_w, head_wv, head_k, head_part,
               out_lo != nullptr ? 1 : 0, out_q, out != nullptr ? 1 : 0};
  const TileMap tm{ceil_div(M, kBM * cg), ceil_div(N, BN), 1};
  const CUtensorMap ta = make_bytes_map(a, K, 3L * M, K, kBKi, kBM, CU_TENSOR_MAP_SWIZZLE_128B);
  const CUtensorMap tq = make_bytes_map(q, Kp, 3L * N, Kp, kBKi, BN / cg, CU_TENSOR_MAP_SWIZZLE_128B);
  if (out == nullptr && (out_lo != nullptr || (out_q == nullptr && head_k <= 0)))
    throw CudaError("gemm_i8x2: missing output plane");
  CUtensorMap to;
  if (out) to = make_f32_out_map(out, N, M, ldo);
  else std::memset(&to, 0, sizeof(to));
  CUtensorMap tl;
  if (out_lo) tl = make_f32_out_map(out_lo, N, M, ldo);
  else std::memset(&tl, 0, sizeof(tl));
  if (BN == 128) run_i8x2_fwd<128, 2>(ta, tq, to, tl, p, tm, stream);
  else run_i8x2_fwd<64, 2>(ta, tq, to, tl, p, tm, stream);
  const int tiles = tm.m_tiles * tm.n_tiles;
  return {BN, 2 * std::min(tiles, num_sms() / 2), tm.n_tiles};
}

void launch_quantize_rows(const float* W, int N, int K, long ldw, int8_t* q, long Kp, float* s,
                          cudaStream_t stream) {
  if (Kp % 16 != 0 || Kp < K) throw CudaError("quantize_rows: Kp must be >= K and a multiple of 16");
  ::tlg::launch_k(quantize_rows_kernel, dim3(N), dim3(256), size_t(0), stream, W, K, ldw, q, Kp, long(N) * Kp, s);
  TLG_CHECK_LAUNCH();
}

LaunchInfo launch_i8_bits_fwd(const uint8_t* bits, long rowb, const int8_t* q, long Kp,
                              const float* scale, const float* bias, int M, int N, int K,
                              float* out, float* out_lo, int ldo, cudaStream_t stream,
                              int8_t* out_q) {
  if (M <= 0 || N <= 0 || K <= 0) throw CudaError("gemm_i8: empty problem");
  if (rowb * 8 < K || Kp < K) throw CudaError("gemm_i8: K exceeds the operand rows");
  // 128-wide tiles (double-buffered accumulators); TLG_I8_BN=256 (experiment): one tile
  // spans N = 256 (the x tiles are expanded once per M tile, accumulators single-buffered)
  const int BN = std::getenv("TLG_I8_BN") && std::atoi(std::getenv("TLG_I8_BN")) == 256 && N > 128
                     ? 256 : 128;
  // CTA pairs (256-row tiles) whenever there are enough of them to fill the GPU
  int cg = (M >= 2 * kBM && long(ceil_div(M, 2 * kBM)) * ceil_div(N, BN) >= num_sms() / 2) ? 2 : 1;
  if (BN == 256) cg = 2;
  if (const char* e = std::getenv("TLG_I8_CG")) cg = std::atoi(e) == 2 ? 2 : 1;
  // TLG_I8_MC=2: two CTA pairs per cluster share the weight-piece tiles (TMA multicast).
  // Correct, but slower at C3 (0.22 vs 0.19 ms): L2 traffic drops 15 %, the per-SM
  // tensor activity does not move, and 4-CTA clusters fit only 132 SMs.
  int mc = 1;
  if (const char* e = std::getenv("TLG_I8_MC"))
    mc = cg == 2 && std::atoi(e) == 2 && M >= 4 * kBM ? 2 : 1;
  if (out_q != nullptr && (N % 32 != 0 || (reinterpret_cast<uintptr_t>(out_q) & 15) != 0))
    throw CudaError("gemm_i8: int8 activation pieces need N % 32 == 0 and 16-B alignment");
  I8Params p{M, N, K, scale, bias, N, out_q, out_lo != nullptr ? 1 : 0};
  const TileMap tm{ceil_div(M, kBM * cg * mc), ceil_div(N, BN), 1};
  // bit rows: box {16 bytes = 128 elements, 128 rows}; pieces: box {128, BN / cg}, SW128
  const CUtensorMap tb = make_bytes_map(bits, rowb, M, rowb, kBKi / 8, kBM, CU_TENSOR_MAP_SWIZZLE_NONE);
  const CUtensorMap tq = make_bytes_map(q, Kp, 3L * N, Kp, kBKi, BN / cg, CU_TENSOR_MAP_SWIZZLE_128B);
  const CUtensorMap to = make_f32_out_map(out, N, M, ldo);
  const CUtensorMap tl = out_lo ? make_f32_out_map(out_lo, N, M, ldo) : CUtensorMap{};
  // Default for CTA pairs without a residual plane and N > 128: 256-column tiles on
  // decoupled operand rings with three epilogue warp groups (gemm_i8_bits_fwd_dec_kernel
  // <256, 2, NQ 2, NX 2, MS 1, EG 3>): x is expanded once per M tile, the N = 256 MMAs
  // read fewer operand bytes per product, and twelve epilogue warps shorten the drain
  // the single-buffered accumulators expose (C3: 0.157 vs 0.188 ms).  TLG_I8_DEC selects
  // the variants measured against it: 0 = coupled stages,
  // 4x3 = decoupled rings at 128 columns, m2e = two M subtiles per CTA, b256 / b256e =
  // one / two epilogue groups.
  int dec = cg == 2 && mc == 1 && out_lo == nullptr && N > 128 && !std::getenv("TLG_I8_BN")
                ? 259 : 0;
  if (const char* e = std::getenv("TLG_I8_DEC"); e && dec != 0)
    dec = std::strcmp(e, "4x3") == 0 ? 43 : std::strcmp(e, "m2e") == 0 ? 3
        : std::strcmp(e, "b256") == 0 ? 256 : std::strcmp(e, "b256e") == 0 ? 257
        : std::strcmp(e, "0") == 0 ? 0 : 259;
  if (dec == 3) {
    // two 128-row M subtiles per CTA share each weight-piece tile (half the L2 -> SM
    // piece traffic per output), accumulators single-buffered
    const TileMap tm2{ceil_div(M, kBM * 2 * 2), ceil_div(N, BN), 1};
    const CUtensorMap tb2 = make_bytes_map(bits, rowb, M, rowb, kBKi / 8, 2 * kBM, CU_TENSOR_MAP_SWIZZLE_NONE);
    run_i8_fwd_dec<128, 2, 2, 2, 2, 2>(tb2, tq, to, tl, p, tm2, stream);
    return {BN, 2 * std::min(tm2.m_tiles * tm2.n_tiles, num_sms() / 2), tm2.n_tiles};
  }
  if (dec == 256 || dec == 257 || dec == 259) {
    const TileMap tmw{ceil_div(M, kBM * 2), ceil_div(N, 256), 1};
    const CUtensorMap tqw = make_bytes_map(q, Kp, 3L * N, Kp, kBKi, 128, CU_TENSOR_MAP_SWIZZLE_128B);
    if (dec == 259) run_i8_fwd_dec<256, 2, 2, 2, 1, 3>(tb, tqw, to, tl, p, tmw, stream);
    else if (dec == 257) run_i8_fwd_dec<256, 2, 2, 2, 1, 2>(tb, tqw, to, tl, p, tmw, stream);
    else run_i8_fwd_dec<256, 2, 2, 2>(tb, tqw, to, tl, p, tmw, stream);
    return {256, 2 * std::min(tmw.m_tiles * tmw.n_tiles, num_sms() / 2), tmw.n_tiles};
  }
  if (dec == 43) run_i8_fwd_dec<128, 2, 4, 3>(tb, tq, to, tl, p, tm, stream);
  else if (BN == 256) run_i8_fwd<256, 2>(tb, tq, to, tl, p, tm, stream);
  else if (mc == 2) run_i8_fwd<128, 2, 2>(tb, tq, to, tl, p, tm, stream);
  else if (cg == 2) run_i8_fwd<128, 2>(tb, tq, to, tl, p, tm, stream);
  else run_i8_fwd<128, 1>(tb, tq, to, tl, p, tm, stream);
  const int tiles = tm.m_tiles * tm.n_tiles;
  const int cl = cg * mc;
  return {BN, cl * std::min(tiles, num_sms() / cl), tm.n_tiles};  // ctas: an upper bound
}

}  // namespace tlg::gemm
