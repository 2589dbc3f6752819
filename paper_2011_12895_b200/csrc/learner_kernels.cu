// Non-GEMM kernels of the B200 learner step (see learner_kernels.cuh).
#include <cmath>
#include <cstdlib>

#include "learner_kernels.cuh"

namespace tlg {

namespace {

constexpr int kMaxA1Limit = 32;  // n_actions + 1 (value) supported by the head kernels

__device__ __forceinline__ bool frame_valid(const BatchDev* b, long f, int* t_out = nullptr) {
  if (b == nullptr) return true;
  const int s = int(f / b->T), t = int(f % b->T);
  if (t_out) *t_out = t;
  return t < b->valid[s];
}

// ---------------------------------------------------------------------------
__global__ void expand_u8_kernel(const uchar4* __restrict__ in, float4* __restrict__ out, long n4) {
  TLG_PDL_ENTRY();
  for (long i = blockIdx.x * long(blockDim.x) + threadIdx.x; i < n4; i += long(gridDim.x) * blockDim.x) {
    const uchar4 u = in[i];
    out[i] = make_float4(u.x, u.y, u.z, u.w);
  }
}

// Bit rows of rowb bytes -> rows of `pitch` bytes (zero padded).  A block stages
// kRepitchRows consecutive rows through shared memory with aligned 16-byte loads (the
// source rows are only 2-byte aligned in general), then writes 16-byte chunks.
constexpr int kRepitchRows = 64;
__global__ void __launch_bounds__(256) repitch_bits_kernel(const uint8_t* __restrict__ bits,
                                                           long rowb, long F,
                                                           uint8_t* __restrict__ out, long pitch) {
  TLG_PDL_ENTRY();
  extern __shared__ uint4 rp_smem[];
  uint8_t* sb = reinterpret_cast<uint8_t*>(rp_smem);
  const long f0 = long(blockIdx.x) * kRepitchRows;
  const int rows = int(F - f0 < kRepitchRows ? F - f0 : long(kRepitchRows));
  const uint8_t* src = bits + f0 * rowb;
  const uintptr_t a0 = reinterpret_cast<uintptr_t>(src) & ~uintptr_t(15);
  const int lead = int(reinterpret_cast<uintptr_t>(src) - a0);
  const int n16 = (lead + rows * int(rowb) + 15) / 16;
  // (the aligned 16-byte chunks stay inside the allocation's 256-byte granules)
  for (int i = threadIdx.x; i < n16; i += blockDim.x)
    rp_smem[i] = __ldg(reinterpret_cast<const uint4*>(a0) + i);
  __syncthreads();
  const int per_row = int(pitch / 16);
  for (int i = threadIdx.x; i < rows * per_row; i += blockDim.x) {
    const int r = i / per_row, j = (i % per_row) * 16;
    uint32_t w[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      uint32_t v = 0;
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        const int col = j + 4 * q + b;
        if (col < rowb) v |= uint32_t(sb[lead + r * int(rowb) + col]) << (8 * b);
      }
      w[q] = v;
    }
    *reinterpret_cast<uint4*>(out + (f0 + r) * pitch + j) = make_uint4(w[0], w[1], w[2], w[3]);
  }
}

// Bit-packed 0/1 observation planes -> uint8 (one thread per packed byte); optionally
// also the same bit rows re-pitched to `pitch` bytes (16-B aligned rows for TMA).
__global__ void unpack_bits_kernel(const uint8_t* __restrict__ bits, long rowb, long F, long D,
                                   uint8_t* __restrict__ out, uint8_t* __restrict__ pitched,
                                   long pitch) {
  TLG_PDL_ENTRY();
  for (long i = blockIdx.x * long(blockDim.x) + threadIdx.x; i < F * rowb;
       i += long(gridDim.x) * blockDim.x) {
    const long f = i / rowb, j = i % rowb;
    const uint32_t v = bits[i];
    if (pitched) pitched[f * pitch + j] = uint8_t(v);
    if (!out) continue;
    uint8_t* o = out + f * D + 8 * j;
    if (8 * j + 8 <= D && ((reinterpret_cast<uintptr_t>(o) & 7) == 0)) {
      uint2 w;
      w.x = (v & 1u) | ((v >> 1) & 1u) << 8 | ((v >> 2) & 1u) << 16 | ((v >> 3) & 1u) << 24;
      w.y = ((v >> 4) & 1u) | ((v >> 5) & 1u) << 8 | ((v >> 6) & 1u) << 16 | ((v >> 7) & 1u) << 24;
      *reinterpret_cast<uint2*>(o) = w;
    } else {
      for (int q = 0; q < 8 && 8 * j + q < D; ++q) o[q] = (v >> q) & 1u;
    }
  }
}

__global__ void split_lo_kernel(const float4* __restrict__ x, float4* __restrict__ lo, long n4) {
  TLG_PDL_ENTRY();
  for (long i = blockIdx.x * long(blockDim.x) + threadIdx.x; i < n4; i += long(gridDim.x) * blockDim.x) {
    const float4 v = x[i];
    lo[i] = make_float4(v.x - tf32_hi(v.x), v.y - tf32_hi(v.y), v.z - tf32_hi(v.z),
                        v.w - tf32_hi(v.w));
  }
}

// ---------------------------------------------------------------------------
// K3a: one warp per frame.  Distribution + ValueEstimate (policy.cpp:73-105) with a
// max-shifted log-sum-exp; writes logits+value [F x (A+1)], the log-prob of the
// taken action (V-trace target logp, learner.cpp:80-84) and optionally probs.
template <int kMaxA1>
__global__ void __launch_bounds__(256) head_forward_kernel(HeadDesc hd, const float* __restrict__ params,
                                                         const float* __restrict__ h, long ldh,
                                                         BatchDev bd, int has_batch, long F,
                                                         float* __restrict__ head_out,
                                                         float* __restrict__ tlogp,
                                                         float* __restrict__ probs_out,
                                                         int* __restrict__ err) {
  TLG_PDL_ENTRY();
  const BatchDev* b = has_batch ? &bd : nullptr;
  const int lane = threadIdx.x & 31;
  const long warps = long(gridDim.x) * (blockDim.x >> 5);
  const int A = hd.A, A1 = hd.A + 1;
  for (long f = blockIdx.x * long(blockDim.x >> 5) + (threadIdx.x >> 5); f < F; f += warps) {
    if (!frame_valid(b, f)) {
      if (lane < A1) head_out[f * A1 + lane] = 0.f;
      if (lane == 0 && tlogp) tlogp[f] = 0.f;
      continue;
    }
    const float* hr = h + f * ldh;
    float acc[kMaxA1];
#pragma unroll
    for (int k = 0; k < kMaxA1; ++k) acc[k] = 0.f;
    int ones = 0, others = 0;
    for (int j = lane; j < hd.H; j += 32) {
      const float x = hr[j];
      if (hd.family == 0) {
        if (x == 1.f) { ++ones; } else if (x != 0.f) { ++others; }
      }
      const float* w = params + hd.wpi + long(j) * hd.wj;
#pragma unroll
      for (int k = 0; k < kMaxA1 - 1; ++k)
        if (k < A) acc[k] = fmaf(__ldg(w + long(k) * hd.wk), x, acc[k]);
      acc[kMaxA1 - 1] = fmaf(__ldg(params + hd.wv + j), x, acc[kMaxA1 - 1]);
    }
#pragma unroll
    for (int k = 0; k < kMaxA1; ++k)
      if (k < A || k == kMaxA1 - 1) acc[k] = warp_sum(acc[k]);
    if (hd.family == 0) {
      ones = __reduce_add_sync(0xffffffffu, ones);
      others = __reduce_add_sync(0xffffffffu, others);
      if (ones != 1 || others != 0) {
        if (lane == 0) atomicOr(err, kErrNotOneHot);
      }
    }
    if (lane == 0) {
      float z[kMaxA1];
      float mx = -INFINITY;
#pragma unroll
      for (int k = 0; k < kMaxA1 - 1; ++k)
        if (k < A) {
          z[k] = acc[k] + (hd.bpi >= 0 ? params[hd.bpi + k] : 0.f);
          mx = fmaxf(mx, z[k]);
        }
      float se = 0.f;
#pragma unroll
      for (int k = 0; k < kMaxA1 - 1; ++k)
        if (k < A) se += expf(z[k] - mx);
      const float lse = mx + logf(se);
      const float v = acc[kMaxA1 - 1] + (hd.bv >= 0 ? params[hd.bv] : 0.f);
#pragma unroll
      for (int k = 0; k < kMaxA1 - 1; ++k)
        if (k < A) {
          head_out[f * A1 + k] = z[k];
          if (probs_out) probs_out[f * A + k] = expf(z[k] - lse);
        }
      head_out[f * A1 + A] = v;
      if (b) {
        const int a = b->action[f];
        if (a < 0 || a >= A) {
          atomicOr(err, kErrActionRange);
          if (tlogp) tlogp[f] = 0.f;
        } else if (tlogp) {
          float za = 0.f;
#pragma unroll
          for (int k = 0; k < kMaxA1 - 1; ++k)
            if (k == a) za = z[k];
          tlogp[f] = za - lse;
        }
      }
    }
  }
}

// K3a (fused form): the last trunk GEMM's epilogue left per-N-tile partial head dot
// products; add them in tile order, add the biases, log-softmax.  Thread per frame.
__global__ void head_finalize_kernel(HeadDesc hd, const float* __restrict__ params,
                                     const float* __restrict__ part, int n_tiles, long F,
                                     long part_rows, BatchDev bd, int has_batch, float* __restrict__ head_out,
                                     float* __restrict__ tlogp, float* __restrict__ logits_out,
                                     float* __restrict__ probs_out, float* __restrict__ value_out,
                                     int* __restrict__ err) {
  TLG_PDL_ENTRY();
  const long f = blockIdx.x * long(blockDim.x) + threadIdx.x;
  if (f >= F) return;
  const int A = hd.A, A1 = A + 1;
  const BatchDev* b = has_batch ? &bd : nullptr;
  if (!frame_valid(b, f)) {
    for (int k = 0; k < A1; ++k) head_out[f * A1 + k] = 0.f;
    if (tlogp) tlogp[f] = 0.f;
    return;
  }
  float z[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    if (k < A1) {
      float acc = 0.f;
      for (int t = 0; t < n_tiles; ++t) acc += part[(long(t) * part_rows + f) * A1 + k];
      const long boff = k < A ? (hd.bpi >= 0 ? hd.bpi + k : -1) : hd.bv;
      z[k] = acc + (boff >= 0 ? params[boff] : 0.f);
    }
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
#pragma unroll
  for (int k = 0; k < 8; ++k)
    if (k < A1) {
      if (head_out) head_out[f * A1 + k] = z[k];
      if (k < A) {
        if (logits_out) logits_out[f * A + k] = z[k];
        if (probs_out) probs_out[f * A + k] = expf(z[k] - lse);
      }
    }
  if (value_out) value_out[f] = z[A < 8 ? A : 7];
  if (b) {
    const int a = b->action[f];
    if (a < 0 || a >= A) {
      atomicOr(err, kErrActionRange);
      if (tlogp) tlogp[f] = 0.f;
    } else if (tlogp) {
      float za = 0.f;
#pragma unroll
      for (int k = 0; k < 8; ++k)
        if (k == a) za = z[k];
      tlogp[f] = za - lse;
    }
  }
}

// ---------------------------------------------------------------------------
// K1: one warp per segment; lanes cover 32 consecutive steps, blocks of 32 steps are
// processed from the end so every warp load/store is one coalesced 128-B row slice.
// Each recursion x_t = a_t x_{t+1} + b_t is a suffix scan of affine maps.
struct Aff {
  float a, b;
};

__device__ __forceinline__ Aff suffix_scan(Aff m, int lane) {
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const float a2 = __shfl_down_sync(0xffffffffu, m.a, d);
    const float b2 = __shfl_down_sync(0xffffffffu, m.b, d);
    if (lane + d < 32) {
      m.b = fmaf(m.a, b2, m.b);
      m.a = m.a * a2;
    }
  }
  return m;
}

// 8 segments (one per warp) per block; the block writes one partial of the adv statistics
constexpr int kRetSegsPerBlock = 8;

__global__ void __launch_bounds__(256) returns_kernel(BatchDev b, int algo, HyperDev hp,
                                                      const float* __restrict__ tlogp,
                                                      float* __restrict__ adv,
                                                      float* __restrict__ target,
                                                      double* __restrict__ seg_partial,
                                                      int* __restrict__ err) {
  TLG_PDL_ENTRY();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int s = blockIdx.x * kRetSegsPerBlock + w;
  double s1 = 0.0, s2 = 0.0;
  int nv = 0;
  if (s < b.S) {
    const int T = b.T;
    int n = b.valid[s];
    if (n > T || n < 0) {
      if (lane == 0) atomicOr(err, kErrValidSteps);
      n = min(max(n, 0), T);
    }
    const long base = long(s) * T;
    const float boot = b.boot[s];
    nv = n;
    const float g = hp.gamma, gl = hp.gamma * hp.lam;
    const int nblk = (T + 31) / 32;
    // carries from the block after the current one (t = (jb+1)*32)
    float carry_v = boot;    // V_{t+1} for lane 31 (bootstrap when t+1 >= n)
    float carry_x = 0.f;     // GAE A / V-trace u at the block start after
    float carry_g = boot;    // lambda-return G
    float carry_vs = boot;   // V-trace vs_{t+1}
    bool bad_adv = false, bad_logp = false;
    for (int jb = nblk - 1; jb >= 0; --jb) {
      const int t = jb * 32 + lane;
      const bool in = t < n;
      const long f = base + t;
      // the row loads depend only on T, not on valid_steps: all of a warp's loads are in
      // flight together (the valid_steps load no longer serialises them); padding masked after
      float r = 0.f, v = 0.f, bl = 0.f, tl = 0.f;
      uint8_t dn = 0;
      if (t < T) {
        r = b.reward[f];
        v = b.value[f];
        dn = b.done[f];
        if (algo != kAlgoPpo) {
          bl = b.blogp[f];
          tl = tlogp[f];
        }
      }
      r = in ? r : 0.f;
      v = in ? v : 0.f;
      const float nt = (in && dn) ? 0.f : 1.f;
      float v_next = __shfl_down_sync(0xffffffffu, v, 1);
      if (lane == 31) v_next = carry_v;
      if (t + 1 >= n) v_next = boot;
      if (algo == kAlgoPpo) {
        // GaeAdvantages (rlmath.cpp:62-78) and LambdaReturn (:45-60)
        Aff ma{in ? gl * nt : 0.f, in ? (r + g * nt * v_next - v) : 0.f};
        Aff mg{in ? gl * nt : 0.f, in ? (r + g * nt * (1.f - hp.lam) * v_next) : boot};
        ma = suffix_scan(ma, lane);
        mg = suffix_scan(mg, lane);
        const float A_t = fmaf(ma.a, carry_x, ma.b);
        const float G_t = fmaf(mg.a, carry_g, mg.b);
        if (t < T) {
          adv[f] = in ? A_t : 0.f;
          target[f] = in ? G_t : 0.f;
        }
        if (in) {
          bad_adv |= !isfinite(A_t);
          s1 += double(A_t);
          s2 += double(A_t) * double(A_t);
        }
        carry_x = __shfl_sync(0xffffffffu, A_t, 0);
        carry_g = __shfl_sync(0xffffffffu, G_t, 0);
      } else {
        // VtraceTargets (rlmath.cpp:80-114): truncated importance weights fused in
        float rho = 0.f, c = 0.f;
        if (in) {
          if (!isfinite(bl) || !isfinite(tl)) bad_logp = true;
          const float w = expf(tl - bl);
          rho = fminf(hp.rho_bar, w);
          c = fminf(hp.c_bar, w);
        }
        const float delta = rho * (r + g * nt * v_next - v);
        Aff mu{in ? g * nt * c : 0.f, in ? delta : 0.f};
        mu = suffix_scan(mu, lane);
        const float u = fmaf(mu.a, carry_x, mu.b);
        const float vs = v + u;
        float vs_next = __shfl_down_sync(0xffffffffu, vs, 1);
        if (lane == 31) vs_next = carry_vs;
        if (t + 1 >= n) vs_next = boot;
        const float pg = rho * (r + g * nt * vs_next - v);
        if (t < T) {
          adv[f] = in ? pg : 0.f;
          target[f] = in ? vs : 0.f;
        }
        if (in) {
          bad_adv |= !isfinite(pg);
          s1 += double(pg);
          s2 += double(pg) * double(pg);
        }
        carry_x = __shfl_sync(0xffffffffu, u, 0);
        carry_vs = __shfl_sync(0xffffffffu, vs, 0);
      }
      carry_v = __shfl_sync(0xffffffffu, v, 0);
    }
    s1 = warp_sum(s1);
    s2 = warp_sum(s2);
    const unsigned anybad = __ballot_sync(0xffffffffu, bad_adv);
    const unsigned anylogp = __ballot_sync(0xffffffffu, bad_logp);
    if (lane == 0) {
      if (anylogp) atomicOr(err, kErrNonFiniteLogp);
      if (anybad) atomicOr(err, kErrNonFiniteAdv);
    }
  }
  // per-block partial {sum A, sum A^2, valid frames}, warps added in fixed order, so the
  // statistics pass reads S/8 partials instead of S (and no valid_steps)
  __shared__ double red[3][kRetSegsPerBlock];
  if (lane == 0) {
    red[0][w] = s1;
    red[1][w] = s2;
    red[2][w] = double(nv);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0.0, c = 0.0, m = 0.0;
    for (int i = 0; i < kRetSegsPerBlock; ++i) { a += red[0][i]; c += red[1][i]; m += red[2][i]; }
    seg_partial[3 * blockIdx.x] = a;
    seg_partial[3 * blockIdx.x + 1] = c;
    seg_partial[3 * blockIdx.x + 2] = m;
  }
}

// K1, vectorised (T % 4 == 0, 16-B aligned rows): 8 lanes per segment, 4 consecutive steps
// per lane (float4 / uchar4 loads and stores), so a warp instruction covers 128 frames.
// Each lane composes its 4 steps' affine maps serially, the 8 lanes of a segment suffix-scan
// the composites (3 shuffle rounds), then each lane expands its 4 values backwards.  Same
// recursions and masking as returns_kernel (rlmath.cpp:45-114), fewer instructions per
// frame: the scalar kernel was issue-bound at ~20 % of HBM bandwidth once the data streams.
constexpr int kRetVecSegsPerBlock = 32;  // 8 warps x 4 segments

struct Aff4 {
  float a[4], b[4];
};

// lane composite of its 4 maps (x_t = a_t x_{t+1} + b_t), suffix scan over the segment's
// 8 lanes; returns x at the lane's first step and at the step after its last (x_next)
__device__ __forceinline__ float scan4(const Aff4& m, float carry, float& x_next) {
  float A = m.a[3], B = m.b[3];
#pragma unroll
  for (int q = 2; q >= 0; --q) {
    B = fmaf(m.a[q], B, m.b[q]);
    A = m.a[q] * A;
  }
  const int j = threadIdx.x & 7;
#pragma unroll
  for (int d = 1; d < 8; d <<= 1) {
    const float a2 = __shfl_down_sync(0xffffffffu, A, d, 8);
    const float b2 = __shfl_down_sync(0xffffffffu, B, d, 8);
    if (j + d < 8) {
      B = fmaf(A, b2, B);
      A = A * a2;
    }
  }
  const float x0 = fmaf(A, carry, B);
  float xn = __shfl_down_sync(0xffffffffu, x0, 1, 8);
  if (j == 7) xn = carry;
  x_next = xn;
  return x0;
}

// Each lane has only ~36-52 B of loads in flight (one chunk at T=32), so bytes in flight per
// SM scale with resident CTAs: PPO is capped at 32 registers (8 CTAs/SM, 20 B spilled to L1),
// V-trace at 40 (6 CTAs/SM).  At 1 M segments (>= 4x L2) this took the kernel from 157 to
// 114 us (PPO) and 180 to 159 us (V-trace) in ncu (profiles/r01_k1_occupancy.md).
template <int kAlgo>
__global__ void __launch_bounds__(256, kAlgo == kAlgoPpo ? 8 : 6) returns_vec_kernel(BatchDev b, HyperDev hp,
                                                          const float* __restrict__ tlogp,
                                                          float* __restrict__ adv,
                                                          float* __restrict__ target,
                                                          double* __restrict__ seg_partial,
                                                          int* __restrict__ err) {
  TLG_PDL_ENTRY();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, j = lane & 7;
  const int s = blockIdx.x * kRetVecSegsPerBlock + w * 4 + (lane >> 3);
  const bool active = s < b.S;
  const int T = b.T;
  int n = 0;
  float boot = 0.f;
  if (active) {
    n = b.valid[s];
    boot = b.boot[s];
    if (n > T || n < 0) {
      if (j == 0) atomicOr(err, kErrValidSteps);
      n = min(max(n, 0), T);
    }
  }
  const long base = long(s) * T;
  const float g = hp.gamma, gl = hp.gamma * hp.lam;
  const int nchunk = (T + 31) / 32;
  float carry_v = boot, carry_x = 0.f, carry_g = boot, carry_vs = boot;
  double s1 = 0.0, s2 = 0.0;
  bool bad_adv = false, bad_logp = false;
  for (int c = nchunk - 1; c >= 0; --c) {
    const int t0 = c * 32 + j * 4;
    const bool row = active && t0 < T;
    float r[4] = {0.f, 0.f, 0.f, 0.f}, v[4] = {0.f, 0.f, 0.f, 0.f};
    float bl[4] = {0.f, 0.f, 0.f, 0.f}, tl[4] = {0.f, 0.f, 0.f, 0.f};
    uchar4 dn = make_uchar4(0, 0, 0, 0);
    if (row) {
      const float4 r4 = *reinterpret_cast<const float4*>(b.reward + base + t0);
      const float4 v4 = *reinterpret_cast<const float4*>(b.value + base + t0);
      dn = *reinterpret_cast<const uchar4*>(b.done + base + t0);
      r[0] = r4.x; r[1] = r4.y; r[2] = r4.z; r[3] = r4.w;
      v[0] = v4.x; v[1] = v4.y; v[2] = v4.z; v[3] = v4.w;
      if (kAlgo != kAlgoPpo) {
        const float4 b4 = *reinterpret_cast<const float4*>(b.blogp + base + t0);
        const float4 l4 = *reinterpret_cast<const float4*>(tlogp + base + t0);
        bl[0] = b4.x; bl[1] = b4.y; bl[2] = b4.z; bl[3] = b4.w;
        tl[0] = l4.x; tl[1] = l4.y; tl[2] = l4.z; tl[3] = l4.w;
      }
    }
    const unsigned char dd[4] = {dn.x, dn.y, dn.z, dn.w};
    bool in[4];
    float nt[4], vn[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      in[q] = t0 + q < n;
      r[q] = in[q] ? r[q] : 0.f;
      v[q] = in[q] ? v[q] : 0.f;
      nt[q] = (in[q] && dd[q]) ? 0.f : 1.f;
    }
    // V_{t+1}: within the lane, then the next lane's first value, then the next chunk's
    float v_after = __shfl_down_sync(0xffffffffu, v[0], 1, 8);
    if (j == 7) v_after = carry_v;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      vn[q] = q < 3 ? v[q + 1] : v_after;
      if (t0 + q + 1 >= n) vn[q] = boot;
    }
    float out_a[4], out_t[4];
    if constexpr (kAlgo == kAlgoPpo) {
      // GaeAdvantages (rlmath.cpp:62-78) and LambdaReturn (:45-60)
      Aff4 ma, mg;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        ma.a[q] = in[q] ? gl * nt[q] : 0.f;
        ma.b[q] = in[q] ? (r[q] + g * nt[q] * vn[q] - v[q]) : 0.f;
        mg.a[q] = ma.a[q];
        mg.b[q] = in[q] ? (r[q] + g * nt[q] * (1.f - hp.lam) * vn[q]) : boot;
      }
      float xa, xg;
      const float a0 = scan4(ma, carry_x, xa);
      const float g0 = scan4(mg, carry_g, xg);
#pragma unroll
      for (int q = 3; q >= 0; --q) {
        xa = fmaf(ma.a[q], xa, ma.b[q]);
        xg = fmaf(mg.a[q], xg, mg.b[q]);
        out_a[q] = in[q] ? xa : 0.f;
        out_t[q] = in[q] ? xg : 0.f;
        if (in[q]) {
          bad_adv |= !isfinite(xa);
          s1 += double(xa);
          s2 += double(xa) * double(xa);
        }
      }
      carry_x = __shfl_sync(0xffffffffu, a0, 0, 8);
      carry_g = __shfl_sync(0xffffffffu, g0, 0, 8);
    } else {
      // VtraceTargets (rlmath.cpp:80-114): truncated importance weights fused in
      Aff4 mu;
      float rho[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        float rh = 0.f, cc = 0.f;
        if (in[q]) {
          if (!isfinite(bl[q]) || !isfinite(tl[q])) bad_logp = true;
          const float wq = expf(tl[q] - bl[q]);
          rh = fminf(hp.rho_bar, wq);
          cc = fminf(hp.c_bar, wq);
        }
        rho[q] = rh;
        mu.a[q] = in[q] ? g * nt[q] * cc : 0.f;
        mu.b[q] = in[q] ? rh * (r[q] + g * nt[q] * vn[q] - v[q]) : 0.f;
      }
      float xu;
      const float u0 = scan4(mu, carry_x, xu);
      float vs[4];
#pragma unroll
      for (int q = 3; q >= 0; --q) {
        xu = fmaf(mu.a[q], xu, mu.b[q]);
        vs[q] = v[q] + xu;
      }
      float vs_after = __shfl_down_sync(0xffffffffu, vs[0], 1, 8);
      if (j == 7) vs_after = carry_vs;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        float vsn = q < 3 ? vs[q + 1] : vs_after;
        if (t0 + q + 1 >= n) vsn = boot;
        const float pg = rho[q] * (r[q] + g * nt[q] * vsn - v[q]);
        out_a[q] = in[q] ? pg : 0.f;
        out_t[q] = in[q] ? vs[q] : 0.f;
        if (in[q]) {
          bad_adv |= !isfinite(pg);
          s1 += double(pg);
          s2 += double(pg) * double(pg);
        }
      }
      carry_x = __shfl_sync(0xffffffffu, u0, 0, 8);
      carry_vs = __shfl_sync(0xffffffffu, vs[0], 0, 8);
    }
    if (row) {
      *reinterpret_cast<float4*>(adv + base + t0) = make_float4(out_a[0], out_a[1], out_a[2], out_a[3]);
      *reinterpret_cast<float4*>(target + base + t0) = make_float4(out_t[0], out_t[1], out_t[2], out_t[3]);
    }
    carry_v = __shfl_sync(0xffffffffu, v[0], 0, 8);
  }
  s1 = warp_sum(s1);
  s2 = warp_sum(s2);
  int nv = j == 0 ? n : 0;
  for (int o = 16; o > 0; o >>= 1) nv += __shfl_xor_sync(0xffffffffu, nv, o);
  const unsigned anybad = __ballot_sync(0xffffffffu, bad_adv);
  const unsigned anylogp = __ballot_sync(0xffffffffu, bad_logp);
  __shared__ double red[3][8];
  if (lane == 0) {
    if (anylogp) atomicOr(err, kErrNonFiniteLogp);
    if (anybad) atomicOr(err, kErrNonFiniteAdv);
    red[0][w] = s1;
    red[1][w] = s2;
    red[2][w] = double(nv);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0.0, c = 0.0, m = 0.0;
    for (int i = 0; i < 8; ++i) { a += red[0][i]; c += red[1][i]; m += red[2][i]; }
    seg_partial[3 * blockIdx.x] = a;
    seg_partial[3 * blockIdx.x + 1] = c;
    seg_partial[3 * blockIdx.x + 2] = m;
  }
}

// EffectiveAdvantages statistics (rlmath.cpp:18-34), fixed-order fp64 reduction.
__global__ void __launch_bounds__(1024) finalize_adv_kernel(const double* __restrict__ seg_partial,
                                                            BatchDev b, int adv_norm,
                                                            StepStatsDev* st, int* err,
                                                            int segs_per_block) {
  TLG_PDL_ENTRY();
  __shared__ double sh1[32], sh2[32];
  __shared__ long long shn[32];
  double s1 = 0.0, s2 = 0.0;
  long long n = 0;
  const int nblk = (b.S + segs_per_block - 1) / segs_per_block;
  for (int i = threadIdx.x; i < nblk; i += blockDim.x) {
    s1 += seg_partial[3 * i];
    s2 += seg_partial[3 * i + 1];
    n += (long long)seg_partial[3 * i + 2];
  }
  s1 = warp_sum(s1);
  s2 = warp_sum(s2);
  for (int o = 16; o > 0; o >>= 1) n += __shfl_xor_sync(0xffffffffu, n, o);
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) { sh1[w] = s1; sh2[w] = s2; shn[w] = n; }
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0.0, c = 0.0;
    long long nn = 0;
    for (int i = 0; i < int(blockDim.x >> 5); ++i) { a += sh1[i]; c += sh2[i]; nn += shn[i]; }
    st->sum_adv = a;
    st->sum_adv2 = c;
    st->n = nn;
    if (nn == 0) {
      atomicOr(err, kErrEmptyBatch);
      st->inv_n = 0.0; st->mean = 0.0; st->sd = 1.0;
      return;
    }
    st->inv_n = 1.0 / double(nn);
    if (adv_norm && nn >= 2) {
      const double mean = a / double(nn);
      double var = c / double(nn) - mean * mean;
      if (var < 0.0) var = 0.0;
      st->mean = mean;
      st->sd = fmax(sqrt(var), 1e-8);
    } else {
      st->mean = 0.0;
      st->sd = 1.0;
    }
  }
}

// ---------------------------------------------------------------------------
// K3b, part 1 (thread per frame): the per-sample PPO / PG body (rlmath.cpp:129-182 /
// 196-220) -> dlogits, dvalue [F][A1]; per-block fp64 loss/stat sums and per-block
// bias-gradient sums (fixed-order warp trees).
// kParts: the logits come straight from the fused-head partial sums of the last trunk
// GEMM (head_finalize_kernel skipped: PPO needs no target log-prob), and the action range
// check (rlmath.cpp:133) happens here.  kKL: teacher KL term compiled in.
template <int kMaxA1, bool kKL, bool kParts>
__global__ void __launch_bounds__(256) loss_math_kernel(
    HeadDesc hd, BatchDev b, const float* __restrict__ head_out, const float* __restrict__ adv,
    const float* __restrict__ target, const StepStatsDev* __restrict__ st, HyperDev hp,
    int loss_kind, float* __restrict__ dzh, double* __restrict__ loss_partial,
    float* __restrict__ bias_partial, const float* __restrict__ teacher_out, int n_tiles,
    const float* __restrict__ params, int* __restrict__ err) {
  TLG_PDL_ENTRY();
  __shared__ double red[5][8];
  __shared__ float bred[kMaxA1][8];
  const int A = hd.A, A1 = A + 1;
  const long F = long(b.S) * b.T;
  const long f = blockIdx.x * long(blockDim.x) + threadIdx.x;
  const float inv_n = float(st->inv_n);
  const double mean = st->mean, sd = st->sd;
  float d[kMaxA1];
#pragma unroll
  for (int k = 0; k < kMaxA1; ++k) d[k] = 0.f;
  double l_loss = 0, l_ratio = 0, l_ent = 0, l_vl = 0, l_clip = 0;
  bool valid = false;
  if (f < F) {
    const int s = int(f / b.T), t = int(f % b.T);
    valid = t < b.valid[s];
  }
  if (valid) {
    float z[kMaxA1];
    if (kParts) {
#pragma unroll
      for (int k = 0; k < kMaxA1; ++k) {
        float acc = 0.f;
        if (k < A1) {
          for (int t = 0; t < n_tiles; ++t) acc += head_out[(long(t) * F + f) * A1 + k];
          const long boff = k < A ? (hd.bpi >= 0 ? hd.bpi + k : -1) : hd.bv;
          if (boff >= 0) acc += params[boff];
        }
        z[k] = acc;
      }
      const int ar = b.action[f];
      if (ar < 0 || ar >= A) atomicOr(err, kErrActionRange);
    } else {
#pragma unroll
      for (int k = 0; k < kMaxA1; ++k) z[k] = k < A1 ? head_out[f * A1 + k] : 0.f;
    }
    float mx = -INFINITY;
#pragma unroll
    for (int k = 0; k < kMaxA1; ++k)
      if (k < A) mx = fmaxf(mx, z[k]);
    float se = 0.f;
#pragma unroll
    for (int k = 0; k < kMaxA1; ++k)
      if (k < A) se += expf(z[k] - mx);
    const float lse = mx + logf(se);
    float pk[kMaxA1], lpk[kMaxA1];
    float ent = 0.f;
#pragma unroll
    for (int k = 0; k < kMaxA1; ++k) {
      lpk[k] = z[k] - lse;
      pk[k] = k < A ? expf(lpk[k]) : 0.f;
      if (k < A && pk[k] > 0.f) ent -= pk[k] * lpk[k];  // Entropy (rlmath.cpp:36-41)
    }
    const int a = min(max(b.action[f], 0), A - 1);  // out-of-range is flagged by K3a
    // teacher KL (rlmath.cpp:145-155, 177-178): KL(p || q) with q the teacher's policy
    float lq[kMaxA1], kl = 0.f;
    const bool kl_on = kKL && loss_kind == 0 && teacher_out != nullptr;
    if (kl_on) {
      float tz[kMaxA1];
#pragma unroll
      for (int k = 0; k < kMaxA1; ++k) tz[k] = k < A ? teacher_out[f * A1 + k] : 0.f;
      float tmx = -INFINITY;
#pragma unroll
      for (int k = 0; k < kMaxA1; ++k)
        if (k < A) tmx = fmaxf(tmx, tz[k]);
      float tse = 0.f;
#pragma unroll
      for (int k = 0; k < kMaxA1; ++k)
        if (k < A) tse += expf(tz[k] - tmx);
      const float tlse = tmx + logf(tse);
#pragma unroll
      for (int k = 0; k < kMaxA1; ++k) {
        lq[k] = tz[k] - tlse;
        if (k < A && pk[k] > 0.f) kl += pk[k] * (lpk[k] - lq[k]);
      }
    }
    float logp = 0.f, V = 0.f;
#pragma unroll
    for (int k = 0; k < kMaxA1; ++k) {
      if (k == a) logp = lpk[k];
      if (k == A) V = z[k];
    }
    const float verr = V - target[f];
    const float ad = float((double(adv[f]) - mean) / sd);
    const float ratio = expf(logp - b.blogp[f]);
    float loss_i;
    if (loss_kind == 0) {
      const float clipped = fminf(fmaxf(ratio, 1.f - hp.clip_eps), 1.f + hp.clip_eps);
      const float t1 = ratio * ad, t2 = clipped * ad;
      loss_i = -fminf(t1, t2) + hp.vf_coef * verr * verr - hp.ent_coef * ent;
      if (kl_on) loss_i += hp.kl_coef * kl;
      if (t2 < t1) l_clip = 1.0;
      const bool surr = t1 <= t2;  // gradient only when the unclipped term is active
#pragma unroll
      for (int k = 0; k < kMaxA1; ++k)
        if (k < A) {
          const float lpz = pk[k] > 0.f ? lpk[k] : 0.f;
          float g = hp.ent_coef * pk[k] * (lpz + ent);
          if (surr) g += -ad * ratio * ((k == a ? 1.f : 0.f) - pk[k]);
          if (kl_on) g += hp.kl_coef * pk[k] * (lpz - lq[k] - kl);
          d[k] = g * inv_n;
        }
    } else {
      loss_i = -ad * logp + hp.vf_coef * verr * verr - hp.ent_coef * ent;
#pragma unroll
      for (int k = 0; k < kMaxA1; ++k)
        if (k < A)
          d[k] = (-ad * ((k == a ? 1.f : 0.f) - pk[k]) +
                  hp.ent_coef * pk[k] * ((pk[k] > 0.f ? lpk[k] : 0.f) + ent)) * inv_n;
    }
#pragma unroll
    for (int k = 0; k < kMaxA1; ++k)
      if (k == A) d[k] = 2.f * hp.vf_coef * verr * inv_n;
    l_loss = loss_i;
    l_ratio = ratio;
    l_ent = ent;
    l_vl = double(verr) * double(verr);
  }
  if (f < F) {
#pragma unroll
    for (int k = 0; k < kMaxA1; ++k)
      if (k < A1) dzh[f * A1 + k] = d[k];
  }
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double v[5] = {l_loss, l_ratio, l_ent, l_vl, l_clip};
#pragma unroll
  for (int q = 0; q < 5; ++q) {
    v[q] = warp_sum(v[q]);
    if (lane == 0) red[q][w] = v[q];
  }
#pragma unroll
  for (int k = 0; k < kMaxA1; ++k) {
    const float t = warp_sum(d[k]);
    if (lane == 0) bred[k][w] = t;
  }
  __syncthreads();
  if (threadIdx.x < 5) {
    double t = 0.0;
    for (int i = 0; i < 8; ++i) t += red[threadIdx.x][i];
    loss_partial[long(blockIdx.x) * 5 + threadIdx.x] = t;
  } else if (threadIdx.x >= 32 && threadIdx.x < 32 + A1) {
    const int k = threadIdx.x - 32;
    float t = 0.f;
    for (int i = 0; i < 8; ++i) t += bred[k][i];
    bias_partial[long(blockIdx.x) * A1 + k] = t;
  }
}

// K3b, part 2: persistent blocks of 256 threads stream chunks of kLossFrames frames
// (thread per head-input column j): dZ_L[f][j] = (sum_k dz_k W_pi[k][j] + dV w_v[j]) *
// (1 - h^2), the head weight gradient sum_f dz_k(f) h[f][j] (AccumulateGrad,
// policy.cpp:122-141) and the last layer's bias gradient sum_f dZ_L[f][j], accumulated in
// registers across the block's chunks; one partial row per block (fixed order).
template <int kMaxA1, int kCPT>
__global__ void __launch_bounds__(256) loss_stream_kernel(
    HeadDesc hd, const float* __restrict__ params, const float* __restrict__ h, long ldh,
    long F, const float* __restrict__ dzh, float* __restrict__ dz, float* __restrict__ dz_lo,
    float* __restrict__ hg_partial, float* __restrict__ db_partial) {
  TLG_PDL_ENTRY();
  extern __shared__ float sdz[];  // [kLossFrames][A1]
  const int A = hd.A, A1 = A + 1;
  const long nchunks = (F + kLossFrames - 1) / kLossFrames;
  const int tid = threadIdx.x;
  float acc[kCPT][kMaxA1];
  float dbacc[kCPT];
  float w[kCPT][kMaxA1];
#pragma unroll
  for (int c = 0; c < kCPT; ++c) {
    const int j = tid + 256 * c;
    dbacc[c] = 0.f;
#pragma unroll
    for (int k = 0; k < kMaxA1; ++k) {
      acc[c][k] = 0.f;
      float wk = 0.f;
      if (j < hd.H) {
        if (k < A) wk = __ldg(params + hd.wpi + long(k) * hd.wk + long(j) * hd.wj);
        else if (k == A) wk = __ldg(params + hd.wv + j);
      }
      w[c][k] = wk;
    }
  }
  for (long ch = blockIdx.x; ch < nchunks; ch += gridDim.x) {
    const long f0 = ch * kLossFrames;
    const int nf = int(F - f0 < long(kLossFrames) ? F - f0 : long(kLossFrames));
    for (int i = tid; i < nf * A1; i += blockDim.x) sdz[i] = dzh[f0 * A1 + i];
    __syncthreads();
#pragma unroll
    for (int c = 0; c < kCPT; ++c) {
      const int j = tid + 256 * c;
      if (j >= hd.H) continue;
      for (int i0 = 0; i0 < nf; i0 += 16) {
        // 16 independent coalesced loads in flight before the math
        float xs[16];
#pragma unroll
        for (int u = 0; u < 16; ++u)
          xs[u] = (i0 + u < nf) ? __ldg(h + (f0 + i0 + u) * ldh + j) : 0.f;
#pragma unroll
        for (int u = 0; u < 16; ++u) {
          if (i0 + u >= nf) break;
          const long f = f0 + i0 + u;
          const float x = xs[u];
          const float* d = sdz + (i0 + u) * A1;
          float dh = 0.f;
#pragma unroll
          for (int k = 0; k < kMaxA1; ++k)
            if (k <= A) {
              dh = fmaf(d[k], w[c][k], dh);
              acc[c][k] = fmaf(d[k], x, acc[c][k]);
            }
          if (dz) {
            const float o = dh * (1.f - x * x);
            dz[f * hd.H + j] = o;
            if (dz_lo) dz_lo[f * hd.H + j] = o - tf32_hi(o);
            dbacc[c] += o;
          }
        }
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int c = 0; c < kCPT; ++c) {
    const int j = tid + 256 * c;
    if (j >= hd.H) continue;
    float* out = hg_partial + long(blockIdx.x) * A1 * hd.H;
#pragma unroll
    for (int k = 0; k < kMaxA1; ++k)
      if (k <= A) out[long(k) * hd.H + j] = acc[c][k];
    if (dz) db_partial[long(blockIdx.x) * hd.H + j] = dbacc[c];
  }
}

// out[c] (+ scatter) = sum over rows r of partial[r*stride + c], in a fixed order:
// warp w of the block sums rows w, w+8, ... for 32 consecutive columns (lane = column,
// coalesced), then the 8 warp sums are added in warp order.  Deterministic.
// K3b, part 2, vectorised (A+1 <= 8, H % 4 == 0): a block owns a contiguous, balanced
// frame range and a slab of up to 1024 columns (blockIdx.y); each thread owns 4 adjacent
// columns (float4) of one frame lane and keeps kU 16-byte loads of h in flight.  The
// frame lanes of a block are folded in shared memory (fixed order) before the block's
// partial row is written, so results do not depend on timing.
template <int kU>
__global__ void __launch_bounds__(256, 2) loss_stream4_kernel(
    HeadDesc hd, const float* __restrict__ params, const float* __restrict__ h, long ldh,
    long F, const float* __restrict__ dzh, float* __restrict__ dz, float* __restrict__ dz_lo,
    float* __restrict__ hg_partial, float* __restrict__ db_partial) {
  TLG_PDL_ENTRY();
  constexpr int kA1 = 8;
  __shared__ float sdz[kLossFrames * kA1];
  __shared__ float red[256 * 4];
  const int A = hd.A, A1 = A + 1;
  const int quads = min(hd.H / 4, 256);            // column quads per slab
  const int lanes = 256 / quads;                    // frame lanes per block (1,2,4,...)
  const int tid = threadIdx.x;
  const int q = tid % quads, lane = tid / quads;
  const bool active = lane < lanes;
  const int j0 = blockIdx.y * quads * 4 + q * 4;    // first column of this thread
  const long fb = F * blockIdx.x / gridDim.x, fe = F * (blockIdx.x + 1) / gridDim.x;
  float w[4][kA1], acc[4][kA1], db[4];
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    db[c] = 0.f;
#pragma unroll
    for (int k = 0; k < kA1; ++k) {
      acc[c][k] = 0.f;
      float wk = 0.f;
      if (active && k < A) wk = __ldg(params + hd.wpi + long(k) * hd.wk + long(j0 + c) * hd.wj);
      else if (active && k == A) wk = __ldg(params + hd.wv + j0 + c);
      w[c][k] = wk;
    }
  }
  for (long f0 = fb; f0 < fe; f0 += kLossFrames) {
    const int nf = int(fe - f0 < long(kLossFrames) ? fe - f0 : long(kLossFrames));
    __syncthreads();
    for (int i = tid; i < nf * kA1; i += 256) {
      const int fi = i / kA1, k = i % kA1;
      sdz[i] = k < A1 ? dzh[(f0 + fi) * A1 + k] : 0.f;
    }
    __syncthreads();
    if (!active) continue;
    for (int i0 = lane; i0 < nf; i0 += lanes * kU) {
      float4 xs[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int i = i0 + u * lanes;
        xs[u] = i < nf ? __ldg(reinterpret_cast<const float4*>(h + (f0 + i) * ldh + j0))
                       : make_float4(0.f, 0.f, 0.f, 0.f);
      }
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int i = i0 + u * lanes;
        if (i >= nf) break;
        const float* d = sdz + i * kA1;
        float dk[kA1];
#pragma unroll
        for (int k = 0; k < kA1; ++k) dk[k] = d[k];
        const float x[4] = {xs[u].x, xs[u].y, xs[u].z, xs[u].w};
        float o[4];
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          float dh = 0.f;
#pragma unroll
          for (int k = 0; k < kA1; ++k) {
            dh = fmaf(dk[k], w[c][k], dh);
            acc[c][k] = fmaf(dk[k], x[c], acc[c][k]);
          }
          o[c] = dh * (1.f - x[c] * x[c]);
          db[c] += o[c];
        }
        if (dz) {
          const long off = (f0 + i) * hd.H + j0;
          *reinterpret_cast<float4*>(dz + off) = make_float4(o[0], o[1], o[2], o[3]);
          if (dz_lo)
            *reinterpret_cast<float4*>(dz_lo + off) =
                make_float4(o[0] - tf32_hi(o[0]), o[1] - tf32_hi(o[1]), o[2] - tf32_hi(o[2]),
                            o[3] - tf32_hi(o[3]));
        }
      }
    }
  }
  // fold the frame lanes (lane 0 + lane 1 + ... in order), one output at a time
  float* out = hg_partial + long(blockIdx.x) * A1 * hd.H;
#pragma unroll
  for (int k = 0; k <= kA1; ++k) {  // k == kA1: the last layer's bias partial
    if (k < kA1 && k >= A1) continue;
    __syncthreads();
#pragma unroll
    for (int c = 0; c < 4; ++c) red[tid * 4 + c] = k < kA1 ? acc[c][k] : db[c];
    __syncthreads();
    if (lane == 0) {
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        float t = red[q * 4 + c];
        for (int l = 1; l < lanes; ++l) t += red[(l * quads + q) * 4 + c];
        if (k < kA1) out[long(k) * hd.H + j0 + c] = t;
        else if (dz) db_partial[long(blockIdx.x) * hd.H + j0 + c] = t;
      }
    }
  }
}

// 32 columns per block, nw = blockDim/32 warps each summing rows w, w + nw, ... in order,
// then the warps' partial sums in warp order (deterministic for a given block size: 32
// warps when few columns must cover many rows, 8 when the grid is already wide)
template <typename Store>
__device__ __forceinline__ void rows_reduce_block(const float* __restrict__ partial, int rows,
                                                  long cols, long stride, Store store,
                                                  long col_block) {
  __shared__ float sh[kRowWarps][33];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = int(blockDim.x >> 5);
  const long c = col_block * 32 + lane;
  float acc = 0.f;
  if (c < cols)
    for (int r = w; r < rows; r += nw) acc += partial[long(r) * stride + c];
  sh[w][lane] = acc;
  __syncthreads();
  if (w == 0 && c < cols) {
    float t = 0.f;
    for (int i = 0; i < nw; ++i) t += sh[i][lane];
    store(c, t);
  }
}

__global__ void __launch_bounds__(1024) rows_reduce_kernel(const float* __restrict__ partial,
                                                          int rows, long cols, long stride,
                                                          float* __restrict__ out) {
  TLG_PDL_ENTRY();
  rows_reduce_block(partial, rows, cols, stride, [&](long c, float v) { out[c] = v; },
                    blockIdx.x);
}

// Head-gradient partials [nblk][A1][H] -> flat gradient (layout-aware, AccumulateGrad
// order of the families, policy.cpp:122-141).
// Blocks past the head columns (db_out set): the top trunk layer's bias gradient from the
// loss kernel's column partials [nblocks][H] -- the same rows, one launch instead of two.
__global__ void __launch_bounds__(1024) head_grad_reduce_kernel(HeadDesc hd,
                                                               const float* __restrict__ hg_partial,
                                                               int nblocks,
                                                               float* __restrict__ grad,
                                                               const float* __restrict__ db_partial,
                                                               float* __restrict__ db_out) {
  TLG_PDL_ENTRY();
  const int A = hd.A, A1 = A + 1;
  const long nw = long(A1) * hd.H;
  const long head_blocks = (nw + 31) / 32;
  if (blockIdx.x >= head_blocks) {
    rows_reduce_block(db_partial, nblocks, hd.H, hd.H, [&](long c, float v) { db_out[c] = v; },
                      long(blockIdx.x) - head_blocks);
    return;
  }
  rows_reduce_block(hg_partial, nblocks, nw, nw, [&](long idx, float v) {
    const int k = int(idx / hd.H), j = int(idx % hd.H);
    if (k < A)
      grad[hd.wpi + long(k) * hd.wk + long(j) * hd.wj] = v;
    else
      grad[hd.wv + j] = v;
  }, blockIdx.x);
}

// Bias partials [nblk][A1] and the loss/stat partials -> gradient + step statistics.
// Warp w < A1 reduces bias column w; warps A1.. reduce the 5 loss sums; each warp sums a
// strided subset then a fixed shuffle tree (deterministic).
// guard (optional): set to 1 when the step failed -- error flags or a non-finite loss --
// so that the optimizer of every rank skips the step (the flag rides the allreduce).
__global__ void head_bias_stats_kernel(HeadDesc hd, const float* __restrict__ bias_partial,
                                       const double* __restrict__ loss_partial, int nblocks,
                                       float* __restrict__ grad, StepStatsDev* st,
                                       const int* __restrict__ err, float* __restrict__ guard) {
  TLG_PDL_ENTRY();
  const int A = hd.A, A1 = A + 1;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (w < A1) {
    float acc = 0.f;
    for (int bk = lane; bk < nblocks; bk += 32) acc += bias_partial[long(bk) * A1 + w];
    acc = warp_sum(acc);
    if (lane == 0) {
      if (w < A && hd.bpi >= 0) grad[hd.bpi + w] = acc;
      if (w == A && hd.bv >= 0) grad[hd.bv] = acc;
    }
  } else if (w < A1 + 5) {
    const int q = w - A1;
    double acc = 0.0;
    for (int bk = lane; bk < nblocks; bk += 32) acc += loss_partial[long(bk) * 5 + q];
    acc = warp_sum(acc);
    if (lane == 0) {
      const double v = acc * st->inv_n;
      if (q == 0 && guard != nullptr && (*err != 0 || !isfinite(v))) guard[0] = 1.f;
      if (q == 0) st->loss = v;
      else if (q == 1) st->ratio = v;
      else if (q == 2) st->entropy = v;
      else if (q == 3) st->vloss = v;
      else st->clip = v;
    }
  }
}

__global__ void dw_reduce_kernel(const float4* __restrict__ ws, int splits, long n4, long stride4,
                                 float4* __restrict__ out) {
  TLG_PDL_ENTRY();
  for (long i = blockIdx.x * long(blockDim.x) + threadIdx.x; i < n4; i += long(gridDim.x) * blockDim.x) {
    float4 a = ws[i];
    for (int s = 1; s < splits; ++s) {
      const float4 b = ws[s * stride4 + i];
      a.x += b.x; a.y += b.y; a.z += b.z; a.w += b.w;
    }
    out[i] = a;
  }
}

__global__ void dw_reduce_scalar_kernel(const float* __restrict__ ws, int splits, long n,
                                        float* __restrict__ out) {
  TLG_PDL_ENTRY();
  for (long i = blockIdx.x * long(blockDim.x) + threadIdx.x; i < n; i += long(gridDim.x) * blockDim.x) {
    float a = ws[i];
    for (int s = 1; s < splits; ++s) a += ws[s * n + i];
    out[i] = a;
  }
}

constexpr int kColRows = 256;  // rows per colsum chunk

__global__ void colsum_partial_kernel(const float* __restrict__ x, long ld, long rows, int cols,
                                      float* __restrict__ partial) {
  TLG_PDL_ENTRY();
  const long r0 = long(blockIdx.y) * kColRows;
  const long r1 = min(rows, r0 + kColRows);
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < cols; j += gridDim.x * blockDim.x) {
    float acc = 0.f;
    for (long r = r0; r < r1; ++r) acc += x[r * ld + j];
    partial[long(blockIdx.y) * cols + j] = acc;
  }
}

__global__ void colsum_reduce_kernel(const float* __restrict__ partial, int chunks, int cols,
                                     float* __restrict__ out) {
  TLG_PDL_ENTRY();
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= cols) return;
  float acc = 0.f;
  for (int c = 0; c < chunks; ++c) acc += partial[long(c) * cols + j];
  out[j] = acc;
}

// K7: fused optimizer over the flat fp32 parameter vector.  Reads p, g, (m, v) and
// writes p, (m, v) and the tf32 residual plane the next step's GEMMs consume.
//   SGD  (rlmath.cpp:229-230):     p -= lr * g
//   Adam (torch.optim.Adam):       m = b1 m + (1-b1) g ; v = b2 v + (1-b2) g^2
//                                  p -= step_size * m / (sqrt(v) / bc2_sqrt + eps)
// g is the allreduced sum times grad_scale (= 1/G, learner.cpp:146-147).
__global__ void optimizer_kernel(float4* __restrict__ p, float4* __restrict__ plo,
                                 const float4* __restrict__ g, float4* __restrict__ m,
                                 float4* __restrict__ v, long n4, float grad_scale, int adam,
                                 float lr, float step_size, float bc2_sqrt, float b1, float b2,
                                 float eps) {
  TLG_PDL_ENTRY();
  for (long i = blockIdx.x * long(blockDim.x) + threadIdx.x; i < n4; i += long(gridDim.x) * blockDim.x) {
    float4 pp = p[i];
    float4 gg = g[i];
    float* pe = &pp.x;
    float* ge = &gg.x;
    if (adam) {
      float4 mm = m[i], vv = v[i];
      float* me = &mm.x;
      float* ve = &vv.x;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const float gq = ge[q] * grad_scale;
        me[q] = b1 * me[q] + (1.f - b1) * gq;
        ve[q] = b2 * ve[q] + (1.f - b2) * gq * gq;
        const float denom = sqrtf(ve[q]) / bc2_sqrt + eps;
        pe[q] -= step_size * me[q] / denom;
      }
      m[i] = mm;
      v[i] = vv;
    } else {
#pragma unroll
      for (int q = 0; q < 4; ++q) pe[q] -= lr * (ge[q] * grad_scale);
    }
    p[i] = pp;
    plo[i] = make_float4(pp.x - tf32_hi(pp.x), pp.y - tf32_hi(pp.y), pp.z - tf32_hi(pp.z),
                         pp.w - tf32_hi(pp.w));
  }
}

int grid_for(long n, int threads, int per_sm = 8) {
  long b = (n + threads - 1) / threads;
  return int(std::max<long>(1, std::min<long>(b, 148L * per_sm)));
}

}  // namespace

void launch_expand_u8(const uint8_t* in, float* out, long n, cudaStream_t s) {
  ::tlg::launch_k(expand_u8_kernel, dim3(grid_for(n / 4, 256)), dim3(256), size_t(0), s, reinterpret_cast<const uchar4*>(in),
                                                        reinterpret_cast<float4*>(out), n / 4);
  TLG_CHECK_LAUNCH();
}

// block per segment: scatter (contiguous i -> slot[i]) or gather (slot[i] -> contiguous i)
__global__ void __launch_bounds__(256) replay_move_kernel(SegArrays src, long src_rowb,
                                                          SegArrays dst, long dst_rowb,
                                                          const uint32_t* __restrict__ slots,
                                                          int T, int scatter) {
  TLG_PDL_ENTRY();
  const long i = blockIdx.x;
  const long si = scatter ? i : long(slots[i]);
  const long di = scatter ? long(slots[i]) : i;
  const uint8_t* so = src.obs + si * T * src_rowb;
  uint8_t* d_o = dst.obs + di * T * dst_rowb;
  if (src_rowb == dst_rowb && (src_rowb & 15) == 0 &&
      ((reinterpret_cast<uintptr_t>(so) | reinterpret_cast<uintptr_t>(d_o)) & 15) == 0) {
    const long n16 = T * src_rowb / 16;
    for (long k = threadIdx.x; k < n16; k += blockDim.x)
      reinterpret_cast<uint4*>(d_o)[k] = reinterpret_cast<const uint4*>(so)[k];
  } else {
    for (long k = threadIdx.x; k < T * dst_rowb; k += blockDim.x) {
      const long t = k / dst_rowb, j = k % dst_rowb;
      d_o[k] = j < src_rowb ? so[t * src_rowb + j] : uint8_t(0);
    }
  }
  for (int t = threadIdx.x; t < T; t += blockDim.x) {
    dst.action[di * T + t] = src.action[si * T + t];
    dst.reward[di * T + t] = src.reward[si * T + t];
    dst.blogp[di * T + t] = src.blogp[si * T + t];
    dst.value[di * T + t] = src.value[si * T + t];
    dst.done[di * T + t] = src.done[si * T + t];
  }
  if (threadIdx.x == 0) {
    dst.boot[di] = src.boot[si];
    dst.valid[di] = src.valid[si];
  }
}

void launch_replay_move(const SegArrays& src, long src_rowb, const SegArrays& dst, long dst_rowb,
                        const uint32_t* slots, int n, int T, bool scatter, cudaStream_t s) {
  if (n <= 0) return;
  ::tlg::launch_k(replay_move_kernel, dim3(n), dim3(256), size_t(0), s, src, src_rowb, dst, dst_rowb, slots, T, scatter ? 1 : 0);
  TLG_CHECK_LAUNCH();
}

void launch_unpack_bits(const uint8_t* bits, long rowb, long F, long D, uint8_t* out,
                        uint8_t* pitched, long pitch,
                        cudaStream_t s) {
  if (out == nullptr) {  // only the re-pitched bit rows
    if (pitch % 16 != 0) throw CudaError("bit-row pitch must be a multiple of 16");
    const size_t smem = size_t(kRepitchRows * rowb + 32);
    if (smem > 48 * 1024) throw CudaError("bit rows too long for the repitch kernel");
    ::tlg::launch_k(repitch_bits_kernel, dim3(ceil_div(F, kRepitchRows)), dim3(256), size_t(smem), s, bits, rowb, F, pitched,
                                                                     pitch);
    TLG_CHECK_LAUNCH();
    return;
  }
  ::tlg::launch_k(unpack_bits_kernel, dim3(grid_for(F * rowb, 256)), dim3(256), size_t(0), s, bits, rowb, F, D, out, pitched,
                                                             pitch);
  TLG_CHECK_LAUNCH();
}

void launch_split_lo(const float* x, float* lo, long n, cudaStream_t s) {
  ::tlg::launch_k(split_lo_kernel, dim3(grid_for(n / 4, 256)), dim3(256), size_t(0), s, reinterpret_cast<const float4*>(x),
                                                       reinterpret_cast<float4*>(lo), n / 4);
  TLG_CHECK_LAUNCH();
}

void launch_head_forward(const HeadDesc& hd, const float* params, const float* h, long ldh,
                         const BatchDev* b, long F, float* head_out, float* tlogp,
                         float* probs_out, int* err, cudaStream_t s) {
  if (hd.A + 1 > kMaxA1Limit) throw CudaError("n_actions exceeds the head kernel limit (31)");
  BatchDev bd{};
  if (b) bd = *b;
  const int blocks = int(std::max<long>(1, std::min<long>((F + 7) / 8, 148L * 16)));
  if (hd.A + 1 <= 8)
    ::tlg::launch_k(head_forward_kernel<8>, dim3(blocks), dim3(256), size_t(0), s, hd, params, h, ldh, bd, b ? 1 : 0, F, head_out,
                                                  tlogp, probs_out, err);
  else
    ::tlg::launch_k(head_forward_kernel<32>, dim3(blocks), dim3(256), size_t(0), s, hd, params, h, ldh, bd, b ? 1 : 0, F,
                                                   head_out, tlogp, probs_out, err);
  TLG_CHECK_LAUNCH();
}

void launch_head_finalize(const HeadDesc& hd, const float* params, const float* part,
                          int n_tiles, long F, const BatchDev* b, float* head_out, float* tlogp,
                          float* logits_out, float* probs_out, float* value_out, int* err,
                          cudaStream_t s, long part_rows) {
  if (hd.A + 1 > 8) throw CudaError("fused head supports n_actions <= 7");
  if (part_rows < F) part_rows = F;  // rows of the GEMM that left the partials
  BatchDev bd{};
  if (b) bd = *b;
  ::tlg::launch_k(head_finalize_kernel, dim3(ceil_div(F, 256)), dim3(256), size_t(0), s, hd, params, part, n_tiles, F, part_rows, bd,
                                                        b ? 1 : 0, head_out, tlogp, logits_out,
                                                        probs_out, value_out, err);
  TLG_CHECK_LAUNCH();
}

static bool aligned(const void* p, uintptr_t a) { return (reinterpret_cast<uintptr_t>(p) & (a - 1)) == 0; }

static bool returns_vec_ok(const BatchDev& b, int algo, const float* tlogp, const float* adv,
                           const float* target) {
  if (b.T % 4 != 0 || std::getenv("TLG_RETURNS_SCALAR")) return false;
  if (!aligned(b.reward, 16) || !aligned(b.value, 16) || !aligned(b.done, 4) ||
      !aligned(adv, 16) || !aligned(target, 16))
    return false;
  return algo == kAlgoPpo || (aligned(b.blogp, 16) && aligned(tlogp, 16));
}

int launch_returns(const BatchDev& b, int algo, const HyperDev& hp, const float* tlogp,
                   float* adv, float* target, double* seg_partial, int* err, cudaStream_t s) {
  int per;
  if (returns_vec_ok(b, algo, tlogp, adv, target)) {
    per = kRetVecSegsPerBlock;
    // one instantiation per algorithm: the PPO kernel drops the V-trace state (56 -> fewer
    // registers, more resident segments per SM for the HBM stream)
    if (algo == kAlgoPpo)
      ::tlg::launch_k(returns_vec_kernel<kAlgoPpo>, dim3(ceil_div(b.S, per)), dim3(256), size_t(0), s, b, hp, tlogp, adv, target,
                                                                    seg_partial, err);
    else
      ::tlg::launch_k(returns_vec_kernel<kAlgoVtrace>, dim3(ceil_div(b.S, per)), dim3(256), size_t(0), s, b, hp, tlogp, adv,
                                                                       target, seg_partial, err);
  } else {
    per = kRetSegsPerBlock;
    ::tlg::launch_k(returns_kernel, dim3(ceil_div(b.S, per)), dim3(32 * per), size_t(0), s, b, algo, hp, tlogp, adv, target,
                                                           seg_partial, err);
  }
  TLG_CHECK_LAUNCH();
  return per;
}

void launch_finalize_adv(const double* seg_partial, const BatchDev& b, int adv_norm,
                         StepStatsDev* st, int* err, cudaStream_t s, int segs_per_block) {
  ::tlg::launch_k(finalize_adv_kernel, dim3(1), dim3(1024), size_t(0), s, seg_partial, b, adv_norm, st, err, segs_per_block);
  TLG_CHECK_LAUNCH();
}

LossLaunch launch_loss_backward(const HeadDesc& hd, const float* params, const float* h,
                                long ldh, const BatchDev& b, const float* head_out,
                                const float* adv, const float* target, const StepStatsDev* st,
                                const HyperDev& hp, int loss_kind, float* dzh, float* dz,
                                float* dz_lo, float* hg_partial, double* loss_partial,
                                float* db_partial, cudaStream_t s, const float* teacher_out,
                                const float* head_part, int n_tiles, int* err) {
  const long F = long(b.S) * b.T;
  const int A1 = hd.A + 1;
  const long nw = long(A1) * hd.H;
  const long nchunks = (F + kLossFrames - 1) / kLossFrames;
  LossLaunch ll;
  const bool vec = A1 <= 8 && hd.H % 4 == 0 && ldh % 4 == 0 &&
                   (reinterpret_cast<uintptr_t>(h) & 15) == 0 && hd.H <= 4096;
  const int slabs = ceil_div(hd.H, 1024);
  // vectorised: 2 resident blocks per SM over all slabs, no more rows than 128-frame chunks
  ll.stream_blocks = vec ? int(std::max<long>(1, std::min<long>(nchunks, 2 * 148 / slabs)))
                         : int(std::min<long>(nchunks, kLossBlocks));
  ll.math_blocks = ceil_div(F, 256);
  float* bias_partial = hg_partial + long(ll.stream_blocks) * nw;
  const float* src = head_part ? head_part : head_out;
#define TLG_MATH(MA, KL, PARTS)                                                              \
  ::tlg::launch_k(loss_math_kernel<MA, KL, PARTS>, dim3(ll.math_blocks), dim3(256), size_t(0), s,                            \
      hd, b, src, adv, target, st, hp, loss_kind, dzh, loss_partial, bias_partial, teacher_out, \
      n_tiles, params, err)
  const bool kl = teacher_out != nullptr;
  if (A1 <= 8) {
    if (head_part) {
      if (kl) TLG_MATH(8, true, true);
      else TLG_MATH(8, false, true);
    } else {
      if (kl) TLG_MATH(8, true, false);
      else TLG_MATH(8, false, false);
    }
  } else {
    if (head_part) throw CudaError("fused-head partials need n_actions + 1 <= 8");
    if (kl) TLG_MATH(32, true, false);
    else TLG_MATH(32, false, false);
  }
#undef TLG_MATH
  TLG_CHECK_LAUNCH();
  if (vec) {
    ::tlg::launch_k(loss_stream4_kernel<8>, dim3(dim3(ll.stream_blocks, slabs)), dim3(256), size_t(0), s, 
        hd, params, h, ldh, F, dzh, dz, dz_lo, hg_partial, db_partial);
    TLG_CHECK_LAUNCH();
    return ll;
  }
  const size_t smem = size_t(kLossFrames) * A1 * sizeof(float);
#define TLG_LOSS(MA, CPT)                                                                  \
  ::tlg::launch_k(loss_stream_kernel<MA, CPT>, dim3(ll.stream_blocks), dim3(256), size_t(smem), s, hd, params, h, ldh, F, dzh, dz, \
                                                                 dz_lo, hg_partial, db_partial)
  const int cpt = (hd.H + 255) / 256;
  if (A1 <= 8) {
    if (cpt <= 1) TLG_LOSS(8, 1);
    else if (cpt <= 2) TLG_LOSS(8, 2);
    else if (cpt <= 4) TLG_LOSS(8, 4);
    else if (cpt <= 8) TLG_LOSS(8, 8);
    else throw CudaError("head input wider than 2048 with the fused loss kernel");
  } else if (A1 <= kMaxA1Limit && cpt <= 1) {
    TLG_LOSS(32, 1);
  } else {
    throw CudaError("n_actions > 7 needs a head input width <= 256");
  }
#undef TLG_LOSS
  TLG_CHECK_LAUNCH();
  return ll;
}

void launch_head_grad_reduce(const HeadDesc& hd, const float* hg_partial,
                             const double* loss_partial, const LossLaunch& ll, float* grad,
                             StepStatsDev* st, cudaStream_t s, const float* bias_partial,
                             const int* err, float* guard, const float* db_partial,
                             float* db_out) {
  const long nw = long(hd.A + 1) * hd.H;
  // (the block size of a separate db reduce over H columns is the same: identical sums)
  if (db_out && rows_reduce_threads(nw) != rows_reduce_threads(hd.H))
    throw CudaError("head_grad_reduce: fused db reduce needs one block size");
  const int blocks = int(ceil_div(nw, 32) + (db_out ? ceil_div(long(hd.H), 32) : 0));
  ::tlg::launch_k(head_grad_reduce_kernel, dim3(blocks), dim3(rows_reduce_threads(nw)), size_t(0), s,
      hd, hg_partial, ll.stream_blocks, grad, db_partial, db_out);
  TLG_CHECK_LAUNCH();
  ::tlg::launch_k(head_bias_stats_kernel, dim3(1), dim3(32 * (hd.A + 1 + 5)), size_t(0), s, 
      hd, bias_partial ? bias_partial : hg_partial + long(ll.stream_blocks) * nw, loss_partial,
      ll.math_blocks, grad, st, err, guard);
  TLG_CHECK_LAUNCH();
}

void launch_rows_reduce(const float* partial, int rows, long cols, long stride, float* out,
                        cudaStream_t s) {
  ::tlg::launch_k(rows_reduce_kernel, dim3(ceil_div(cols, 32)), dim3(rows_reduce_threads(cols)), size_t(0), s, partial, rows, cols,
                                                                             stride, out);
  TLG_CHECK_LAUNCH();
}

void launch_dw_reduce(const float* ws, int splits, long n, float* grad, cudaStream_t s) {
  // few columns per partial row: warp-parallel fixed-order reduction over the rows;
  // otherwise one float4 per thread walks the splits in order
  if (splits > 32 || (splits > 8 && n < 4L * 148 * 256)) {
    launch_rows_reduce(ws, splits, n, n, grad, s);
    return;
  }
  if ((n & 3) == 0 && (reinterpret_cast<uintptr_t>(grad) & 15) == 0) {
    ::tlg::launch_k(dw_reduce_kernel, dim3(grid_for(n / 4, 256)), dim3(256), size_t(0), s, reinterpret_cast<const float4*>(ws),
                                                          splits, n / 4, n / 4,
                                                          reinterpret_cast<float4*>(grad));
  } else {
    ::tlg::launch_k(dw_reduce_scalar_kernel, dim3(grid_for(n, 256)), dim3(256), size_t(0), s, ws, splits, n, grad);
  }
  TLG_CHECK_LAUNCH();
}

void launch_colsum(const float* x, long ld, long rows, int cols, float* partial, float* grad,
                   cudaStream_t s) {
  const int chunks = ceil_div(rows, kColRows);
  dim3 grid(ceil_div(cols, 256), chunks);
  ::tlg::launch_k(colsum_partial_kernel, dim3(grid), dim3(256), size_t(0), s, x, ld, rows, cols, partial);
  TLG_CHECK_LAUNCH();
  ::tlg::launch_k(colsum_reduce_kernel, dim3(ceil_div(cols, 256)), dim3(256), size_t(0), s, partial, chunks, cols, grad);
  TLG_CHECK_LAUNCH();
}

void launch_optimizer(float* params, float* params_lo, const float* grad, float* m, float* v,
                      long n, float grad_scale, int adam, float lr, float step_size,
                      float bc2_sqrt, float b1, float b2, float eps, cudaStream_t s) {
  // n is padded to a multiple of 4 by the allocator
  ::tlg::launch_k(optimizer_kernel, dim3(grid_for(n / 4, 256, 4)), dim3(256), size_t(0), s, 
      reinterpret_cast<float4*>(params), reinterpret_cast<float4*>(params_lo),
      reinterpret_cast<const float4*>(grad), reinterpret_cast<float4*>(m),
      reinterpret_cast<float4*>(v), n / 4, grad_scale, adam, lr, step_size, bc2_sqrt, b1, b2,
      eps);
  TLG_CHECK_LAUNCH();
}

}  // namespace tlg
