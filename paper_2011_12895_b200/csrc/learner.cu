// B200 learner step + InfServer forward behind the C ABI of include/tlg_b200.h.
//
// One tlg_learner owns one GPU's shard of Learner::TrainStep (learner.cpp:104-158):
//
//   stage batch (H2D or device) -> obs tf32 residual
//   forward trunk GEMMs   (tcgen05 3xTF32, tanh epilogue writes x and its residual)
//   K3a heads             (logits, value, target logp)
//   K1 returns            (GAE + lambda-return | V-trace), adv-norm statistics
//   K3b loss + dlogits    (PPO / PG), head gradients, tanh' of the last layer
//   backward trunk GEMMs  (dW split-K + fixed-order reduce, db column sums, dX with tanh')
//   [NCCL sum-allreduce of the flat fp32 gradient + failure guard]
//   K7 optimizer          (Adam | SGD; skipped on any rank's failure)
//
// All reductions have a fixed order, so a step is bit-reproducible run to run.
#include "nccl_dyn.h"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/tlg_b200.h"
#include "gemm_i8.cuh"
#include "learner_kernels.cuh"

namespace {

thread_local std::string g_err;

struct InvalidArg : std::invalid_argument {
  using std::invalid_argument::invalid_argument;
};
struct RuntimeErr : std::runtime_error {
  using std::runtime_error::runtime_error;
};

template <typename F>
int Guard(F&& f) {
  try {
    f();
    return TLG_OK;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return TLG_INVALID_ARGUMENT;
  } catch (const tlg::CudaError& e) {
    g_err = e.what();
    return TLG_CUDA_ERROR;
  } catch (const std::exception& e) {
    g_err = e.what();
    return TLG_RUNTIME_ERROR;
  }
}

// Run-to-run determinism of the gradient sum (the reference's determinism contract,
// docs/architecture.md:83-89): NCCL's per-size algorithm / protocol choice is
// pinned unless the caller set it (TLG_NCCL_PIN=0 leaves NCCL's tuner alone).
void pin_nccl() {
  const char* pin = std::getenv("TLG_NCCL_PIN");
  if (pin && std::strcmp(pin, "0") == 0) return;
  setenv("NCCL_ALGO", "Ring", 0);
}

#define NCCL_CHECK(expr)                                                              \
  do {                                                                                \
    ncclResult_t _r = (expr);                                                         \
    if (_r != ncclSuccess)                                                            \
      throw tlg::CudaError(std::string(#expr) + ": " + tlg::nccl::api().GetErrorString(_r)); \
  } while (0)

// Fused-head partial slices per row a trunk GEMM can write (LaunchInfo::head_slices):
// ceil(H / BN) tiles x epilogue groups, at most ceil(H / 64) + 2 for the tile plans of
// gemm_sm100.cu (64-column tiles; 128 / 256 with up to 2 groups) and the int8 kernels.
long head_slices_max(long H) { return (H + 63) / 64 + 2; }

// Parameter layout of the three families (policy.cpp:23-27,78-104).
struct Net {
  uint32_t family, D, A, L;
  // GEMM row length of the observations: D rounded up to 4 floats (16-B rows for TMA).
  // The flat parameters keep the reference layout [h_1 x D]; when D_pad != D the first
  // trunk layer runs on zero-padded copies (obs rows, W_1) and its dW is compacted back.
  uint32_t D_pad;
  std::vector<uint32_t> dims;
  std::vector<long> w_off, b_off;
  long P = 0;
  tlg::HeadDesc head{};

  explicit Net(const tlg_policy_shape& s) {
    if (s.obs_dim == 0 || s.n_actions == 0)
      throw InvalidArg("policy shape dimensions must be positive");
    if (s.family > TLG_FAMILY_MLP) throw InvalidArg("unknown policy family");
    if (s.n_actions + 1 > 32) throw InvalidArg("n_actions > 31 is not supported on the GPU path");
    family = s.family;
    D = s.obs_dim;
    D_pad = family == TLG_FAMILY_MLP ? (D + 3) / 4 * 4 : D;
    A = s.n_actions;
    L = family == TLG_FAMILY_MLP ? s.n_hidden : 0;
    if (L > 8) throw InvalidArg("at most 8 hidden layers");
    dims.push_back(D);
    long off = 0;
    for (uint32_t l = 0; l < L; ++l) {
      const uint32_t h = s.hidden[l];
      if (h == 0) throw InvalidArg("hidden width must be positive");
      if (h % 4 != 0)
        throw InvalidArg("mlp hidden widths must be multiples of 4 on the GPU path");
      w_off.push_back(off);
      off += long(h) * dims.back();
      b_off.push_back(off);
      off += h;
      dims.push_back(h);
    }
    const int H = int(dims.back());
    head.family = int(family);
    head.A = int(A);
    head.H = H;
    if (family == TLG_FAMILY_MLP) {
      head.wpi = off; head.wk = H; head.wj = 1; off += long(A) * H;
      head.bpi = off; off += A;
      head.wv = off; off += H;
      head.bv = off; off += 1;
    } else {
      head.wpi = 0;
      head.wk = family == TLG_FAMILY_LINEAR ? int(D) : 1;   // linear W[k][j]  (policy.cpp:86)
      head.wj = family == TLG_FAMILY_LINEAR ? 1 : int(A);   // tabular T[row][k] (policy.cpp:80)
      head.bpi = -1;
      head.wv = long(A) * D;
      head.bv = -1;
      off = long(A) * D + D;
    }
    P = off;
  }
  bool padded() const { return L > 0 && D_pad != D; }
  // K extent of trunk layer l's GEMMs (its input width, padded for layer 0)
  int gin(uint32_t l) const { return l == 0 ? int(D_pad) : int(dims[l]); }
};

// Zero-padded copy of a row-major [rows x cols] matrix into [rows x cols_pad].
__global__ void pad_rows_kernel(const float* __restrict__ src, long rows, int cols, int cols_pad,
                                float* __restrict__ dst) {
  TLG_PDL_ENTRY();
  const long n = rows * cols_pad;
  for (long i = blockIdx.x * long(blockDim.x) + threadIdx.x; i < n;
       i += long(gridDim.x) * blockDim.x) {
    const long r = i / cols_pad;
    const int c = int(i - r * cols_pad);
    dst[i] = c < cols ? src[r * cols + c] : 0.f;
  }
}

void pad_rows(const float* src, long rows, int cols, int cols_pad, float* dst, cudaStream_t st) {
  const long n = rows * cols_pad;
  ::tlg::launch_k(pad_rows_kernel, dim3(int(std::min<long>((n + 255) / 256, 148L * 8))), dim3(256), size_t(0), st, src, rows, cols,
                                                                               cols_pad, dst);
  TLG_CHECK_LAUNCH();
}

template <typename T>
T* dalloc(size_t n) {
  void* p = nullptr;
  if (n == 0) n = 1;
  TLG_CUDA(cudaMalloc(&p, n * sizeof(T)));
  TLG_CUDA(cudaMemset(p, 0, n * sizeof(T)));
  return static_cast<T*>(p);
}

struct DevFree {
  std::vector<void*> ptrs;
  ~DevFree() {
    for (void* p : ptrs) cudaFree(p);
  }
  template <typename T>
  T* add(size_t n) {
    T* p = dalloc<T>(n);
    ptrs.push_back(p);
    return p;
  }
};

long pad4(long n) { return (n + 3) & ~3L; }

}  // namespace

// ===========================================================================
struct tlg_learner {
  tlg_learner_config cfg{};
  Net net;
  int S_max, T;
  long F_max;
  long P_pad;
  cudaStream_t stream = nullptr;
  DevFree mem;
  // parameters / optimizer (flat, fp32); grad has 4 trailing guard slots
  static constexpr int kMaxLocalShards = 64;
  static constexpr int kMaxSplits = 128;
  float *params, *params_lo, *grad, *grad_tmp, *adam_m, *adam_v;
  float grad_scale = 1.f;
  // batch
  float *obs, *obs_lo;
  // net.padded(): observation rows, W_1 (student / teacher) and dW_1 at D_pad columns
  float *obs_pad = nullptr, *w1p = nullptr, *w1p_lo = nullptr, *tw1p = nullptr,
        *tw1p_lo = nullptr, *dw1p = nullptr;
  uint8_t* obs_u8;
  uint8_t* obs_bits;       // bit planes, row pitch bits_pitch (16-B aligned rows)
  long bits_pitch = 0;
  uint8_t* obs_bits_lin;    // host bit rows as shipped (ceil(D/8) bytes per frame)
  // layer-1 weights as fixed-point int8 pieces for the exact binary-plane GEMM
  int8_t* wq = nullptr;
  float* wq_scale = nullptr;
  long wq_kp = 0;
  const bool i8_disabled = std::getenv("TLG_NO_I8") != nullptr;
  const bool i8_dw_disabled = std::getenv("TLG_NO_I8_DW") != nullptr;
  // layer-1 dW on the int8 tensor cores: dZ_1 as per-split fixed-point pieces
  int8_t* dzq = nullptr;
  unsigned* colmax = nullptr;
  static constexpr int kMaxI8Splits = 148;
  // parameter plane the int8 pieces in wq were quantized from during this step (the
  // student's or the teacher's); null = stale.  Shards alternate teacher and student
  // forwards, so the pieces are rebuilt whenever the plane differs.
  const float* wq_src = nullptr;
  // layer 2 on int8 x int8 (tanh activations as pieces, W_2 as row pieces).  Opt-in
  // (TLG_I8X2=1): measured at C3 its forward is L2->SM-bound at 64-column tiles and the
  // extra piece plane costs layer 1 more than layer 2 saves (profiles/r01_ncu_i8x2.md)
  const bool i8x2_disabled = std::getenv("TLG_I8X2") == nullptr;
  int8_t* act_q = nullptr;  // [3][F][h_1]
  int8_t* w2q = nullptr;    // [3][h_2][h_1]
  float* w2_scale = nullptr;
  int32_t* action;
  float *reward, *blogp, *value;
  uint8_t* done;
  float* boot;
  int32_t* valid;
  // activations
  std::vector<float*> act, act_lo, dz, dz_lo;
  // tf32 residual (lo = x - trunc_tf32(x)) of the fp32 GEMM operands: derived in shared
  // memory by the consuming GEMM (Operand::lo_smem, the default), or -- TLG_LO_HBM=1, the
  // round-1 scheme kept for A/B runs -- planes written by each producer and re-read from
  // HBM.  Only dZ_1 keeps a plane when layer 1's dW runs on uint8 planes (that kernel's
  // converter warps expand the bytes, so it reads the residual plane).
  const bool lo_hbm = std::getenv("TLG_LO_HBM") != nullptr;
  bool x0_has_lo = false;  // this shard's observations are inexact in tf32 (fp32 values)
  tlg::gemm::Operand lo_op(const float* hi, const float* plane, long ld, bool mn) const {
    tlg::gemm::Operand o{hi, nullptr, ld, mn};
    if (lo_hbm) o.lo = plane;
    else o.lo_smem = true;
    return o;
  }
  // dZ_l's residual plane has a reader: the tf32 layer-1 dW over uint8 planes
  bool dz_lo_plane(int l, const uint8_t* x0u8) const {
    return lo_hbm || (l == 0 && x0u8 != nullptr);
  }
  float *head_out, *head_part, *tlogp, *adv, *target, *dzh;
  // teacher policy for the PPO KL term (rlmath.cpp:145-155; tlg_learner_set_teacher)
  float* teacher = nullptr;
  float* teacher_lo = nullptr;
  float* t_head_out = nullptr;
  bool has_teacher = false;
  // the reference's learner passes no teacher (learner.cpp:127); with one set, PPO losses
  // carry the KL term (V-trace's PgLossAndGrad has none, rlmath.cpp:187-222)
  bool teacher_active() const { return has_teacher && cfg.algo != TLG_ALGO_VTRACE; }
  double* seg_partial;
  tlg::StepStatsDev* stats;
  int* err;
  float* hg_partial;
  double* loss_partial;
  float* ws;
  long ws_elems;
  float* col_partial;
  // host
  tlg_hyper hp{};
  bool hp_set = false;
  uint64_t adam_t = 0;
  uint64_t steps_done = 0;
  ncclComm_t comm = nullptr;
  int nranks = 1, rank = 0;
  // ---- gradient buckets (TLG_OVERLAP=1, nranks > 1, one local shard per rank): each
  // layer's dW/db region of the flat gradient is sum-allreduced on comm_stream as soon as
  // the backward has written it, overlapping the layers below (learner.cpp:138-149,
  // SURVEY 8(e)).  The last bucket travels in one NCCL group with the failure guard; the
  // optimizer waits for comm_done.  Default: one allreduce after the whole backward.
  cudaStream_t comm_stream = nullptr;
  static constexpr int kMaxBuckets = 12;
  cudaEvent_t bucket_ev[kMaxBuckets]{};
  cudaEvent_t comm_done = nullptr;
  int n_buckets = 0;
  bool overlap_active = false;
  long pend_off = 0, pend_count = 0;
  bool pend_guard = false;
  // Bucketed overlap is opt-in (TLG_OVERLAP=1): measured on NVLink B200s, NCCL kernels
  // competing with the persistent dW GEMMs for SMs (dW2 71 -> 89 us at N = 2) cost more
  // than one allreduce of the whole gradient after the backward (C3 weak step 0.81-0.86
  // vs 0.77-0.80 ms at N = 2 / 4, tools/overlap_probe.sh).
  const bool overlap_requested = std::getenv("TLG_OVERLAP") != nullptr;
  void issue_bucket(long off, long count, bool with_guard);
  // grad[off, off + count) (and the failure guard, with_guard) is final on `stream`:
  // allreduce it now, or -- the last bucket of the step -- in bucket_flush()
  void bucket_ready(long off, long count, bool last, bool with_guard = false) {
    if (!overlap_active) return;
    if (last) {
      pend_off = off;
      pend_count = count;
      pend_guard = with_guard;
    } else {
      issue_bucket(off, count, with_guard);
    }
  }
  void bucket_flush();
  tlg::StepStatsDev* h_stats = nullptr;
  int* h_flags = nullptr;  // [0] err bits, [1..] guard as float bits
  cudaEvent_t ev[8]{};
  // per-GEMM events (timing mode): [kind 0 fwd | 1 dW | 2 dX][layer][begin,end]
  cudaEvent_t kev[3][8][2]{};
  int launches = 0;
  int S_last = 0;

  tlg_learner(const tlg_learner_config& c, const tlg_policy_shape& s) : cfg(c), net(s) {
    if (c.max_segments == 0 || c.unroll_len == 0)
      throw InvalidArg("max_segments and unroll_len must be >= 1");
    if (c.algo > TLG_ALGO_PPO_VTRACE) throw InvalidArg("unknown algo");
    for (uint32_t l = 1; l < net.L; ++l)  // dZ column sums are fused into the dX epilogue
      if (net.dims[l] > uint32_t(tlg::gemm::kColMax))
        throw InvalidArg("mlp hidden widths below the top layer must be <= 2048 on the GPU path");
    TLG_CUDA(cudaSetDevice(c.device));
    S_max = int(c.max_segments);
    T = int(c.unroll_len);
    F_max = long(S_max) * T;
    P_pad = pad4(net.P);
    TLG_CUDA(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking));
    params = mem.add<float>(P_pad);
    params_lo = mem.add<float>(P_pad);
    grad = mem.add<float>(P_pad + 4);
    grad_tmp = mem.add<float>(P_pad + 4);
    adam_m = mem.add<float>(P_pad);
    adam_v = mem.add<float>(P_pad);
    adam_t_dev = mem.add<uint64_t>(1);
    opt_done = mem.add<unsigned>(4);
    TLG_CUDA(cudaMemset(opt_done, 0, 16));
    const long D = net.D;
    obs = mem.add<float>(F_max * D);
    obs_lo = lo_hbm ? mem.add<float>(F_max * long(net.D_pad)) : nullptr;
    if (net.padded()) {
      obs_pad = mem.add<float>(F_max * long(net.D_pad));
      w1p = mem.add<float>(long(net.dims[1]) * net.D_pad);
      w1p_lo = mem.add<float>(long(net.dims[1]) * net.D_pad);
      dw1p = mem.add<float>(long(net.dims[1]) * net.D_pad);
    }
    obs_u8 = cfg.obs_dtype != TLG_OBS_F32 ? mem.add<uint8_t>(F_max * D + 16) : nullptr;
    bits_pitch = ((D + 7) / 8 + 15) / 16 * 16;
    obs_bits = cfg.obs_dtype != TLG_OBS_F32 ? mem.add<uint8_t>(F_max * bits_pitch + 16) : nullptr;
    if (obs_bits) TLG_CUDA(cudaMemset(obs_bits, 0, F_max * bits_pitch + 16));
    obs_bits_lin = cfg.obs_dtype != TLG_OBS_F32 ? mem.add<uint8_t>(F_max * ((D + 7) / 8) + 16)
                                                : nullptr;
    if (obs_bits && net.L >= 2) {
      wq_kp = (D + 15) / 16 * 16;
      wq = mem.add<int8_t>(3 * long(net.dims[1]) * wq_kp);
      wq_scale = mem.add<float>(net.dims[1]);
      if (net.dims[1] % 16 == 0) {
        dzq = mem.add<int8_t>(3 * F_max * long(net.dims[1]));
        colmax = mem.add<unsigned>(long(kMaxI8Splits) * net.dims[1]);
      }
      if (net.dims[1] % 32 == 0 && net.A + 1 <= 8) {
        act_q = mem.add<int8_t>(3 * F_max * long(net.dims[1]));
        w2q = mem.add<int8_t>(3 * long(net.dims[2]) * net.dims[1]);
        w2_scale = mem.add<float>(net.dims[2]);
      }
    }
    action = mem.add<int32_t>(F_max);
    reward = mem.add<float>(F_max);
    blogp = mem.add<float>(F_max);
    value = mem.add<float>(F_max);
    done = mem.add<uint8_t>(F_max);
    boot = mem.add<float>(S_max);
    valid = mem.add<int32_t>(S_max);
    for (uint32_t l = 0; l < net.L; ++l) {
      const long n = F_max * net.dims[l + 1];
      act.push_back(mem.add<float>(n));
      act_lo.push_back(lo_hbm ? mem.add<float>(n) : nullptr);
      dz.push_back(mem.add<float>(n));
      dz_lo.push_back(lo_hbm || (l == 0 && cfg.obs_dtype != TLG_OBS_F32) ? mem.add<float>(n)
                                                                         : nullptr);
    }
    const int A1 = int(net.A) + 1;
    head_out = mem.add<float>(F_max * A1);
    head_part = mem.add<float>(F_max * A1 * head_slices_max(net.head.H));
    tlogp = mem.add<float>(F_max);
    adv = mem.add<float>(F_max);
    target = mem.add<float>(F_max);
    seg_partial = mem.add<double>(3 * ((S_max + 7) / 8));  // one {s1, s2, n} per returns block
    stats = mem.add<tlg::StepStatsDev>(kMaxLocalShards);
    err = mem.add<int>(4);
    // partial rows: one per loss block, or one per persistent CTA of the fused loss GEMM
    const long nblk = std::max<long>((F_max + tlg::kLossFrames - 1) / tlg::kLossFrames,
                                     tlg::gemm::num_sms());
    hg_partial = mem.add<float>(nblk * A1 * long(net.head.H) + nblk * A1);
    loss_partial = mem.add<double>(nblk * 5);
    dzh = mem.add<float>(F_max * A1);
    ws_elems = 0;
    long max_cols = 1;
    for (uint32_t l = 0; l < net.L; ++l) {
      const int out = int(net.dims[l + 1]), in = net.gin(l);
      const int sp = tlg::gemm::pick_splits(out, in, int(F_max), kMaxSplits);
      ws_elems = std::max(ws_elems, long(sp) * out * in);
      max_cols = std::max<long>(max_cols, out);
    }
    if (dzq) ws_elems = std::max(ws_elems, long(kMaxI8Splits) * net.dims[1] * net.D_pad);
    ws = ws_elems ? mem.add<float>(ws_elems) : nullptr;
    // rows: the loss kernel's blocks, or one per persistent GEMM CTA (the dX epilogue's
    // fused column sums), whichever is more
    const long cp_rows = std::max<long>((F_max + tlg::kLossFrames - 1) / tlg::kLossFrames + 1,
                                        tlg::gemm::num_sms());
    col_partial = mem.add<float>(cp_rows * std::max<long>(max_cols, net.head.H));
    TLG_CUDA(cudaMallocHost(&h_stats, kMaxLocalShards * sizeof(tlg::StepStatsDev)));
    TLG_CUDA(cudaMallocHost(&h_flags, 16));
    for (auto& e : ev) TLG_CUDA(cudaEventCreate(&e));
    for (auto& a : kev)
      for (auto& b : a)
        for (auto& e : b) TLG_CUDA(cudaEventCreate(&e));
  }

  ~tlg_learner() {
    if (stream) cudaStreamSynchronize(stream);
    for (auto& g : graphs)
      if (g.exec) cudaGraphExecDestroy(g.exec);
    if (copy_stream) {
      cudaStreamSynchronize(copy_stream);
      cudaStreamDestroy(copy_stream);
    }
    for (auto& sl : slots) {
      if (sl.ready) cudaEventDestroy(sl.ready);
      if (sl.consumed) cudaEventDestroy(sl.consumed);
    }
    if (comm_stream) {
      cudaStreamSynchronize(comm_stream);
      cudaStreamDestroy(comm_stream);
    }
    for (auto& e : bucket_ev)
      if (e) cudaEventDestroy(e);
    if (comm_done) cudaEventDestroy(comm_done);
    if (comm) tlg::nccl::api().CommDestroy(comm);
    for (auto& e : ev)
      if (e) cudaEventDestroy(e);
    for (auto& a : kev)
      for (auto& b : a)
        for (auto& e : b)
          if (e) cudaEventDestroy(e);
    if (h_stats) cudaFreeHost(h_stats);
    if (h_flags) cudaFreeHost(h_flags);
    if (stream) cudaStreamDestroy(stream);
  }

  void make_comm_stream() {
    if (comm_stream) return;
    int lo = 0, hi = 0;
    TLG_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    // highest priority: a bucket's NCCL kernel is scheduled as soon as SMs free up
    TLG_CUDA(cudaStreamCreateWithPriority(&comm_stream, cudaStreamNonBlocking, hi));
  }

  void mark(int i) {
    if (cfg.timing) TLG_CUDA(cudaEventRecord(ev[i], stream));
  }
  void kmark(int kind, int layer, int end) {
    if (cfg.timing) TLG_CUDA(cudaEventRecord(kev[kind][layer][end], stream));
  }

  // uint8 observations feed the first trunk GEMM and its dW directly (converted in smem)
  bool direct_u8() const { return net.L > 0 && net.D % 16 == 0; }
  const uint8_t* x0_u8 = nullptr;
  const uint8_t* x0_bits = nullptr;  // bit planes (pitch bits_pitch) for the int8 layer-1 GEMM

  // binary planes take the exact int8 tensor-core path for layer 1 (L >= 2: the fused
  // heads stay on the last trunk layer's tf32 epilogue)
  bool i8_layer1() const { return wq != nullptr && !i8_disabled; }
  bool i8_dw1() const { return i8_layer1() && dzq != nullptr && !i8_dw_disabled; }
  bool i8_fwd2(long F) const { return i8_layer1() && act_q != nullptr && !i8x2_disabled && F >= 256; }

  // split-K plan of the int8 layer-1 dW: as many splits as fill one wave of CTA pairs,
  // an even number of 128-frame k-blocks per split (the dX epilogue's 256-row tiles
  // never straddle a split), <= 1024 k-blocks per split (exact int32 accumulators)
  void i8_dw_plan(long F, int& splits, int& kb_per_split) const {
    const int kb_total = int((F + 127) / 128);
    const int cg = net.dims[1] >= 256 ? 2 : 1;
    const int tiles = ((int(net.dims[1]) + 128 * cg - 1) / (128 * cg)) *
                      ((int(net.D) + 128 * cg - 1) / (128 * cg));
    const int units = cg == 2 ? tlg::gemm::num_sms() / 2 : tlg::gemm::num_sms();
    splits = std::max(1, std::min(units / std::max(1, tiles), kMaxI8Splits));
    kb_per_split = (kb_total + splits - 1) / splits;
    kb_per_split = std::max(2, std::min(1024, (kb_per_split + 1) / 2 * 2));
    splits = (kb_total + kb_per_split - 1) / kb_per_split;
  }

  void stage(const tlg_segment_batch& b, int on_device, tlg::BatchDev& bd, const float** obs_f32,
             bool& obs_exact, bool internal = false) {
    x0_u8 = nullptr;
    x0_bits = nullptr;
    if (b.n_segments == 0) throw InvalidArg("empty minibatch");
    if (int(b.n_segments) > S_max) throw InvalidArg("batch exceeds the learner's max_segments");
    if (int(b.unroll_len) != T) throw InvalidArg("unroll_len mismatch");
    if (b.obs_dim != net.D) throw InvalidArg("observation size does not match policy shape");
    if (b.obs_dtype != TLG_OBS_F32 && b.obs_dtype != TLG_OBS_U8 && b.obs_dtype != TLG_OBS_BITS)
      throw InvalidArg("unknown obs dtype");
    if (b.obs_dtype != TLG_OBS_F32 && obs_u8 == nullptr)
      throw InvalidArg("learner not configured for uint8 / bit-packed observations");
    const long S = b.n_segments, F = S * T, D = net.D;
    bd.S = int(S);
    bd.T = T;
    if (b.obs_dtype == TLG_OBS_BITS) {
      // bit-packed 0/1 planes (LSB first, obs_pitch or ceil(D/8) bytes per frame)
      const long rowb_min = (D + 7) / 8;
      const long rowb = b.obs_pitch ? long(b.obs_pitch) : rowb_min;
      if (rowb != rowb_min && rowb != bits_pitch)
        throw InvalidArg("obs_pitch must be 0, ceil(obs_dim/8) or that rounded up to 16 bytes");
      const uint8_t* bits = static_cast<const uint8_t*>(b.obs);
      const bool pitched = rowb == bits_pitch;  // rows already 16-B multiples
      if (!on_device) {
        uint8_t* dst = pitched ? obs_bits : obs_bits_lin;
        TLG_CUDA(cudaMemcpyAsync(dst, bits, size_t(F * rowb), cudaMemcpyHostToDevice, stream));
        bits = dst;
      } else if (pitched && (internal || (reinterpret_cast<uintptr_t>(bits) & 15) != 0)) {
        // graph replays read the learner's own buffer
        TLG_CUDA(cudaMemcpyAsync(obs_bits, bits, size_t(F * rowb), cudaMemcpyDeviceToDevice,
                                 stream));
        bits = obs_bits;
      }
      if (pitched) {
        if (i8_layer1()) x0_bits = bits;
        if (!i8_dw1()) {  // the tf32 layer-1 dW (or a non-MLP family) reads uint8 planes
          tlg::launch_unpack_bits(bits, rowb, F, D, obs_u8, nullptr, 0, stream);
          ++launches;
        }
      } else {
        // one pass: rows re-pitched to 16 B for the int8 GEMM's TMA (pad bytes zero) and,
        // when the tf32 layer-1 dW runs, expanded to the uint8 planes it reads
        tlg::launch_unpack_bits(bits, rowb, F, D, i8_dw1() ? nullptr : obs_u8,
                                i8_layer1() ? obs_bits : nullptr, bits_pitch, stream);
        if (i8_layer1()) x0_bits = obs_bits;
        ++launches;
      }
      tlg_segment_batch u = b;
      u.obs_dtype = TLG_OBS_U8;
      u.obs = obs_u8;
      // the remaining arrays follow the caller's residency; obs now lives on the device
      stage_rest(u, on_device, internal, bd, obs_f32, obs_exact, /*obs_on_device=*/true);
      return;
    }
    stage_rest(b, on_device, internal, bd, obs_f32, obs_exact, on_device != 0);
  }

  void stage_rest(const tlg_segment_batch& b, int on_device, bool internal, tlg::BatchDev& bd,
                  const float** obs_f32, bool& obs_exact, bool obs_on_device) {
    const long S = b.n_segments, F = S * T, D = net.D;
    if (on_device && !internal) {
      bd.action = b.action;
      bd.reward = b.reward;
      bd.blogp = b.behavior_logp;
      bd.value = b.value_est;
      bd.done = b.done;
      bd.boot = b.bootstrap;
      bd.valid = b.valid_steps;
      if (b.obs_dtype == TLG_OBS_U8) {
        if (direct_u8() && (reinterpret_cast<uintptr_t>(b.obs) & 15) == 0) {
          x0_u8 = static_cast<const uint8_t*>(b.obs);
        } else {
          tlg::launch_expand_u8(static_cast<const uint8_t*>(b.obs), obs, F * D, stream);
          ++launches;
        }
        *obs_f32 = obs;
        obs_exact = true;
      } else {
        *obs_f32 = static_cast<const float*>(b.obs);
        obs_exact = false;
      }
      return;
    }
    auto h2d = [&](void* dst, const void* src, size_t bytes) {
      TLG_CUDA(cudaMemcpyAsync(dst, src, bytes,
                               on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice,
                               stream));
    };
    if (b.obs_dtype == TLG_OBS_U8) {
      if (b.obs != obs_u8)
        TLG_CUDA(cudaMemcpyAsync(obs_u8, b.obs, size_t(F * D),
                                 obs_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice,
                                 stream));
      if (direct_u8()) {
        x0_u8 = obs_u8;
      } else {
        tlg::launch_expand_u8(obs_u8, obs, F * D, stream);
        ++launches;
      }
      obs_exact = true;
    } else {
      h2d(obs, b.obs, size_t(F * D) * 4);
      obs_exact = false;
    }
    *obs_f32 = obs;
    h2d(action, b.action, F * 4);
    h2d(reward, b.reward, F * 4);
    h2d(blogp, b.behavior_logp, F * 4);
    h2d(value, b.value_est, F * 4);
    h2d(done, b.done, F);
    h2d(boot, b.bootstrap, S * 4);
    h2d(valid, b.valid_steps, S * 4);
    bd.action = action;
    bd.reward = reward;
    bd.blogp = blogp;
    bd.value = value;
    bd.done = done;
    bd.boot = boot;
    bd.valid = valid;
  }

  struct Staged {
    tlg::BatchDev bd{};
    const float* x0 = nullptr;
    const uint8_t* x0_u8 = nullptr;
    const uint8_t* x0_bits = nullptr;
    bool exact = false;
  };

  Staged stage_shard(const tlg_segment_batch& b, int on_device, bool internal) {
    Staged sg;
    stage(b, on_device, sg.bd, &sg.x0, sg.exact, internal);
    sg.x0_u8 = x0_u8;
    sg.x0_bits = x0_bits;
    return sg;
  }

  // One shard's forward/backward; its gradient lands in `gtarget` (learner.cpp:117-134).
  void run_shard(const tlg_segment_batch& b, int on_device, int shard, float* gtarget) {
    compute_shard(stage_shard(b, on_device, false), shard, gtarget);
  }

  // Trunk forward + policy/value heads with the parameter set P (the student's, or a
  // teacher's for the KL term, rlmath.cpp:145-155): head outputs [F][A+1] -> out,
  // log-prob of the taken action -> out_tlogp (may be null).
  // PPO with fused heads: the loss kernel reads the head partial sums directly (no target
  // log-prob is needed, so head_finalize_kernel is skipped)
  bool loss_reads_parts() const {
    return cfg.algo == TLG_ALGO_PPO && net.L > 0 && fused_head();
  }
  // PPO without a teacher: the top trunk GEMM's epilogue also runs the loss and writes
  // dZ_L directly (gemm kEpiFwdLoss; h_L never reaches HBM).  Opt-in (TLG_FUSED_LOSS=1):
  // correct, but at C3 the two-pass epilogue makes that GEMM epilogue-bound (276 us vs
  // 208 us for forward + loss kernels, profiles/r01_fused_loss.md).
  const bool fused_loss_disabled = std::getenv("TLG_FUSED_LOSS") == nullptr;
  bool fused_loss_ok(long F) const {
    return loss_reads_parts() && !teacher_active() && !fused_loss_disabled &&
           net.head.H <= 256 && F >= 256;
  }
  const tlg::gemm::LossEpi* fuse_loss_epi = nullptr;  // set while the fused step runs
  int fused_ctas = 0;

  void forward_heads(const Staged& sg, const float* P, const float* P_lo, const float* x0,
                     const float* x0_lo, float* out, float* out_tlogp, bool timed,
                     bool finalize = true) {
    const tlg::BatchDev bd = sg.bd;
    const long F = long(bd.S) * T;
    // ---- forward trunk
    using tlg::gemm::Operand;
    for (uint32_t l = 0; l < net.L; ++l) {
      const int in = net.gin(l), outw = int(net.dims[l + 1]);
      Operand A = l > 0       ? lo_op(act[l - 1], act_lo[l - 1], in, false)
                  : x0_has_lo ? lo_op(x0, x0_lo, in, false)
                              : Operand{x0, nullptr, in, false, x0_u8};
      Operand B{P + net.w_off[l], P_lo + net.w_off[l], in, false};
      if (l == 0 && net.padded()) {  // the padded copy of this plane's W_1
        B.hi = P == params ? w1p : tw1p;
        B.lo = P == params ? w1p_lo : tw1p_lo;
      }
      tlg::gemm::Params p{};
      p.out_hi = act[l];
      // the top layer's residual plane has no reader (heads and loss read the full plane)
      p.out_lo = l + 1 == net.L ? nullptr : act_lo[l];  // null unless TLG_LO_HBM
      p.ldo = outw;
      p.bias = P + net.b_off[l];
      const bool fuse_head = l + 1 == net.L && fused_head();
      if (fuse_head) {  // policy/value heads in the last trunk GEMM's epilogue
        p.head_w = P + net.head.wpi;
        p.head_wv = P + net.head.wv;
        p.head_k = int(net.A) + 1;
        p.head_part = head_part;
      }
      const bool fuse_loss = fuse_head && fuse_loss_epi != nullptr;
      if (fuse_loss) {  // ... and the PPO loss: the epilogue writes dZ_L instead of h_L
        p.loss = *fuse_loss_epi;
        p.out_hi = dz[l];
        p.out_lo = dz_lo_plane(int(l), x0_u8) ? dz_lo[l] : nullptr;
      }
      if (l == 0 && sg.x0_bits != nullptr && wq_src != P) {
        // this step's layer-1 weights of plane P -> int8 pieces (once per step and plane)
        tlg::gemm::launch_quantize_rows(P + net.w_off[0], outw, int(net.D), int(net.D), wq, wq_kp,
                                        wq_scale, stream);
        wq_src = P;
        ++launches;
      }
      if (timed) kmark(0, int(l), 0);
      int slices;  // fused heads: the launch's partial slices per row
      if (l == 0 && sg.x0_bits != nullptr) {
        // binary planes x int8 weight pieces: exact integer tensor-core GEMM (+ the
        // activations as int8 pieces when layer 2 takes the int8 path too)
        slices = tlg::gemm::launch_i8_bits_fwd(sg.x0_bits, bits_pitch, wq, wq_kp, wq_scale, p.bias,
                                           int(F), outw, int(net.D), act[0],
                                           net.L > 1 ? act_lo[0] : nullptr, outw,
                                           stream,
                                           i8_fwd2(F) ? act_q : nullptr).head_slices;
      } else if (l == 1 && sg.x0_bits != nullptr && i8_fwd2(F)) {
        tlg::gemm::launch_quantize_rows(P + net.w_off[1], outw, in, in, w2q, in, w2_scale,
                                        stream);
        ++launches;
        slices = tlg::gemm::launch_i8x2_fwd(act_q, w2q, in, w2_scale, p.bias, int(F), outw, in,
                                        act[1], p.out_lo, outw, p.head_w, p.head_wv, p.head_k,
                                        p.head_part, stream).head_slices;
      } else if (fuse_loss) {
        const tlg::gemm::LaunchInfo li =
            tlg::gemm::launch(A, B, int(F), outw, in, tlg::gemm::kEpiFwdLoss, p, 1, stream);
        slices = li.head_slices;
        fused_ctas = li.ctas;
      } else {
        slices = tlg::gemm::launch(A, B, int(F), outw, in, tlg::gemm::kEpiFwdTanh, p, 1, stream)
                     .head_slices;
      }
      if (timed) kmark(0, int(l), 1);
      if (fuse_head) head_tiles = slices;
      ++launches;
    }
    const float* hL = net.L ? act[net.L - 1] : x0;
    const long ldh = net.head.H;
    if (net.L > 0 && fused_head()) {
      if (!finalize) return;
      tlg::launch_head_finalize(net.head, P, head_part, head_tiles, F, &bd, out, out_tlogp,
                                nullptr, nullptr, nullptr, err, stream);
    } else {
      tlg::launch_head_forward(net.head, P, hL, ldh, &bd, F, out, out_tlogp, nullptr, err, stream);
    }
    launches += 1;
  }

  // Trunk backward from dZ_L: dW / db per layer (split-K, fixed-order reductions), dX with
  // tanh' for the layer below, then the rank-ordered shard accumulation and failure guard.
  // Trunk backward from dZ_L.  (1) the dX chain top down -- dZ_{l-1} = (dZ_l . W_l) *
  // (1 - X_{l-1}^2) -- with db_{l-1} reduced right after each dX from the column partials
  // its epilogue wrote; (2) the weight gradients bottom up (dW split-K + fixed-order
  // reduce), so the widest bucket (layer 1 holds ~88 % of C3's parameters) reaches the
  // comm stream first and its allreduce runs under the remaining dW GEMMs; then the
  // rank-ordered shard accumulation.
  void backward_trunk(const Staged& sg, int shard, float* gtarget, const float* x0,
                      const float* x0_lo, long F) {
    using tlg::gemm::Operand;
    const bool i8dw = sg.x0_bits != nullptr && i8_dw1();
    for (int l = int(net.L) - 1; l >= 1; --l) {
      const int in = int(net.dims[l]), outw = int(net.dims[l + 1]);
      Operand A2 = lo_op(dz[l], dz_lo[l], outw, false);
      Operand B2{params + net.w_off[l], params_lo + net.w_off[l], in, true};
      tlg::gemm::Params p2{};
      p2.out_hi = dz[l - 1];
      p2.out_lo = dz_lo_plane(l - 1, sg.x0_u8) ? dz_lo[l - 1] : nullptr;
      p2.ldo = in;
      p2.act_hi = act[l - 1];
      p2.ld_act = in;
      p2.colsum = col_partial;
      if (l == 1 && i8dw) {
        // dZ_1 feeds only the int8 dW: column maxima per split instead of a residual plane
        int sp_i8, kbps;
        i8_dw_plan(F, sp_i8, kbps);
        TLG_CUDA(cudaMemsetAsync(colmax, 0, size_t(sp_i8) * in * sizeof(unsigned), stream));
        p2.colmax = colmax;
        p2.colmax_rows = kbps * 128;
        p2.out_lo = nullptr;
      }
      if (shard == 0) kmark(2, l, 0);
      colsum_rows = tlg::gemm::launch(A2, B2, int(F), in, outw, tlg::gemm::kEpiBwdTanh, p2, 1,
                                      stream).ctas;
      if (shard == 0) kmark(2, l, 1);
      // db_{l-1} = column sums of dZ_{l-1} (col_partial is reused by the next dX)
      tlg::launch_rows_reduce(col_partial, colsum_rows, in, in, gtarget + net.b_off[l - 1],
                              stream);
      launches += 2;
    }
    for (int l = 0; l < int(net.L); ++l) {
      const int in = int(net.dims[l]), outw = int(net.dims[l + 1]);
      if (l == 0 && i8dw) {
        // dW_1 = dZ_1^T . X on the int8 tensor cores (exact int32 per split)
        int sp_i8, kbps;
        i8_dw_plan(F, sp_i8, kbps);
        tlg::gemm::launch_quantize_cols(dz[0], F, outw, outw, colmax, long(kbps) * 128, dzq,
                                        stream);
        // N = D_pad: the bit rows are zero past obs_dim, so the pad columns come out zero
        const int gin = net.gin(0);
        if (shard == 0) kmark(1, l, 0);
        tlg::gemm::launch_i8_bits_dw(dzq, sg.x0_bits, bits_pitch, colmax, outw, gin, int(F), kbps,
                                     ws, stream);
        if (shard == 0) kmark(1, l, 1);
        tlg::launch_dw_reduce(ws, sp_i8, long(outw) * gin,
                              net.padded() ? dw1p : gtarget + net.w_off[0], stream);
        if (net.padded())  // [h_1 x D_pad] -> the flat layout's [h_1 x D]
          TLG_CUDA(cudaMemcpy2DAsync(gtarget + net.w_off[0], size_t(in) * 4, dw1p,
                                     size_t(gin) * 4, size_t(in) * 4, size_t(outw),
                                     cudaMemcpyDeviceToDevice, stream));
        launches += 3;
      } else {
        // dW_l = dZ_l^T . X_{l-1}   (K = frames, split-K partials reduced in fixed order)
        const float* xin = l == 0 ? x0 : act[l - 1];
        const float* xin_lo = l == 0 ? x0_lo : act_lo[l - 1];
        const bool pad = l == 0 && net.padded();
        const int gin = net.gin(uint32_t(l));
        int sp = tlg::gemm::pick_splits(outw, gin, int(F), kMaxSplits);
        while (long(sp) * outw * gin > ws_elems && sp > 1) --sp;
        // layer 1 over uint8 planes (converted in smem, exact): dZ_1's residual plane
        const bool u8b = l == 0 && x0_u8 != nullptr;
        Operand A = u8b ? Operand{dz[0], dz_lo[0], outw, true} : lo_op(dz[l], dz_lo[l], outw, true);
        Operand B = u8b ? Operand{nullptr, nullptr, gin, true, x0_u8}
                    : (l > 0 || x0_has_lo) ? lo_op(xin, xin_lo, gin, true)
                                           : Operand{xin, nullptr, gin, true};
        tlg::gemm::Params p{};
        p.ws = ws;
        p.ws_split_stride = long(outw) * gin;
        const int kb = (int(F) + tlg::gemm::kBK - 1) / tlg::gemm::kBK;
        const int per = (kb + sp - 1) / sp;
        const int sp_eff = (kb + per - 1) / per;  // launch() drops empty splits the same way
        if (shard == 0) kmark(1, l, 0);
        tlg::gemm::launch(A, B, outw, gin, int(F), tlg::gemm::kEpiStore, p, sp, stream);
        if (shard == 0) kmark(1, l, 1);
        tlg::launch_dw_reduce(ws, sp_eff, long(outw) * gin, pad ? dw1p : gtarget + net.w_off[l],
                              stream);
        if (pad)  // [h_1 x D_pad] -> the flat layout's [h_1 x D]
          TLG_CUDA(cudaMemcpy2DAsync(gtarget + net.w_off[0], size_t(in) * 4, dw1p,
                                     size_t(gin) * 4, size_t(in) * 4, size_t(outw),
                                     cudaMemcpyDeviceToDevice, stream));
        launches += 2;
      }
      // W_l and b_l are contiguous in the flat layout: one bucket, allreduced while the
      // dW GEMMs of the layers above run
      bucket_ready(net.w_off[l], long(outw) * in + outw, l + 1 == int(net.L));
    }
    if (gtarget != grad) {
      accumulate_grad();  // grad += shard gradient, in rank order (learner.cpp:145-147)
    }
  }

  void compute_shard(const Staged& sg, int shard, float* gtarget) {
    tlg::StepStatsDev* st = stats + shard;
    const tlg::BatchDev bd = sg.bd;
    const float* x0 = sg.x0;
    const bool obs_exact = sg.exact;
    x0_u8 = sg.x0_u8;
    S_last = bd.S;
    const long F = long(bd.S) * T;
    const long D = net.D;
    const float* x0_lo = nullptr;
    x0_has_lo = net.L > 0 && !obs_exact;
    if (net.padded() && !(sg.x0_bits != nullptr && i8_dw1())) {
      // observation rows at D_pad floats for the tf32 GEMMs that read them (pad columns
      // stay zero from allocation); the int8 layer-1 kernels read the bit rows instead
      TLG_CUDA(cudaMemcpy2DAsync(obs_pad, size_t(net.D_pad) * 4, x0, size_t(D) * 4,
                                 size_t(D) * 4, size_t(F), cudaMemcpyDeviceToDevice, stream));
      x0 = obs_pad;
    }
    if (x0_has_lo && lo_hbm) {
      tlg::launch_split_lo(x0, obs_lo, F * long(net.gin(0)), stream);
      ++launches;
      x0_lo = obs_lo;
    }
    if (shard == 0) mark(1);
    if (teacher_active()) {
      // the teacher's head outputs first (the student's forward then reuses the buffers)
      forward_heads(sg, teacher, teacher_lo, x0, x0_lo, t_head_out, nullptr, false);
    }
    const bool parts = loss_reads_parts();
    tlg::HyperDev hd{float(hp.gamma), float(hp.lam), float(hp.clip_eps), float(hp.vf_coef),
                     float(hp.ent_coef), float(hp.rho_bar), float(hp.c_bar), hp.adv_norm,
                     float(hp.kl_teacher_coef)};
    const int algo = int(cfg.algo);
    if (fused_loss_ok(F)) {
      // GAE + advantage statistics need no forward output (rlmath.cpp:62-78, 18-34)
      const int rpb = tlg::launch_returns(bd, algo, hd, tlogp, adv, target, seg_partial, err, stream);
      tlg::launch_finalize_adv(seg_partial, bd, hp.adv_norm, st, err, stream, rpb);
      tlg::gemm::LossEpi le{};
      le.action = bd.action;
      le.blogp = bd.blogp;
      le.valid = bd.valid;
      le.T = T;
      le.adv = adv;
      le.target = target;
      le.stats = reinterpret_cast<const double*>(st);
      le.clip_eps = hd.clip_eps;
      le.vf_coef = hd.vf_coef;
      le.ent_coef = hd.ent_coef;
      le.bpi = net.head.bpi;
      le.bv = net.head.bv;
      le.params = params;
      le.hg_partial = hg_partial;
      le.db_partial = col_partial;
      le.loss_partial = loss_partial;
      le.err = err;
      // the CTA count is known only at launch: bias partials follow the weight partials of
      // at most num_sms() rows
      const long nw = long(net.A + 1) * net.head.H;
      le.bias_partial = hg_partial + long(tlg::gemm::num_sms()) * nw;
      fuse_loss_epi = &le;
      forward_heads(sg, params, params_lo, x0, x0_lo, head_out, tlogp, shard == 0, false);
      fuse_loss_epi = nullptr;
      if (shard == 0) mark(2);
      tlg::LossLaunch ll{fused_ctas, fused_ctas};
      // (+ the failure guard: the shard's loss and error flags are final here)
      tlg::launch_head_grad_reduce(net.head, hg_partial, loss_partial, ll, gtarget, st, stream,
                                   le.bias_partial, err, grad + P_pad);
      bucket_ready(net.head.wpi, net.P - net.head.wpi, net.L == 0, /*with_guard=*/true);
      tlg::launch_rows_reduce(col_partial, fused_ctas, net.head.H, net.head.H,
                              gtarget + net.b_off[net.L - 1], stream);
      launches += 5;
      if (shard == 0) mark(3);
      backward_trunk(sg, shard, gtarget, x0, x0_lo, F);
      return;
    }
    forward_heads(sg, params, params_lo, x0, x0_lo, head_out, tlogp, shard == 0, !parts);
    if (shard == 0) mark(2);
    // ---- heads, returns, loss
    const float* hL = net.L ? act[net.L - 1] : x0;
    const long ldh = net.head.H;
    const int rpb = tlg::launch_returns(bd, algo, hd, tlogp, adv, target, seg_partial, err, stream);
    tlg::launch_finalize_adv(seg_partial, bd, hp.adv_norm, st, err, stream, rpb);
    const int loss_kind = algo == TLG_ALGO_VTRACE ? 1 : 0;
    const tlg::LossLaunch ll = tlg::launch_loss_backward(
        net.head, params, hL, ldh, bd, head_out, adv, target, st, hd, loss_kind, dzh,
        net.L ? dz[net.L - 1] : nullptr,
        net.L && dz_lo_plane(int(net.L) - 1, x0_u8) ? dz_lo[net.L - 1] : nullptr, hg_partial,
        loss_partial, col_partial, stream, teacher_active() ? t_head_out : nullptr,
        parts ? head_part : nullptr, head_tiles, err);
    // (+ the failure guard: the shard's loss and error flags are final here)
    // (+ db of the top trunk layer from the loss kernel's column partials, same launch)
    const bool fuse_db = net.L > 0 && tlg::rows_reduce_threads(long(net.A + 1) * net.head.H) ==
                                          tlg::rows_reduce_threads(net.head.H);
    tlg::launch_head_grad_reduce(net.head, hg_partial, loss_partial, ll, gtarget, st, stream,
                                 nullptr, err, grad + P_pad, fuse_db ? col_partial : nullptr,
                                 fuse_db ? gtarget + net.b_off[net.L - 1] : nullptr);
    bucket_ready(net.head.wpi, net.P - net.head.wpi, net.L == 0, /*with_guard=*/true);
    launches += 6;
    if (net.L > 0 && !fuse_db) {  // db of the top trunk layer from the loss kernel's partials
      tlg::launch_rows_reduce(col_partial, ll.stream_blocks, net.head.H, net.head.H,
                              gtarget + net.b_off[net.L - 1], stream);
      ++launches;
    }
    if (shard == 0) mark(3);
    backward_trunk(sg, shard, gtarget, x0, x0_lo, F);
  }

  // Learner::TrainStep over `n` local shards (+ the communicator's other ranks).
  // Small steps are launch-bound: after staging into the learner's own buffers, the
  // whole device step (kernels, allreduce, optimizer, stats D2H) replays as one CUDA graph.
  bool use_graph(const tlg_segment_batch*, int n) const {
    return !cfg.timing && n == 1 && !graph_disabled && comm_warm;
  }
  // NCCL connects its transports lazily at a communicator's first collectives, which
  // must not happen under stream capture: the first step after comm init runs eagerly
  bool comm_warm = true;
  // graph of a step over an external device-resident batch, keyed by its pointers
  struct ExtGraph {
    const void* ptrs[8] = {};
    uint32_t S = 0, dtype = 0, pitch = 0;
    int slot = 0;  // index into graphs[]
    uint64_t last_use = 0;
  };
  static void batch_ptrs(const tlg_segment_batch& b, const void* out[8]) {
    out[0] = b.obs;
    out[1] = b.action;
    out[2] = b.reward;
    out[3] = b.behavior_logp;
    out[4] = b.value_est;
    out[5] = b.done;
    out[6] = b.bootstrap;
    out[7] = b.valid_steps;
  }
  // graphs[] slot for this external batch (LRU over kExtGraphs entries)
  int ext_graph_slot(const tlg_segment_batch& b) {
    const void* ptrs[8];
    batch_ptrs(b, ptrs);
    ++graph_clock;
    for (auto& e : ext)
      if (std::equal(ptrs, ptrs + 8, e.ptrs) && e.S == b.n_segments && e.dtype == b.obs_dtype &&
          e.pitch == b.obs_pitch) {
        e.last_use = graph_clock;
        return e.slot;
      }
    ExtGraph* v = nullptr;
    if (int(ext.size()) < kExtGraphs) {
      ext.push_back(ExtGraph{});
      v = &ext.back();
      v->slot = 3 + int(ext.size()) - 1;
    } else {
      v = &*std::min_element(ext.begin(), ext.end(), [](const ExtGraph& x, const ExtGraph& y) {
        return x.last_use < y.last_use;
      });
      Graph& g = graphs[v->slot];
      if (g.exec) cudaGraphExecDestroy(g.exec);
      g = Graph{};
    }
    std::copy(ptrs, ptrs + 8, v->ptrs);
    v->S = b.n_segments;
    v->dtype = b.obs_dtype;
    v->pitch = b.obs_pitch;
    v->last_use = graph_clock;
    return v->slot;
  }

  void step(const tlg_segment_batch* bs, int n, int on_device, tlg_step_stats* out,
            cudaEvent_t consumed = nullptr, const tlg_segment_batch* stage_next = nullptr) {
    if (!hp_set) throw InvalidArg("hyperparameters not set");
    // PpoLossAndGrad (rlmath.cpp:119-120); the PG (V-trace) loss takes no teacher
    if (hp.kl_teacher_coef > 0.0 && cfg.algo != TLG_ALGO_VTRACE && !has_teacher)
      throw InvalidArg("teacher params required when kl_teacher_coef > 0");
    if (n < 1 || n > kMaxLocalShards) throw InvalidArg("1..64 local shards per call");
    launches = 0;
    TLG_CUDA(cudaSetDevice(cfg.device));
    if (use_graph(bs, n)) {
      // a batch staged by stage_async is read in place (its slot's graph), as is any other
      // device-resident batch (a graph per batch address, LRU); host batches are copied
      // into the learner's own buffers first (binding 0)
      int bind = 0;
      if (on_device) {
        for (int k = 0; k < 2; ++k)
          if (slots[k].ready && bs[0].action == slots[k].action) bind = 1 + k;
        if (bind == 0) bind = ext_graph_slot(bs[0]);
      }
      const Staged sg = stage_shard(bs[0], on_device, /*internal=*/bind == 0);
      const long key = long(sg.bd.S) * 8 + (sg.x0_u8 ? 1 : 0) + (sg.exact ? 2 : 0) +
                       (sg.x0_bits ? 4 : 0);
      Graph& gr = graphs[bind];
      const bool slot_bind = bind == 1 || bind == 2;  // staging slots (3.. = external)
      if (!gr.exec || key != gr.key || gr.hyper != hyper_version ||
          (slot_bind && gr.obs != slots[bind - 1].obs)) {
        if (gr.exec) cudaGraphExecDestroy(gr.exec);
        gr.exec = nullptr;
        cudaGraph_t g;
        TLG_CUDA(cudaStreamBeginCapture(stream, cudaStreamCaptureModeThreadLocal));
        try {
          enqueue_device_step(&sg, 1);
        } catch (...) {
          // leave the stream usable: end (and drop) the partial capture before reporting
          cudaGraph_t partial = nullptr;
          cudaStreamEndCapture(stream, &partial);
          if (partial) cudaGraphDestroy(partial);
          cudaGetLastError();
          throw;
        }
        TLG_CUDA(cudaStreamEndCapture(stream, &g));
        TLG_CUDA(cudaGraphInstantiate(&gr.exec, g, 0));
        cudaGraphDestroy(g);
        gr.key = key;
        gr.hyper = hyper_version;
        gr.launches = launches;
        gr.obs = slot_bind ? slots[bind - 1].obs : nullptr;
      }
      TLG_CUDA(cudaGraphLaunch(gr.exec, stream));
      launches = gr.launches;
      S_last = sg.bd.S;  // host code of the captured step ran only at capture
    } else {
      enqueue_device_step(nullptr, n, bs, on_device);
    }
    if (consumed) TLG_CUDA(cudaEventRecord(consumed, stream));
    // host-side staging of the next batch while this step runs on the device; the step
    // has already been launched, so its results are checked before a staging error is
    // reported (the parameters have moved: the caller must see the step's own outcome)
    if (stage_next) {
      try {
        stage_async(*stage_next);
      } catch (...) {
        finish(n, out);
        throw;
      }
    }
    finish(n, out);
  }

  // ---- asynchronous staging: H2D of the next batch overlaps the current step
  struct Slot {
    void* obs = nullptr;
    size_t obs_bytes = 0;
    int32_t* action = nullptr;
    float *reward = nullptr, *blogp = nullptr, *value = nullptr, *boot = nullptr;
    uint8_t* done = nullptr;
    int32_t* valid = nullptr;
    cudaEvent_t ready = nullptr, consumed = nullptr;
    tlg_segment_batch dev{};
  };
  Slot slots[2];
  int slot_next = 0, slot_count = 0, slot_head = 0;
  cudaStream_t copy_stream = nullptr;

  // everything stage() would reject, checked before any copy is queued (the copy sizes
  // derive from obs_dim / obs_dtype / obs_pitch, so a mismatch would over-read the host)
  void check_stage(const tlg_segment_batch& b) const {
    if (int(b.n_segments) > S_max || b.n_segments == 0) throw InvalidArg("bad batch size");
    if (int(b.unroll_len) != T) throw InvalidArg("unroll_len mismatch");
    if (b.obs_dim != net.D) throw InvalidArg("observation size does not match policy shape");
    if (b.obs_dtype != TLG_OBS_F32 && b.obs_dtype != TLG_OBS_U8 && b.obs_dtype != TLG_OBS_BITS)
      throw InvalidArg("unknown obs dtype");
    if (b.obs_dtype != TLG_OBS_F32 && obs_u8 == nullptr)
      throw InvalidArg("learner not configured for uint8 / bit-packed observations");
    if (b.obs_dtype == TLG_OBS_BITS && b.obs_pitch != 0 &&
        long(b.obs_pitch) != (long(net.D) + 7) / 8 && long(b.obs_pitch) != bits_pitch)
      throw InvalidArg("obs_pitch must be 0, ceil(obs_dim/8) or that rounded up to 16 bytes");
  }

  void stage_async(const tlg_segment_batch& b) {
    if (slot_count == 2) throw InvalidArg("both staging slots hold untrained batches");
    check_stage(b);
    if (!copy_stream) TLG_CUDA(cudaStreamCreateWithFlags(&copy_stream, cudaStreamNonBlocking));
    Slot& sl = slots[slot_next];
    const long S = b.n_segments, F = S * T, D = net.D;
    const size_t ob = b.obs_dtype == TLG_OBS_F32 ? size_t(F * D) * 4
                      : b.obs_dtype == TLG_OBS_U8 ? size_t(F * D)
                                                  : size_t(F * (b.obs_pitch ? long(b.obs_pitch)
                                                                             : (D + 7) / 8));
    if (!sl.ready) {
      TLG_CUDA(cudaEventCreateWithFlags(&sl.ready, cudaEventDisableTiming));
      TLG_CUDA(cudaEventCreateWithFlags(&sl.consumed, cudaEventDisableTiming));
      sl.action = mem.add<int32_t>(F_max);
      sl.reward = mem.add<float>(F_max);
      sl.blogp = mem.add<float>(F_max);
      sl.value = mem.add<float>(F_max);
      sl.done = mem.add<uint8_t>(F_max);
      sl.boot = mem.add<float>(S_max);
      sl.valid = mem.add<int32_t>(S_max);
    }
    if (sl.obs_bytes < ob) {
      sl.obs = mem.add<uint8_t>(ob + 16);
      sl.obs_bytes = ob;
    }
    TLG_CUDA(cudaStreamWaitEvent(copy_stream, sl.consumed, 0));
    auto cp = [&](void* dst, const void* src, size_t bytes) {
      TLG_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, copy_stream));
    };
    cp(sl.obs, b.obs, ob);
    cp(sl.action, b.action, F * 4);
    cp(sl.reward, b.reward, F * 4);
    cp(sl.blogp, b.behavior_logp, F * 4);
    cp(sl.value, b.value_est, F * 4);
    cp(sl.done, b.done, F);
    cp(sl.boot, b.bootstrap, S * 4);
    cp(sl.valid, b.valid_steps, S * 4);
    TLG_CUDA(cudaEventRecord(sl.ready, copy_stream));
    sl.dev = b;
    sl.dev.obs = sl.obs;
    sl.dev.action = sl.action;
    sl.dev.reward = sl.reward;
    sl.dev.behavior_logp = sl.blogp;
    sl.dev.value_est = sl.value;
    sl.dev.done = sl.done;
    sl.dev.bootstrap = sl.boot;
    sl.dev.valid_steps = sl.valid;
    slot_next ^= 1;
    ++slot_count;
  }

  void train_staged(tlg_step_stats* out, const tlg_segment_batch* next = nullptr) {
    if (slot_count == 0) throw InvalidArg("no staged batch");
    if (next) check_stage(*next);  // fail before the step is launched
    Slot& sl = slots[slot_head];
    slot_head ^= 1;
    --slot_count;
    TLG_CUDA(cudaStreamWaitEvent(stream, sl.ready, 0));
    step(&sl.dev, 1, /*on_device=*/1, out, sl.consumed, next);
  }


  // Everything after staging: per-shard compute, allreduce, optimizer, stats D2H.
  void enqueue_device_step(const Staged* staged, int n, const tlg_segment_batch* bs = nullptr,
                           int on_device = 0) {
    launches = 0;
    wq_src = nullptr;  // the parameters changed since the last step
    if (net.padded()) {  // this step's W_1 planes at D_pad columns
      pad_rows(params + net.w_off[0], net.dims[1], int(net.D), int(net.D_pad), w1p, stream);
      pad_rows(params_lo + net.w_off[0], net.dims[1], int(net.D), int(net.D_pad), w1p_lo, stream);
      launches += 2;
    }
    overlap_active = nranks > 1 && n == 1 && overlap_requested;
    n_buckets = 0;
    pend_count = 0;
    pend_guard = false;
    mark(0);
    TLG_CUDA(cudaMemsetAsync(err, 0, 16, stream));
    TLG_CUDA(cudaMemsetAsync(grad + P_pad, 0, 16, stream));
    for (int r = 0; r < n; ++r) {
      if (staged) compute_shard(staged[r], r, r == 0 ? grad : grad_tmp);
      else run_shard(bs[r], on_device, r, r == 0 ? grad : grad_tmp);
    }
    mark(4);
    // ---- allreduce over ranks (learner.cpp:138-149); the guard slot rides along
    if (nranks > 1) {
      if (overlap_active) {
        bucket_flush();
      } else {
        NCCL_CHECK(tlg::nccl::api().AllReduce(grad, grad, size_t(P_pad + 4), ncclFloat, ncclSum,
                                              comm, stream));
      }
    }
    mark(5);
    // ---- optimizer (skipped on device when any shard of any rank failed); the Adam step
    // counter lives on the device so a captured graph replays correctly
    const bool adam = cfg.optimizer == TLG_OPT_ADAM;
    grad_scale = 1.f / float(n * nranks);
    launch_guarded_optimizer(adam, float(hp.learning_rate));
    mark(6);
    // ---- results
    TLG_CUDA(cudaMemcpyAsync(h_stats, stats, n * sizeof(tlg::StepStatsDev),
                             cudaMemcpyDeviceToHost, stream));
    TLG_CUDA(cudaMemcpyAsync(h_flags, err, 4, cudaMemcpyDeviceToHost, stream));
    TLG_CUDA(cudaMemcpyAsync(h_flags + 1, grad + P_pad, 4, cudaMemcpyDeviceToHost, stream));
  }

  void finish(int n, tlg_step_stats* out) {
    const bool adam = cfg.optimizer == TLG_OPT_ADAM;
    TLG_CUDA(cudaStreamSynchronize(stream));
    const int e = h_flags[0];
    float guard;
    std::memcpy(&guard, &h_flags[1], 4);
    const uint64_t k = steps_done + 1;
    if (e & tlg::kErrValidSteps) throw InvalidArg("valid_steps exceeds unroll_len");
    if (e & tlg::kErrEmptyBatch) throw InvalidArg("empty minibatch");
    if (e & tlg::kErrNotOneHot) throw InvalidArg("tabular observation must be one-hot");
    if (e & tlg::kErrActionRange) throw InvalidArg("action out of range");
    if (e & tlg::kErrNonFiniteLogp) throw InvalidArg("non-finite log probability");
    if (e & tlg::kErrNonFiniteAdv) throw InvalidArg("non-finite advantage");
    for (int r = 0; r < n; ++r)
      if (!std::isfinite(h_stats[r].loss))
        throw RuntimeErr("non-finite loss at update step " + std::to_string(k));
    if (guard != 0.f)
      throw RuntimeErr("learner shard failed on another rank at update step " + std::to_string(k));
    if (adam) ++adam_t;
    steps_done = k;
    comm_warm = true;
    if (out) {
      for (int r = 0; r < n; ++r) {
        const tlg::StepStatsDev& h = h_stats[r];
        out[r].loss = h.loss;
        out[r].clip_fraction = cfg.algo == TLG_ALGO_VTRACE ? 0.0 : h.clip;
        out[r].mean_ratio = h.ratio;
        out[r].entropy = h.entropy;
        out[r].value_loss = h.vloss;
        out[r].n_samples = uint64_t(h.n);
      }
    }
  }

  void accumulate_grad();
  bool fused_head() const { return net.A + 1 <= 8; }
  int colsum_rows = 0;
  int head_tiles = 1;
  void launch_guarded_optimizer(bool adam, float lr);
  struct Graph {
    cudaGraphExec_t exec = nullptr;
    long key = -1;
    uint64_t hyper = ~0ull;
    int launches = 0;
    const void* obs = nullptr;  // slot obs buffer the graph reads (slot bindings)
  };
  static constexpr int kExtGraphs = 64;
  // learner's own buffers, staging slot 0, staging slot 1, external device batches
  Graph graphs[3 + kExtGraphs];
  std::vector<ExtGraph> ext;
  uint64_t graph_clock = 0;
  uint64_t hyper_version = 0;
  bool graph_disabled = std::getenv("TLG_NO_GRAPH") != nullptr;
  uint64_t* adam_t_dev = nullptr;
  unsigned* opt_done = nullptr;  // blocks of the optimizer launch done (the last advances t)
};

namespace {

// guard[0] > 0 iff some shard raised an error bit or produced a non-finite loss; it is
// summed by the allreduce together with the gradient, so every rank agrees to skip.
__global__ void accumulate_kernel(float4* __restrict__ g, const float4* __restrict__ t, long n4) {
  TLG_PDL_ENTRY();
  for (long i = blockIdx.x * long(blockDim.x) + threadIdx.x; i < n4;
       i += long(gridDim.x) * blockDim.x) {
    float4 a = g[i];
    const float4 b = t[i];
    a.x += b.x; a.y += b.y; a.z += b.z; a.w += b.w;
    g[i] = a;
  }
}

// The block that finishes last advances the Adam step counter (when the step applied),
// after every block has read it: one launch instead of an optimizer + a counter kernel.
__device__ __forceinline__ void optimizer_block_done(bool applied, uint64_t* adam_t,
                                                     unsigned* done) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(done, 1u) == gridDim.x - 1) {
      if (applied) *adam_t += 1;
      *done = 0;  // ready for the next step (graph replays included)
      __threadfence();
    }
  }
}

__global__ void optimizer_guarded_kernel(float4* __restrict__ p, float4* __restrict__ plo,
                                         const float4* __restrict__ g, float4* __restrict__ m,
                                         float4* __restrict__ v, long n4, const float* guard,
                                         float grad_scale, int adam, float lr,
                                         uint64_t* adam_t, double b1d, double b2d,
                                         float eps, unsigned* done) {
  TLG_PDL_ENTRY();
  if (*guard != 0.f) {  // some shard failed: parameters stay untouched
    optimizer_block_done(false, adam_t, done);
    return;
  }
  // torch.optim.Adam bias corrections for step t = (completed steps) + 1
  const double t = double(*adam_t + 1);
  const float step_size = float(double(lr) / (1.0 - pow(b1d, t)));
  const float bc2_sqrt = float(sqrt(1.0 - pow(b2d, t)));
  const float b1 = float(b1d), b2 = float(b2d);
  for (long i = blockIdx.x * long(blockDim.x) + threadIdx.x; i < n4;
       i += long(gridDim.x) * blockDim.x) {
    float4 pp = p[i];
    const float4 gg = g[i];
    float* pe = &pp.x;
    const float* ge = &gg.x;
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
    plo[i] = make_float4(pp.x - tlg::tf32_hi(pp.x), pp.y - tlg::tf32_hi(pp.y),
                         pp.z - tlg::tf32_hi(pp.z), pp.w - tlg::tf32_hi(pp.w));
  }
  optimizer_block_done(true, adam_t, done);
}

__global__ void split_lo_flat(const float* x, float* lo, long n) {
  TLG_PDL_ENTRY();
  long i = blockIdx.x * long(blockDim.x) + threadIdx.x;
  if (i < n) lo[i] = x[i] - tlg::tf32_hi(x[i]);
}

}  // namespace

void tlg_learner::issue_bucket(long off, long count, bool with_guard) {
  if (n_buckets >= kMaxBuckets) throw RuntimeErr("too many gradient buckets");
  cudaEvent_t& e = bucket_ev[n_buckets++];
  if (!e) TLG_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  TLG_CUDA(cudaEventRecord(e, stream));
  TLG_CUDA(cudaStreamWaitEvent(comm_stream, e, 0));
  const auto& nc = tlg::nccl::api();
  if (with_guard && count > 0) NCCL_CHECK(nc.GroupStart());
  if (count > 0)
    NCCL_CHECK(nc.AllReduce(grad + off, grad + off, size_t(count), ncclFloat, ncclSum, comm,
                            comm_stream));
  if (with_guard) {
    NCCL_CHECK(nc.AllReduce(grad + P_pad, grad + P_pad, 4, ncclFloat, ncclSum, comm,
                            comm_stream));
    if (count > 0) NCCL_CHECK(nc.GroupEnd());
  }
}

void tlg_learner::bucket_flush() {
  issue_bucket(pend_off, pend_count, pend_guard);
  if (!comm_done) TLG_CUDA(cudaEventCreateWithFlags(&comm_done, cudaEventDisableTiming));
  TLG_CUDA(cudaEventRecord(comm_done, comm_stream));
  TLG_CUDA(cudaStreamWaitEvent(stream, comm_done, 0));  // joins the capture, if any
}

void tlg_learner::accumulate_grad() {
  const long n4 = P_pad / 4;
  ::tlg::launch_k(accumulate_kernel, dim3(int(std::max<long>(1, std::min<long>((n4 + 255) / 256, 148L * 4)))), dim3(256), size_t(0), stream, reinterpret_cast<float4*>(grad),
                                reinterpret_cast<const float4*>(grad_tmp), n4);
  TLG_CHECK_LAUNCH();
  ++launches;
}

void tlg_learner::launch_guarded_optimizer(bool adam, float lr) {
  const long n4 = P_pad / 4;
  const int blocks = int(std::max<long>(1, std::min<long>((n4 + 255) / 256, 148L * 4)));
  ::tlg::launch_k(optimizer_guarded_kernel, dim3(blocks), dim3(256), size_t(0), stream, 
      reinterpret_cast<float4*>(params), reinterpret_cast<float4*>(params_lo),
      reinterpret_cast<const float4*>(grad), reinterpret_cast<float4*>(adam_m),
      reinterpret_cast<float4*>(adam_v), n4, grad + P_pad, grad_scale, adam ? 1 : 0, lr,
      adam_t_dev, cfg.adam_beta1, cfg.adam_beta2, float(cfg.adam_eps), opt_done);
  TLG_CHECK_LAUNCH();
  launches += 1;
}

// ===========================================================================
struct tlg_policy {
  Net net;
  int device;
  long max_batch;
  cudaStream_t stream = nullptr;
  DevFree mem;
  float *params, *params_lo, *obs, *obs_lo, *head_out, *head_part, *logits, *probs, *value;
  std::vector<float*> act, act_lo;
  // net.padded(): observation rows and W_1 at D_pad columns (see Net)
  float *obs_pad = nullptr, *w1p = nullptr, *w1p_lo = nullptr;
  void pad_w1() {
    if (!net.padded()) return;
    pad_rows(params + net.w_off[0], net.dims[1], int(net.D), int(net.D_pad), w1p, stream);
    pad_rows(params_lo + net.w_off[0], net.dims[1], int(net.D), int(net.D_pad), w1p_lo, stream);
  }
  int* err;
  long P_pad;
  int head_tiles = 1;
  // Layers >= 2 as exact int8 x int8 tensor-core GEMMs (gemm_i8x2_fwd_kernel): each
  // layer's tanh outputs leave its epilogue as three fixed-scale int8 pieces (1/127) and the
  // weights of layers >= 2 as per-row-scaled pieces (quantized when the parameters are
  // set), so the 1024-wide layers run at the int8 instruction rate instead of three tf32
  // passes.  The pair kernel tiles 256 rows: batches are evaluated on at least kMinRows
  // rows (the extra rows are scratch), so every batch size takes the same path and a row's
  // outputs do not depend on the batch it came in.  Opt-in (TLG_POLICY_I8=1): at C4 the
  // int8 x int8 kernel streams its operands from L2 at 64-column tiles (three accumulators
  // fill TMEM) and the layer-1 epilogue pays for the piece stores, 0.73 ms per batch
  // against 0.62 ms for 3xTF32.
  static constexpr long kMinRows = 256;
  bool i8 = false;
  long rows_cap = 0;                // max(max_batch, kMinRows)
  int8_t* act_q[2] = {nullptr, nullptr};  // ping-pong [3][rows][h_l]
  std::vector<int8_t*> wq;          // [l] pieces [3][h_{l+1}][h_l], l >= 1
  std::vector<float*> wscale;       // [l] row scales [h_{l+1}]
  bool i8_eligible() const {
    if (net.L < 2) return false;
    const char* e = std::getenv("TLG_POLICY_I8");
    if (!e || std::atoi(e) != 1) return false;
    for (uint32_t l = 1; l < net.L; ++l)  // pieces need 32-column chunks, K % 16
      if (net.dims[l] % 32 != 0) return false;
    return true;
  }
  // parameters changed: padded W_1 and the int8 weight pieces of layers >= 2
  void prepare_params() {
    pad_w1();
    if (!i8) return;
    for (uint32_t l = 1; l < net.L; ++l) {
      const int in = int(net.dims[l]), outw = int(net.dims[l + 1]);
      tlg::gemm::launch_quantize_rows(params + net.w_off[l], outw, in, in, wq[l], in, wscale[l],
                                      stream);
    }
  }
  // pipelined batches (tlg_policy_forward_async): two slots of device inputs / outputs, an
  // H2D and a D2H stream around the compute stream, events ordering slot reuse
  struct Slot {
    float *obs = nullptr, *logits = nullptr, *probs = nullptr, *value = nullptr;
    int* err = nullptr;       // this batch's error flags (device), read back with its outputs
    int* err_host = nullptr;  // pinned
    cudaEvent_t h2d = nullptr, computed = nullptr, d2h = nullptr;
    uint64_t ticket = 0;
  };
  Slot pipe[2];
  cudaStream_t h2d_stream = nullptr, d2h_stream = nullptr;
  uint64_t next_ticket = 1, done_ticket = 0;

  tlg_policy(const tlg_policy_shape& s, int dev, long mb) : net(s), device(dev), max_batch(mb) {
    if (mb <= 0) throw InvalidArg("max_batch must be >= 1");
    TLG_CUDA(cudaSetDevice(dev));
    TLG_CUDA(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking));
    P_pad = pad4(net.P);
    params = mem.add<float>(P_pad);
    params_lo = mem.add<float>(P_pad);
    i8 = i8_eligible();
    rows_cap = i8 ? std::max(mb, kMinRows) : mb;
    obs = mem.add<float>(rows_cap * net.D);
    obs_lo = nullptr;
    if (i8) {
      long widest = 0;
      for (uint32_t l = 1; l < net.L; ++l) widest = std::max(widest, long(net.dims[l]));
      for (int8_t*& q : act_q) q = mem.add<int8_t>(3 * rows_cap * widest);
      wq.assign(net.L, nullptr);
      wscale.assign(net.L, nullptr);
      for (uint32_t l = 1; l < net.L; ++l) {
        wq[l] = mem.add<int8_t>(3 * long(net.dims[l + 1]) * net.dims[l]);
        wscale[l] = mem.add<float>(net.dims[l + 1]);
      }
      // scratch rows start as zeros (finite); they never reach a caller's outputs
      TLG_CUDA(cudaMemsetAsync(obs, 0, size_t(rows_cap * net.D) * 4, stream));
    }
    if (net.padded()) {
      obs_pad = mem.add<float>(rows_cap * net.D_pad);
      if (i8) TLG_CUDA(cudaMemsetAsync(obs_pad, 0, size_t(rows_cap * net.D_pad) * 4, stream));
      w1p = mem.add<float>(long(net.dims[1]) * net.D_pad);
      w1p_lo = mem.add<float>(long(net.dims[1]) * net.D_pad);
    }
    head_out = mem.add<float>(mb * (net.A + 1));
    head_part = mem.add<float>(rows_cap * (net.A + 1) * head_slices_max(net.head.H));
    logits = mem.add<float>(mb * net.A);
    probs = mem.add<float>(mb * net.A);
    value = mem.add<float>(mb);
    err = mem.add<int>(4);
    for (uint32_t l = 0; l < net.L; ++l) {
      // int8 layers keep their activations as pieces only; the top layer's fp32 plane is
      // only read when the heads are not fused
      const bool plane = !i8 || (l + 1 == net.L && net.A + 1 > 8);
      act.push_back(plane ? mem.add<float>(mb * net.dims[l + 1]) : nullptr);
      act_lo.push_back(nullptr);
    }
  }
  // Enqueue one forward of n device-resident observations on `stream`; error flags are
  // or-ed into errp (default: `err`).
  void enqueue(const float* x0, long n, float* lg, float* pr, float* vv, int* errp = nullptr);
  void open_pipe() {
    if (h2d_stream) return;
    TLG_CUDA(cudaStreamCreateWithFlags(&h2d_stream, cudaStreamNonBlocking));
    TLG_CUDA(cudaStreamCreateWithFlags(&d2h_stream, cudaStreamNonBlocking));
    for (Slot& sl : pipe) {
      sl.obs = mem.add<float>(rows_cap * net.D);
      sl.logits = mem.add<float>(max_batch * net.A);
      sl.probs = mem.add<float>(max_batch * net.A);
      sl.value = mem.add<float>(max_batch);
      sl.err = mem.add<int>(4);
      TLG_CUDA(cudaMallocHost(&sl.err_host, 16));
      TLG_CUDA(cudaEventCreateWithFlags(&sl.h2d, cudaEventDisableTiming));
      TLG_CUDA(cudaEventCreateWithFlags(&sl.computed, cudaEventDisableTiming));
      TLG_CUDA(cudaEventCreateWithFlags(&sl.d2h, cudaEventDisableTiming));
    }
  }
  ~tlg_policy() {
    for (Slot& sl : pipe) {
      if (sl.h2d) cudaEventSynchronize(sl.d2h), cudaEventDestroy(sl.h2d);
      if (sl.computed) cudaEventDestroy(sl.computed);
      if (sl.d2h) cudaEventDestroy(sl.d2h);
      if (sl.err_host) cudaFreeHost(sl.err_host);
    }
    if (h2d_stream) cudaStreamDestroy(h2d_stream);
    if (d2h_stream) cudaStreamDestroy(d2h_stream);
    if (stream) {
      cudaStreamSynchronize(stream);
      cudaStreamDestroy(stream);
    }
  }
};

namespace {

__global__ void unpack_head_kernel(const float* head_out, int A, long n, float* logits,
                                   float* value) {
  TLG_PDL_ENTRY();
  const long i = blockIdx.x * long(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  for (int k = 0; k < A; ++k) logits[i * A + k] = head_out[i * (A + 1) + k];
  value[i] = head_out[i * (A + 1) + A];
}

void set_params_common(float* params, float* params_lo, long P, long P_pad, const double* values,
                       size_t n, cudaStream_t stream) {
  if (long(n) != P) throw InvalidArg("parameter count mismatch");
  std::vector<float> h(P_pad, 0.f);
  for (long i = 0; i < P; ++i) h[i] = float(values[i]);
  TLG_CUDA(cudaMemcpyAsync(params, h.data(), P_pad * 4, cudaMemcpyHostToDevice, stream));
  ::tlg::launch_k(split_lo_flat, dim3(int((P_pad + 255) / 256)), dim3(256), size_t(0), stream, params, params_lo, P_pad);
  TLG_CHECK_LAUNCH();
  TLG_CUDA(cudaStreamSynchronize(stream));
}

}  // namespace

void tlg_policy::enqueue(const float* x0, long n, float* lg, float* pr, float* vv, int* errp) {
  const long D = net.D, A = net.A;
  int* err = errp ? errp : this->err;
  // rows the GEMMs evaluate: the int8 pair kernels tile 256 rows (see kMinRows)
  const long m = i8 ? std::max(n, kMinRows) : n;
  if (net.padded()) {
    TLG_CUDA(cudaMemcpy2DAsync(obs_pad, size_t(net.D_pad) * 4, x0, size_t(D) * 4, size_t(D) * 4,
                               size_t(n), cudaMemcpyDeviceToDevice, stream));
    x0 = obs_pad;
  } else if (m > n && x0 != obs) {
    TLG_CUDA(cudaMemcpyAsync(obs, x0, size_t(n * D) * 4, cudaMemcpyDeviceToDevice, stream));
    x0 = obs;
  }
  // the tf32 residuals of the observations and activations are derived in the GEMMs'
  // shared memory (Operand::lo_smem): no residual planes
  using tlg::gemm::Operand;
  for (uint32_t l = 0; l < net.L; ++l) {
    const int in = net.gin(l), outw = int(net.dims[l + 1]);
    Operand Aop{l == 0 ? x0 : act[l - 1], nullptr, in, false};
    Aop.lo_smem = true;
    Operand Bop{params + net.w_off[l], params_lo + net.w_off[l], in, false};
    if (l == 0 && net.padded()) {
      Bop.hi = w1p;
      Bop.lo = w1p_lo;
    }
    tlg::gemm::Params gp{};
    const bool fuse = l + 1 == net.L && net.A + 1 <= 8;
    // with fused heads nothing reads the top layer's plane
    gp.out_hi = fuse ? nullptr : act[l];
    gp.out_lo = nullptr;
    gp.ldo = outw;
    gp.bias = params + net.b_off[l];
    if (fuse) {
      gp.head_w = params + net.head.wpi;
      gp.head_wv = params + net.head.wv;
      gp.head_k = int(A) + 1;
      gp.head_part = head_part;
    }
    int8_t* q_out = i8 && l + 1 < net.L ? act_q[l & 1] : nullptr;
    int slices;  // fused heads: the launch's partial slices per row
    if (i8 && l >= 1) {
      slices = tlg::gemm::launch_i8x2_fwd(act_q[(l - 1) & 1], wq[l], in, wscale[l], gp.bias,
                                          int(m), outw, in, gp.out_hi, nullptr, outw, gp.head_w,
                                          gp.head_wv, gp.head_k, gp.head_part, stream, q_out)
                   .head_slices;
    } else {
      gp.out_q = q_out;
      if (q_out) gp.out_hi = nullptr;  // the next layer reads the pieces
      slices = tlg::gemm::launch(Aop, Bop, int(m), outw, in, tlg::gemm::kEpiFwdTanh, gp, 1, stream)
                   .head_slices;
    }
    if (fuse) head_tiles = slices;
  }
  const float* hL = net.L ? act[net.L - 1] : x0;
  if (net.L > 0 && net.A + 1 <= 8) {
    tlg::launch_head_finalize(net.head, params, head_part, head_tiles, n, nullptr, nullptr,
                              nullptr, lg, pr, vv, err, stream, m);
  } else {
    tlg::launch_head_forward(net.head, params, hL, net.head.H, nullptr, n, head_out, nullptr, pr,
                             err, stream);
    ::tlg::launch_k(unpack_head_kernel, dim3(int((n + 255) / 256)), dim3(256), size_t(0), stream,
                    head_out, int(A), n, lg, vv);
  }
}

// ===========================================================================
extern "C" {

const char* tlg_last_error(void) { return g_err.c_str(); }
const char* tlg_version(void) { return "tlg_b200 0.2 (sm_100a, tcgen05 3xTF32 / int8)"; }

int tlg_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

void* tlg_host_alloc(size_t bytes) {
  void* p = nullptr;
  if (cudaMallocHost(&p, bytes ? bytes : 1) != cudaSuccess) {
    g_err = "cudaMallocHost failed";
    return nullptr;
  }
  return p;
}

void tlg_host_free(void* p) {
  if (p) cudaFreeHost(p);
}

int tlg_learner_create(const tlg_learner_config* cfg, const tlg_policy_shape* shape,
                       tlg_learner** out) {
  return Guard([&] {
    if (!cfg || !shape || !out) throw InvalidArg("null argument");
    *out = new tlg_learner(*cfg, *shape);
  });
}

void tlg_learner_destroy(tlg_learner* l) { delete l; }

size_t tlg_learner_param_count(const tlg_learner* l) { return l ? size_t(l->net.P) : 0; }

int tlg_learner_set_params(tlg_learner* l, const double* values, size_t n) {
  return Guard([&] {
    TLG_CUDA(cudaSetDevice(l->cfg.device));
    set_params_common(l->params, l->params_lo, l->net.P, l->P_pad, values, n, l->stream);
    TLG_CUDA(cudaMemsetAsync(l->adam_m, 0, l->P_pad * 4, l->stream));
    TLG_CUDA(cudaMemsetAsync(l->adam_v, 0, l->P_pad * 4, l->stream));
    TLG_CUDA(cudaMemsetAsync(l->adam_t_dev, 0, 8, l->stream));
    TLG_CUDA(cudaStreamSynchronize(l->stream));
    l->adam_t = 0;
  });
}

int tlg_learner_set_teacher(tlg_learner* l, const double* values, size_t n) {
  return Guard([&] {
    TLG_CUDA(cudaSetDevice(l->cfg.device));
    if (values == nullptr) {
      l->has_teacher = false;
    } else {
      if (!l->teacher) {
        l->teacher = l->mem.add<float>(l->P_pad);
        l->teacher_lo = l->mem.add<float>(l->P_pad);
        l->t_head_out = l->mem.add<float>(l->F_max * (l->net.A + 1));
      }
      set_params_common(l->teacher, l->teacher_lo, l->net.P, l->P_pad, values, n, l->stream);
      if (l->net.padded()) {
        const long n1 = long(l->net.dims[1]) * l->net.D_pad;
        if (!l->tw1p) {
          l->tw1p = l->mem.add<float>(n1);
          l->tw1p_lo = l->mem.add<float>(n1);
        }
        pad_rows(l->teacher + l->net.w_off[0], l->net.dims[1], int(l->net.D), int(l->net.D_pad),
                 l->tw1p, l->stream);
        pad_rows(l->teacher_lo + l->net.w_off[0], l->net.dims[1], int(l->net.D),
                 int(l->net.D_pad), l->tw1p_lo, l->stream);
      }
      TLG_CUDA(cudaStreamSynchronize(l->stream));
      l->has_teacher = true;
    }
    ++l->hyper_version;  // captured graphs include (or not) the teacher pass
  });
}

int tlg_learner_get_params(tlg_learner* l, double* values, size_t n) {
  return Guard([&] {
    if (long(n) != l->net.P) throw InvalidArg("parameter count mismatch");
    std::vector<float> h(l->net.P);
    TLG_CUDA(cudaMemcpyAsync(h.data(), l->params, l->net.P * 4, cudaMemcpyDeviceToHost,
                             l->stream));
    TLG_CUDA(cudaStreamSynchronize(l->stream));
    for (long i = 0; i < l->net.P; ++i) values[i] = double(h[i]);
  });
}

int tlg_learner_get_grad(tlg_learner* l, double* values, size_t n) {
  return Guard([&] {
    if (long(n) != l->net.P) throw InvalidArg("parameter count mismatch");
    std::vector<float> h(l->net.P);
    TLG_CUDA(cudaMemcpyAsync(h.data(), l->grad, l->net.P * 4, cudaMemcpyDeviceToHost,
                             l->stream));
    TLG_CUDA(cudaStreamSynchronize(l->stream));
    // the summed gradient times 1/(local shards x ranks) of the last step
    for (long i = 0; i < l->net.P; ++i) values[i] = double(h[i]) * double(l->grad_scale);
  });
}

int tlg_learner_get_returns(tlg_learner* l, float* adv, float* target, size_t n_frames) {
  return Guard([&] {
    const long F = long(l->S_last) * l->T;
    if (long(n_frames) < F) throw InvalidArg("buffer too small");
    TLG_CUDA(cudaMemcpyAsync(adv, l->adv, F * 4, cudaMemcpyDeviceToHost, l->stream));
    TLG_CUDA(cudaMemcpyAsync(target, l->target, F * 4, cudaMemcpyDeviceToHost, l->stream));
    TLG_CUDA(cudaStreamSynchronize(l->stream));
  });
}

int tlg_learner_set_hyper(tlg_learner* l, const tlg_hyper* hp) {
  return Guard([&] {
    // HyperParams::Validate subset (types.cpp:17-35)
    if (!(std::isfinite(hp->learning_rate) && hp->learning_rate > 0))
      throw InvalidArg("hyperparams: learning_rate must be > 0");
    if (!(hp->gamma > 0 && hp->gamma <= 1)) throw InvalidArg("hyperparams: gamma must be in (0, 1]");
    if (!(hp->lam >= 0 && hp->lam <= 1)) throw InvalidArg("hyperparams: lam must be in [0, 1]");
    if (!(hp->clip_eps > 0)) throw InvalidArg("hyperparams: clip_eps must be > 0");
    if (!(hp->rho_bar > 0) || !(hp->c_bar > 0) || hp->c_bar > hp->rho_bar)
      throw InvalidArg("hyperparams: need 0 < c_bar <= rho_bar");
    if (!(hp->kl_teacher_coef >= 0)) throw InvalidArg("kl_teacher_coef must be >= 0");
    l->hp = *hp;
    l->hp_set = true;
    ++l->hyper_version;
  });
}

int tlg_comm_unique_id(uint8_t out[128]) {
  return Guard([&] {
    ncclUniqueId id;
    NCCL_CHECK(tlg::nccl::api().GetUniqueId(&id));
    static_assert(sizeof(id) == 128, "ncclUniqueId size");
    std::memcpy(out, &id, 128);
  });
}

int tlg_learner_comm_init(tlg_learner* l, const uint8_t unique_id[128], int nranks, int rank) {
  return Guard([&] {
    if (nranks < 1 || rank < 0 || rank >= nranks) throw InvalidArg("bad rank / nranks");
    TLG_CUDA(cudaSetDevice(l->cfg.device));
    if (l->comm) {
      tlg::nccl::api().CommDestroy(l->comm);
      l->comm = nullptr;
    }
    l->nranks = nranks;
    l->rank = rank;
    l->comm_warm = nranks == 1;
    ++l->hyper_version;  // re-capture: the step graph embeds the communicator
    if (nranks > 1) {
      pin_nccl();
      ncclUniqueId id;
      std::memcpy(&id, unique_id, 128);
      NCCL_CHECK(tlg::nccl::api().CommInitRank(&l->comm, nranks, id, rank));
      l->make_comm_stream();
    }
  });
}

int tlg_learner_comm_init_all(tlg_learner* const* learners, int n) {
  return Guard([&] {
    if (!learners || n < 1 || n > 64) throw InvalidArg("1..64 learners");
    std::vector<int> devs(n);
    for (int i = 0; i < n; ++i) {
      if (!learners[i]) throw InvalidArg("null learner");
      devs[i] = learners[i]->cfg.device;
      for (int j = 0; j < i; ++j)
        if (devs[j] == devs[i]) throw InvalidArg("learners must be on distinct devices");
      if (learners[i]->net.P != learners[0]->net.P)
        throw InvalidArg("learners must share one policy shape");
    }
    for (int i = 0; i < n; ++i) {
      tlg_learner* l = learners[i];
      TLG_CUDA(cudaSetDevice(l->cfg.device));
      if (l->comm) {
        tlg::nccl::api().CommDestroy(l->comm);
        l->comm = nullptr;
      }
      l->nranks = n;
      l->rank = i;
      l->comm_warm = n == 1;
      ++l->hyper_version;
    }
    if (n == 1) return;
    pin_nccl();
    std::vector<ncclComm_t> comms(n);
    NCCL_CHECK(tlg::nccl::api().CommInitAll(comms.data(), n, devs.data()));
    for (int i = 0; i < n; ++i) {
      learners[i]->comm = comms[i];
      TLG_CUDA(cudaSetDevice(learners[i]->cfg.device));
      learners[i]->make_comm_stream();
    }
  });
}

// ---------------------------------------------------------------------------
// Device-resident replay ring
struct tlg_replay {
  tlg_learner* l = nullptr;
  // ingest runs on its own stream (a put does not wait for an in-flight step); a step's
  // gather waits for the last put through `ready`
  cudaStream_t stream = nullptr;
  cudaEvent_t ready = nullptr;
  uint32_t cap = 0, dtype = 0;
  long rowb = 0;  // bytes per frame row in the ring and the gathered batches
  DevFree mem;
  tlg::SegArrays ring{}, stage{}, gath{};
  long stage_segs = 0, stage_rowb = 0, gath_segs = 0;
  uint32_t *d_put_slots = nullptr, *d_gather_slots = nullptr;
  long put_slots_cap = 0, gather_slots_cap = 0;

  std::mutex alloc_mu;  // puts (ingest thread) and steps (trainer thread) both allocate

  tlg::SegArrays alloc(long segs, long rb) {
    std::lock_guard<std::mutex> g(alloc_mu);
    const int T = l->T;
    tlg::SegArrays a{};
    a.obs = mem.add<uint8_t>(segs * T * rb + 16);
    a.action = mem.add<int32_t>(segs * T);
    a.reward = mem.add<float>(segs * T);
    a.blogp = mem.add<float>(segs * T);
    a.value = mem.add<float>(segs * T);
    a.done = mem.add<uint8_t>(segs * T);
    a.boot = mem.add<float>(segs);
    a.valid = mem.add<int32_t>(segs);
    return a;
  }
  uint32_t* slots_to_device(uint32_t*& buf, long& capn, const uint32_t* h, long n,
                            cudaStream_t st) {
    for (long i = 0; i < n; ++i)
      if (h[i] >= cap) throw InvalidArg("replay slot out of range");
    if (capn < n) {
      std::lock_guard<std::mutex> g(alloc_mu);
      buf = mem.add<uint32_t>(n);
      capn = n;
    }
    TLG_CUDA(cudaMemcpyAsync(buf, h, n * 4, cudaMemcpyHostToDevice, st));
    return buf;
  }
  ~tlg_replay() {
    if (stream) {
      cudaStreamSynchronize(stream);
      cudaStreamDestroy(stream);
    }
    if (ready) cudaEventDestroy(ready);
  }
};

int tlg_replay_create(tlg_learner* l, uint32_t capacity, uint32_t obs_dtype, tlg_replay** out) {
  return Guard([&] {
    if (!l || !out) throw InvalidArg("null argument");
    if (capacity == 0) throw InvalidArg("replay capacity must be >= 1");
    if (obs_dtype != TLG_OBS_F32 && obs_dtype != TLG_OBS_BITS)
      throw InvalidArg("device replay stores fp32 or bit-packed observations");
    if (obs_dtype == TLG_OBS_BITS && l->obs_bits == nullptr)
      throw InvalidArg("learner not configured for bit-packed observations");
    TLG_CUDA(cudaSetDevice(l->cfg.device));
    auto r = std::make_unique<tlg_replay>();
    r->l = l;
    r->cap = capacity;
    r->dtype = obs_dtype;
    r->rowb = obs_dtype == TLG_OBS_BITS ? l->bits_pitch : long(l->net.D) * 4;
    r->ring = r->alloc(capacity, r->rowb);
    TLG_CUDA(cudaStreamCreateWithFlags(&r->stream, cudaStreamNonBlocking));
    TLG_CUDA(cudaEventCreateWithFlags(&r->ready, cudaEventDisableTiming));
    *out = r.release();
  });
}

void tlg_replay_destroy(tlg_replay* r) {
  if (r && r->l && r->l->stream) cudaStreamSynchronize(r->l->stream);  // no gather in flight
  delete r;
}

int tlg_replay_put(tlg_replay* r, const uint32_t* slots, const tlg_segment_batch* b) {
  return Guard([&] {
    if (!r || !slots || !b) throw InvalidArg("null argument");
    tlg_learner* l = r->l;
    TLG_CUDA(cudaSetDevice(l->cfg.device));
    const int T = l->T;
    const long n = b->n_segments, D = l->net.D;
    if (n == 0) return;
    if (int(b->unroll_len) != T) throw InvalidArg("unroll_len mismatch");
    if (b->obs_dim != l->net.D) throw InvalidArg("observation size does not match policy shape");
    if (b->obs_dtype != r->dtype) throw InvalidArg("observation format differs from the replay's");
    const long src_rowb = r->dtype == TLG_OBS_BITS
                              ? (b->obs_pitch ? long(b->obs_pitch) : (D + 7) / 8)
                              : D * 4;
    if (r->dtype == TLG_OBS_BITS && (src_rowb < (D + 7) / 8 || src_rowb > r->rowb))
      throw InvalidArg("bad obs_pitch");
    if (r->stage_segs < n || r->stage_rowb < src_rowb) {
      r->stage = r->alloc(n, std::max(src_rowb, r->rowb));
      r->stage_segs = n;
      r->stage_rowb = std::max(src_rowb, r->rowb);
    }
    const long F = n * T;
    auto h2d = [&](void* dst, const void* src, size_t bytes) {
      TLG_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, r->stream));
    };
    h2d(r->stage.obs, b->obs, size_t(F * src_rowb));
    h2d(r->stage.action, b->action, F * 4);
    h2d(r->stage.reward, b->reward, F * 4);
    h2d(r->stage.blogp, b->behavior_logp, F * 4);
    h2d(r->stage.value, b->value_est, F * 4);
    h2d(r->stage.done, b->done, F);
    h2d(r->stage.boot, b->bootstrap, n * 4);
    h2d(r->stage.valid, b->valid_steps, n * 4);
    const uint32_t* ds =
        r->slots_to_device(r->d_put_slots, r->put_slots_cap, slots, n, r->stream);
    tlg::launch_replay_move(r->stage, src_rowb, r->ring, r->rowb, ds, int(n), T, true, r->stream);
    TLG_CUDA(cudaEventRecord(r->ready, r->stream));
    TLG_CUDA(cudaStreamSynchronize(r->stream));  // the host batch may be reused on return
  });
}

int tlg_learner_train_step_replay(tlg_learner* l, tlg_replay* r, const uint32_t* slots,
                                  uint32_t n_shards, uint32_t per_shard, tlg_step_stats* stats) {
  return Guard([&] {
    if (!l || !r || !slots) throw InvalidArg("null argument");
    if (r->l != l) throw InvalidArg("replay belongs to another learner");
    if (n_shards == 0 || per_shard == 0) throw InvalidArg("empty minibatch");
    if (int(per_shard) > l->S_max) throw InvalidArg("batch exceeds the learner's max_segments");
    TLG_CUDA(cudaSetDevice(l->cfg.device));
    const long total = long(n_shards) * per_shard;
    const int T = l->T;
    if (r->gath_segs < total) {
      r->gath = r->alloc(total, r->rowb);
      r->gath_segs = total;
    }
    const uint32_t* ds =
        r->slots_to_device(r->d_gather_slots, r->gather_slots_cap, slots, total, l->stream);
    TLG_CUDA(cudaStreamWaitEvent(l->stream, r->ready, 0));
    tlg::launch_replay_move(r->ring, r->rowb, r->gath, r->rowb, ds, int(total), T, false,
                            l->stream);
    std::vector<tlg_segment_batch> bs(n_shards);
    for (uint32_t k = 0; k < n_shards; ++k) {
      const long s0 = long(k) * per_shard, f0 = s0 * T;
      tlg_segment_batch& b = bs[k];
      b.n_segments = per_shard;
      b.unroll_len = T;
      b.obs_dim = l->net.D;
      b.obs_dtype = r->dtype;
      b.obs_pitch = r->dtype == TLG_OBS_BITS ? uint32_t(r->rowb) : 0;
      b.obs = r->gath.obs + f0 * r->rowb;
      b.action = r->gath.action + f0;
      b.reward = r->gath.reward + f0;
      b.behavior_logp = r->gath.blogp + f0;
      b.value_est = r->gath.value + f0;
      b.done = r->gath.done + f0;
      b.bootstrap = r->gath.boot + s0;
      b.valid_steps = r->gath.valid + s0;
    }
    l->step(bs.data(), int(n_shards), /*on_device=*/1, stats);
  });
}

int tlg_learner_train_step(tlg_learner* l, const tlg_segment_batch* batch, int on_device,
                           tlg_step_stats* stats) {
  return Guard([&] {
    if (!l || !batch) throw InvalidArg("null argument");
    l->step(batch, 1, on_device, stats);
  });
}

int tlg_learner_train_step_shards(tlg_learner* l, const tlg_segment_batch* shards, int n_shards,
                                  int on_device, tlg_step_stats* stats) {
  return Guard([&] {
    if (!l || !shards) throw InvalidArg("null argument");
    l->step(shards, n_shards, on_device, stats);
  });
}

int tlg_learner_stage(tlg_learner* l, const tlg_segment_batch* host_batch) {
  return Guard([&] {
    TLG_CUDA(cudaSetDevice(l->cfg.device));
    l->stage_async(*host_batch);
  });
}

int tlg_learner_train_staged(tlg_learner* l, tlg_step_stats* stats) {
  return Guard([&] {
    TLG_CUDA(cudaSetDevice(l->cfg.device));
    l->train_staged(stats);
  });
}

int tlg_learner_train_staged_next(tlg_learner* l, const tlg_segment_batch* next_host_batch,
                                  tlg_step_stats* stats) {
  return Guard([&] {
    TLG_CUDA(cudaSetDevice(l->cfg.device));
    l->train_staged(stats, next_host_batch);
  });
}

void* tlg_learner_stream(tlg_learner* l) { return l ? static_cast<void*>(l->stream) : nullptr; }

int tlg_learner_phase_ms(tlg_learner* l, float* out, int n) {
  return Guard([&] {
    if (!l->cfg.timing) throw InvalidArg("learner created without timing");
    const int pairs[7][2] = {{0, 1}, {1, 2}, {2, 3}, {3, 4}, {4, 5}, {5, 6}, {0, 6}};
    for (int i = 0; i < n && i < 7; ++i)
      TLG_CUDA(cudaEventElapsedTime(&out[i], l->ev[pairs[i][0]], l->ev[pairs[i][1]]));
  });
}

int tlg_learner_last_launches(tlg_learner* l) { return l ? l->launches : 0; }

int tlg_learner_set_timing(tlg_learner* l, int on) {
  return Guard([&] { l->cfg.timing = on ? 1 : 0; });
}

int tlg_learner_kernel_ms(tlg_learner* l, int kind, int layer, float* ms) {
  return Guard([&] {
    if (!l->cfg.timing) throw InvalidArg("learner created without timing");
    if (kind < 0 || kind > 2 || layer < 0 || layer >= int(l->net.L))
      throw InvalidArg("no such GEMM");
    if (kind == 2 && layer == 0) throw InvalidArg("layer 1 has no dX GEMM");
    TLG_CUDA(cudaEventElapsedTime(ms, l->kev[kind][layer][0], l->kev[kind][layer][1]));
  });
}

int tlg_policy_create(const tlg_policy_shape* shape, int32_t device, uint32_t max_batch,
                      tlg_policy** out) {
  return Guard([&] { *out = new tlg_policy(*shape, device, long(max_batch)); });
}

void tlg_policy_destroy(tlg_policy* p) { delete p; }

int tlg_policy_set_params(tlg_policy* p, const double* values, size_t n) {
  return Guard([&] {
    TLG_CUDA(cudaSetDevice(p->device));
    set_params_common(p->params, p->params_lo, p->net.P, p->P_pad, values, n, p->stream);
    p->prepare_params();
    TLG_CUDA(cudaStreamSynchronize(p->stream));
  });
}

int tlg_policy_set_params_from_learner(tlg_policy* p, tlg_learner* l) {
  return Guard([&] {
    if (!p || !l) throw InvalidArg("null argument");
    if (p->net.P != l->net.P || p->net.dims != l->net.dims || p->net.A != l->net.A ||
        p->net.family != l->net.family)
      throw InvalidArg("policy and learner shapes differ");
    // learner stream -> policy stream: the copy sees the learner's last step; policy
    // stream -> learner stream: the learner's next optimizer step waits for the copy.
    // No host synchronisation; the planes (params and their tf32 residuals, kept in step
    // by the optimizer) cross NVLink peer-to-peer when the devices differ.
    cudaEvent_t ev_l, ev_p;
    TLG_CUDA(cudaSetDevice(l->cfg.device));
    TLG_CUDA(cudaEventCreateWithFlags(&ev_l, cudaEventDisableTiming));
    TLG_CUDA(cudaEventRecord(ev_l, l->stream));
    TLG_CUDA(cudaSetDevice(p->device));
    TLG_CUDA(cudaEventCreateWithFlags(&ev_p, cudaEventDisableTiming));
    TLG_CUDA(cudaStreamWaitEvent(p->stream, ev_l, 0));
    const size_t bytes = size_t(p->P_pad) * 4;
    if (p->device == int(l->cfg.device)) {
      TLG_CUDA(cudaMemcpyAsync(p->params, l->params, bytes, cudaMemcpyDeviceToDevice, p->stream));
      TLG_CUDA(cudaMemcpyAsync(p->params_lo, l->params_lo, bytes, cudaMemcpyDeviceToDevice,
                               p->stream));
    } else {
      TLG_CUDA(cudaMemcpyPeerAsync(p->params, p->device, l->params, int(l->cfg.device), bytes,
                                   p->stream));
      TLG_CUDA(cudaMemcpyPeerAsync(p->params_lo, p->device, l->params_lo, int(l->cfg.device),
                                   bytes, p->stream));
    }
    TLG_CUDA(cudaSetDevice(p->device));
    p->prepare_params();
    TLG_CUDA(cudaEventRecord(ev_p, p->stream));
    TLG_CUDA(cudaSetDevice(l->cfg.device));
    TLG_CUDA(cudaStreamWaitEvent(l->stream, ev_p, 0));
    TLG_CUDA(cudaEventDestroy(ev_l));  // destruction is deferred until the event completes
    TLG_CUDA(cudaEventDestroy(ev_p));
  });
}

int tlg_policy_forward(tlg_policy* p, const float* obs, size_t n, float* logits, float* probs,
                       float* value, int on_device) {
  return Guard([&] {
    if (n == 0) return;
    if (long(n) > p->max_batch) throw InvalidArg("batch exceeds max_batch");
    TLG_CUDA(cudaSetDevice(p->device));
    const long D = p->net.D, A = p->net.A;
    const float* x0 = obs;
    if (!on_device) {
      TLG_CUDA(cudaMemcpyAsync(p->obs, obs, n * D * 4, cudaMemcpyHostToDevice, p->stream));
      x0 = p->obs;
    }
    float* lg = on_device ? logits : p->logits;
    float* pr = on_device ? probs : p->probs;
    float* vv = on_device ? value : p->value;
    TLG_CUDA(cudaMemsetAsync(p->err, 0, 4, p->stream));
    p->enqueue(x0, long(n), lg, pr, vv);
    if (!on_device) {
      TLG_CUDA(cudaMemcpyAsync(logits, p->logits, n * A * 4, cudaMemcpyDeviceToHost, p->stream));
      TLG_CUDA(cudaMemcpyAsync(probs, p->probs, n * A * 4, cudaMemcpyDeviceToHost, p->stream));
      TLG_CUDA(cudaMemcpyAsync(value, p->value, n * 4, cudaMemcpyDeviceToHost, p->stream));
    }
    int e = 0;
    TLG_CUDA(cudaMemcpyAsync(&e, p->err, 4, cudaMemcpyDeviceToHost, p->stream));
    TLG_CUDA(cudaStreamSynchronize(p->stream));
    if (e & tlg::kErrNotOneHot) throw InvalidArg("tabular observation must be one-hot");
  });
}

int tlg_policy_forward_async(tlg_policy* p, const float* obs, size_t n, float* logits,
                             float* probs, float* value, uint64_t* ticket) {
  return Guard([&] {
    if (!p || !obs || !logits || !probs || !value || !ticket) throw InvalidArg("null argument");
    if (n == 0 || long(n) > p->max_batch) throw InvalidArg("batch must hold 1..max_batch rows");
    TLG_CUDA(cudaSetDevice(p->device));
    p->open_pipe();
    const uint64_t t = p->next_ticket;
    tlg_policy::Slot& sl = p->pipe[t & 1];
    // the slot's previous batch must have drained (its D2H read the slot's outputs)
    if (sl.ticket != 0) TLG_CUDA(cudaEventSynchronize(sl.d2h));
    const long D = p->net.D, A = p->net.A;
    // H2D (page-locked host memory overlaps the forward of the previous batch)
    TLG_CUDA(cudaStreamWaitEvent(p->h2d_stream, sl.computed, 0));  // the slot's obs are free
    TLG_CUDA(cudaMemcpyAsync(sl.obs, obs, n * D * 4, cudaMemcpyHostToDevice, p->h2d_stream));
    TLG_CUDA(cudaEventRecord(sl.h2d, p->h2d_stream));
    // forward on the policy stream
    TLG_CUDA(cudaStreamWaitEvent(p->stream, sl.h2d, 0));
    TLG_CUDA(cudaMemsetAsync(sl.err, 0, 4, p->stream));
    p->enqueue(sl.obs, long(n), sl.logits, sl.probs, sl.value, sl.err);
    TLG_CUDA(cudaEventRecord(sl.computed, p->stream));
    // D2H overlaps the next batch's forward
    TLG_CUDA(cudaStreamWaitEvent(p->d2h_stream, sl.computed, 0));
    TLG_CUDA(cudaMemcpyAsync(logits, sl.logits, n * A * 4, cudaMemcpyDeviceToHost, p->d2h_stream));
    TLG_CUDA(cudaMemcpyAsync(probs, sl.probs, n * A * 4, cudaMemcpyDeviceToHost, p->d2h_stream));
    TLG_CUDA(cudaMemcpyAsync(value, sl.value, n * 4, cudaMemcpyDeviceToHost, p->d2h_stream));
    TLG_CUDA(cudaMemcpyAsync(sl.err_host, sl.err, 4, cudaMemcpyDeviceToHost, p->d2h_stream));
    TLG_CUDA(cudaEventRecord(sl.d2h, p->d2h_stream));
    sl.ticket = t;
    p->next_ticket = t + 1;
    *ticket = t;
  });
}

int tlg_policy_wait(tlg_policy* p, uint64_t ticket) {
  return Guard([&] {
    if (!p) throw InvalidArg("null argument");
    if (ticket == 0 || ticket >= p->next_ticket) throw InvalidArg("unknown ticket");
    if (ticket <= p->done_ticket) return;
    if (ticket + 2 < p->next_ticket) throw InvalidArg("ticket no longer tracked (2 in flight)");
    TLG_CUDA(cudaSetDevice(p->device));
    tlg_policy::Slot& sl = p->pipe[ticket & 1];
    if (sl.ticket != ticket) throw InvalidArg("ticket no longer tracked");
    // the batch's outputs and error flags arrived together; the compute stream (already
    // running the next batch) is not synchronised
    TLG_CUDA(cudaEventSynchronize(sl.d2h));
    p->done_ticket = ticket;
    if (sl.err_host[0] & tlg::kErrNotOneHot)
      throw InvalidArg("tabular observation must be one-hot");
  });
}

void* tlg_policy_stream(tlg_policy* p) { return p ? static_cast<void*>(p->stream) : nullptr; }

int tlg_returns(uint32_t algo, const tlg_hyper* hp, uint32_t n_segments, uint32_t unroll_len,
                const float* reward, const float* value_est, const uint8_t* done,
                const float* bootstrap, const int32_t* valid_steps, const float* behavior_logp,
                const float* target_logp, float* adv, float* target, void* stream) {
  return Guard([&] {
    if (n_segments == 0 || unroll_len == 0) throw InvalidArg("segment length must be >= 1");
    if (algo != TLG_ALGO_PPO && target_logp == nullptr)
      throw InvalidArg("V-trace needs target log-probabilities");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    tlg::BatchDev bd{};
    bd.S = int(n_segments);
    bd.T = int(unroll_len);
    bd.reward = reward;
    bd.value = value_est;
    bd.done = done;
    bd.boot = bootstrap;
    bd.valid = valid_steps;
    bd.blogp = behavior_logp;
    tlg::HyperDev hd{float(hp->gamma), float(hp->lam), float(hp->clip_eps), float(hp->vf_coef),
                     float(hp->ent_coef), float(hp->rho_bar), float(hp->c_bar), hp->adv_norm};
    // per-device scratch, grown on demand (a per-call allocation costs more than the
    // kernels at small sizes); calls on one device are serialised by its mutex
    struct Scratch {
      std::mutex mu;
      void* buf = nullptr;
      size_t bytes = 0;
      int* host_err = nullptr;
    };
    static Scratch scratch[64];
    int dev = 0;
    TLG_CUDA(cudaGetDevice(&dev));
    Scratch& sc = scratch[dev & 63];
    std::lock_guard<std::mutex> lk(sc.mu);
    const size_t need = 64 + 24 * ((size_t(n_segments) + 7) / 8);
    if (sc.bytes < need) {
      if (sc.buf) TLG_CUDA(cudaFree(sc.buf));
      sc.buf = nullptr;
      sc.bytes = 0;
      TLG_CUDA(cudaMalloc(&sc.buf, need));
      sc.bytes = need;
    }
    if (!sc.host_err) TLG_CUDA(cudaMallocHost(reinterpret_cast<void**>(&sc.host_err), 4));
    int* err = static_cast<int*>(sc.buf);
    double* part = reinterpret_cast<double*>(static_cast<char*>(sc.buf) + 64);
    TLG_CUDA(cudaMemsetAsync(err, 0, 4, s));
    tlg::launch_returns(bd, int(algo == TLG_ALGO_PPO ? tlg::kAlgoPpo : tlg::kAlgoVtrace), hd,
                        target_logp, adv, target, part, err, s);
    TLG_CUDA(cudaMemcpyAsync(sc.host_err, err, 4, cudaMemcpyDeviceToHost, s));
    TLG_CUDA(cudaStreamSynchronize(s));
    const int e = *sc.host_err;
    if (e & tlg::kErrNonFiniteLogp) throw InvalidArg("non-finite log probability");
    if (e & tlg::kErrValidSteps) throw InvalidArg("valid_steps exceeds unroll_len");
  });
}

}  // extern "C"
