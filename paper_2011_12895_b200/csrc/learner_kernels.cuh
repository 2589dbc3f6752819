// Non-GEMM kernels of the B200 learner step and InfServer forward.
//
//   K1  returns_kernel      GAE + lambda-return | V-trace (rho/c clip fused), one warp per
//                           segment, reverse affine warp scans over T      rlmath.cpp:45-114
//   K3a head_forward        policy/value heads, log-softmax, target logp  policy.cpp:73-105
//   K3b loss_backward       PPO / PG loss + dlogits/dvalue + head grads + tanh' of the
//                           last trunk layer                               rlmath.cpp:116-222
//   K7  optimizer_kernel    fused Adam (torch semantics) | SGD             rlmath.cpp:224-232
// plus deterministic (fixed-order) reductions for advantage normalisation
// (rlmath.cpp:18-34), split-K dW partials and bias column sums.
#pragma once

#include "common.cuh"

namespace tlg {

// Error bits raised on device, mapped to the reference's exceptions on the host.
enum ErrBits : int {
  kErrNonFiniteLogp = 1,    // rlmath.cpp:90-91   invalid_argument
  kErrActionRange = 2,      // rlmath.cpp:133     invalid_argument
  kErrNotOneHot = 4,        // policy.cpp:57-71   invalid_argument
  kErrNonFiniteAdv = 8,     // rlmath.cpp:22      invalid_argument
  kErrEmptyBatch = 16,      // rlmath.cpp:118     invalid_argument
  kErrValidSteps = 32,      // valid_steps > unroll_len
};

enum Algo : int { kAlgoPpo = 0, kAlgoVtrace = 1, kAlgoPpoVtrace = 2 };

// Policy/value head over the head input h (the last trunk activation, or the raw
// observation for the tabular/linear families).
struct HeadDesc {
  int family;   // 0 tabular, 1 linear, 2 mlp
  int A;        // n_actions
  int H;        // head input width
  long wpi;     // W_pi(k, j) = params[wpi + k*wk + j*wj]
  int wk, wj;
  long bpi;     // -1: no bias
  long wv;      // w_v(j) = params[wv + j]
  long bv;      // -1: no bias
};

struct BatchDev {
  int S, T;
  const int32_t* action;
  const float* reward;
  const float* blogp;
  const float* value;
  const uint8_t* done;
  const float* boot;
  const int32_t* valid;
};

struct HyperDev {
  float gamma, lam, clip_eps, vf_coef, ent_coef, rho_bar, c_bar;
  int adv_norm;
  float kl_coef;  // kl_teacher_coef (PPO with a teacher)
};

// Device-side per-step statistics (written by finalize kernels, read once by host).
struct StepStatsDev {
  double sum_adv, sum_adv2;
  double mean, sd;
  double inv_n;
  long long n;
  double loss, ratio, entropy, vloss, clip;
};

constexpr int kLossFrames = 128;  // frames per loss_backward chunk
constexpr int kLossBlocks = 444;  // persistent loss_backward blocks (3 per SM): partial rows

void launch_expand_u8(const uint8_t* in, float* out, long n, cudaStream_t s);
void launch_split_lo(const float* x, float* lo, long n, cudaStream_t s);
// Device-resident replay (learner.cu tlg_replay): scatter n segments of a contiguous
// staged batch into ring slots, or gather slots into a contiguous batch.  obs rows are
// copied byte-exactly (src_rowb -> dst_rowb bytes per frame, zero padded).
struct SegArrays {
  uint8_t* obs;
  int32_t* action;
  float *reward, *blogp, *value;
  uint8_t* done;
  float* boot;
  int32_t* valid;
};
void launch_replay_move(const SegArrays& src, long src_rowb, const SegArrays& dst, long dst_rowb,
                        const uint32_t* slots, int n, int T, bool scatter, cudaStream_t s);

void launch_unpack_bits(const uint8_t* bits, long rowb, long F, long D, uint8_t* out,
                        uint8_t* pitched, long pitch,
                        cudaStream_t s);
void launch_head_forward(const HeadDesc& hd, const float* params, const float* h, long ldh,
                         const BatchDev* b, long F, float* head_out, float* tlogp,
                         float* probs_out, int* err, cudaStream_t s);
// Fused-head finalisation (n_actions <= 7): part = [n_tiles][F][A+1] partial dot products
// from the last trunk GEMM epilogue.  Writes head_out [F][A+1] (+ tlogp with a batch),
// and/or logits/probs/value for inference.
void launch_head_finalize(const HeadDesc& hd, const float* params, const float* part,
                          int n_tiles, long F, const BatchDev* b, float* head_out, float* tlogp,
                          float* logits_out, float* probs_out, float* value_out, int* err,
                          cudaStream_t s, long part_rows = 0);
// returns the segments per block of the kernel it chose (the layout of seg_partial)
int launch_returns(const BatchDev& b, int algo, const HyperDev& hp, const float* tlogp,
                   float* adv, float* target, double* seg_partial, int* err, cudaStream_t s);
void launch_finalize_adv(const double* seg_partial, const BatchDev& b, int adv_norm,
                         StepStatsDev* st, int* err, cudaStream_t s, int segs_per_block);
struct LossLaunch {
  int stream_blocks;  // rows of the head-weight / last-layer-bias partials
  int math_blocks;    // rows of the loss/stat and head-bias partials
};
// dz/dz_lo may be null (no trunk).  dzh: scratch [F][A+1] (dlogits, dvalue).
LossLaunch launch_loss_backward(const HeadDesc& hd, const float* params, const float* h,
                                long ldh, const BatchDev& b, const float* head_out,
                                const float* adv, const float* target, const StepStatsDev* st,
                                const HyperDev& hp, int loss_kind, float* dzh, float* dz,
                                float* dz_lo, float* hg_partial, double* loss_partial,
                                float* db_partial, cudaStream_t s,
                                const float* teacher_out = nullptr,
                                const float* head_part = nullptr, int n_tiles = 0,
                                int* err = nullptr);
void launch_head_grad_reduce(const HeadDesc& hd, const float* hg_partial,
                             const double* loss_partial, const LossLaunch& ll, float* grad,
                             StepStatsDev* st, cudaStream_t s,
                             const float* bias_partial = nullptr, const int* err = nullptr,
                             float* guard = nullptr, const float* db_partial = nullptr,
                             float* db_out = nullptr);
// Fixed-order column reductions: warps of the block sum rows w, w + nw, ...; the block
// size (so the summation order) depends on the column count only.
constexpr int kRowWarps = 32;
inline int rows_reduce_threads(long cols) { return cols >= 8192 ? 256 : 32 * kRowWarps; }
// out[c] = sum_r partial[r*stride + c] for c < cols, fixed order (deterministic).
void launch_rows_reduce(const float* partial, int rows, long cols, long stride, float* out,
                        cudaStream_t s);
void launch_dw_reduce(const float* ws, int splits, long n, float* grad, cudaStream_t s);
// grad[j] = sum over rows of x[row][j] (fixed order); partial: scratch [chunks x cols]
void launch_colsum(const float* x, long ld, long rows, int cols, float* partial, float* grad,
                   cudaStream_t s);
void launch_optimizer(float* params, float* params_lo, const float* grad, float* m, float* v,
                      long n, float grad_scale, int adam, float lr, float step_size,
                      float bc2_sqrt, float b1, float b2, float eps, cudaStream_t s);

}  // namespace tlg
