/* tlg_b200.h -- C ABI of the B200-native TLeague learner / InferenceServer hot path.
 *
 * libtlg_b200.so (paper_2011_12895_b200/_lib/) is a plain C-ABI shared library:
 * no C++ or torch types cross it, every call returns an int status (0 = ok) and
 * never throws; tlg_last_error() holds the message of the last failure on the
 * calling thread.  Status codes map one to one onto the exceptions the reference
 * throws at the same boundary:
 *
 *   TLG_OK                0
 *   TLG_INVALID_ARGUMENT  1   std::invalid_argument   (rlmath.cpp:11-15,22,90-91,118-120,133;
 *                                                       policy.cpp:11-19,57-71)
 *   TLG_RUNTIME_ERROR     2   std::runtime_error      ("non-finite loss at update step k",
 *                                                       learner.cpp:141-144)
 *   TLG_CUDA_ERROR        3   device / driver failure (fail-stop)
 *
 * The entry points replace, one for one, the reference interfaces below
 * (paths relative to /root/reference/proj):
 *
 *   tlg_learner_*            learner::Learner::TrainStep math            src/learner/learner.cpp:56-158
 *     tlg_learner_train_step   BuildMinibatch + Ppo/PgLossAndGrad per shard,
 *                              rank-ordered gradient mean, SgdStep       learner.cpp:56-152
 *     tlg_learner_set_params   StartPeriod's params_ = record.params     learner.cpp:31-43
 *     tlg_learner_get_params   Publish's record.params = params_         learner.cpp:160-169
 *   tlg_policy_*             InfServer::BatchLoop per-batch evaluation    src/infserver/inf_server.cpp:125-144
 *                            (Distribution + ValueEstimate, policy.cpp:73-105)
 *   tlg_returns_*            rlmath::GaeAdvantages / LambdaReturn /
 *                            VtraceTargets over a [S][T] batch            src/rlmath/rlmath.cpp:45-114
 *
 * Data layout (host or device pointers as stated per call): a segment batch is
 * SoA, segment-major and t-minor ([S][T], frame f = s*T + t), the GPU mirror of
 * TrajectorySegment (types.hpp:82-104): only the first valid_steps[s] steps of
 * a segment are real; padding steps are excluded from every loss term.
 * Parameters cross as the reference's flat fp64 ParamBlob::values
 * (types.hpp:26-34) and live on the device as fp32.
 */
#ifndef TLG_B200_H_
#define TLG_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TLG_OK 0
#define TLG_INVALID_ARGUMENT 1
#define TLG_RUNTIME_ERROR 2
#define TLG_CUDA_ERROR 3

/* PolicyFamily (types.hpp:14); TLG_FAMILY_MLP is the appended wire tag 2. */
#define TLG_FAMILY_TABULAR 0
#define TLG_FAMILY_LINEAR 1
#define TLG_FAMILY_MLP 2

/* learner::Algo (learner.hpp:18); PPO_VTRACE = PPO clipped surrogate over V-trace
 * targets (config C5, appended). */
#define TLG_ALGO_PPO 0
#define TLG_ALGO_VTRACE 1
#define TLG_ALGO_PPO_VTRACE 2

#define TLG_OPT_SGD 0  /* rlmath::SgdStep, the reference optimizer */
#define TLG_OPT_ADAM 1 /* torch.optim.Adam semantics (north star) */

#define TLG_OBS_F32 0
#define TLG_OBS_U8 1 /* exact integer planes (e.g. Pommerman 0/1 features) */
#define TLG_OBS_BITS 2 /* 0/1 planes bit-packed LSB-first, ceil(obs_dim/8) bytes per frame */

/* Flat layout (family MLP): [W_1 (h1 x d), b_1, ..., W_L, b_L | W_pi (A x hL), b_pi |
 * w_v (hL), b_v], W row-major [out x in].  Tabular/linear keep the reference layout
 * (policy.cpp:23-27, 78-104). */
typedef struct tlg_policy_shape {
  uint32_t family;
  uint32_t obs_dim;
  uint32_t n_actions;
  uint32_t n_hidden; /* MLP trunk depth (tanh layers), <= 8 */
  uint32_t hidden[8];
} tlg_policy_shape;

/* tleague::HyperParams (types.hpp:36-57), learner-relevant fields. */
typedef struct tlg_hyper {
  double learning_rate, gamma, lam, clip_eps, vf_coef, ent_coef, kl_teacher_coef, rho_bar,
      c_bar;
  uint32_t batch_size, unroll_len, max_reuse;
  int32_t adv_norm;
} tlg_hyper;

typedef struct tlg_learner_config {
  uint32_t algo;           /* TLG_ALGO_* */
  uint32_t optimizer;      /* TLG_OPT_* */
  double adam_beta1, adam_beta2, adam_eps;
  uint32_t max_segments;   /* per-shard capacity S (the shard's batch_size) */
  uint32_t unroll_len;     /* T */
  int32_t device;          /* CUDA ordinal */
  uint32_t obs_dtype;      /* TLG_OBS_* accepted by train_step */
  uint32_t timing;         /* 1: record per-phase CUDA events each step */
} tlg_learner_config;

/* One shard's slice of the replay draw, SoA [S][T]. */
typedef struct tlg_segment_batch {
  uint32_t n_segments, unroll_len, obs_dim, obs_dtype;
  const void* obs;              /* [S][T][obs_dim] f32 or u8, or TLG_OBS_BITS: [S][T] rows of
                                   ceil(obs_dim / 8) bytes, 0/1 planes LSB first */
  const int32_t* action;        /* [S][T] */
  const float* reward;          /* [S][T] */
  const float* behavior_logp;   /* [S][T] */
  const float* value_est;       /* [S][T] */
  const uint8_t* done;          /* [S][T] */
  const float* bootstrap;       /* [S] */
  const int32_t* valid_steps;   /* [S] */
  uint32_t obs_pitch;           /* TLG_OBS_BITS: bytes per frame row, >= ceil(obs_dim / 8);
                                   0 = ceil(obs_dim / 8).  A multiple of 16 lets a device-
                                   resident batch feed the int8 GEMM without re-pitching. */
} tlg_segment_batch;

/* rlmath::LossStats (rlmath.hpp:52-57) plus the loss itself (mean over the shard's
 * valid samples) and the sample count.  Under data parallelism these are this
 * rank's own shard values. */
typedef struct tlg_step_stats {
  double loss, clip_fraction, mean_ratio, entropy, value_loss;
  uint64_t n_samples;
} tlg_step_stats;

typedef struct tlg_learner tlg_learner;
typedef struct tlg_policy tlg_policy;

const char* tlg_last_error(void);
const char* tlg_version(void);
/* CUDA devices visible to this process (0 without a driver / GPU). */
int tlg_device_count(void);
/* Page-locked host staging memory for the host-pointer calls (NULL on failure). */
void* tlg_host_alloc(size_t bytes);
void tlg_host_free(void* p);

/* ---- learner ------------------------------------------------------------ */
int tlg_learner_create(const tlg_learner_config* cfg, const tlg_policy_shape* shape,
                       tlg_learner** out);
void tlg_learner_destroy(tlg_learner* l);
size_t tlg_learner_param_count(const tlg_learner* l);
/* f64 -> device f32; also resets the optimizer state (StartPeriod). */
int tlg_learner_set_params(tlg_learner* l, const double* values, size_t n);
/* Teacher policy for the PPO KL penalty (rlmath.cpp:116-185, PpoLossAndGrad's `teacher`;
 * hyper kl_teacher_coef): f64 flat blob of the same shape; NULL clears it.  Without a
 * teacher, kl_teacher_coef > 0 fails the step with TLG_INVALID_ARGUMENT
 * ("teacher params required when kl_teacher_coef > 0", rlmath.cpp:119-120).  The V-trace
 * (PG) loss has no KL term, as in the reference. */
int tlg_learner_set_teacher(tlg_learner* l, const double* values, size_t n);
int tlg_learner_get_params(tlg_learner* l, double* values, size_t n);
int tlg_learner_set_hyper(tlg_learner* l, const tlg_hyper* hp);
/* Multi-GPU: join an NCCL communicator of `nranks` learner shards (one process or
 * thread per GPU).  `unique_id` is the 128-byte ncclUniqueId from
 * tlg_comm_unique_id on rank 0, distributed by the caller. */
int tlg_comm_unique_id(uint8_t out[128]);
int tlg_learner_comm_init(tlg_learner* l, const uint8_t unique_id[128], int nranks, int rank);
/* In-process data parallelism (one host thread per GPU, the reference's shard threads of
 * learner.cpp:117-134 mapped onto devices): one ncclCommInitAll over n learners created
 * on n distinct devices; learners[i] becomes rank i.  Steps must then be issued for all
 * n learners concurrently (one host thread each).  With one local shard per rank, each
 * layer's gradient bucket is allreduced on a high-priority comm stream as soon as the
 * backward has produced it, overlapping the layers below; NCCL_ALGO / NCCL_PROTO are
 * pinned (Ring; LL128,Simple) for run-to-run determinism unless already set or
 * TLG_NCCL_PIN=0. */
int tlg_learner_comm_init_all(tlg_learner* const* learners, int n);
/* One synchronized update over this rank's shard.  `batch` pointers are host
 * memory (copied in on the learner's stream; pinned memory is used as-is) when
 * on_device == 0, else device memory.  The gradient is averaged over the
 * communicator's ranks in a single fp32 sum-allreduce (learner.cpp:138-149),
 * then every rank applies the identical optimizer step. */
int tlg_learner_train_step(tlg_learner* l, const tlg_segment_batch* batch, int on_device,
                           tlg_step_stats* stats);
/* Learner::TrainStep with `n_shards` in-process shards on this GPU (the reference's
 * num_shards shard threads, learner.cpp:117-134): shard r's gradient is computed over
 * shards[r] with its own advantage normalisation and 1/n (rlmath.cpp:18-34,122), the
 * shard gradients are summed in rank order, allreduced with the other ranks, and
 * scaled by 1/(n_shards * nranks).  stats receives one entry per local shard. */
int tlg_learner_train_step_shards(tlg_learner* l, const tlg_segment_batch* shards, int n_shards,
                                  int on_device, tlg_step_stats* stats);
/* Pipelined host input: tlg_learner_stage queues an asynchronous H2D copy of a host
 * batch (pinned memory; it must stay valid until the step that consumes it returns)
 * into one of two device staging slots on a copy stream, so the transfer of step k+1
 * overlaps step k; tlg_learner_train_staged runs one step on the oldest staged batch. */
int tlg_learner_stage(tlg_learner* l, const tlg_segment_batch* host_batch);
int tlg_learner_train_staged(tlg_learner* l, tlg_step_stats* stats);
/* tlg_learner_train_staged, and — when next_host_batch is not NULL — tlg_learner_stage of
 * that batch issued while the step runs (after its launch, before its results are read),
 * so the host-side staging work leaves the critical path: one call per step. */
int tlg_learner_train_staged_next(tlg_learner* l, const tlg_segment_batch* next_host_batch,
                                  tlg_step_stats* stats);

/* Device-resident replay: segments are copied to HBM once, at ingest,
 * into `capacity` slots; a training step then names its segments by slot and the batch
 * is gathered on the device (replay_mem.cpp:14-49 keeps the draw decisions on the host:
 * the caller maps its draw to slots).  obs_dtype: TLG_OBS_F32 or TLG_OBS_BITS (rows
 * stored 16-byte pitched).  tlg_replay_put copies b->n_segments host segments into
 * slots[0..n); tlg_learner_train_step_replay runs one step over n_shards shards of
 * `per_shard` slots each (slots[r * per_shard + i], the reference's shard slices,
 * learner.cpp:122-124) and writes stats[n_shards]; results equal
 * tlg_learner_train_step_shards on the same segments.  Puts run on the replay's own
 * stream and may overlap a step on another host thread (puts themselves must be
 * serialised, and must not target slots of a step in flight). */
typedef struct tlg_replay tlg_replay;
int tlg_replay_create(tlg_learner* l, uint32_t capacity, uint32_t obs_dtype, tlg_replay** out);
void tlg_replay_destroy(tlg_replay* r);
int tlg_replay_put(tlg_replay* r, const uint32_t* slots, const tlg_segment_batch* host_batch);
int tlg_learner_train_step_replay(tlg_learner* l, tlg_replay* r, const uint32_t* slots,
                                  uint32_t n_shards, uint32_t per_shard, tlg_step_stats* stats);
/* The averaged gradient of the last step (f32 -> f64), for parity checks. */
int tlg_learner_get_grad(tlg_learner* l, double* out, size_t n);
/* Per-frame advantages / value targets of the last step ([S][T], f32, padding = 0). */
int tlg_learner_get_returns(tlg_learner* l, float* adv, float* target, size_t n_frames);
/* CUDA stream (cudaStream_t) the learner launches on. */
void* tlg_learner_stream(tlg_learner* l);
/* Per-phase device times (ms) of the last step when cfg.timing = 1:
 * [0] H2D staging, [1] forward GEMMs, [2] heads+returns+loss, [3] backward GEMMs+reductions,
 * [4] allreduce, [5] optimizer, [6] whole step.  n <= 7. */
int tlg_learner_phase_ms(tlg_learner* l, float* out, int n);
/* Toggle per-phase / per-GEMM event timing (timed steps launch eagerly, not as a graph). */
int tlg_learner_set_timing(tlg_learner* l, int on);
/* Kernel launches issued by the last train_step (this library's kernels only). */
int tlg_learner_last_launches(tlg_learner* l);
/* Device time (ms) of one trunk GEMM of the last step (timing mode): kind 0 = forward,
 * 1 = dW (split-K, without its reduce), 2 = dX; layer is 0-based. */
int tlg_learner_kernel_ms(tlg_learner* l, int kind, int layer, float* ms);

/* ---- inference (InfServer batched forward) ----------------------------- */
int tlg_policy_create(const tlg_policy_shape* shape, int32_t device, uint32_t max_batch,
                      tlg_policy** out);
void tlg_policy_destroy(tlg_policy* p);
int tlg_policy_set_params(tlg_policy* p, const double* values, size_t n);
/* Co-located refresh (replaces the fp64 blob round trip of
 * InfServer::RefreshNow, inf_server.cpp:41-48, when learner and server share a node):
 * copies the learner's fp32 parameter planes device-to-device (peer-to-peer across
 * GPUs), stream-ordered after the learner's last step and before its next one; no host
 * synchronisation.  Same result as tlg_policy_set_params(tlg_learner_get_params(l)).
 * Shapes must match (else TLG_INVALID_ARGUMENT). */
int tlg_policy_set_params_from_learner(tlg_policy* p, tlg_learner* l);
/* obs [n][obs_dim] f32; logits/probs [n][A] f32; value [n] f32.  Host pointers
 * when on_device == 0 (copied on the policy's stream), else device pointers.
 * Each row is evaluated independently of the others (batch-invariant). */
int tlg_policy_forward(tlg_policy* p, const float* obs, size_t n, float* logits, float* probs,
                       float* value, int on_device);
/* Pipelined batches from host memory (the InfServer's stream of request batches): enqueue
 * one batch -- H2D on a copy stream, the forward on the policy's stream, D2H on a second
 * copy stream -- and return at once with a ticket; batch k+1's H2D overlaps batch k's
 * forward and batch k-1's D2H (page-locked host buffers overlap; pageable ones still
 * work).  Two batches are in flight at most (enqueuing a third waits for the oldest).  A
 * batch's host buffers must stay valid until tlg_policy_wait(ticket) returns; results are
 * the same as tlg_policy_forward's.  tlg_policy_wait reports that batch's own errors
 * (TLG_INVALID_ARGUMENT: a tabular observation that is not one-hot) and never waits for
 * the batch enqueued after it. */
int tlg_policy_forward_async(tlg_policy* p, const float* obs, size_t n, float* logits,
                             float* probs, float* value, uint64_t* ticket);
int tlg_policy_wait(tlg_policy* p, uint64_t ticket);
void* tlg_policy_stream(tlg_policy* p);

/* ---- returns (K1) standalone -------------------------------------------- */
/* Device pointers, [S][T].  algo PPO: adv = GAE, target = lambda-return;
 * VTRACE / PPO_VTRACE: adv = pg_adv, target = vs (target_logp required). */
int tlg_returns(uint32_t algo, const tlg_hyper* hp, uint32_t n_segments, uint32_t unroll_len,
                const float* reward, const float* value_est, const uint8_t* done,
                const float* bootstrap, const int32_t* valid_steps, const float* behavior_logp,
                const float* target_logp, float* adv, float* target, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* TLG_B200_H_ */
