/* TEST INFRASTRUCTURE ONLY -- the CPU oracle (checker) for the B200 learner path.
 *
 * A plain fp64 restatement of the reference's hot-path arithmetic
 * (/root/reference/proj/src/{rlmath,policy,learner}), extended to the MLP
 * family, PPO-over-V-trace and Adam that the north star adds but the reference
 * cannot run.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference arm may load this library; the product path
 * (paper_2011_12895_b200) never links or calls it.
 *
 * Parity pinning: the tabular/linear families, GAE, lambda-return, V-trace,
 * PPO/PG loss+grad and SGD are pinned against the reference library itself
 * (oracle/_ref, built from the reference's own sources) and against the golden
 * fixtures in tests/golden/ generated from it.  The MLP family and Adam are
 * pinned by central finite differences (the reference's own FD pattern,
 * rlmath_test.cpp:268-365) and by torch-CPU float64 autograd.
 */
#ifndef TLG_ORACLE_H_
#define TLG_ORACLE_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* family: 0 tabular_softmax, 1 linear_softmax (types.hpp:14), 2 mlp (appended). */
typedef struct orc_shape {
  uint32_t family;
  uint32_t obs_dim;
  uint32_t n_actions;
  uint32_t n_hidden; /* mlp: number of tanh trunk layers */
  uint32_t hidden[8];
} orc_shape;

/* Mirrors tleague::HyperParams (types.hpp:36-57) minus the league-only Elo knobs. */
typedef struct orc_hyper {
  double learning_rate, gamma, lam, clip_eps, vf_coef, ent_coef, kl_teacher_coef, rho_bar,
      c_bar;
  uint32_t batch_size, unroll_len, max_reuse;
  int32_t adv_norm;
} orc_hyper;

/* SoA view of a slice of segments, [S][T] frame-major (segment-major, t-minor). */
typedef struct orc_segments {
  uint32_t n_segments, unroll_len, obs_dim;
  const double* obs;           /* [S][T][obs_dim] */
  const uint32_t* action;      /* [S][T] */
  const double* reward;        /* [S][T] */
  const double* behavior_logp; /* [S][T] */
  const double* value_est;     /* [S][T] */
  const uint8_t* done;         /* [S][T] */
  const double* bootstrap;     /* [S] */
  const uint32_t* valid_steps; /* [S] */
} orc_segments;

/* clip_fraction, mean_ratio, entropy, value_loss (rlmath.hpp:52-57) */
typedef struct orc_stats {
  double loss, clip_fraction, mean_ratio, entropy, value_loss;
  uint64_t n_samples;
} orc_stats;

const char* orc_last_error(void);

size_t orc_param_count(const orc_shape* s);
int orc_init_params(const orc_shape* s, double scale, uint64_t seed, double* out);
int orc_forward(const orc_shape* s, const double* params, const double* obs, size_t n,
                double* logits, double* probs, double* value);

int orc_gae(const double* r, const double* v, const uint8_t* done, size_t n, double boot,
            double gamma, double lam, double* adv);
int orc_lambda_return(const double* r, const double* v, const uint8_t* done, size_t n,
                      double boot, double gamma, double lam, double* ret);
int orc_vtrace(const double* bl, const double* tl, const double* r, const double* v,
               const uint8_t* done, size_t n, double boot, double gamma, double rho_bar,
               double c_bar, double* vs, double* pg_adv);

/* Per-minibatch losses over compacted samples (n >= 1). grad has orc_param_count entries. */
int orc_ppo_loss_grad(const orc_shape* s, const double* params, const double* teacher,
                      size_t n, const double* obs, const uint32_t* action, const double* blogp,
                      const double* adv, const double* vtarget, const orc_hyper* hp,
                      double* grad, orc_stats* stats);
int orc_pg_loss_grad(const orc_shape* s, const double* params, size_t n, const double* obs,
                     const uint32_t* action, const double* blogp, const double* adv,
                     const double* vtarget, const orc_hyper* hp, double* grad,
                     orc_stats* stats);

/* One shard of Learner::TrainStep (learner.cpp:56-102 + :126-128):
 * algo 0 = PPO (GAE + lambda-return, clipped surrogate),
 *      1 = V-trace (PG loss over V-trace targets, target logps under params),
 *      2 = PPO+V-trace (clipped surrogate over V-trace pg_adv / vs; config C5). */
int orc_shard_loss_grad(const orc_shape* s, const double* params, const orc_hyper* hp,
                        uint32_t algo, const orc_segments* segs, double* grad,
                        orc_stats* stats);

/* Optional per-frame outputs of the batch assembly (for kernel-level parity):
 * adv/target in [S][T] layout (padding frames left 0). */
int orc_shard_returns(const orc_shape* s, const double* params, const orc_hyper* hp,
                      uint32_t algo, const orc_segments* segs, double* adv, double* target);

int orc_sgd_step(const double* params, const double* grad, size_t n, double lr, double* out);
/* torch.optim.Adam semantics (no amsgrad, no weight decay); step is 1-based. */
int orc_adam_step(double* params, const double* grad, double* m, double* v, size_t n,
                  uint64_t step, double lr, double beta1, double beta2, double eps);

#ifdef __cplusplus
}
#endif
#endif /* TLG_ORACLE_H_ */
