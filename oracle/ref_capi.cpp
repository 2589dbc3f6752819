// TEST INFRASTRUCTURE ONLY (oracle checker). Never linked into the product.
//
// extern "C" shim over the UNMODIFIED reference library compiled from
// /root/reference/proj/src by oracle/Makefile into oracle/_ref/.  It lets the
// Python tests, the golden-fixture generator and bench.py's cpu_baseline call
// the reference's own routines on identical inputs:
//
//   ref_gae / ref_lambda_return / ref_vtrace  -> rlmath.cpp:62-78, 45-60, 80-114
//   ref_init_params / ref_distribution / ref_value_estimate -> policy.cpp:29-105
//   ref_ppo_loss_grad / ref_pg_loss_grad       -> rlmath.cpp:116-185, 187-222
//   ref_sgd_step                               -> rlmath.cpp:224-232
//   ref_replay_*                               -> replay_mem.cpp:14-49
//   ref_learner_*                              -> learner.cpp:21-176 driven through
//                                                 LeagueState + DirectPool (as the
//                                                 reference's learner_test.cpp rig does)
//
// Errors: every entry point returns 0 on success, 1 for std::invalid_argument,
// 2 for std::runtime_error / other std::exception; ref_last_error() holds the
// message (thread-local).
#include <cstdint>
#include <cstring>
#include <memory>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "tleague/league/league_state.hpp"
#include "tleague/learner/learner.hpp"
#include "tleague/learner/replay_mem.hpp"
#include "tleague/policy/policy.hpp"
#include "tleague/pool/model_store.hpp"
#include "tleague/pool/pool_iface.hpp"
#include "tleague/rlmath/rlmath.hpp"

using namespace tleague;

namespace {

thread_local std::string g_err;

template <typename F>
int Guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 1;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 2;
  }
}

struct BoolArr {
  std::unique_ptr<bool[]> buf;
  std::span<const bool> span;
  BoolArr(const uint8_t* d, std::size_t n) : buf(new bool[n ? n : 1]) {
    for (std::size_t i = 0; i < n; ++i) buf[i] = d[i] != 0;
    span = std::span<const bool>(buf.get(), n);
  }
};

ParamBlob MakeBlob(uint32_t family, uint32_t obs_dim, uint32_t n_actions, const double* values) {
  ParamBlob b;
  b.family = static_cast<PolicyFamily>(family);
  b.shape = {obs_dim, n_actions};
  b.values.assign(values, values + policy::ParamCount(b.family, b.shape));
  return b;
}

}  // namespace

extern "C" {

// Mirrors tleague::HyperParams field for field (types.hpp:36-57).
struct ref_hyper {
  double learning_rate, gamma, lam, clip_eps, vf_coef, ent_coef, kl_teacher_coef, rho_bar,
      c_bar;
  uint32_t batch_size, unroll_len, max_reuse;
  int32_t adv_norm;
};

static HyperParams ToHyper(const ref_hyper* h) {
  HyperParams hp;
  hp.learning_rate = h->learning_rate;
  hp.gamma = h->gamma;
  hp.lam = h->lam;
  hp.clip_eps = h->clip_eps;
  hp.vf_coef = h->vf_coef;
  hp.ent_coef = h->ent_coef;
  hp.kl_teacher_coef = h->kl_teacher_coef;
  hp.rho_bar = h->rho_bar;
  hp.c_bar = h->c_bar;
  hp.batch_size = h->batch_size;
  hp.unroll_len = h->unroll_len;
  hp.max_reuse = h->max_reuse;
  hp.adv_norm = h->adv_norm != 0;
  return hp;
}

const char* ref_last_error() { return g_err.c_str(); }

int ref_gae(const double* r, const double* v, const uint8_t* done, std::size_t n, double boot,
            double gamma, double lam, double* out) {
  return Guard([&] {
    BoolArr d(done, n);
    auto a = rlmath::GaeAdvantages({r, n}, {v, n}, boot, d.span, gamma, lam);
    std::memcpy(out, a.data(), n * sizeof(double));
  });
}

int ref_lambda_return(const double* r, const double* v, const uint8_t* done, std::size_t n,
                      double boot, double gamma, double lam, double* out) {
  return Guard([&] {
    BoolArr d(done, n);
    auto a = rlmath::LambdaReturn({r, n}, {v, n}, boot, d.span, gamma, lam);
    std::memcpy(out, a.data(), n * sizeof(double));
  });
}

int ref_vtrace(const double* bl, const double* tl, const double* r, const double* v,
               const uint8_t* done, std::size_t n, double boot, double gamma, double rho_bar,
               double c_bar, double* vs, double* pg) {
  return Guard([&] {
    BoolArr d(done, n);
    auto res = rlmath::VtraceTargets({bl, n}, {tl, n}, {r, n}, {v, n}, boot, d.span, gamma,
                                     rho_bar, c_bar);
    std::memcpy(vs, res.vs.data(), n * sizeof(double));
    std::memcpy(pg, res.pg_adv.data(), n * sizeof(double));
  });
}

std::size_t ref_param_count(uint32_t family, uint32_t obs_dim, uint32_t n_actions) {
  return policy::ParamCount(static_cast<PolicyFamily>(family), {obs_dim, n_actions});
}

int ref_init_params(uint32_t family, uint32_t obs_dim, uint32_t n_actions, double scale,
                    uint64_t seed, double* out) {
  return Guard([&] {
    auto b = policy::InitParams(static_cast<PolicyFamily>(family), {obs_dim, n_actions}, scale,
                                seed);
    std::memcpy(out, b.values.data(), b.values.size() * sizeof(double));
  });
}

// Batched forward exactly as InfServer::BatchLoop evaluates each request
// (inf_server.cpp:132-144): Distribution + ValueEstimate per observation.
int ref_batch_forward(uint32_t family, uint32_t obs_dim, uint32_t n_actions,
                      const double* params, const double* obs, std::size_t n, double* logits,
                      double* probs, double* values) {
  return Guard([&] {
    ParamBlob b = MakeBlob(family, obs_dim, n_actions, params);
    for (std::size_t i = 0; i < n; ++i) {
      std::span<const double> o(obs + i * obs_dim, obs_dim);
      auto dist = policy::Distribution(b, o);
      std::memcpy(logits + i * n_actions, dist.logits.data(), n_actions * sizeof(double));
      std::memcpy(probs + i * n_actions, dist.probs.data(), n_actions * sizeof(double));
      values[i] = policy::ValueEstimate(b, o);
    }
  });
}

// stats_out: clip_fraction, mean_ratio, entropy, value_loss (rlmath.hpp:52-57)
int ref_ppo_loss_grad(uint32_t family, uint32_t obs_dim, uint32_t n_actions,
                      const double* params, const double* teacher, std::size_t n,
                      const double* obs, const uint32_t* action, const double* blogp,
                      const double* adv, const double* vtarget, const ref_hyper* hyper,
                      double* loss_out, double* grad_out, double* stats_out) {
  return Guard([&] {
    ParamBlob b = MakeBlob(family, obs_dim, n_actions, params);
    ParamBlob t;
    if (teacher) t = MakeBlob(family, obs_dim, n_actions, teacher);
    rlmath::Minibatch mb;
    for (std::size_t i = 0; i < n; ++i) {
      rlmath::Sample s;
      s.obs.assign(obs + i * obs_dim, obs + (i + 1) * obs_dim);
      s.action = action[i];
      s.behavior_logp = blogp[i];
      s.advantage = adv[i];
      s.value_target = vtarget[i];
      mb.samples.push_back(std::move(s));
    }
    auto res = rlmath::PpoLossAndGrad(b, teacher ? &t : nullptr, mb, ToHyper(hyper));
    *loss_out = res.loss;
    std::memcpy(grad_out, res.grad.data(), res.grad.size() * sizeof(double));
    stats_out[0] = res.stats.clip_fraction;
    stats_out[1] = res.stats.mean_ratio;
    stats_out[2] = res.stats.entropy;
    stats_out[3] = res.stats.value_loss;
  });
}

int ref_pg_loss_grad(uint32_t family, uint32_t obs_dim, uint32_t n_actions,
                     const double* params, std::size_t n, const double* obs,
                     const uint32_t* action, const double* blogp, const double* adv,
                     const double* vtarget, const ref_hyper* hyper, double* loss_out,
                     double* grad_out, double* stats_out) {
  return Guard([&] {
    ParamBlob b = MakeBlob(family, obs_dim, n_actions, params);
    rlmath::Minibatch mb;
    for (std::size_t i = 0; i < n; ++i) {
      rlmath::Sample s;
      s.obs.assign(obs + i * obs_dim, obs + (i + 1) * obs_dim);
      s.action = action[i];
      s.behavior_logp = blogp[i];
      s.advantage = adv[i];
      s.value_target = vtarget[i];
      mb.samples.push_back(std::move(s));
    }
    auto res = rlmath::PgLossAndGrad(b, mb, ToHyper(hyper));
    *loss_out = res.loss;
    std::memcpy(grad_out, res.grad.data(), res.grad.size() * sizeof(double));
    stats_out[0] = res.stats.clip_fraction;
    stats_out[1] = res.stats.mean_ratio;
    stats_out[2] = res.stats.entropy;
    stats_out[3] = res.stats.value_loss;
  });
}

int ref_sgd_step(uint32_t family, uint32_t obs_dim, uint32_t n_actions, const double* params,
                 const double* grad, double lr, double* out) {
  return Guard([&] {
    ParamBlob b = MakeBlob(family, obs_dim, n_actions, params);
    auto next = rlmath::SgdStep(b, {grad, b.values.size()}, lr);
    std::memcpy(out, next.values.data(), next.values.size() * sizeof(double));
  });
}

// ---------------------------------------------------------------------------
// Segments cross this shim as SoA [n_seg][unroll] arrays (the layout the GPU
// path consumes); they are expanded into the reference's AoS TrajectorySegment
// (types.hpp:82-104) here.
struct ref_segments {
  uint32_t n_segments, unroll_len, obs_dim;
  const double* obs;         // [S][T][obs_dim]
  const uint32_t* action;    // [S][T]
  const double* reward;      // [S][T]
  const double* behavior_logp;
  const double* value_est;
  const uint8_t* done;       // [S][T]
  const double* bootstrap;   // [S]
  const uint32_t* valid_steps;  // [S]
  const uint64_t* segment_seq;  // [S] (nullable)
};

static TrajectorySegment ToSegment(const ref_segments* s, std::size_t i, const std::string& key) {
  TrajectorySegment seg;
  seg.model_key = key;
  seg.valid_steps = s->valid_steps[i];
  seg.bootstrap_value = s->bootstrap[i];
  seg.segment_seq = s->segment_seq ? s->segment_seq[i] : i;
  seg.steps.resize(s->unroll_len);
  for (uint32_t t = 0; t < s->unroll_len; ++t) {
    const std::size_t f = i * s->unroll_len + t;
    SegmentStep& st = seg.steps[t];
    st.obs.assign(s->obs + f * s->obs_dim, s->obs + (f + 1) * s->obs_dim);
    st.action = s->action[f];
    st.reward = s->reward[f];
    st.behavior_logp = s->behavior_logp[f];
    st.value_est = s->value_est[f];
    st.done = s->done[f] != 0;
  }
  return seg;
}

// ReplayMem (replay_mem.cpp): segments are identified by segment_seq so the
// caller can compare draw order bit for bit.
void* ref_replay_create(std::size_t capacity, uint32_t max_reuse, uint64_t seed) {
  void* out = nullptr;
  Guard([&] { out = new learner::ReplayMem(capacity, max_reuse, seed); });
  return out;
}
void ref_replay_destroy(void* r) { delete static_cast<learner::ReplayMem*>(r); }
int ref_replay_push(void* r, uint64_t seq, uint32_t valid_steps) {
  return Guard([&] {
    TrajectorySegment seg;
    seg.segment_seq = seq;
    seg.valid_steps = valid_steps;
    static_cast<learner::ReplayMem*>(r)->Push(std::move(seg));
  });
}
int ref_replay_sample(void* r, std::size_t n, uint64_t* seq_out) {
  return Guard([&] {
    auto segs = static_cast<learner::ReplayMem*>(r)->SampleBlocking(n);
    for (std::size_t i = 0; i < segs.size(); ++i) seq_out[i] = segs[i].segment_seq;
  });
}
uint64_t ref_replay_consumed(void* r) {
  return static_cast<learner::ReplayMem*>(r)->consumed_steps();
}
std::size_t ref_replay_size(void* r) { return static_cast<learner::ReplayMem*>(r)->size(); }

// The reference Learner behind its own league/pool rig (learner_test.cpp:16-31).
struct RefRig {
  pool::ModelStore store;
  pool::DirectPool pool{store};
  std::unique_ptr<league::LeagueState> league;
  std::unique_ptr<learner::Learner> lrn;
};

void* ref_learner_create(uint32_t family, uint32_t obs_dim, uint32_t n_actions,
                         double init_scale, uint64_t league_seed, const ref_hyper* hyper,
                         uint32_t num_shards, uint32_t algo, uint32_t publish_interval,
                         std::size_t replay_capacity, uint64_t seed) {
  RefRig* rig = nullptr;
  int rc = Guard([&] {
    auto r = std::make_unique<RefRig>();
    league::LearnerGroupConfig g;
    g.family = static_cast<PolicyFamily>(family);
    g.shape = {obs_dim, n_actions};
    g.init_scale = init_scale;
    g.hyper = ToHyper(hyper);
    r->league = std::make_unique<league::LeagueState>(
        std::vector<league::LearnerGroupConfig>{g}, r->pool, league_seed);
    learner::LearnerConfig cfg;
    cfg.num_shards = num_shards;
    cfg.algo = algo == 0 ? learner::Algo::kPpo : learner::Algo::kVtrace;
    cfg.publish_interval = publish_interval;
    cfg.replay_capacity = replay_capacity;
    cfg.seed = seed;
    r->lrn = std::make_unique<learner::Learner>(cfg, *r->league, r->pool);
    rig = r.release();
  });
  return rc == 0 ? rig : nullptr;
}
void ref_learner_destroy(void* h) { delete static_cast<RefRig*>(h); }
int ref_learner_push(void* h, const ref_segments* segs) {
  return Guard([&] {
    auto* rig = static_cast<RefRig*>(h);
    for (std::size_t i = 0; i < segs->n_segments; ++i)
      rig->lrn->PushSegment(ToSegment(segs, i, rig->lrn->current_key()));
  });
}
int ref_learner_train_step(void* h, int32_t* ok) {
  return Guard([&] { *ok = static_cast<RefRig*>(h)->lrn->TrainStep() ? 1 : 0; });
}
std::size_t ref_learner_param_count(void* h) {
  return static_cast<RefRig*>(h)->lrn->params().values.size();
}
int ref_learner_params(void* h, double* out) {
  return Guard([&] {
    const auto& v = static_cast<RefRig*>(h)->lrn->params().values;
    std::memcpy(out, v.data(), v.size() * sizeof(double));
  });
}
int ref_learner_pool_params(void* h, const char* key, double* out) {
  return Guard([&] {
    auto rec = static_cast<RefRig*>(h)->store.Get(key);
    std::memcpy(out, rec->params.values.data(), rec->params.values.size() * sizeof(double));
  });
}
uint64_t ref_learner_consumed(void* h) {
  return static_cast<RefRig*>(h)->lrn->replay().consumed_steps();
}
std::size_t ref_learner_replay_size(void* h) {
  return static_cast<RefRig*>(h)->lrn->replay().size();
}

}  // extern "C"
