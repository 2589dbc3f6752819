// Drop-in acceptance of the B200 Learner / InfServer against the reference's own
// services (LeagueState, ModelStore/DirectPool, ReplayMem, net, run::RunBench), in the
// scenarios of the reference's learner_test.cpp and infserver_test.cpp.  Numeric
// checks compare with the reference's fp64 rlmath/policy routines (linked unchanged)
// in the reference's Close() metric (acceptance.cpp:439-441).
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <filesystem>
#include <cstdio>
#include <functional>
#include <limits>
#include <memory>
#include <random>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "tleague/infserver/inf_server.hpp"
#include "tleague/league/league_state.hpp"
#include "tleague/learner/learner.hpp"
#include "tleague/policy/policy.hpp"
#include "tleague/pool/model_store.hpp"
#include "tleague/rlmath/rlmath.hpp"
#include "tleague/learner/learner_service.hpp"
#include "tleague/pool/model_pool_service.hpp"
#include "tleague/proto/codec.hpp"
#include "tleague/proto/wire_ext.hpp"
#include "tleague/run/bench.hpp"
#include "tleague/run/config.hpp"
#include "tleague/run/local_run.hpp"
#include "tleague/run/model_io.hpp"
#include "tlg_b200.h"

using namespace tleague;

// ---------------------------------------------------------------------------
// minimal test harness
namespace {
struct Case {
  const char* name;
  std::function<void()> fn;
};
std::vector<Case>& Cases() {
  static std::vector<Case> c;
  return c;
}
int g_fail = 0, g_checks = 0;
struct Reg {
  Reg(const char* n, std::function<void()> f) { Cases().push_back({n, std::move(f)}); }
};
#define TEST(name)                         \
  static void name();                      \
  static Reg reg_##name(#name, name);      \
  static void name()
#define CHECK(cond)                                                              \
  do {                                                                           \
    ++g_checks;                                                                  \
    if (!(cond)) {                                                               \
      ++g_fail;                                                                  \
      std::printf("  CHECK failed %s:%d: %s\n", __FILE__, __LINE__, #cond);       \
    }                                                                            \
  } while (0)
#define CHECK_THROWS_AS(expr, type)                                              \
  do {                                                                           \
    ++g_checks;                                                                  \
    bool ok_ = false;                                                            \
    try {                                                                        \
      expr;                                                                      \
    } catch (const type&) {                                                      \
      ok_ = true;                                                                \
    } catch (...) {                                                              \
    }                                                                            \
    if (!ok_) {                                                                  \
      ++g_fail;                                                                  \
      std::printf("  CHECK_THROWS_AS failed %s:%d: %s\n", __FILE__, __LINE__, #expr); \
    }                                                                            \
  } while (0)

bool Close(double a, double b, double tol) {
  return std::abs(a - b) <= tol * std::max({1.0, std::abs(a), std::abs(b)});
}
bool AllClose(const std::vector<double>& a, const std::vector<double>& b, double tol,
              double* worst = nullptr) {
  if (a.size() != b.size()) return false;
  double w = 0;
  bool ok = true;
  for (std::size_t i = 0; i < a.size(); ++i) {
    const double e = std::abs(a[i] - b[i]) / std::max({1.0, std::abs(a[i]), std::abs(b[i])});
    w = std::max(w, e);
    ok &= Close(a[i], b[i], tol);
  }
  if (worst) *worst = w;
  return ok;
}

// ---------------------------------------------------------------------------
// learner_test.cpp-style rig and synthetic segments (3-step episodes, one state)
struct Rig {
  pool::ModelStore store;
  pool::DirectPool pool{store};
  league::LeagueState league;
  explicit Rig(HyperParams hyper, std::uint64_t seed = 42) : league(Groups(hyper), pool, seed) {}
  static std::vector<league::LearnerGroupConfig> Groups(HyperParams hyper) {
    league::LearnerGroupConfig cfg;
    cfg.shape = {1, 3};
    cfg.init_scale = 0.3;
    cfg.hyper = hyper;
    return {cfg};
  }
};

HyperParams TestHyper() {
  HyperParams hp;
  hp.learning_rate = 0.05;
  hp.batch_size = 4;
  hp.max_reuse = 1;
  hp.unroll_len = 3;
  return hp;
}

TrajectorySegment MakeSegment(const std::string& key, std::mt19937_64& rng, std::uint64_t seq) {
  TrajectorySegment seg;
  seg.model_key = key;
  seg.segment_seq = seq;
  seg.valid_steps = 3;
  seg.steps.resize(3);
  std::uniform_real_distribution<double> real(-1.0, 1.0);
  for (auto& step : seg.steps) {
    step.obs = {1.0};
    step.action = static_cast<std::uint32_t>(rng() % 3);
    // fp32-representable so the fp64 oracle and the fp32 device path see the same data
    step.reward = double(float(real(rng)));
    step.behavior_logp = double(float(std::log(1.0 / 3) + 0.1 * real(rng)));
    step.value_est = double(float(real(rng)));
  }
  seg.steps.back().done = true;
  return seg;
}

// the reference's consume-time batch assembly, run serially in fp64 (learner.cpp:56-102)
rlmath::Minibatch OracleBatch(const std::vector<TrajectorySegment>& segments, bool vtrace,
                              const ParamBlob& params, const HyperParams& hp) {
  rlmath::Minibatch batch;
  for (const auto& seg : segments) {
    const std::size_t n = seg.valid_steps;
    std::vector<double> r(n), v(n), bl(n), tl(n);
    std::unique_ptr<bool[]> d(new bool[n]);
    for (std::size_t t = 0; t < n; ++t) {
      r[t] = seg.steps[t].reward;
      v[t] = seg.steps[t].value_est;
      bl[t] = seg.steps[t].behavior_logp;
      d[t] = seg.steps[t].done;
      if (vtrace)
        tl[t] = std::log(policy::Distribution(params, seg.steps[t].obs).probs[seg.steps[t].action]);
    }
    std::span<const bool> dones(d.get(), n);
    std::vector<double> adv, tgt;
    if (!vtrace) {
      adv = rlmath::GaeAdvantages(r, v, seg.bootstrap_value, dones, hp.gamma, hp.lam);
      tgt = rlmath::LambdaReturn(r, v, seg.bootstrap_value, dones, hp.gamma, hp.lam);
    } else {
      auto vt = rlmath::VtraceTargets(bl, tl, r, v, seg.bootstrap_value, dones, hp.gamma,
                                      hp.rho_bar, hp.c_bar);
      adv = std::move(vt.pg_adv);
      tgt = std::move(vt.vs);
    }
    for (std::size_t t = 0; t < n; ++t) {
      rlmath::Sample s;
      s.obs = seg.steps[t].obs;
      s.action = seg.steps[t].action;
      s.behavior_logp = bl[t];
      s.advantage = adv[t];
      s.value_target = tgt[t];
      batch.samples.push_back(std::move(s));
    }
  }
  return batch;
}

}  // namespace

// ---------------------------------------------------------------------------
TEST(stale_model_keys_are_dropped) {
  Rig rig(TestHyper());
  learner::LearnerConfig cfg;
  cfg.seed = 7;
  learner::Learner lrn(cfg, rig.league, rig.pool);
  std::mt19937_64 rng(1);
  lrn.PushSegment(MakeSegment("main:0099", rng, 0));
  lrn.PushSegment(MakeSegment("other:0000", rng, 1));
  CHECK(lrn.replay().size() == 0);
  CHECK(lrn.Counters().stale_dropped == 2);
  lrn.PushSegment(MakeSegment(lrn.current_key(), rng, 2));
  CHECK(lrn.replay().size() == 1);
}

TEST(two_shards_match_the_serial_fp64_reference) {
  for (auto algo : {learner::Algo::kPpo, learner::Algo::kVtrace}) {
    HyperParams hyper = TestHyper();
    const bool vtrace = algo == learner::Algo::kVtrace;
    if (vtrace) hyper.max_reuse = 2;
    Rig rig(hyper);
    learner::LearnerConfig cfg;
    cfg.num_shards = 2;
    cfg.algo = algo;
    cfg.publish_interval = 1;
    cfg.seed = 99;
    learner::Learner lrn(cfg, rig.league, rig.pool);
    learner::ReplayMem oracle_replay(cfg.replay_capacity, hyper.max_reuse, cfg.seed);
    ParamBlob oracle = rig.store.Get(lrn.current_key())->params;
    CHECK(oracle == lrn.params());
    std::mt19937_64 feed_a(2024), feed_b(2024);
    std::uint64_t seq = 0;
    const std::size_t draw = hyper.batch_size * 2;
    double worst_all = 0;
    for (int step = 0; step < 30; ++step) {
      for (std::size_t i = 0; i < draw; ++i) {
        lrn.PushSegment(MakeSegment(lrn.current_key(), feed_a, seq + i));
        oracle_replay.Push(MakeSegment(lrn.current_key(), feed_b, seq + i));
      }
      seq += draw;
      CHECK(lrn.TrainStep());
      auto segs = oracle_replay.SampleBlocking(draw);  // same ring, same seed: same draw
      std::vector<double> avg(oracle.values.size(), 0.0);
      for (int r = 0; r < 2; ++r) {
        std::vector<TrajectorySegment> slice(segs.begin() + r * hyper.batch_size,
                                             segs.begin() + (r + 1) * hyper.batch_size);
        auto batch = OracleBatch(slice, vtrace, oracle, hyper);
        auto res = vtrace ? rlmath::PgLossAndGrad(oracle, batch, hyper)
                          : rlmath::PpoLossAndGrad(oracle, nullptr, batch, hyper);
        for (std::size_t i = 0; i < avg.size(); ++i) avg[i] += res.grad[i];
      }
      for (double& g : avg) g *= 0.5;
      oracle = rlmath::SgdStep(oracle, avg, hyper.learning_rate);
      double worst = 0;
      CHECK(AllClose(lrn.params().values, oracle.values, 1e-4, &worst));
      worst_all = std::max(worst_all, worst);
      // publish_interval = 1: the pool copy is the learner's parameters
      CHECK(rig.store.Get(lrn.current_key())->params.values == lrn.params().values);
      CHECK(lrn.replay().consumed_steps() == oracle_replay.consumed_steps());
    }
    std::printf("  %s: 30 steps, worst Close() error vs fp64 reference %.2e\n",
                vtrace ? "vtrace" : "ppo", worst_all);
  }
}

TEST(publishing_follows_the_configured_cadence) {
  Rig rig(TestHyper());
  learner::LearnerConfig cfg;
  cfg.publish_interval = 3;
  cfg.seed = 5;
  learner::Learner lrn(cfg, rig.league, rig.pool);
  const ParamBlob seed_params = rig.store.Get(lrn.current_key())->params;
  std::mt19937_64 rng(9);
  std::uint64_t seq = 0;
  auto feed_and_step = [&] {
    for (int i = 0; i < 4; ++i) lrn.PushSegment(MakeSegment(lrn.current_key(), rng, seq++));
    CHECK(lrn.TrainStep());
  };
  feed_and_step();
  feed_and_step();
  CHECK(lrn.params().values != seed_params.values);
  CHECK(rig.store.Get(lrn.current_key())->params.values == seed_params.values);
  feed_and_step();
  CHECK(rig.store.Get(lrn.current_key())->params.values == lrn.params().values);
  CHECK(lrn.update_steps() == 3);
}

TEST(finishing_a_period_freezes_rolls_the_key_and_clears_the_ring) {
  Rig rig(TestHyper());
  learner::LearnerConfig cfg;
  cfg.publish_interval = 100;
  cfg.seed = 6;
  learner::Learner lrn(cfg, rig.league, rig.pool);
  CHECK(lrn.current_key() == "main:0000");
  std::mt19937_64 rng(13);
  for (int i = 0; i < 4; ++i) lrn.PushSegment(MakeSegment("main:0000", rng, i));
  CHECK(lrn.TrainStep());
  lrn.PushSegment(MakeSegment("main:0000", rng, 99));
  std::string successor = lrn.FinishPeriod();
  CHECK(successor == "main:0001");
  CHECK(lrn.current_key() == "main:0001");
  CHECK(lrn.replay().size() == 0);
  auto frozen = rig.store.Get("main:0000");
  CHECK(frozen->frozen);
  CHECK(frozen->params.values == lrn.params().values);
  lrn.PushSegment(MakeSegment("main:0000", rng, 100));
  CHECK(lrn.replay().size() == 0);
  CHECK(lrn.Counters().stale_dropped == 1);
}

TEST(a_non_finite_loss_aborts_the_training_step_loudly) {
  Rig rig(TestHyper());
  learner::LearnerConfig cfg;
  cfg.seed = 8;
  learner::Learner lrn(cfg, rig.league, rig.pool);
  const ParamBlob before = lrn.params();
  std::mt19937_64 rng(3);
  for (int i = 0; i < 4; ++i) {
    auto seg = MakeSegment(lrn.current_key(), rng, i);
    seg.steps[0].reward = std::numeric_limits<double>::quiet_NaN();
    lrn.PushSegment(seg);
  }
  CHECK_THROWS_AS(lrn.TrainStep(), std::invalid_argument);  // "non-finite advantage"
  CHECK(lrn.params() == before);
  CHECK(lrn.update_steps() == 0);
}

TEST(shutdown_releases_a_blocked_train_step) {
  Rig rig(TestHyper());
  learner::LearnerConfig cfg;
  cfg.seed = 9;
  learner::Learner lrn(cfg, rig.league, rig.pool);
  bool result = true;
  std::thread trainer([&] { result = lrn.TrainStep(); });
  std::this_thread::sleep_for(std::chrono::milliseconds(30));
  lrn.Shutdown();
  trainer.join();
  CHECK(!result);
}

// ---------------------------------------------------------------------------
namespace {
ModelRecord LinearModel(const std::string& key, std::uint64_t seed) {
  ModelRecord rec;
  rec.model_key = key;
  rec.params = policy::InitParams(PolicyFamily::kLinearSoftmax, {4, 3}, 1.0, seed);
  for (double& v : rec.params.values) v = double(float(v));
  return rec;
}
std::vector<double> RandomObs(std::mt19937_64& rng) {
  std::normal_distribution<double> n(0.0, 1.0);
  std::vector<double> obs(4);
  for (double& x : obs) x = double(float(n(rng)));
  return obs;
}
}  // namespace

TEST(remote_inference_equals_local_gpu_bit_for_bit_and_fp64_within_tolerance) {
  pool::ModelStore store;
  pool::DirectPool pool(store);
  auto rec = LinearModel("main:0000", 3);
  pool.PutModel(rec);
  infserver::InfServer server({"main:0000"}, pool, "127.0.0.1", 0);
  infserver::InferenceClient client(server.endpoint());
  std::mt19937_64 rng(17);
  double worst = 0;
  for (int i = 0; i < 2000; ++i) {
    auto obs = RandomObs(rng);
    auto reply = client.Infer(obs);
    auto local = server.EvaluateLocal(obs);
    CHECK(reply.logits == local.logits);
    CHECK(reply.probs == local.probs);
    CHECK(reply.value == local.value);
    auto ref = policy::Distribution(rec.params, obs);
    double w1 = 0, w2 = 0;
    CHECK(AllClose(reply.logits, ref.logits, 1e-5, &w1));
    CHECK(AllClose(reply.probs, ref.probs, 1e-5, &w2));
    CHECK(Close(reply.value, policy::ValueEstimate(rec.params, obs), 1e-5));
    worst = std::max({worst, w1, w2});
  }
  std::printf("  worst Close() error vs fp64 policy::Distribution %.2e\n", worst);
  server.Stop();
}

TEST(batched_requests_from_many_clients_are_routed_to_the_right_caller) {
  pool::ModelStore store;
  pool::DirectPool pool(store);
  auto rec = LinearModel("main:0000", 9);
  pool.PutModel(rec);
  infserver::InfServer::Config cfg{"main:0000"};
  cfg.max_batch = 8;
  cfg.flush_timeout_ms = 5.0;
  infserver::InfServer server(cfg, pool, "127.0.0.1", 0);
  std::atomic<int> mismatches{0};
  std::vector<std::thread> threads;
  for (int t = 0; t < 12; ++t) {
    threads.emplace_back([&, t] {
      infserver::InferenceClient client(server.endpoint());
      std::mt19937_64 rng(1000 + t);
      for (int i = 0; i < 200; ++i) {
        auto obs = RandomObs(rng);
        auto reply = client.Infer(obs);
        auto local = server.EvaluateLocal(obs);  // batch invariance: same bits alone
        if (reply.logits != local.logits || reply.value != local.value) mismatches.fetch_add(1);
      }
    });
  }
  for (auto& t : threads) t.join();
  CHECK(mismatches.load() == 0);
  server.Stop();
}

TEST(the_tracked_key_follows_pool_updates_with_a_monotonic_version) {
  pool::ModelStore store;
  pool::DirectPool pool(store);
  pool.PutModel(LinearModel("main:0000", 1));
  infserver::InfServer::Config cfg{"latest:main"};
  cfg.refresh_interval_ms = 5;
  infserver::InfServer server(cfg, pool, "127.0.0.1", 0);
  const std::uint64_t v0 = server.model_version();
  server.RefreshNow();
  CHECK(server.model_version() == v0);
  pool.PutModel(LinearModel("main:0001", 2));
  server.RefreshNow();
  CHECK(server.model_version() == v0 + 1);
  pool.PutModel(LinearModel("main:0002", 3));
  for (int i = 0; i < 200 && server.model_version() == v0 + 1; ++i)
    std::this_thread::sleep_for(std::chrono::milliseconds(5));
  CHECK(server.model_version() == v0 + 2);
  server.Stop();
}

TEST(replies_stay_self_consistent_under_concurrent_blob_refresh) {
  pool::ModelStore store;
  pool::DirectPool pool(store);
  auto rec_a = LinearModel("main:0000", 11);
  auto rec_b = LinearModel("main:0000", 22);
  // device evaluations of each blob alone (batch-invariant forward)
  tlg_policy_shape s{};
  s.family = TLG_FAMILY_LINEAR;
  s.obs_dim = 4;
  s.n_actions = 3;
  tlg_policy *pa = nullptr, *pb = nullptr;
  CHECK(tlg_policy_create(&s, 0, 1, &pa) == 0);
  CHECK(tlg_policy_create(&s, 0, 1, &pb) == 0);
  CHECK(tlg_policy_set_params(pa, rec_a.params.values.data(), rec_a.params.values.size()) == 0);
  CHECK(tlg_policy_set_params(pb, rec_b.params.values.data(), rec_b.params.values.size()) == 0);
  pool.PutModel(rec_a);
  infserver::InfServer::Config cfg{"main:0000"};
  cfg.refresh_interval_ms = 1;
  infserver::InfServer server(cfg, pool, "127.0.0.1", 0);
  std::atomic<bool> stop{false};
  std::thread writer([&] {
    bool a = false;
    while (!stop.load()) {
      pool.PutModel(a ? rec_a : rec_b);
      a = !a;
      std::this_thread::sleep_for(std::chrono::milliseconds(1));
    }
  });
  infserver::InferenceClient client(server.endpoint());
  std::mt19937_64 rng(5);
  int matched_a = 0, matched_b = 0, torn = 0;
  for (int i = 0; i < 2000; ++i) {
    auto obs = RandomObs(rng);
    auto reply = client.Infer(obs);
    float o[4], la[3], pa_[3], va, lb[3], pb_[3], vb;
    for (int j = 0; j < 4; ++j) o[j] = float(obs[j]);
    tlg_policy_forward(pa, o, 1, la, pa_, &va, 0);
    tlg_policy_forward(pb, o, 1, lb, pb_, &vb, 0);
    auto eq = [&](const float* l, float v) {
      for (int k = 0; k < 3; ++k)
        if (reply.logits[k] != double(l[k])) return false;
      return reply.value == double(v);
    };
    if (eq(la, va)) ++matched_a;
    else if (eq(lb, vb)) ++matched_b;
    else ++torn;
  }
  stop.store(true);
  writer.join();
  CHECK(torn == 0);
  CHECK(matched_a > 0);
  CHECK(matched_b > 0);
  server.Stop();
  tlg_policy_destroy(pa);
  tlg_policy_destroy(pb);
}

TEST(constructing_against_a_missing_key_fails_fast) {
  pool::ModelStore store;
  pool::DirectPool pool(store);
  CHECK_THROWS_AS(infserver::InfServer({"absent:0000"}, pool, "127.0.0.1", 0), std::exception);
}

TEST(device_resident_replay_matches_the_host_replay_path) {
  // LearnerConfig::device_replay: segments live in HBM slots from PushSegment on and the
  // draw is gathered on the device; draws (the reference ReplayMem's) and parameters must
  // equal the host-packing path exactly, through FIFO eviction and reuse.
  for (auto algo : {learner::Algo::kPpo, learner::Algo::kVtrace}) {
    HyperParams hyper = TestHyper();
    hyper.max_reuse = algo == learner::Algo::kVtrace ? 2 : 1;
    Rig rig_a(hyper), rig_b(hyper);
    learner::LearnerConfig cfg;
    cfg.num_shards = 2;
    cfg.algo = algo;
    cfg.publish_interval = 1;
    cfg.seed = 5;
    cfg.replay_capacity = 12;  // small: pushes evict through the FIFO
    learner::LearnerConfig cfg_dev = cfg;
    cfg_dev.device_replay = true;
    learner::Learner host(cfg, rig_a.league, rig_a.pool);
    learner::Learner dev(cfg_dev, rig_b.league, rig_b.pool);
    std::mt19937_64 feed_a(77), feed_b(77);
    std::uint64_t seq = 0;
    for (int step = 0; step < 20; ++step) {
      const int pushes = 8 + step % 5;  // >= one draw (2 shards x 4 segments)
      for (int i = 0; i < pushes; ++i, ++seq) {
        host.PushSegment(MakeSegment(host.current_key(), feed_a, seq));
        dev.PushSegment(MakeSegment(dev.current_key(), feed_b, seq));
      }
      CHECK(host.replay().size() == dev.replay().size());
      CHECK(host.TrainStep());
      CHECK(dev.TrainStep());
      CHECK(host.params().values == dev.params().values);
      CHECK(host.replay().consumed_steps() == dev.replay().consumed_steps());
    }
  }
}

// the SoA layout of the C ABI for a group of segments (what a bulk message would carry)
struct SoaBatch {
  std::vector<std::uint8_t> obs8, done;
  std::vector<float> obs32, reward, blogp, value, boot;
  std::vector<std::int32_t> action, valid;
  tlg_segment_batch c{};
};

std::unique_ptr<SoaBatch> ToSoa(const std::vector<TrajectorySegment>& segs, std::uint32_t T,
                                std::uint32_t D, bool bits) {
  auto b = std::make_unique<SoaBatch>();
  const std::size_t n = segs.size(), rowb = (D + 7) / 8;
  if (bits) b->obs8.assign(n * T * rowb, 0);
  else b->obs32.assign(n * T * D, 0.f);
  b->done.assign(n * T, 0);
  b->reward.assign(n * T, 0.f);
  b->blogp.assign(n * T, 0.f);
  b->value.assign(n * T, 0.f);
  b->action.assign(n * T, 0);
  for (std::size_t i = 0; i < n; ++i) {
    const TrajectorySegment& sg = segs[i];
    b->boot.push_back(float(sg.bootstrap_value));
    b->valid.push_back(std::int32_t(sg.valid_steps));
    for (std::uint32_t t = 0; t < sg.valid_steps; ++t) {
      const std::size_t f = i * T + t;
      const SegmentStep& st = sg.steps[t];
      for (std::uint32_t j = 0; j < D; ++j) {
        if (bits) b->obs8[f * rowb + j / 8] |= std::uint8_t((st.obs[j] == 1.0) << (j % 8));
        else b->obs32[f * D + j] = float(st.obs[j]);
      }
      b->action[f] = std::int32_t(st.action);
      b->reward[f] = float(st.reward);
      b->blogp[f] = float(st.behavior_logp);
      b->value[f] = float(st.value_est);
      b->done[f] = st.done ? 1 : 0;
    }
  }
  tlg_segment_batch& c = b->c;
  c.n_segments = std::uint32_t(n);
  c.unroll_len = T;
  c.obs_dim = D;
  c.obs_dtype = bits ? TLG_OBS_BITS : TLG_OBS_F32;
  c.obs = bits ? static_cast<const void*>(b->obs8.data()) : static_cast<const void*>(b->obs32.data());
  c.action = b->action.data();
  c.reward = b->reward.data();
  c.behavior_logp = b->blogp.data();
  c.value_est = b->value.data();
  c.done = b->done.data();
  c.bootstrap = b->boot.data();
  c.valid_steps = b->valid.data();
  return b;
}

TEST(bulk_soa_ingest_matches_per_segment_pushes) {
  // Learner::PushSegmentBatch (one SoA copy into the device ring per group) draws and
  // trains exactly like the same segments pushed one by one; in host-replay mode too.
  for (auto algo : {learner::Algo::kPpo, learner::Algo::kVtrace}) {
    HyperParams hyper = TestHyper();
    hyper.max_reuse = algo == learner::Algo::kVtrace ? 2 : 1;
    Rig rig_a(hyper), rig_b(hyper), rig_c(hyper);
    learner::LearnerConfig cfg;
    cfg.num_shards = 2;
    cfg.algo = algo;
    cfg.publish_interval = 1;
    cfg.seed = 9;
    cfg.replay_capacity = 12;
    cfg.device_replay = true;
    learner::LearnerConfig cfg_host = cfg;
    cfg_host.device_replay = false;
    learner::Learner one(cfg, rig_a.league, rig_a.pool);
    learner::Learner bulk(cfg, rig_b.league, rig_b.pool);
    learner::Learner bulk_host(cfg_host, rig_c.league, rig_c.pool);
    std::mt19937_64 feed(123);
    std::uint64_t seq = 0;
    for (int step = 0; step < 16; ++step) {
      const int pushes = 8 + step % 4;
      std::vector<TrajectorySegment> group;
      for (int i = 0; i < pushes; ++i, ++seq) {
        TrajectorySegment sg = MakeSegment(one.current_key(), feed, seq);
        if (seq % 3 == 1) {  // ragged
          sg.valid_steps = 2;
          sg.steps.resize(2);
        }
        one.PushSegment(sg);
        group.push_back(std::move(sg));
      }
      auto soa_bits = ToSoa(group, hyper.unroll_len, 1, true);
      auto soa_f32 = ToSoa(group, hyper.unroll_len, 1, false);
      bulk.PushSegmentBatch(bulk.current_key(), soa_bits->c);
      bulk_host.PushSegmentBatch(bulk_host.current_key(), soa_f32->c);
      CHECK(one.replay().size() == bulk.replay().size());
      CHECK(one.replay().size() == bulk_host.replay().size());
      CHECK(one.TrainStep());
      CHECK(bulk.TrainStep());
      CHECK(bulk_host.TrainStep());
      CHECK(one.params().values == bulk.params().values);
      CHECK(one.params().values == bulk_host.params().values);
      CHECK(one.replay().consumed_steps() == bulk.replay().consumed_steps());
    }
    // stale keys are dropped as a whole, oversize groups rejected
    std::vector<TrajectorySegment> stale{MakeSegment("other:0000", feed, 0)};
    auto st = ToSoa(stale, hyper.unroll_len, 1, true);
    const auto before = bulk.Counters().stale_dropped;
    bulk.PushSegmentBatch("other:0000", st->c);
    CHECK(bulk.Counters().stale_dropped == before + 1);
    std::vector<TrajectorySegment> big;
    for (int i = 0; i < 13; ++i) big.push_back(MakeSegment(bulk.current_key(), feed, 0));
    auto bg = ToSoa(big, hyper.unroll_len, 1, true);
    bool threw = false;
    try {
      bulk.PushSegmentBatch(bulk.current_key(), bg->c);
    } catch (const std::invalid_argument&) {
      threw = true;
    }
    CHECK(threw);
  }
}

TEST(a_rejected_push_leaves_the_device_replay_mirror_in_step) {
  // A push that fails (a non-binary observation in a bit-packed period, a bad obs_pitch)
  // must leave the HBM slot map exactly in step with the reference ReplayMem, which never
  // saw the segment: later draws and parameters equal a host-replay learner's that was
  // never offered the bad pushes.
  HyperParams hyper = TestHyper();
  Rig rig_a(hyper), rig_b(hyper);
  learner::LearnerConfig cfg;
  cfg.num_shards = 2;
  cfg.publish_interval = 1;
  cfg.seed = 3;
  cfg.replay_capacity = 12;
  learner::LearnerConfig cfg_dev = cfg;
  cfg_dev.device_replay = true;
  learner::Learner host(cfg, rig_a.league, rig_a.pool);
  learner::Learner dev(cfg_dev, rig_b.league, rig_b.pool);
  std::mt19937_64 feed_a(31), feed_b(31), junk(5);
  std::uint64_t seq = 0;
  for (int step = 0; step < 8; ++step) {
    for (int i = 0; i < 10; ++i, ++seq) {  // the ring is full from step 1 on: pushes evict
      host.PushSegment(MakeSegment(host.current_key(), feed_a, seq));
      dev.PushSegment(MakeSegment(dev.current_key(), feed_b, seq));
      if (i % 4 == 1) {
        TrajectorySegment bad = MakeSegment(dev.current_key(), junk, 0);
        bad.steps[1].obs = {0.5};  // not a 0/1 plane: rejected in a bit-packed period
        CHECK_THROWS_AS(dev.PushSegment(bad), std::invalid_argument);
        std::vector<TrajectorySegment> grp{MakeSegment(dev.current_key(), junk, 0)};
        auto soa = ToSoa(grp, hyper.unroll_len, 1, true);
        soa->c.obs_pitch = 64;  // wider than a 16-B padded row
        CHECK_THROWS_AS(dev.PushSegmentBatch(dev.current_key(), soa->c), std::invalid_argument);
      }
    }
    CHECK(host.replay().size() == dev.replay().size());
    CHECK(host.TrainStep());
    CHECK(dev.TrainStep());
    CHECK(host.params().values == dev.params().values);
    CHECK(host.replay().consumed_steps() == dev.replay().consumed_steps());
  }
}

TEST(devices_spread_the_shards_over_gpus_like_local_shards) {
  // LearnerConfig::devices: num_shards shards over G GPUs in this process (one host thread
  // per device, NCCL allreduce in per-layer buckets).  With 2 ranks the NCCL sum a + b is
  // the same fp32 operation as the single-GPU rank-ordered local sum, so parameters match
  // the 2-local-shard learner bit for bit, step after step.
  if (tlg_device_count() < 2) {
    std::printf("  skipped: needs 2 GPUs\n");
    return;
  }
  for (auto algo : {learner::Algo::kPpo, learner::Algo::kVtrace}) {
    HyperParams hyper = TestHyper();
    Rig rig_a(hyper), rig_b(hyper);
    learner::LearnerConfig cfg;
    cfg.num_shards = 2;
    cfg.algo = algo;
    cfg.publish_interval = 1;
    cfg.seed = 11;
    cfg.optimizer = learner::Optimizer::kAdam;
    learner::LearnerConfig cfg2 = cfg;
    cfg2.devices = {0, 1};
    learner::Learner one(cfg, rig_a.league, rig_a.pool);
    learner::Learner two(cfg2, rig_b.league, rig_b.pool);
    std::mt19937_64 feed_a(8), feed_b(8);
    std::uint64_t seq = 0;
    for (int step = 0; step < 12; ++step) {
      for (int i = 0; i < 8; ++i, ++seq) {
        one.PushSegment(MakeSegment(one.current_key(), feed_a, seq));
        two.PushSegment(MakeSegment(two.current_key(), feed_b, seq));
      }
      CHECK(one.TrainStep());
      CHECK(two.TrainStep());
      CHECK(one.params().values == two.params().values);
    }
  }
  learner::LearnerConfig bad;
  bad.num_shards = 3;
  bad.devices = {0, 1};
  Rig rig(TestHyper());
  CHECK_THROWS_AS(learner::Learner(bad, rig.league, rig.pool), std::invalid_argument);
}

// ---------------------------------------------------------------------------
// The MLP policy family registered at the reference's extension seam (wire tag 2,
// integration/patches/mlp_family.py + integration/policy_mlp.cpp).
namespace {
const PolicyShape kGridMlp{50, 6, {256, 256}};  // grid_duel's obs/actions, 2x256 trunk

league::LearnerGroupConfig MlpGroup(HyperParams hyper, PolicyShape shape) {
  league::LearnerGroupConfig cfg;
  cfg.family = PolicyFamily::kMlp;
  cfg.shape = shape;
  cfg.init_scale = 0.1;
  cfg.hyper = hyper;
  return cfg;
}

TrajectorySegment MakeSegmentD(const std::string& key, std::mt19937_64& rng, std::uint64_t seq,
                               std::uint32_t D, std::uint32_t A, std::uint32_t T, bool binary) {
  TrajectorySegment seg;
  seg.model_key = key;
  seg.segment_seq = seq;
  seg.valid_steps = T - (seq % 5 == 2 ? 1 : 0);  // some ragged
  seg.steps.resize(seg.valid_steps);
  std::uniform_real_distribution<double> real(-1.0, 1.0);
  std::normal_distribution<double> gauss(0.0, 1.0);
  for (auto& step : seg.steps) {
    step.obs.resize(D);
    for (double& x : step.obs) x = binary ? double(rng() % 10 == 0) : double(float(gauss(rng)));
    step.action = static_cast<std::uint32_t>(rng() % A);
    step.reward = double(float(real(rng)));
    step.behavior_logp = double(float(std::log(1.0 / A) + 0.1 * real(rng)));
    step.value_est = double(float(real(rng)));
  }
  seg.bootstrap_value = double(float(real(rng)));
  return seg;
}
}  // namespace

TEST(mlp_family_learner_matches_the_fp64_reference_on_grid_duel_shape) {
  // A league seeded with MLP blobs (InitParams of the registered family), the B200 learner
  // training them through StartPeriod / PushSegment / TrainStep, against the reference's
  // own fp64 rlmath losses back-propagated through policy::mlp; obs 50 is not a multiple
  // of 4, so the device pads its rows internally.  Gaussian observations ship as fp32,
  // 0/1 planes bit-packed (int8 layer-1 kernels).
  for (bool binary : {false, true})
    for (auto algo : {learner::Algo::kPpo, learner::Algo::kVtrace}) {
      HyperParams hyper = TestHyper();
      hyper.unroll_len = 5;
      const bool vtrace = algo == learner::Algo::kVtrace;
      pool::ModelStore store;
      pool::DirectPool pool(store);
      league::LeagueState league({MlpGroup(hyper, kGridMlp)}, pool, 42);
      learner::LearnerConfig cfg;
      cfg.num_shards = 2;
      cfg.algo = algo;
      cfg.publish_interval = 1;
      cfg.seed = 99;
      learner::Learner lrn(cfg, league, pool);
      learner::ReplayMem oracle_replay(cfg.replay_capacity, hyper.max_reuse, cfg.seed);
      ParamBlob oracle = store.Get(lrn.current_key())->params;
      CHECK(oracle.family == PolicyFamily::kMlp);
      CHECK(oracle.values.size() == policy::ParamCount(PolicyFamily::kMlp, kGridMlp));
      CHECK(oracle == lrn.params());
      std::mt19937_64 feed_a(2025), feed_b(2025);
      std::uint64_t seq = 0;
      const std::size_t draw = hyper.batch_size * 2;
      double worst_all = 0;
      for (int step = 0; step < 8; ++step) {
        for (std::size_t i = 0; i < draw; ++i) {
          lrn.PushSegment(MakeSegmentD(lrn.current_key(), feed_a, seq + i, 50, 6, 5, binary));
          oracle_replay.Push(MakeSegmentD(lrn.current_key(), feed_b, seq + i, 50, 6, 5, binary));
        }
        seq += draw;
        CHECK(lrn.TrainStep());
        auto segs = oracle_replay.SampleBlocking(draw);
        std::vector<double> avg(oracle.values.size(), 0.0);
        for (int r = 0; r < 2; ++r) {
          std::vector<TrajectorySegment> slice(segs.begin() + r * hyper.batch_size,
                                               segs.begin() + (r + 1) * hyper.batch_size);
          auto batch = OracleBatch(slice, vtrace, oracle, hyper);
          auto res = vtrace ? rlmath::PgLossAndGrad(oracle, batch, hyper)
                            : rlmath::PpoLossAndGrad(oracle, nullptr, batch, hyper);
          for (std::size_t i = 0; i < avg.size(); ++i) avg[i] += res.grad[i];
        }
        for (double& g : avg) g *= 0.5;
        oracle = rlmath::SgdStep(oracle, avg, hyper.learning_rate);
        double worst = 0;
        CHECK(AllClose(lrn.params().values, oracle.values, 1e-4, &worst));
        worst_all = std::max(worst_all, worst);
        CHECK(store.Get(lrn.current_key())->params.family == PolicyFamily::kMlp);
      }
      std::printf("  %s %s obs: 8 steps, worst Close() error vs fp64 reference %.2e\n",
                  vtrace ? "vtrace" : "ppo", binary ? "0/1" : "gaussian", worst_all);
    }
}

TEST(mlp_blobs_travel_as_wire_tag_2_and_serve_from_the_b200_infserver) {
  // ParamBlob of family kMlp: codec round trip (model files are ParamPut frames,
  // docs/protocol.md:91-93), remote == local GPU inference bit for bit, and within 1e-5 of
  // the fp64 host family (what actors use for frozen MLP opponents, actor_loop.cpp:81-84).
  ModelRecord rec;
  rec.model_key = "mlp:0000";
  rec.params = policy::InitParams(PolicyFamily::kMlp, kGridMlp, 0.1, 5);
  for (double& v : rec.params.values) v = double(float(v));
  const std::string path = "/tmp/tlg_dropin_mlp.model";
  run::SaveModel(path, rec);
  ModelRecord back = run::LoadModel(path);
  CHECK(back.params == rec.params);
  CHECK(back.params.shape.hidden == kGridMlp.hidden);
  std::remove(path.c_str());
  pool::ModelStore store;
  pool::DirectPool pool(store);
  pool.PutModel(rec);
  infserver::InfServer server({"mlp:0000"}, pool, "127.0.0.1", 0);
  infserver::InferenceClient client(server.endpoint());
  std::mt19937_64 rng(3);
  std::normal_distribution<double> n(0.0, 1.0);
  double worst = 0;
  for (int i = 0; i < 300; ++i) {
    std::vector<double> obs(50);
    for (double& x : obs) x = double(float(n(rng)));
    auto reply = client.Infer(obs);
    auto local = server.EvaluateLocal(obs);
    CHECK(reply.logits == local.logits);
    CHECK(reply.probs == local.probs);
    auto ref = policy::Distribution(rec.params, obs);
    double w1 = 0, w2 = 0;
    CHECK(AllClose(reply.logits, ref.logits, 1e-5, &w1));
    CHECK(AllClose(reply.probs, ref.probs, 1e-5, &w2));
    CHECK(Close(reply.value, policy::ValueEstimate(rec.params, obs), 1e-5));
    worst = std::max({worst, w1, w2});
  }
  std::printf("  MLP 50-256-256-(6,1): worst Close() error vs fp64 policy::mlp %.2e\n", worst);
  server.Stop();
}

TEST(mlp_host_gradient_matches_central_finite_differences) {
  // policy::mlp::AccumulateGrad in the reference's FD pattern (policy_test.cpp:144-194):
  // d(c . logits + c_v * value)/d(theta) at h = 1e-6.
  const PolicyShape shape{7, 4, {5, 6}};
  ParamBlob p = policy::InitParams(PolicyFamily::kMlp, shape, 0.5, 11);
  std::mt19937_64 rng(1);
  std::normal_distribution<double> n(0.0, 1.0);
  std::vector<double> obs(7), c(4);
  for (double& x : obs) x = n(rng);
  for (double& x : c) x = n(rng);
  const double cv = 0.7;
  auto f = [&](const ParamBlob& q) {
    auto d = policy::Distribution(q, obs);
    double s = cv * policy::ValueEstimate(q, obs);
    for (int k = 0; k < 4; ++k) s += c[k] * d.logits[k];
    return s;
  };
  std::vector<double> g(p.values.size(), 0.0);
  policy::AccumulateGrad(p, obs, c, cv, g);
  double worst = 0;
  for (std::size_t i = 0; i < p.values.size(); ++i) {
    ParamBlob a = p, b = p;
    a.values[i] += 1e-6;
    b.values[i] -= 1e-6;
    const double fd = (f(a) - f(b)) / 2e-6;
    worst = std::max(worst, std::abs(fd - g[i]) / std::max(1.0, std::abs(fd)));
  }
  CHECK(worst < 1e-5);
  std::printf("  %zu parameters, worst FD error %.2e\n", p.values.size(), worst);
}

TEST(local_run_trains_an_mlp_league_on_grid_duel) {
  // run::LocalRun (lockstep) on grid_duel with `family: mlp`: actors act with the MLP
  // family against frozen MLP opponents, the B200 learner trains, frozen models are
  // written as tag-2 model files.
  const std::string text =
      "env: grid_duel\nmode: lockstep\nalgo: ppo\nseed: 5\nperiods: 3\nperiod_steps: 4\n"
      "publish_interval: 2\nactors: 2\nshards: 1\ninit_scale: 0.1\nfamily: mlp\n"
      "hidden: 64,32\nbatch_size: 4\nunroll_len: 8\nlearning_rate: 0.01\n";
  run::RunConfig cfg = run::ParseRunConfigText(text, "mlp.conf");
  CHECK(cfg.groups.at(0).family == PolicyFamily::kMlp);
  const std::string dir = "/tmp/tlg_dropin_mlp_run";
  std::filesystem::remove_all(dir);
  auto res = run::LocalRun(cfg, dir);
  CHECK(res.frozen_keys.size() == 3);
  for (const auto& key : res.frozen_keys) {
    auto rec = run::LoadModel(dir + "/models/" + run::ModelFileName(key));
    CHECK(rec.params.family == PolicyFamily::kMlp);
    CHECK((rec.params.shape.hidden == std::vector<std::uint32_t>{64, 32}));
    CHECK(rec.params.shape.obs_dim == 50);
    CHECK(rec.frozen);
  }
  CHECK(!res.group_counters.empty() && res.group_counters[0].update_steps > 0);
  std::filesystem::remove_all(dir);
}

// ---------------------------------------------------------------------------
// Wire extensions (message kinds 17 SegmentBatchPush, 18 ParamChunk; wire_ext.hpp).
TEST(bulk_segment_messages_over_tcp_train_like_single_pushes) {
  // learner::LearnerClient::PushSegmentBatch -> TCP -> LearnerService -> the B200
  // learner's bulk ingest (one frame per group, observations bit-packed or fp32), against
  // a learner fed the same segments one PushSegment at a time: identical draws and
  // parameters, in host-replay and device-replay mode.
  for (bool dev : {false, true})
    for (bool binary : {true, false}) {
      HyperParams hyper = TestHyper();
      hyper.unroll_len = 5;
      pool::ModelStore store_a, store_b;
      pool::DirectPool pool_a(store_a), pool_b(store_b);
      const PolicyShape shape{20, 6, {32, 32}};
      league::LeagueState league_a({MlpGroup(hyper, shape)}, pool_a, 7);
      league::LeagueState league_b({MlpGroup(hyper, shape)}, pool_b, 7);
      learner::LearnerConfig cfg;
      cfg.num_shards = 2;
      cfg.seed = 4;
      cfg.replay_capacity = 24;
      cfg.device_replay = dev;
      learner::Learner one(cfg, league_a, pool_a);
      learner::Learner bulk(cfg, league_b, pool_b);
      learner::LearnerService svc(bulk, "127.0.0.1", 0);
      learner::LearnerClient client(svc.endpoint());
      std::mt19937_64 feed(17);
      std::uint64_t seq = 0;
      for (int step = 0; step < 6; ++step) {
        std::vector<TrajectorySegment> group;
        for (int i = 0; i < 10; ++i, ++seq) {
          TrajectorySegment sg = MakeSegmentD(one.current_key(), feed, seq, 20, 6, 5, binary);
          one.PushSegment(sg);
          group.push_back(std::move(sg));
        }
        const SegmentBatch b = PackSegmentBatch(group, 5);
        CHECK(b.obs_format == (binary ? SegmentBatch::kObsBits : SegmentBatch::kObsF32));
        client.PushSegmentBatch(b);
        CHECK(one.replay().size() == bulk.replay().size());
        CHECK(one.TrainStep());
        CHECK(bulk.TrainStep());
        CHECK(one.params().values == bulk.params().values);
        CHECK(one.replay().consumed_steps() == bulk.replay().consumed_steps());
      }
      // codec round trip of the message itself
      auto group = std::vector<TrajectorySegment>{
          MakeSegmentD(one.current_key(), feed, 1, 20, 6, 5, binary)};
      proto::Message m = proto::MakeMessage(3, proto::SegmentBatchPushBody{PackSegmentBatch(group, 5)});
      CHECK(proto::Decode(proto::Encode(m)) == m);
      svc.Stop();
    }
}

TEST(c5_size_models_publish_and_travel_in_chunks) {
  // C5's 4x2048 MLP: 12.7M fp64 parameters = 102 MB, over the 64 MiB frame and the
  // reference ModelStore's 32 MiB blob cap.  Seeded by the league, trained and published
  // by the B200 learner, put / got over TCP in ParamChunk slices, saved as a chunked
  // model file, served by the B200 InfServer through a remote pool.
  const PolicyShape c5{64, 6, {2048, 2048, 2048, 2048}};
  HyperParams hyper = TestHyper();
  hyper.batch_size = 2;
  hyper.unroll_len = 4;
  pool::ModelPoolService svc("127.0.0.1", 0, {});
  pool::ModelPoolClient remote({svc.endpoint()});
  league::LeagueState league({MlpGroup(hyper, c5)}, remote, 9);  // chunked put of the seed
  const std::string key = league.RequestLearnerTask(0, 0).learning_model_key;
  ModelRecord seed = remote.GetModel(key);  // chunked get
  CHECK(seed.params.values.size() == policy::ParamCount(PolicyFamily::kMlp, c5));
  CHECK(seed.params.values.size() * sizeof(double) > proto::kMaxFrameBytes);
  learner::LearnerConfig cfg;
  cfg.publish_interval = 1;
  learner::Learner lrn(cfg, league, remote);
  std::mt19937_64 feed(2);
  for (int i = 0; i < 2; ++i) lrn.PushSegment(MakeSegmentD(lrn.current_key(), feed, i, 64, 6, 4, false));
  CHECK(lrn.TrainStep());  // publishes (publish_interval = 1): a chunked put
  ModelRecord back = remote.GetModel(key);
  CHECK(back.params == lrn.params());
  CHECK(back.params.values != seed.params.values);
  const std::string path = "/tmp/tlg_dropin_c5.model";
  run::SaveModel(path, back);
  CHECK(run::LoadModel(path) == back);
  std::remove(path.c_str());
  infserver::InfServer server({key}, remote, "127.0.0.1", 0);
  std::normal_distribution<double> n(0.0, 1.0);
  double worst = 0;
  for (int i = 0; i < 8; ++i) {
    std::vector<double> obs(64);
    for (double& x : obs) x = double(float(n(feed)));
    auto reply = server.EvaluateLocal(obs);
    auto ref = policy::Distribution(back.params, obs);
    double w = 0;
    // four 2048-wide fp32 layers (3xTF32): the 1e-4 class of forward-derived values
    CHECK(AllClose(reply.probs, ref.probs, 1e-4, &w));
    worst = std::max(worst, w);
  }
  std::printf("  C5 record %.1f MB in %zu-byte chunks; InfServer vs fp64 %.2e\n",
              back.params.values.size() * 8.0 / 1e6, proto::ext::kChunkBytes, worst);
  server.Stop();
  svc.Stop();
}

TEST(reference_run_bench_runs_on_the_b200_learner) {
  // run::RunBench (bench.cpp:60-162) builds learner::Learner -- here the B200 drop-in --
  // next to the reference's own actors, league and pool.
  run::BenchOptions opts;
  opts.duration_s = 1.0;
  opts.warmup_s = 0.3;
  auto res = run::RunBench("grid-1x2x8", opts);
  std::printf("  RunBench grid-1x2x8 on the B200 learner: rfps %.0f cfps %.0f\n", res.rfps,
              res.cfps);
  CHECK(res.cfps > 0.0);
  CHECK(res.rfps > 0.0);
}

int main(int argc, char** argv) {
  int ran = 0;
  for (const auto& c : Cases()) {
    if (argc > 1 && std::string(c.name).find(argv[1]) == std::string::npos) continue;
    const int before = g_fail;
    std::printf("[ RUN  ] %s\n", c.name);
    try {
      c.fn();
    } catch (const std::exception& e) {
      ++g_fail;
      std::printf("  uncaught exception: %s\n", e.what());
    }
    std::printf("[ %s ] %s\n", g_fail == before ? " OK " : "FAIL", c.name);
    ++ran;
  }
  std::printf("%d tests, %d checks, %d failures\n", ran, g_checks, g_fail);
  return g_fail ? 1 : 0;
}
