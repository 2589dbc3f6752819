// Throughput of the drop-in learner::Learner at BASELINE config C3 through the
// reference-facing C++ API, in the pattern of the reference's run::RunBench
// (bench.cpp:115-151: frames consumed per second of TrainStep): a league seeded with the
// MLP family (obs 11x11x16 = 1936 binary planes, 1936-256-256-(6,1), PPO, T=32, a draw of
// 4096 segments, Adam), segments pushed as the reference's AoS TrajectorySegment.
//
//   host replay   : TrainStep = ReplayMem draw + parallel SoA/bit packing of the fp64 AoS
//                   draw + H2D + the device step
//   device replay : PushSegment stages each segment into HBM (coalesced puts); TrainStep
//                   = draw + device gather + the device step
//
// Prints one JSON line.  Usage: dropin_bench [segments=4096] [steps=4]
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <string>
#include <vector>

#include "tleague/league/league_state.hpp"
#include "tleague/learner/learner.hpp"
#include "tleague/pool/model_store.hpp"

using namespace tleague;
using Clock = std::chrono::steady_clock;

namespace {

double Secs(Clock::time_point a, Clock::time_point b) {
  return std::chrono::duration<double>(b - a).count();
}

std::vector<TrajectorySegment> MakePool(std::size_t n, std::uint32_t T, std::uint32_t D,
                                        std::uint64_t seed) {
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<double> real(-1.0, 1.0);
  std::vector<TrajectorySegment> pool(n);
  for (auto& seg : pool) {
    seg.valid_steps = T;
    seg.steps.resize(T);
    for (auto& st : seg.steps) {
      st.obs.resize(D);
      for (double& x : st.obs) x = (rng() % 10 == 0) ? 1.0 : 0.0;  // Bernoulli(0.1) planes
      st.action = std::uint32_t(rng() % 6);
      st.reward = double(float(real(rng)));
      st.behavior_logp = double(float(std::log(1.0 / 6) + 0.1 * real(rng)));
      st.value_est = double(float(real(rng)));
      st.done = rng() % 100 == 0;
    }
    seg.bootstrap_value = double(float(real(rng)));
  }
  return pool;
}

struct Result {
  double cfps = 0, push_sps = 0, step_s = 0;
};

Result Run(bool device_replay, std::uint32_t S, int steps, const std::vector<TrajectorySegment>& pool) {
  const std::uint32_t T = 32, D = 1936;
  HyperParams hp;
  hp.batch_size = S;
  hp.unroll_len = T;
  hp.max_reuse = 1;
  hp.learning_rate = 3e-4;
  league::LearnerGroupConfig g;
  g.family = PolicyFamily::kMlp;
  g.shape = PolicyShape{D, 6, {256, 256}};
  g.init_scale = 0.05;
  g.hyper = hp;
  pool::ModelStore store;
  pool::DirectPool dpool(store);
  league::LeagueState league({g}, dpool, 7);
  learner::LearnerConfig cfg;
  cfg.num_shards = 1;
  cfg.publish_interval = 1000000;
  cfg.replay_capacity = 2 * S;
  cfg.optimizer = learner::Optimizer::kAdam;
  cfg.device_replay = device_replay;
  learner::Learner lrn(cfg, league, dpool);
  Result r;
  double push_s = 0, train_s = 0;
  std::size_t pushed = 0, frames = 0;
  std::size_t k = 0;
  for (int step = 0; step < steps + 1; ++step) {  // step 0: warm-up (allocations, graphs)
    auto t0 = Clock::now();
    for (std::uint32_t i = 0; i < S; ++i, ++k) {
      TrajectorySegment seg = pool[k % pool.size()];
      seg.model_key = lrn.current_key();
      seg.segment_seq = k;
      lrn.PushSegment(seg);
    }
    auto t1 = Clock::now();
    const auto c0 = lrn.replay().consumed_steps();
    lrn.TrainStep();
    auto t2 = Clock::now();
    if (step > 0) {
      push_s += Secs(t0, t1);
      train_s += Secs(t1, t2);
      pushed += S;
      frames += lrn.replay().consumed_steps() - c0;
    }
  }
  r.cfps = double(frames) / train_s;
  r.push_sps = double(pushed) / push_s;
  r.step_s = train_s / steps;
  return r;
}

}  // namespace

int main(int argc, char** argv) {
  const std::uint32_t S = argc > 1 ? std::uint32_t(std::atoi(argv[1])) : 4096;
  const int steps = argc > 2 ? std::atoi(argv[2]) : 4;
  const auto pool = MakePool(std::min<std::uint32_t>(S, 1024), 32, 1936, 11);
  const Result host = Run(false, S, steps, pool);
  const Result dev = Run(true, S, steps, pool);
  std::printf(
      "{\"workload\": \"C3 drop-in learner::Learner::TrainStep (MLP family 1936-256-256, PPO, "
      "T=32, %u segments per step, Adam)\", \"host_replay\": {\"cfps\": %.1f, "
      "\"train_step_ms\": %.3f, \"push_segments_per_s\": %.1f}, \"device_replay\": {\"cfps\": "
      "%.1f, \"train_step_ms\": %.3f, \"push_segments_per_s\": %.1f}, \"steps\": %d, "
      "\"unit\": \"frames/s\"}\n",
      S, host.cfps, host.step_s * 1e3, host.push_sps, dev.cfps, dev.step_s * 1e3, dev.push_sps,
      steps);
  return 0;
}
