// B200 drop-in for tleague's learner::Learner (reference: include/tleague/learner/learner.hpp).
//
// Same public interface, same semantics: a maintainer replaces src/learner/learner.cpp
// with integration/learner_b200.cpp and puts this header ahead of the reference's on the
// include path; callers (run::LocalRun, run::RunBench, the CLI learner) recompile
// unchanged.  The replay ring, stale-key filter, publish cadence and period rollover
// stay on the host exactly as in the reference (ReplayMem is the reference's own,
// replay_mem.cpp); the per-shard batch assembly, returns, loss fwd/bwd, rank-ordered
// gradient mean and optimizer run on the GPU through the C ABI of include/tlg_b200.h.
//
// Additions (defaulted, so existing aggregate initialisation keeps compiling): the CUDA
// device, the optimizer (SGD = the reference's rlmath::SgdStep, or Adam), and the MLP
// trunk widths for the appended MLP policy family.
#pragma once

#include <atomic>
#include <cstdint>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "tleague/league/league_iface.hpp"
#include "tleague/learner/replay_mem.hpp"
#include "tleague/learner/segment_sink.hpp"
#include "tleague/pool/pool_iface.hpp"
#include "tleague/types.hpp"

struct tlg_segment_batch;  // include/tlg_b200.h (SoA segment batch of the C ABI)

namespace tleague::learner {

enum class Algo { kPpo, kVtrace, kPpoVtrace };

// "ppo" | "vtrace" | "ppo_vtrace"; throws std::invalid_argument otherwise.
Algo ParseAlgo(const std::string& name);

enum class Optimizer { kSgd, kAdam };

struct LearnerConfig {
  std::uint32_t group = 0;
  std::uint32_t num_shards = 1;
  Algo algo = Algo::kPpo;
  std::uint32_t publish_interval = 10;
  std::uint32_t period_steps = 100;
  std::size_t replay_capacity = 4096;
  std::uint64_t seed = 0;
  std::uint32_t step_delay_ms = 0;
  // ---- B200 additions
  int device = 0;
  // More than one entry: data-parallel over these devices in this process (one learner
  // and one host thread per device, NCCL over NVLink); num_shards must be a multiple of
  // devices.size(), each device taking num_shards / devices.size() consecutive shards.
  std::vector<int> devices;
  Optimizer optimizer = Optimizer::kSgd;
  double adam_beta1 = 0.9, adam_beta2 = 0.999, adam_eps = 1e-8;
  // Non-empty: the blob is an MLP (flat [W_1,b_1,...,W_L,b_L | W_pi,b_pi | w_v,b_v])
  // over ParamBlob::shape {obs_dim, n_actions}.
  std::vector<std::uint32_t> mlp_hidden;
  // Device-resident replay: PushSegment copies each segment into an HBM slot once; the
  // host ReplayMem keeps making the (bit-identical) draw decisions over entries whose
  // observations are dropped, and TrainStep gathers the drawn slots on the device (no
  // per-step packing or observation H2D).  Within a period all observations must be
  // 0/1 planes or all fp32 values, fixed by the first segment.
  bool device_replay = false;
};

struct ThroughputStats {
  double rfps = 0.0;
  double cfps = 0.0;
  std::uint64_t update_steps = 0;
  std::uint64_t stale_dropped = 0;
};

class Learner : public SegmentSink {
 public:
  Learner(LearnerConfig config, league::LeagueIface& league, pool::ModelPoolIface& pool);
  ~Learner() override;

  Learner(const Learner&) = delete;
  Learner& operator=(const Learner&) = delete;

  void StartPeriod();
  void PushSegment(const TrajectorySegment& segment) override;
  // Bulk SoA ingest (an extension): `batch.n_segments` segments of one
  // model key in the C ABI's SoA layout (TLG_OBS_F32 or TLG_OBS_BITS) — what a bulk
  // segment message would carry.  Same replay bookkeeping and draws as that many
  // PushSegment calls in order; with device_replay the observations go to their HBM
  // slots in one copy instead of one per segment.  At most replay_capacity segments.
  void PushSegmentBatch(const std::string& model_key, const tlg_segment_batch& batch);
  // The same for the bulk segment message (message kind 17, SegmentSink extension): the
  // batch's SoA arrays are handed to the device ring without unpacking.
  void PushSegmentBatch(const SegmentBatch& batch) override;
  bool TrainStep();
  std::string FinishPeriod();
  std::string RunPeriod();
  void Shutdown();

  const std::string& current_key() const { return current_key_; }
  // Host fp64 mirror of the device parameters, refreshed lazily after updates.
  const ParamBlob& params() const;
  const HyperParams& hyper() const { return hyper_; }
  std::uint64_t update_steps() const { return update_steps_; }
  ReplayMem& replay() { return replay_; }

  ThroughputStats Counters() const;
  void LogMetricsLine(std::string& out);

 private:
  struct Gpu;
  void Publish();
  bool TrainStepDeviceReplay(std::size_t per_shard);
  void SyncParams() const;

  LearnerConfig config_;
  league::LeagueIface& league_;
  pool::ModelPoolIface& pool_;
  ReplayMem replay_;

  std::mutex task_mu_;
  std::string current_key_;
  HyperParams hyper_;
  mutable ParamBlob params_;
  mutable bool params_stale_ = false;
  std::string parent_key_;
  std::uint64_t created_at_us_ = 0;
  std::uint64_t update_steps_ = 0;
  std::atomic<std::uint64_t> stale_dropped_{0};
  std::unique_ptr<Gpu> gpu_;

  std::uint64_t last_metric_recv_ = 0;
  std::uint64_t last_metric_cons_ = 0;
  double last_metric_ts_ = 0.0;
};

}  // namespace tleague::learner
