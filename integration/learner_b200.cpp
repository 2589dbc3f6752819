// B200 drop-in implementation of tleague::learner::Learner (replaces the reference's
// src/learner/learner.cpp).  Host control flow mirrors learner.cpp line for line; the
// math of TrainStep (learner.cpp:117-152) runs on the GPU via include/tlg_b200.h.
#include "tleague/learner/learner.hpp"

#include <algorithm>
#include <atomic>
#include <exception>
#include <chrono>
#include <cmath>
#include <condition_variable>
#include <cstdio>
#include <cstring>
#include <deque>
#include <stdexcept>
#include <string_view>
#include <thread>
#include <unordered_map>
#include <unordered_set>

#include "tlg_b200.h"

namespace tleague::learner {

namespace {

// C-ABI status -> the reference's exception types (learner.cpp:129-144, rlmath.cpp).
void Check(int rc) {
  if (rc == TLG_OK) return;
  const std::string msg = tlg_last_error();
  if (rc == TLG_INVALID_ARGUMENT) throw std::invalid_argument(msg);
  throw std::runtime_error(msg);
}

// The device-side shape of a blob: PolicyFamily::kMlp carries its trunk widths in
// PolicyShape::hidden (wire tag 2); `hidden` (the config's mlp_hidden) is the older
// spelling for an MLP-layout blob tagged with another family, and must agree otherwise.
tlg_policy_shape DeviceShape(const ParamBlob& b, const std::vector<std::uint32_t>& hidden) {
  tlg_policy_shape s{};
  const bool mlp = b.family == PolicyFamily::kMlp;
  const std::vector<std::uint32_t>& h = mlp ? b.shape.hidden : hidden;
  if (mlp && !hidden.empty() && hidden != b.shape.hidden)
    throw std::invalid_argument("mlp_hidden does not match the blob's trunk widths");
  s.family = (mlp || !hidden.empty()) ? TLG_FAMILY_MLP : std::uint32_t(b.family);
  s.obs_dim = b.shape.obs_dim;
  s.n_actions = b.shape.n_actions;
  if (h.size() > 8) throw std::invalid_argument("at most 8 hidden layers");
  s.n_hidden = std::uint32_t(h.size());
  for (std::uint32_t l = 0; l < s.n_hidden; ++l) s.hidden[l] = h[l];
  return s;
}

// fn(lo, hi) over [0, n) split into contiguous ranges on up to 32 host threads (fewer
// when the work is small); the first exception (in range order) is rethrown.
template <typename F>
void ParallelRanges(std::size_t n, std::size_t work, F&& fn) {
  const std::size_t nth = std::max<std::size_t>(
      1, std::min<std::size_t>({32, std::size_t(std::max(1u, std::thread::hardware_concurrency())),
                                work / (1u << 16) + 1, n}));
  if (nth <= 1) {
    fn(std::size_t(0), n);
    return;
  }
  std::vector<std::thread> pool;
  std::vector<std::exception_ptr> errs(nth);
  for (std::size_t w = 0; w < nth; ++w)
    pool.emplace_back([&, w] {
      try {
        fn(n * w / nth, n * (w + 1) / nth);
      } catch (...) {
        errs[w] = std::current_exception();
      }
    });
  for (auto& t : pool) t.join();
  for (auto& e : errs)
    if (e) std::rethrow_exception(e);
}

// The device-replay entry the reference ReplayMem holds for a segment whose data lives in
// an HBM slot: ReplayMem reads only valid_steps (received / consumed counters,
// replay_mem.cpp:16,40), so the steps themselves are not copied; segment_seq carries the
// private id of the slot mirror.
TrajectorySegment ReplayEntry(const std::string& key, std::uint32_t valid_steps, double boot) {
  TrajectorySegment e;
  e.model_key = key;
  e.valid_steps = valid_steps;
  e.bootstrap_value = boot;
  return e;
}

template <typename T>
struct Pinned {
  T* p = nullptr;
  std::size_t n = 0;
  void ensure(std::size_t count) {
    if (count <= n) return;
    tlg_host_free(p);
    p = static_cast<T*>(tlg_host_alloc(count * sizeof(T)));
    if (!p) throw std::runtime_error("pinned host allocation failed");
    n = count;
  }
  ~Pinned() { tlg_host_free(p); }
};

}  // namespace

Algo ParseAlgo(const std::string& name) {
  // the reference's two names (learner.cpp:14-18) plus C5's PPO-over-V-trace
  static constexpr std::pair<std::string_view, Algo> kNames[] = {
      {"ppo", Algo::kPpo}, {"vtrace", Algo::kVtrace}, {"ppo_vtrace", Algo::kPpoVtrace}};
  for (const auto& [n, a] : kNames)
    if (n == name) return a;
  throw std::invalid_argument("unknown algo: " + name);
}

// One GPU learner plus pinned SoA staging for `shards` slices of the replay draw.
struct Learner::Gpu {
  tlg_learner* h = nullptr;
  // LearnerConfig::devices with G > 1: one learner per device (hs[0] == h), joined by one
  // ncclCommInitAll; each device takes num_shards / G consecutive shards of the draw
  std::vector<tlg_learner*> hs;
  tlg_policy_shape shape{};
  std::uint32_t S = 0, T = 0, shards = 0;
  std::size_t P = 0;
  Pinned<float> obs, reward, blogp, value, boot;
  Pinned<std::int32_t> action, valid;
  Pinned<std::uint8_t> done, bits;
  bool binary = false;  // this draw's observations are all 0/1: shipped bit-packed
  std::vector<tlg_segment_batch> batches;
  std::vector<tlg_step_stats> stats;

  // ---- device-resident replay (LearnerConfig::device_replay)
  // The host ReplayMem holds observation-less copies tagged with a private id (their
  // segment_seq); `live` mirrors its FIFO (Push evicts the oldest live entry exactly when
  // ReplayMem pops its front) and its reuse counts (an entry leaves after max_reuse
  // draws), so every live entry's HBM slot is known.  Pushes and draws are serialised
  // under `mu`; slots of the step in flight are pinned and freed after it.
  struct Live {
    std::uint32_t slot, uses;
  };
  tlg_replay* ring = nullptr;
  std::uint32_t ring_dtype = 0, ring_cap = 0;
  bool ring_decided = false;
  std::mutex mu;
  std::condition_variable cv;
  bool shutting_down = false;
  std::uint64_t next_id = 0;
  std::deque<std::uint64_t> fifo;                   // ids in push order (lazy deletion)
  std::unordered_map<std::uint64_t, Live> live;     // id -> slot, draws so far
  std::vector<std::uint32_t> free_slots, deferred;  // deferred: freed while pinned
  std::unordered_set<std::uint32_t> pinned;

  void ResetRing(std::size_t capacity) {
    if (ring) tlg_replay_destroy(ring);
    ring = nullptr;
    ring_decided = false;
    ring_cap = std::uint32_t(capacity) + 1;  // + the trash slot of Flush
    trash_slot = ring_cap - 1;
    stg_slots.clear();
    fifo.clear();
    live.clear();
    pinned.clear();
    deferred.clear();
    free_slots.clear();
    for (std::uint32_t i = trash_slot; i-- > 0;) free_slots.push_back(i);
  }
  void Release(std::uint32_t slot) {
    if (pinned.count(slot)) deferred.push_back(slot);
    else free_slots.push_back(slot);
  }
  // Undo log of a group of admissions: the mirror changes only when ReplayMem::Push
  // really happens, so a push that fails after Admit (a bad segment, a failed copy) is
  // rolled back before the error reaches the caller.
  struct Undo {
    std::vector<std::pair<std::uint64_t, Live>> evicted;  // in eviction order
    std::vector<std::uint32_t> taken;                      // slots handed out
    std::uint64_t first_id = 0;                            // ids >= this were added
  };
  Undo BeginAdmit() const {
    Undo u;
    u.first_id = next_id;
    return u;
  }
  // mirrors ReplayMem::Push (replay_mem.cpp:14-20) before the stripped copy is pushed
  std::uint32_t Admit(std::size_t capacity, Undo& u) {
    if (live.size() == capacity) {
      while (!fifo.empty() && !live.count(fifo.front())) fifo.pop_front();
      const std::uint64_t id = fifo.front();
      const Live e = live.at(id);
      u.evicted.emplace_back(id, e);
      Release(e.slot);
      live.erase(id);
      fifo.pop_front();
    }
    if (free_slots.empty()) throw std::runtime_error("device replay ring exhausted");
    const std::uint32_t slot = free_slots.back();
    free_slots.pop_back();
    u.taken.push_back(slot);
    return slot;
  }
  // Register an admitted segment under a fresh id (after its slot holds the data).
  std::uint64_t Enter(std::uint32_t slot) {
    live.emplace(next_id, Live{slot, 0});
    fifo.push_back(next_id);
    return next_id++;
  }
  static void Unfree(std::vector<std::uint32_t>& v, std::uint32_t slot) {
    for (std::size_t i = v.size(); i-- > 0;)
      if (v[i] == slot) {
        v.erase(v.begin() + std::ptrdiff_t(i));
        return;
      }
  }
  // Restore the mirror to its state before BeginAdmit.
  void Rollback(Undo& u) {
    while (next_id > u.first_id) {
      --next_id;
      live.erase(next_id);
      if (!fifo.empty() && fifo.back() == next_id) fifo.pop_back();
    }
    for (std::size_t i = u.taken.size(); i-- > 0;) free_slots.push_back(u.taken[i]);
    for (std::size_t i = u.evicted.size(); i-- > 0;) {
      const auto& [id, e] = u.evicted[i];
      Unfree(free_slots, e.slot);
      Unfree(deferred, e.slot);
      live.emplace(id, e);
      fifo.push_front(id);
    }
    u = Undo{};
  }
  // ---- coalesced ingest: PushSegment packs each segment (SoA, the same packing as Pack)
  // into a pinned staging batch and records its slot; the staged segments reach their HBM
  // slots in one tlg_replay_put (one copy per array, one synchronisation) when the stage
  // fills, before every draw and before a bulk push.  A slot staged twice (its entry was
  // evicted and the slot handed out again before the flush) keeps only its newest
  // segment: older copies are redirected to a trash slot past the ring's live slots.
  static constexpr std::uint32_t kStageSegs = 512;
  Pinned<std::uint8_t> stg_bits, stg_done;
  Pinned<float> stg_obs, stg_f;  // f32 obs; reward | blogp | value per frame, bootstrap
  Pinned<std::int32_t> stg_i;    // action per frame, valid_steps per segment
  std::vector<std::uint32_t> stg_slots;
  std::uint32_t trash_slot = 0;

  // Validate and pack `seg` into the next free stage position (the caller flushes a full
  // stage first); nothing is recorded until Commit, so a throw leaves no trace.
  void Prepare(const TrajectorySegment& seg) {
    const std::size_t D = shape.obs_dim, rowb = (D + 7) / 8;
    const bool bitsfmt = ring_dtype == TLG_OBS_BITS;
    if (stg_slots.size() == kStageSegs) Flush();
    const std::size_t k = stg_slots.size(), f0 = k * T;
    if (bitsfmt) stg_bits.ensure(std::size_t(kStageSegs) * T * rowb);
    else stg_obs.ensure(std::size_t(kStageSegs) * T * D);
    stg_f.ensure(std::size_t(kStageSegs) * (3 * T + 1));
    stg_i.ensure(std::size_t(kStageSegs) * (T + 1));
    stg_done.ensure(std::size_t(kStageSegs) * T);
    float* rw = stg_f.p + f0;
    float* bl = stg_f.p + std::size_t(kStageSegs) * T + f0;
    float* va = stg_f.p + 2 * std::size_t(kStageSegs) * T + f0;
    float* bo = stg_f.p + 3 * std::size_t(kStageSegs) * T + k;
    std::int32_t* ac = stg_i.p + f0;
    std::int32_t* vs = stg_i.p + std::size_t(kStageSegs) * T + k;
    std::uint8_t* dn = stg_done.p + f0;
    if (seg.valid_steps > T || seg.valid_steps > seg.steps.size())
      throw std::invalid_argument("segment valid_steps exceeds its steps / unroll_len");
    for (std::uint32_t t = 0; t < T; ++t) {
      std::uint8_t* brow = bitsfmt ? stg_bits.p + (f0 + t) * rowb : nullptr;
      float* orow = bitsfmt ? nullptr : stg_obs.p + (f0 + t) * D;
      if (bitsfmt) std::memset(brow, 0, rowb);
      if (t < seg.valid_steps) {
        const SegmentStep& st = seg.steps[t];
        if (st.obs.size() != D)
          throw std::invalid_argument("observation size does not match policy shape");
        if (bitsfmt) {
          for (std::size_t j = 0; j < D; ++j) {
            if (st.obs[j] == 1.0) brow[j >> 3] |= std::uint8_t(1u << (j & 7));
            else if (st.obs[j] != 0.0)
              throw std::invalid_argument("device replay: non-binary observation in a "
                                          "bit-packed period");
          }
        } else {
          for (std::size_t j = 0; j < D; ++j) orow[j] = float(st.obs[j]);
        }
        ac[t] = std::int32_t(st.action);
        rw[t] = float(st.reward);
        bl[t] = float(st.behavior_logp);
        va[t] = float(st.value_est);
        dn[t] = st.done ? 1 : 0;
      } else {
        if (!bitsfmt) std::memset(orow, 0, D * sizeof(float));
        ac[t] = 0;
        rw[t] = bl[t] = va[t] = 0.f;
        dn[t] = 0;
      }
    }
    *bo = float(seg.bootstrap_value);
    *vs = std::int32_t(seg.valid_steps);
  }
  // The prepared segment belongs in `slot`.
  void Commit(std::uint32_t slot) { stg_slots.push_back(slot); }
  // Staged segments -> their HBM slots (one put).  Must run before the slots are read.
  void Flush() {
    const std::size_t n = stg_slots.size();
    if (n == 0) return;
    std::vector<std::uint32_t> sl(stg_slots);
    std::unordered_set<std::uint32_t> seen;
    for (std::size_t i = n; i-- > 0;)
      if (!seen.insert(sl[i]).second) sl[i] = trash_slot;  // an older copy of a reused slot
    tlg_segment_batch b{};
    b.n_segments = std::uint32_t(n);
    b.unroll_len = T;
    b.obs_dim = shape.obs_dim;
    b.obs_dtype = ring_dtype;
    b.obs = ring_dtype == TLG_OBS_BITS ? static_cast<const void*>(stg_bits.p)
                                       : static_cast<const void*>(stg_obs.p);
    b.action = stg_i.p;
    b.reward = stg_f.p;
    b.behavior_logp = stg_f.p + std::size_t(kStageSegs) * T;
    b.value_est = stg_f.p + 2 * std::size_t(kStageSegs) * T;
    b.done = stg_done.p;
    b.bootstrap = stg_f.p + 3 * std::size_t(kStageSegs) * T;
    b.valid_steps = stg_i.p + std::size_t(kStageSegs) * T;
    stg_slots.clear();  // cleared first: a failed copy is a device error (fail-stop)
    Check(tlg_replay_put(ring, sl.data(), &b));
  }

  ~Gpu() {
    if (ring) tlg_replay_destroy(ring);
    DestroyLearners();
  }
  void DestroyLearners() {
    for (tlg_learner* x : hs) tlg_learner_destroy(x);
    hs.clear();
    h = nullptr;
  }

  bool Matches(const tlg_policy_shape& s, std::uint32_t S_, std::uint32_t T_,
               std::uint32_t sh) const {
    return h && std::memcmp(&s, &shape, sizeof(s)) == 0 && S_ == S && T_ == T && sh == shards;
  }

  // SoA packing of the reference's AoS segments (types.hpp:82-104), padding zeroed.
  // Observations made only of 0/1 planes (Pommerman-style) travel bit-packed
  // (TLG_OBS_BITS, exact, 32x fewer bytes than fp32) and take the int8 tensor-core
  // layer-1 path; anything else travels as fp32.
  void Pack(const std::vector<TrajectorySegment>& segs) {
    const std::size_t D = shape.obs_dim, F = std::size_t(S) * T * shards;
    const std::size_t rowb = (D + 7) / 8;
    // the format is decided over the whole draw first (a parallel scan)
    std::atomic<bool> all_binary{true};
    ParallelRanges(segs.size(), segs.size() * T * D, [&](std::size_t lo, std::size_t hi) {
      for (std::size_t i = lo; i < hi && all_binary.load(std::memory_order_relaxed); ++i) {
        const TrajectorySegment& seg = segs[i];
        const std::uint32_t n =
            std::min<std::uint32_t>(seg.valid_steps, std::uint32_t(seg.steps.size()));
        for (std::uint32_t t = 0; t < n; ++t)
          for (double x : seg.steps[t].obs)
            if (x != 0.0 && x != 1.0) {
              all_binary = false;
              return;
            }
      }
    });
    binary = all_binary.load();
    if (binary) bits.ensure(F * rowb);
    else obs.ensure(F * D);
    reward.ensure(F);
    blogp.ensure(F);
    value.ensure(F);
    action.ensure(F);
    done.ensure(F);
    boot.ensure(std::size_t(S) * shards);
    valid.ensure(std::size_t(S) * shards);
    // segments are independent: pack them on up to 16 host threads (a C3 draw is 4096
    // segments x 32 steps x 1936 doubles = 2 GB of fp64 observations)
    ParallelRanges(segs.size(), segs.size() * T * D,
                   [&](std::size_t lo, std::size_t hi) { PackRange(segs, lo, hi, rowb); });
    batches.assign(shards, tlg_segment_batch{});
    for (std::uint32_t r = 0; r < shards; ++r) {
      tlg_segment_batch& b = batches[r];
      const std::size_t f0 = std::size_t(r) * S * T, s0 = std::size_t(r) * S;
      b.n_segments = S;
      b.unroll_len = T;
      b.obs_dim = shape.obs_dim;
      b.obs_dtype = binary ? TLG_OBS_BITS : TLG_OBS_F32;
      b.obs = binary ? static_cast<const void*>(bits.p + f0 * rowb)
                     : static_cast<const void*>(obs.p + f0 * D);
      b.action = action.p + f0;
      b.reward = reward.p + f0;
      b.behavior_logp = blogp.p + f0;
      b.value_est = value.p + f0;
      b.done = done.p + f0;
      b.bootstrap = boot.p + s0;
      b.valid_steps = valid.p + s0;
    }
  }

  void PackRange(const std::vector<TrajectorySegment>& segs, std::size_t lo, std::size_t hi,
                 std::size_t rowb) {
    const std::size_t D = shape.obs_dim;
    for (std::size_t i = lo; i < hi; ++i) {
      const TrajectorySegment& seg = segs[i];
      if (seg.valid_steps > T || seg.valid_steps > seg.steps.size())
        throw std::invalid_argument("segment valid_steps exceeds its steps / unroll_len");
      boot.p[i] = float(seg.bootstrap_value);
      valid.p[i] = std::int32_t(seg.valid_steps);
      for (std::uint32_t t = 0; t < T; ++t) {
        const std::size_t f = i * T + t;
        if (t < seg.valid_steps) {
          const SegmentStep& st = seg.steps[t];
          if (st.obs.size() != D)
            throw std::invalid_argument("observation size does not match policy shape");
          if (binary) {
            // eight planes per byte, LSB first, without branches (vectorises)
            std::uint8_t* row = bits.p + f * rowb;
            const double* x = st.obs.data();
            const std::size_t full = D / 8;
            for (std::size_t b = 0; b < full; ++b, x += 8) {
              unsigned v = 0;
              for (int k = 0; k < 8; ++k) v |= unsigned(x[k] != 0.0) << k;
              row[b] = std::uint8_t(v);
            }
            unsigned v = 0;
            for (std::size_t j = full * 8; j < D; ++j) v |= unsigned(st.obs[j] != 0.0) << (j & 7);
            if (full * 8 < D) row[full] = std::uint8_t(v);
            std::memset(row + (D + 7) / 8, 0, rowb - (D + 7) / 8);
          } else {
            for (std::size_t j = 0; j < D; ++j) obs.p[f * D + j] = float(st.obs[j]);
          }
          action.p[f] = std::int32_t(st.action);
          reward.p[f] = float(st.reward);
          blogp.p[f] = float(st.behavior_logp);
          value.p[f] = float(st.value_est);
          done.p[f] = st.done ? 1 : 0;
        } else {  // padding (segmenter.cpp:26-31): all zero
          if (binary) std::memset(bits.p + f * rowb, 0, rowb);
          else std::memset(obs.p + f * D, 0, D * sizeof(float));
          action.p[f] = 0;
          reward.p[f] = blogp.p[f] = value.p[f] = 0.f;
          done.p[f] = 0;
        }
      }
    }
  }

  // One training step over the packed shards: on one device a single call; on G devices
  // one host thread per device issues its num_shards / G shards (the reference's shard
  // threads, learner.cpp:117-134), the gradient sum crossing NVLink in NCCL buckets.
  // The first failure (in device order) is rethrown, as learner.cpp:134-136 does.
  void Train() {
    stats.assign(shards, tlg_step_stats{});
    const int G = int(hs.size());
    if (G <= 1) {
      Check(tlg_learner_train_step_shards(h, batches.data(), int(shards), /*on_device=*/0,
                                          stats.data()));
      return;
    }
    const int per = int(shards) / G;
    std::vector<int> rc(G, TLG_OK);
    std::vector<std::string> msg(G);
    std::vector<std::thread> th;
    for (int g = 0; g < G; ++g)
      th.emplace_back([&, g] {
        rc[g] = tlg_learner_train_step_shards(hs[g], batches.data() + g * per, per, 0,
                                              stats.data() + g * per);
        if (rc[g] != TLG_OK) msg[g] = tlg_last_error();  // thread-local message
      });
    for (auto& t : th) t.join();
    for (int g = 0; g < G; ++g)
      if (rc[g] != TLG_OK) {
        if (rc[g] == TLG_INVALID_ARGUMENT) throw std::invalid_argument(msg[g]);
        throw std::runtime_error(msg[g]);
      }
  }
};

Learner::Learner(LearnerConfig config, league::LeagueIface& league, pool::ModelPoolIface& pool)
    : config_(std::move(config)),
      league_(league),
      pool_(pool),
      replay_(config_.replay_capacity, /*max_reuse set per task*/ 1, config_.seed),
      gpu_(std::make_unique<Gpu>()) {
  if (config_.num_shards == 0) throw std::invalid_argument("num_shards must be >= 1");
  if (config_.devices.size() > 1) {
    if (config_.num_shards % config_.devices.size() != 0)
      throw std::invalid_argument("num_shards must be a multiple of the number of devices");
    if (config_.device_replay)
      throw std::invalid_argument("device_replay runs on a single device");
  }
  StartPeriod();
}

Learner::~Learner() = default;

void Learner::StartPeriod() {
  Task task = league_.RequestLearnerTask(config_.group, 0);
  ModelRecord record = pool_.GetModel(task.learning_model_key);
  std::lock_guard lock(task_mu_);
  current_key_ = task.learning_model_key;
  hyper_ = task.hyperparams;
  params_ = std::move(record.params);
  params_stale_ = false;
  parent_key_ = record.parent_key;
  created_at_us_ = record.created_at_us;
  replay_.Clear();
  replay_.SetMaxReuse(hyper_.max_reuse);

  // (Re)configure the device learner for this period's blob and hyperparameters.
  const tlg_policy_shape s = DeviceShape(params_, config_.mlp_hidden);
  const std::uint32_t S = hyper_.batch_size, T = hyper_.unroll_len;
  if (gpu_->ring) {  // the ring belongs to the device learner: drop it first
    std::lock_guard dl(gpu_->mu);
    tlg_replay_destroy(gpu_->ring);
    gpu_->ring = nullptr;
  }
  if (!gpu_->Matches(s, S, T, config_.num_shards)) {
    gpu_->DestroyLearners();
    tlg_learner_config c{};
    c.algo = config_.algo == Algo::kPpo      ? TLG_ALGO_PPO
             : config_.algo == Algo::kVtrace ? TLG_ALGO_VTRACE
                                             : TLG_ALGO_PPO_VTRACE;
    c.optimizer = config_.optimizer == Optimizer::kAdam ? TLG_OPT_ADAM : TLG_OPT_SGD;
    c.adam_beta1 = config_.adam_beta1;
    c.adam_beta2 = config_.adam_beta2;
    c.adam_eps = config_.adam_eps;
    c.max_segments = S;
    c.unroll_len = T;
    c.obs_dtype = TLG_OBS_BITS;  // accepts fp32 and bit-packed batches
    const std::vector<int> devs =
        config_.devices.size() > 1 ? config_.devices : std::vector<int>{config_.device};
    for (int d : devs) {
      c.device = d;
      tlg_learner* x = nullptr;
      Check(tlg_learner_create(&c, &s, &x));
      gpu_->hs.push_back(x);
    }
    gpu_->h = gpu_->hs[0];
    if (gpu_->hs.size() > 1)
      Check(tlg_learner_comm_init_all(gpu_->hs.data(), int(gpu_->hs.size())));
    gpu_->shape = s;
    gpu_->S = S;
    gpu_->T = T;
    gpu_->shards = config_.num_shards;
    gpu_->P = tlg_learner_param_count(gpu_->h);
  }
  tlg_hyper hp{hyper_.learning_rate, hyper_.gamma, hyper_.lam, hyper_.clip_eps,
               hyper_.vf_coef, hyper_.ent_coef, hyper_.kl_teacher_coef, hyper_.rho_bar,
               hyper_.c_bar, hyper_.batch_size, hyper_.unroll_len, hyper_.max_reuse,
               hyper_.adv_norm ? 1 : 0};
  for (tlg_learner* x : gpu_->hs) {  // identical parameters and optimizer state everywhere
    Check(tlg_learner_set_hyper(x, &hp));
    Check(tlg_learner_set_params(x, params_.values.data(), params_.values.size()));
  }
  if (config_.device_replay) {
    std::lock_guard dl(gpu_->mu);
    // replay_capacity live entries + the slots pinned by one draw
    gpu_->ResetRing(config_.replay_capacity + std::size_t(S) * config_.num_shards);
  }
}

void Learner::Shutdown() {
  replay_.Shutdown();
  std::lock_guard dl(gpu_->mu);
  gpu_->shutting_down = true;
  gpu_->cv.notify_all();
}

void Learner::PushSegment(const TrajectorySegment& segment) {
  {
    std::lock_guard lock(task_mu_);
    if (segment.model_key != current_key_) {
      stale_dropped_.fetch_add(1, std::memory_order_relaxed);
      return;
    }
  }
  if (!config_.device_replay) {
    replay_.Push(segment);
    return;
  }
  Gpu& g = *gpu_;
  std::lock_guard dl(g.mu);
  if (!g.ring_decided) {  // the period's first segment fixes the ring's format
    bool binary = true;
    const std::uint32_t n = std::min<std::uint32_t>(segment.valid_steps,
                                                    std::uint32_t(segment.steps.size()));
    for (std::uint32_t t = 0; t < n && binary; ++t)
      for (double x : segment.steps[t].obs)
        if (x != 0.0 && x != 1.0) {
          binary = false;
          break;
        }
    g.ring_dtype = binary ? TLG_OBS_BITS : TLG_OBS_F32;
    Check(tlg_replay_create(g.h, g.ring_cap, g.ring_dtype, &g.ring));
    g.ring_decided = true;
  }
  g.Prepare(segment);  // throws on a bad segment before the mirror changes
  TrajectorySegment stripped = ReplayEntry(segment.model_key, segment.valid_steps,
                                           segment.bootstrap_value);
  Gpu::Undo undo = g.BeginAdmit();
  try {
    const std::uint32_t slot = g.Admit(config_.replay_capacity, undo);
    g.Commit(slot);
    stripped.segment_seq = g.Enter(slot);
    replay_.Push(std::move(stripped));
  } catch (...) {
    g.Rollback(undo);
    throw;
  }
  g.cv.notify_all();
}

namespace {
// one SoA segment -> a TrajectorySegment (observations widened exactly to f64)
TrajectorySegment SegmentFromSoa(const tlg_segment_batch& b, std::uint32_t i,
                                 const std::string& key) {
  const std::uint32_t T = b.unroll_len, D = b.obs_dim;
  const std::size_t rowb = b.obs_pitch ? b.obs_pitch : (D + 7) / 8;
  TrajectorySegment seg;
  seg.model_key = key;
  seg.valid_steps = std::uint32_t(b.valid_steps[i]);
  seg.bootstrap_value = b.bootstrap[i];
  seg.steps.resize(seg.valid_steps);
  for (std::uint32_t t = 0; t < seg.valid_steps; ++t) {
    const std::size_t f = std::size_t(i) * T + t;
    SegmentStep& st = seg.steps[t];
    st.obs.resize(D);
    if (b.obs_dtype == TLG_OBS_BITS) {
      const auto* row = static_cast<const std::uint8_t*>(b.obs) + f * rowb;
      for (std::uint32_t j = 0; j < D; ++j) st.obs[j] = (row[j >> 3] >> (j & 7)) & 1u;
    } else {
      const float* row = static_cast<const float*>(b.obs) + f * D;
      for (std::uint32_t j = 0; j < D; ++j) st.obs[j] = row[j];
    }
    st.action = std::uint32_t(b.action[f]);
    st.reward = b.reward[f];
    st.behavior_logp = b.behavior_logp[f];
    st.value_est = b.value_est[f];
    st.done = b.done[f] != 0;
  }
  return seg;
}
}  // namespace

void Learner::PushSegmentBatch(const std::string& model_key, const tlg_segment_batch& b) {
  if (b.obs_dtype != TLG_OBS_F32 && b.obs_dtype != TLG_OBS_BITS)
    throw std::invalid_argument("PushSegmentBatch: observations must be f32 or bit planes");
  if (b.n_segments == 0) return;
  if (b.n_segments > config_.replay_capacity)
    throw std::invalid_argument("PushSegmentBatch: more segments than replay_capacity");
  for (std::uint32_t i = 0; i < b.n_segments; ++i)
    if (b.valid_steps[i] < 0 || std::uint32_t(b.valid_steps[i]) > b.unroll_len)
      throw std::invalid_argument("segment valid_steps exceeds its steps / unroll_len");
  {
    std::lock_guard lock(task_mu_);
    if (model_key != current_key_) {
      stale_dropped_.fetch_add(b.n_segments, std::memory_order_relaxed);
      return;
    }
  }
  if (!config_.device_replay) {
    for (std::uint32_t i = 0; i < b.n_segments; ++i) replay_.Push(SegmentFromSoa(b, i, model_key));
    return;
  }
  Gpu& g = *gpu_;
  std::lock_guard dl(g.mu);
  if (b.unroll_len != g.T || b.obs_dim != g.shape.obs_dim)
    throw std::invalid_argument("PushSegmentBatch: unroll_len / obs_dim do not match");
  if (!g.ring_decided) {
    g.ring_dtype = b.obs_dtype;
    Check(tlg_replay_create(g.h, g.ring_cap, g.ring_dtype, &g.ring));
    g.ring_decided = true;
  }
  if (b.obs_dtype != g.ring_dtype)
    throw std::invalid_argument("PushSegmentBatch: observation format differs from the period's");
  g.Flush();  // staged single pushes land first: this batch may reuse their slots
  if (b.obs_dtype == TLG_OBS_BITS && b.obs_pitch != 0 &&
      (b.obs_pitch < (b.obs_dim + 7) / 8 || b.obs_pitch > ((b.obs_dim + 7) / 8 + 15) / 16 * 16))
    throw std::invalid_argument("PushSegmentBatch: bad obs_pitch");
  // observation-less entries first (nothing below can fail on the caller's data)
  std::vector<TrajectorySegment> stripped(b.n_segments);
  for (std::uint32_t i = 0; i < b.n_segments; ++i) {
    stripped[i] = ReplayEntry(model_key, std::uint32_t(b.valid_steps[i]), b.bootstrap[i]);
  }
  // admit in order (mirrors n ReplayMem::Push evictions), one device copy, then the
  // entries in the same order; any failure restores the mirror
  std::vector<std::uint32_t> slots(b.n_segments);
  Gpu::Undo undo = g.BeginAdmit();
  try {
    // each admission sees the previous ones (the FIFO evicts as n single pushes would)
    for (std::uint32_t i = 0; i < b.n_segments; ++i) {
      slots[i] = g.Admit(config_.replay_capacity, undo);
      stripped[i].segment_seq = g.Enter(slots[i]);
    }
    Check(tlg_replay_put(g.ring, slots.data(), &b));
  } catch (...) {
    g.Rollback(undo);
    throw;
  }
  for (std::uint32_t i = 0; i < b.n_segments; ++i) replay_.Push(std::move(stripped[i]));
  g.cv.notify_all();
}

void Learner::PushSegmentBatch(const SegmentBatch& b) {
  if (b.n_segments == 0) return;
  const std::size_t F = std::size_t(b.n_segments) * b.unroll_len;
  if (b.action.size() != F || b.valid_steps.size() != b.n_segments)
    throw std::invalid_argument("PushSegmentBatch: inconsistent segment batch");
  tlg_segment_batch v{};
  v.n_segments = b.n_segments;
  v.unroll_len = b.unroll_len;
  v.obs_dim = b.obs_dim;
  v.obs_dtype = b.obs_format == SegmentBatch::kObsBits ? TLG_OBS_BITS : TLG_OBS_F32;
  v.obs = b.obs.data();
  v.action = b.action.data();
  v.reward = b.reward.data();
  v.behavior_logp = b.behavior_logp.data();
  v.value_est = b.value_est.data();
  v.done = b.done.data();
  v.bootstrap = b.bootstrap.data();
  v.valid_steps = b.valid_steps.data();
  PushSegmentBatch(b.model_key, v);
}

bool Learner::TrainStep() {
  if (config_.step_delay_ms > 0)
    std::this_thread::sleep_for(std::chrono::milliseconds(config_.step_delay_ms));
  const std::size_t per_shard = hyper_.batch_size;
  if (config_.device_replay) return TrainStepDeviceReplay(per_shard);
  auto segments = replay_.SampleBlocking(per_shard * config_.num_shards);
  if (segments.empty()) return false;
  gpu_->Pack(segments);
  // Per-shard gradients, rank-ordered mean, optimizer.  Errors come back as the
  // reference's exception types; on failure the parameters are unchanged.
  gpu_->Train();
  ++update_steps_;
  params_stale_ = true;
  if (config_.publish_interval > 0 && update_steps_ % config_.publish_interval == 0) Publish();
  return true;
}

// TrainStep over the device-resident ring: the same ReplayMem draw (pushes are held off
// while it happens, so the live-entry mirror stays exact), then a device gather by slot.
bool Learner::TrainStepDeviceReplay(std::size_t per_shard) {
  Gpu& g = *gpu_;
  const std::size_t n = per_shard * config_.num_shards;
  std::vector<std::uint32_t> slots;
  {
    std::unique_lock dl(g.mu);
    g.cv.wait(dl, [&] { return g.shutting_down || replay_.size() >= n; });
    if (g.shutting_down) return false;
    g.Flush();  // every live entry's observations are in HBM before the gather
    auto segments = replay_.SampleBlocking(n);  // cannot block: pushes are held off
    if (segments.empty()) return false;
    slots.reserve(n);
    for (const TrajectorySegment& seg : segments) {
      Gpu::Live& e = g.live.at(seg.segment_seq);
      slots.push_back(e.slot);
      g.pinned.insert(e.slot);
      if (++e.uses >= hyper_.max_reuse) {  // ReplayMem erased it (replay_mem.cpp:41-44)
        g.Release(e.slot);
        g.live.erase(seg.segment_seq);
      }
    }
  }
  g.stats.assign(config_.num_shards, tlg_step_stats{});
  int rc = tlg_learner_train_step_replay(g.h, g.ring, slots.data(), config_.num_shards,
                                         std::uint32_t(per_shard), g.stats.data());
  {
    std::lock_guard dl(g.mu);
    g.pinned.clear();
    g.free_slots.insert(g.free_slots.end(), g.deferred.begin(), g.deferred.end());
    g.deferred.clear();
  }
  Check(rc);
  ++update_steps_;
  params_stale_ = true;
  if (config_.publish_interval > 0 && update_steps_ % config_.publish_interval == 0) Publish();
  return true;
}

void Learner::SyncParams() const {
  if (!params_stale_) return;
  Check(tlg_learner_get_params(gpu_->h, params_.values.data(), params_.values.size()));
  params_stale_ = false;
}

const ParamBlob& Learner::params() const {
  SyncParams();
  return params_;
}

// The record the pool holds for the learning model: the current parameters (mirrored
// from the device) under the period's key, lineage and hyperparameters, not frozen
// (learner.cpp:160-172).
void Learner::Publish() {
  const ParamBlob& now = params();
  pool_.PutModel(ModelRecord{.model_key = current_key_,
                             .params = now,
                             .hyperparams = hyper_,
                             .parent_key = parent_key_,
                             .created_at_us = created_at_us_,
                             .frozen = false});
}

// Period rollover (learner.cpp:174-186): the final parameters reach the pool before the
// league freezes the member; then the successor period begins.
std::string Learner::FinishPeriod() {
  Publish();
  const std::string successor = league_.EndLearningPeriod(config_.group);
  StartPeriod();
  return successor;
}

std::string Learner::RunPeriod() {
  std::uint32_t done = 0;
  while (done < config_.period_steps && TrainStep()) ++done;
  // a shut-down replay ends the period early: no rollover, empty key
  return done == config_.period_steps ? FinishPeriod() : std::string();
}

ThroughputStats Learner::Counters() const {
  // cumulative step counts (not rates), as the reference reports them
  return ThroughputStats{double(replay_.received_steps()), double(replay_.consumed_steps()),
                         update_steps_, stale_dropped_.load(std::memory_order_relaxed)};
}

// `ts=<unix s> group=<g> rfps=<r> cfps=<c> steps=<k>` with the receive / consume rates
// since the previous call (zero on the first), learner.cpp:197-218.
void Learner::LogMetricsLine(std::string& out) {
  const double t = std::chrono::duration<double>(
                       std::chrono::steady_clock::now().time_since_epoch()).count();
  const std::uint64_t got = replay_.received_steps(), used = replay_.consumed_steps();
  const double span = t - last_metric_ts_;
  const bool have_rate = last_metric_ts_ > 0.0 && span > 0.0;
  const double rfps = have_rate ? double(got - last_metric_recv_) / span : 0.0;
  const double cfps = have_rate ? double(used - last_metric_cons_) / span : 0.0;
  last_metric_ts_ = t;
  last_metric_recv_ = got;
  last_metric_cons_ = used;
  const long long unix_s = std::chrono::duration_cast<std::chrono::seconds>(
                               std::chrono::system_clock::now().time_since_epoch()).count();
  char line[160];
  std::snprintf(line, sizeof(line), "ts=%lld group=%u rfps=%.1f cfps=%.1f steps=%llu\n", unix_s,
                config_.group, rfps, cfps, static_cast<unsigned long long>(update_steps_));
  out.append(line);
}

}  // namespace tleague::learner
