// The drop-in ReplayMem (integration/replay_mem_b200.cpp) against the reference's own
// (src/learner/replay_mem.cpp, compiled into this test under another class name): random
// push / sample / clear sequences at several capacities and reuse bounds must give the
// same segments in the same order and the same counters.  CPU only; built with the
// reference sources present (integration/Makefile).
#include <chrono>
#include <cstdio>
#include <random>
#include <string>

#include "tleague/learner/replay_mem.hpp"  // the drop-in (integration/include first)

#define ReplayMem RefReplayMem
#include TLG_REF_REPLAY_HPP
#include TLG_REF_REPLAY_CPP
#undef ReplayMem

using namespace tleague;

namespace {

int failures = 0;

void Expect(bool ok, const char* what, int round) {
  if (!ok) {
    ++failures;
    if (failures < 20) std::printf("  MISMATCH %s (round %d)\n", what, round);
  }
}

TrajectorySegment Seg(std::uint64_t seq, std::uint32_t valid) {
  TrajectorySegment s;
  s.model_key = "k";
  s.segment_seq = seq;
  s.valid_steps = valid;
  return s;
}

void Fuzz(std::size_t capacity, std::uint32_t max_reuse, std::uint64_t seed, int rounds) {
  learner::ReplayMem ours(capacity, max_reuse, seed);
  learner::RefReplayMem ref(capacity, max_reuse, seed);
  std::mt19937_64 ops(seed * 7 + capacity);
  std::uint64_t seq = 0;
  for (int r = 0; r < rounds; ++r) {
    const int op = int(ops() % 100);
    if (op < 55) {
      const int k = 1 + int(ops() % (capacity + 2));
      for (int i = 0; i < k; ++i) {
        const std::uint32_t valid = std::uint32_t(ops() % 33);
        ours.Push(Seg(seq, valid));
        ref.Push(Seg(seq, valid));
        ++seq;
      }
    } else if (op < 97) {
      if (ref.size() == 0) continue;
      const std::size_t n = 1 + std::size_t(ops() % ref.size());
      auto a = ours.SampleBlocking(n), b = ref.SampleBlocking(n);
      bool same = a.size() == b.size();
      for (std::size_t i = 0; same && i < a.size(); ++i)
        same = a[i].segment_seq == b[i].segment_seq && a[i].valid_steps == b[i].valid_steps;
      Expect(same, "sampled segments", r);
    } else {
      ours.Clear();
      ref.Clear();
      const std::uint32_t m = 1 + std::uint32_t(ops() % 3);
      ours.SetMaxReuse(m);
      ref.SetMaxReuse(m);
    }
    Expect(ours.size() == ref.size(), "size", r);
    Expect(ours.received_steps() == ref.received_steps(), "received_steps", r);
    Expect(ours.consumed_steps() == ref.consumed_steps(), "consumed_steps", r);
  }
}

}  // namespace

int main() {
  for (std::size_t cap : {1, 2, 5, 17, 64, 300})
    for (std::uint32_t reuse : {1u, 2u, 3u})
      for (std::uint64_t seed : {1ull, 99ull}) Fuzz(cap, reuse, seed, 4000);
  // the C3 shape: 4096-segment draws from an 8192-entry ring, max_reuse 1
  {
    learner::ReplayMem ours(8192, 1, 5);
    learner::RefReplayMem ref(8192, 1, 5);
    double t_ours = 0, t_ref = 0;
    std::uint64_t seq = 0;
    for (int step = 0; step < 6; ++step) {
      for (int i = 0; i < 4096 + 512 * step; ++i, ++seq) {
        ours.Push(Seg(seq, 32));
        ref.Push(Seg(seq, 32));
      }
      const auto t0 = std::chrono::steady_clock::now();
      auto a = ours.SampleBlocking(4096);
      const auto t1 = std::chrono::steady_clock::now();
      auto b = ref.SampleBlocking(4096);
      const auto t2 = std::chrono::steady_clock::now();
      t_ours += std::chrono::duration<double>(t1 - t0).count();
      t_ref += std::chrono::duration<double>(t2 - t1).count();
      bool same = a.size() == b.size();
      for (std::size_t i = 0; same && i < a.size(); ++i) same = a[i].segment_seq == b[i].segment_seq;
      Expect(same, "C3 draw", step);
    }
    std::printf("C3 draw (4096 of <= 8192, max_reuse 1): drop-in %.3f ms, reference %.3f ms\n",
                t_ours / 6 * 1e3, t_ref / 6 * 1e3);
  }
  std::printf("%s (%d mismatches)\n", failures ? "REPLAY MEM TEST FAILED" : "REPLAY MEM TEST PASSED",
              failures);
  return failures ? 1 : 0;
}
