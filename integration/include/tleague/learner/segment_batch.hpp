// A group of trajectory segments of one model key in columnar (SoA) form: the payload of
// the bulk segment message (MsgKind::kSegmentBatchPush, wire tag 17, appended by
// integration/patches/wire_ext.py) and the host mirror of the C ABI's tlg_segment_batch
// (include/tlg_b200.h).  Compared with n SegmentPush frames of fp64 AoS steps
// (codec.cpp:199-213: 8 bytes per observation element plus per-step headers), a batch
// carries fp32 values -- or 0/1 observation planes bit-packed, 1 bit per element -- in
// one frame, and the B200 learner copies it into its HBM replay ring as is.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "tleague/types.hpp"

namespace tleague {

struct SegmentBatch {
  static constexpr std::uint32_t kObsF32 = 0;   // obs: [n][T][obs_dim] float32
  static constexpr std::uint32_t kObsBits = 2;  // obs: [n][T] rows of ceil(obs_dim/8) bytes
  std::string model_key;
  std::uint32_t n_segments = 0, unroll_len = 0, obs_dim = 0, obs_format = kObsF32;
  std::vector<std::uint8_t> obs;
  std::vector<std::int32_t> action;       // [n][T]
  std::vector<float> reward;              // [n][T]
  std::vector<float> behavior_logp;       // [n][T]
  std::vector<float> value_est;           // [n][T]
  std::vector<std::uint8_t> done;         // [n][T]
  std::vector<float> bootstrap;           // [n]
  std::vector<std::int32_t> valid_steps;  // [n]
  std::vector<std::uint64_t> segment_seq; // [n]
  bool operator==(const SegmentBatch&) const = default;
};

// AoS -> SoA.  Steps past valid_steps are zero (segmenter.cpp:26-31).  With
// allow_bits, a group whose observations are all 0/1 travels bit-packed.  Values are
// rounded to fp32.  Throws std::invalid_argument on inconsistent segments.
SegmentBatch PackSegmentBatch(const std::vector<TrajectorySegment>& segs,
                              std::uint32_t unroll_len, bool allow_bits = true);
// SoA -> AoS (observations widened exactly to fp64); valid_steps steps per segment.
std::vector<TrajectorySegment> UnpackSegmentBatch(const SegmentBatch& b);

}  // namespace tleague
