// Wire extensions (message kinds 17 SegmentBatchPush and 18 ParamChunk): see
// tleague/proto/wire_ext.hpp.  Compiled into the services archive next to the patched
// reference codec / pool / learner-service translation units.
#include "tleague/proto/wire_ext.hpp"

#include <cstring>
#include <fstream>
#include <map>
#include <mutex>
#include <random>
#include <stdexcept>
#include <tuple>

#include "tleague/net/tcp.hpp"
#include "tleague/pool/model_store.hpp"
#include "tleague/proto/codec.hpp"

namespace tleague {

// ---------------------------------------------------------------------------
// SegmentBatch <-> TrajectorySegment
SegmentBatch PackSegmentBatch(const std::vector<TrajectorySegment>& segs,
                              std::uint32_t unroll_len, bool allow_bits) {
  SegmentBatch b;
  const std::uint32_t T = unroll_len;
  if (T == 0) throw std::invalid_argument("unroll_len must be >= 1");
  b.n_segments = static_cast<std::uint32_t>(segs.size());
  b.unroll_len = T;
  if (!segs.empty()) b.model_key = segs.front().model_key;
  for (const auto& s : segs) {
    if (s.model_key != b.model_key)
      throw std::invalid_argument("a segment batch carries one model key");
    if (s.valid_steps > T || s.valid_steps > s.steps.size())
      throw std::invalid_argument("segment valid_steps exceeds its steps / unroll_len");
    for (std::uint32_t t = 0; t < s.valid_steps; ++t) {
      if (b.obs_dim == 0) b.obs_dim = static_cast<std::uint32_t>(s.steps[t].obs.size());
      if (s.steps[t].obs.size() != b.obs_dim)
        throw std::invalid_argument("observation sizes differ within a segment batch");
    }
  }
  bool bits = allow_bits;
  for (const auto& s : segs)
    for (std::uint32_t t = 0; t < s.valid_steps && bits; ++t)
      for (double x : s.steps[t].obs)
        if (x != 0.0 && x != 1.0) {
          bits = false;
          break;
        }
  b.obs_format = bits ? SegmentBatch::kObsBits : SegmentBatch::kObsF32;
  const std::size_t n = segs.size(), F = n * T, D = b.obs_dim, rowb = (D + 7) / 8;
  b.obs.assign(bits ? F * rowb : F * D * sizeof(float), 0);
  b.action.assign(F, 0);
  b.reward.assign(F, 0.f);
  b.behavior_logp.assign(F, 0.f);
  b.value_est.assign(F, 0.f);
  b.done.assign(F, 0);
  b.bootstrap.assign(n, 0.f);
  b.valid_steps.assign(n, 0);
  b.segment_seq.assign(n, 0);
  for (std::size_t i = 0; i < n; ++i) {
    const TrajectorySegment& s = segs[i];
    b.bootstrap[i] = static_cast<float>(s.bootstrap_value);
    b.valid_steps[i] = static_cast<std::int32_t>(s.valid_steps);
    b.segment_seq[i] = s.segment_seq;
    for (std::uint32_t t = 0; t < s.valid_steps; ++t) {
      const std::size_t f = i * T + t;
      const SegmentStep& st = s.steps[t];
      if (bits) {
        std::uint8_t* row = b.obs.data() + f * rowb;
        for (std::size_t j = 0; j < D; ++j)
          if (st.obs[j] != 0.0) row[j >> 3] |= static_cast<std::uint8_t>(1u << (j & 7));
      } else {
        float* row = reinterpret_cast<float*>(b.obs.data()) + f * D;
        for (std::size_t j = 0; j < D; ++j) row[j] = static_cast<float>(st.obs[j]);
      }
      b.action[f] = static_cast<std::int32_t>(st.action);
      b.reward[f] = static_cast<float>(st.reward);
      b.behavior_logp[f] = static_cast<float>(st.behavior_logp);
      b.value_est[f] = static_cast<float>(st.value_est);
      b.done[f] = st.done ? 1 : 0;
    }
  }
  return b;
}

std::vector<TrajectorySegment> UnpackSegmentBatch(const SegmentBatch& b) {
  const std::size_t n = b.n_segments, T = b.unroll_len, D = b.obs_dim, rowb = (D + 7) / 8;
  const bool bits = b.obs_format == SegmentBatch::kObsBits;
  std::vector<TrajectorySegment> out(n);
  for (std::size_t i = 0; i < n; ++i) {
    TrajectorySegment& s = out[i];
    s.model_key = b.model_key;
    s.valid_steps = static_cast<std::uint32_t>(b.valid_steps[i]);
    s.bootstrap_value = b.bootstrap[i];
    s.segment_seq = b.segment_seq[i];
    s.steps.resize(s.valid_steps);
    for (std::size_t t = 0; t < s.valid_steps; ++t) {
      const std::size_t f = i * T + t;
      SegmentStep& st = s.steps[t];
      st.obs.resize(D);
      if (bits) {
        const std::uint8_t* row = b.obs.data() + f * rowb;
        for (std::size_t j = 0; j < D; ++j) st.obs[j] = (row[j >> 3] >> (j & 7)) & 1u;
      } else {
        const float* row = reinterpret_cast<const float*>(b.obs.data()) + f * D;
        for (std::size_t j = 0; j < D; ++j) st.obs[j] = row[j];
      }
      st.action = static_cast<std::uint32_t>(b.action[f]);
      st.reward = b.reward[f];
      st.behavior_logp = b.behavior_logp[f];
      st.value_est = b.value_est[f];
      st.done = b.done[f] != 0;
    }
  }
  return out;
}

namespace proto::ext {

namespace {

// little-endian scalar / array packing (the reference codec's byte order, codec.cpp:10-40)
template <typename T>
void PutScalar(std::string& s, T v) {
  for (std::size_t i = 0; i < sizeof(T); ++i)
    s.push_back(static_cast<char>(static_cast<std::uint64_t>(v) >> (8 * i)));
}
template <typename T>
void PutArray(std::string& s, const std::vector<T>& v) {
  PutScalar<std::uint64_t>(s, v.size());
  const std::size_t bytes = v.size() * sizeof(T);
  const std::size_t at = s.size();
  s.resize(at + bytes);
  if (bytes) std::memcpy(s.data() + at, v.data(), bytes);  // little-endian host
}

struct Cursor {
  const std::string& s;
  std::size_t pos = 0;
  void Need(std::size_t n) const {
    if (s.size() - pos < n) throw DecodeError("truncated segment batch");
  }
  template <typename T>
  T Scalar() {
    Need(sizeof(T));
    std::uint64_t v = 0;
    for (std::size_t i = 0; i < sizeof(T); ++i)
      v |= static_cast<std::uint64_t>(static_cast<std::uint8_t>(s[pos + i])) << (8 * i);
    pos += sizeof(T);
    return static_cast<T>(v);
  }
  template <typename T>
  std::vector<T> Array(std::size_t expect) {
    const std::uint64_t n = Scalar<std::uint64_t>();
    if (n != expect) throw DecodeError("segment batch array length mismatch");
    Need(n * sizeof(T));
    std::vector<T> v(n);
    if (n) std::memcpy(v.data(), s.data() + pos, n * sizeof(T));
    pos += n * sizeof(T);
    return v;
  }
};

std::uint64_t Fnv1a(std::span<const std::uint8_t> b) {
  std::uint64_t h = 1469598103934665603ull;
  for (std::uint8_t c : b) h = (h ^ c) * 1099511628211ull;
  return h | 1u;  // never 0 (0 = "no stamp yet")
}

std::string Slice(const std::vector<std::uint8_t>& bytes, std::uint32_t index) {
  const std::size_t lo = std::size_t(index) * kChunkBytes;
  const std::size_t hi = std::min(bytes.size(), lo + kChunkBytes);
  return std::string(reinterpret_cast<const char*>(bytes.data()) + lo, hi - lo);
}

std::uint32_t ChunkCount(std::size_t bytes) {
  return static_cast<std::uint32_t>((bytes + kChunkBytes - 1) / kChunkBytes);
}

}  // namespace

std::string EncodeSegmentBatch(const SegmentBatch& b) {
  std::string s;
  PutScalar<std::uint32_t>(s, static_cast<std::uint32_t>(b.model_key.size()));
  s += b.model_key;
  PutScalar(s, b.n_segments);
  PutScalar(s, b.unroll_len);
  PutScalar(s, b.obs_dim);
  PutScalar(s, b.obs_format);
  PutArray(s, b.obs);
  PutArray(s, b.action);
  PutArray(s, b.reward);
  PutArray(s, b.behavior_logp);
  PutArray(s, b.value_est);
  PutArray(s, b.done);
  PutArray(s, b.bootstrap);
  PutArray(s, b.valid_steps);
  PutArray(s, b.segment_seq);
  return s;
}

SegmentBatch DecodeSegmentBatch(const std::string& bytes) {
  Cursor c{bytes};
  SegmentBatch b;
  const std::uint32_t klen = c.Scalar<std::uint32_t>();
  c.Need(klen);
  b.model_key = bytes.substr(c.pos, klen);
  c.pos += klen;
  b.n_segments = c.Scalar<std::uint32_t>();
  b.unroll_len = c.Scalar<std::uint32_t>();
  b.obs_dim = c.Scalar<std::uint32_t>();
  b.obs_format = c.Scalar<std::uint32_t>();
  if (b.obs_format != SegmentBatch::kObsF32 && b.obs_format != SegmentBatch::kObsBits)
    throw DecodeError("unknown segment batch observation format");
  const std::size_t F = std::size_t(b.n_segments) * b.unroll_len;
  const std::size_t ob = b.obs_format == SegmentBatch::kObsBits ? F * ((b.obs_dim + 7) / 8)
                                                                : F * b.obs_dim * sizeof(float);
  b.obs = c.Array<std::uint8_t>(ob);
  b.action = c.Array<std::int32_t>(F);
  b.reward = c.Array<float>(F);
  b.behavior_logp = c.Array<float>(F);
  b.value_est = c.Array<float>(F);
  b.done = c.Array<std::uint8_t>(F);
  b.bootstrap = c.Array<float>(b.n_segments);
  b.valid_steps = c.Array<std::int32_t>(b.n_segments);
  b.segment_seq = c.Array<std::uint64_t>(b.n_segments);
  if (c.pos != bytes.size()) throw DecodeError("trailing bytes after segment batch");
  for (std::int32_t v : b.valid_steps)
    if (v < 0 || std::uint32_t(v) > b.unroll_len)
      throw DecodeError("segment batch valid_steps out of range");
  return b;
}

// ---------------------------------------------------------------------------
// Chunked parameter records
bool NeedsChunks(const ModelRecord& record) {
  // values dominate the encoding; 1 MiB covers keys, shape and hyperparameters
  return record.params.values.size() * sizeof(double) + (1u << 20) > kMaxFrameBytes;
}

bool IsTooLarge(const Message& reply) {
  const auto* err = std::get_if<ErrorBody>(&reply.payload);
  return err != nullptr && err->code == kErrTooLarge;
}

void PutChunked(net::RpcClient& rpc, const ModelRecord& record) {
  const std::vector<std::uint8_t> bytes = EncodeModelRecord(record);
  std::random_device rd;
  const std::uint64_t stamp = ((std::uint64_t(rd()) << 32) ^ rd()) | 1u;
  const std::uint32_t count = ChunkCount(bytes.size());
  for (std::uint32_t i = 0; i < count; ++i)
    net::Expect<AckBody>(rpc.Call(ParamChunkBody{record.model_key, stamp, i, count, Slice(bytes, i)}));
}

ModelRecord GetChunked(net::RpcClient& rpc, const std::string& key) {
  for (int attempt = 0; attempt < 3; ++attempt) {
    const auto first = net::Expect<ParamChunkBody>(rpc.Call(ParamChunkBody{key, 0, 0, 0, {}}));
    std::vector<std::uint8_t> bytes(first.bytes.begin(), first.bytes.end());
    bool changed = false;
    for (std::uint32_t i = 1; i < first.count && !changed; ++i) {
      const Message reply = rpc.Call(ParamChunkBody{key, first.stamp, i, 0, {}});
      if (const auto* err = std::get_if<ErrorBody>(&reply.payload);
          err != nullptr && err->code == kErrProtocol) {
        changed = true;  // replaced mid-transfer: start over
        break;
      }
      const auto& c = net::Expect<ParamChunkBody>(reply);
      bytes.insert(bytes.end(), c.bytes.begin(), c.bytes.end());
    }
    if (!changed) return DecodeModelRecord(bytes);
  }
  throw std::runtime_error("model record kept changing during a chunked get: " + key);
}

Message HandleParamChunk(pool::ModelStore& store, const ParamChunkBody& chunk,
                         std::uint64_t corr,
                         const std::function<void(const ModelRecord&)>& forward) {
  if (chunk.count == 0 && chunk.bytes.empty()) {
    // get: slice `index` of the record's encoding (the last encoding is cached per store)
    struct Cached {
      std::shared_ptr<const ModelRecord> rec;
      std::vector<std::uint8_t> bytes;
      std::uint64_t stamp = 0;
    };
    static std::mutex mu;
    static std::map<const pool::ModelStore*, Cached> cache;
    auto rec = store.Get(chunk.key);
    std::lock_guard lock(mu);
    Cached& c = cache[&store];
    if (c.rec != rec) {
      c.rec = rec;
      c.bytes = EncodeModelRecord(*rec);
      c.stamp = Fnv1a(c.bytes);
    }
    if (chunk.stamp != 0 && chunk.stamp != c.stamp)
      return MakeError(corr, kErrProtocol, "record changed during a chunked get");
    const std::uint32_t count = ChunkCount(c.bytes.size());
    if (chunk.index >= count) return MakeError(corr, kErrBadRequest, "chunk index out of range");
    return MakeMessage(corr, ParamChunkBody{chunk.key, c.stamp, chunk.index, count,
                                            Slice(c.bytes, chunk.index)});
  }
  // put: chunks of one transfer arrive in order on one connection
  struct Partial {
    std::uint32_t next = 0, count = 0;
    std::vector<std::uint8_t> bytes;
  };
  static std::mutex mu;
  static std::map<std::tuple<const pool::ModelStore*, std::string, std::uint64_t>, Partial> open;
  ModelRecord record;
  {
    std::lock_guard lock(mu);
    auto key = std::make_tuple(&store, chunk.key, chunk.stamp);
    Partial& p = open[key];
    if (chunk.index != p.next || (p.count != 0 && p.count != chunk.count) || chunk.count == 0) {
      open.erase(key);
      return MakeError(corr, kErrProtocol, "out-of-order parameter chunk");
    }
    p.count = chunk.count;
    p.bytes.insert(p.bytes.end(), chunk.bytes.begin(), chunk.bytes.end());
    if (++p.next < p.count) return MakeAck(corr);
    std::vector<std::uint8_t> bytes = std::move(p.bytes);
    open.erase(key);
    record = DecodeModelRecord(bytes);
  }
  if (record.model_key != chunk.key) return MakeError(corr, kErrProtocol, "chunk key mismatch");
  store.Put(record);
  forward(record);
  return MakeAck(corr);
}

bool SaveChunked(const std::string& path, const ModelRecord& record) {
  if (!NeedsChunks(record)) return false;
  const std::vector<std::uint8_t> bytes = EncodeModelRecord(record);
  const std::uint32_t count = ChunkCount(bytes.size());
  std::ofstream out(path, std::ios::binary | std::ios::trunc);
  if (!out) throw std::runtime_error("cannot write model file: " + path);
  for (std::uint32_t i = 0; i < count; ++i) {
    const auto frame = Encode(MakeMessage(0, ParamChunkBody{record.model_key, Fnv1a(bytes), i,
                                                            count, Slice(bytes, i)}));
    out.write(reinterpret_cast<const char*>(frame.data()), std::streamsize(frame.size()));
  }
  if (!out) throw std::runtime_error("short write to model file: " + path);
  return true;
}

std::optional<ModelRecord> LoadChunked(std::span<const std::uint8_t> file) {
  if (file.size() < 4) return std::nullopt;
  std::uint32_t len0 = 0;
  for (int i = 0; i < 4; ++i) len0 |= std::uint32_t(file[i]) << (8 * i);
  if (std::size_t(len0) + 4 >= file.size()) return std::nullopt;  // one frame: not chunked
  FrameSplitter fs;
  fs.Feed(file);
  std::vector<std::uint8_t> frame, bytes;
  std::uint32_t expect = 0, count = 0;
  while (fs.Next(frame)) {
    const Message m = Decode(frame);
    const auto* c = std::get_if<ParamChunkBody>(&m.payload);
    if (c == nullptr || c->index != expect || (count != 0 && c->count != count))
      throw std::runtime_error("not a chunked model file");
    count = c->count;
    bytes.insert(bytes.end(), c->bytes.begin(), c->bytes.end());
    ++expect;
  }
  if (expect == 0 || expect != count || fs.buffered() != 0)
    throw std::runtime_error("truncated chunked model file");
  return DecodeModelRecord(bytes);
}

}  // namespace proto::ext
}  // namespace tleague
