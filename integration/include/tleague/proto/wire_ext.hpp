// Wire extensions appended at the reference's protocol seam (proj/docs/extending.md
// "Wire compatibility": new message kinds take the next tags; existing frames and golden
// files are unchanged).  Registered by integration/patches/wire_ext.py:
//
//   17 SegmentBatchPush  a columnar group of segments (tleague::SegmentBatch) for the
//                        learner's bulk ingest
//   18 ParamChunk        a slice of an encoded ModelRecord, for parameter blobs larger
//                        than a frame (C5's 12.7M fp64 parameters are 102 MB
//                        against the 64 MiB frame, message.hpp:13)
//
// ParamChunk: a put sends count chunks {key, stamp = transfer id, index, count, bytes};
// the pool reassembles and Puts the record once the last chunk arrived.  A get first
// tries ParamGet; a record too large for one reply frame answers kErrTooLarge, and the
// client then fetches chunk i with {key, stamp = 0, index = i, count = 0, bytes = ""}
// (the reply's stamp is a hash of the whole encoding, so a record replaced mid-transfer
// is detected and the transfer restarts).  Model files of such records are the put
// chunks' frames back to back.
#pragma once

#include <cstdint>
#include <functional>
#include <optional>
#include <span>
#include <string>
#include <vector>

#include "tleague/learner/segment_batch.hpp"
#include "tleague/types.hpp"

namespace tleague::net {
class RpcClient;
}
namespace tleague::pool {
class ModelStore;
}

namespace tleague::proto {
struct Message;
struct ParamChunkBody;
}  // namespace tleague::proto

namespace tleague::proto::ext {

inline constexpr std::size_t kChunkBytes = 32ull << 20;   // encoded bytes per chunk
inline constexpr std::uint32_t kErrTooLarge = 8;          // ErrorBody code (appended)

std::string EncodeSegmentBatch(const SegmentBatch& b);
SegmentBatch DecodeSegmentBatch(const std::string& bytes);

// true when the record's single-frame encoding would exceed the frame limit
bool NeedsChunks(const ModelRecord& record);
void PutChunked(net::RpcClient& rpc, const ModelRecord& record);
ModelRecord GetChunked(net::RpcClient& rpc, const std::string& key);
bool IsTooLarge(const Message& reply);

// ModelPoolService side: a put chunk (stores the record after the last one, then
// `forward` replicates it) or a get chunk request (replies with the slice).
Message HandleParamChunk(pool::ModelStore& store, const ParamChunkBody& chunk,
                         std::uint64_t correlation_id,
                         const std::function<void(const ModelRecord&)>& forward);

// model_io: oversized records as put-chunk frames; false / nullopt when not applicable
bool SaveChunked(const std::string& path, const ModelRecord& record);
std::optional<ModelRecord> LoadChunked(std::span<const std::uint8_t> file_bytes);

}  // namespace tleague::proto::ext
