#!/usr/bin/env python3
"""Appends two message kinds at the reference's wire seam (proj/docs/extending.md "Wire
compatibility": new kinds take the next tags, existing encodings and golden frames stay
byte-identical), the way a maintainer would edit the reference tree:

  17 SegmentBatchPush   bulk columnar segment ingest:
                        message.hpp/codec.cpp body, SegmentSink::PushSegmentBatch (default:
                        one PushSegment per segment), LearnerService / LearnerClient
  18 ParamChunk         parameter records larger than a 64 MiB frame:
                        chunked put / get in ModelPoolService / ModelPoolClient, chunked
                        model files (model_io.cpp), and ModelStore's blob cap lifted from
                        half a frame (model_store.cpp:16-17) to kMaxBlobBytes

The logic lives in integration/wire_ext.cpp (tleague::proto::ext); the edits below only
hook it in.  Like mlp_family.py, the patched copies are build outputs under
oracle/_ref/dropin/patched/ and every edit is anchored on an exact reference line.

    python integration/patches/wire_ext.py <reference proj dir> <out dir>
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from mlp_family import patch  # noqa: E402

EXT = '#include "tleague/proto/wire_ext.hpp"\n'


def main(ref, out, base=None):
    """base: an already patched copy of a file (mlp_family.py output) to edit further."""
    def src(rel):
        b = f"{out}/{rel}"
        return b if os.path.exists(b) and rel in (base or ()) else f"{ref}/{rel}"

    patch(src("include/tleague/proto/message.hpp"), f"{out}/include/tleague/proto/message.hpp", [
        ('#include "tleague/types.hpp"\n',
         '#include "tleague/learner/segment_batch.hpp"\n#include "tleague/types.hpp"\n'),
        ("inline constexpr std::size_t kMaxFrameBytes = 64ull * 1024 * 1024;\n",
         "inline constexpr std::size_t kMaxFrameBytes = 64ull * 1024 * 1024;\n"
         "// pool records (larger than a frame: ParamChunk on the wire and in model files)\n"
         "inline constexpr std::size_t kMaxBlobBytes = 4ull << 30;\n"),
        ("  kError = 16,\n};",
         "  kError = 16,\n  kSegmentBatchPush = 17,\n  kParamChunk = 18,\n};"),
        ("// Error codes carried in ErrorBody.",
         "// A columnar group of segments of one model key (bulk ingest).\n"
         "struct SegmentBatchPushBody {\n"
         "  SegmentBatch batch;\n"
         "  bool operator==(const SegmentBatchPushBody&) const = default;\n"
         "};\n\n"
         "// A slice of an encoded ModelRecord (see tleague/proto/wire_ext.hpp).\n"
         "struct ParamChunkBody {\n"
         "  std::string key;\n"
         "  std::uint64_t stamp = 0;\n"
         "  std::uint32_t index = 0, count = 0;\n"
         "  std::string bytes;\n"
         "  bool operator==(const ParamChunkBody&) const = default;\n"
         "};\n\n"
         "// Error codes carried in ErrorBody."),
        ("  kErrNoModelLoaded = 7,\n",
         "  kErrNoModelLoaded = 7,\n  kErrTooLarge = 8,  // record exceeds one frame: use ParamChunk\n"),
        ("    AckBody, ErrorBody>;",
         "    AckBody, ErrorBody, SegmentBatchPushBody, ParamChunkBody>;"),
    ])
    patch(f"{ref}/include/tleague/proto/codec.hpp", f"{out}/include/tleague/proto/codec.hpp", [
        ("Message Decode(std::span<const std::uint8_t> frame);\n",
         "Message Decode(std::span<const std::uint8_t> frame);\n\n"
         "// The ModelRecord encoding of ParamPut / ParamReply bodies without a frame around it\n"
         "// (chunked transfers of records larger than a frame, ParamChunk).\n"
         "std::vector<std::uint8_t> EncodeModelRecord(const ModelRecord& record);\n"
         "ModelRecord DecodeModelRecord(std::span<const std::uint8_t> bytes);\n"),
    ])
    patch(src("src/proto/codec.cpp"), f"{out}/src/proto/codec.cpp", [
        ('#include "tleague/proto/codec.hpp"\n', '#include "tleague/proto/codec.hpp"\n' + EXT),
        ("  void operator()(const ErrorBody& b) {\n    w.U32(b.code);\n    w.Str(b.message);\n  }\n",
         "  void operator()(const ErrorBody& b) {\n    w.U32(b.code);\n    w.Str(b.message);\n  }\n"
         "  void operator()(const SegmentBatchPushBody& b) { w.Str(ext::EncodeSegmentBatch(b.batch)); }\n"
         "  void operator()(const ParamChunkBody& b) {\n"
         "    w.Str(b.key);\n    w.U64(b.stamp);\n    w.U32(b.index);\n    w.U32(b.count);\n"
         "    w.Str(b.bytes);\n  }\n"),
        ("    case MsgKind::kAck:\n      return AckBody{r.Str()};",
         "    case MsgKind::kSegmentBatchPush:\n"
         "      return SegmentBatchPushBody{ext::DecodeSegmentBatch(r.Str())};\n"
         "    case MsgKind::kParamChunk: {\n"
         "      ParamChunkBody b;\n      b.key = r.Str();\n      b.stamp = r.U64();\n"
         "      b.index = r.U32();\n      b.count = r.U32();\n      b.bytes = r.Str();\n"
         "      return b;\n    }\n"
         "    case MsgKind::kAck:\n      return AckBody{r.Str()};"),
        ('    case MsgKind::kError: return "Error";\n',
         '    case MsgKind::kError: return "Error";\n'
         '    case MsgKind::kSegmentBatchPush: return "SegmentBatchPush";\n'
         '    case MsgKind::kParamChunk: return "ParamChunk";\n'),
        ("  if (kind < 1 || kind > 16) throw DecodeError(\"unknown message kind\");",
         "  if (kind < 1 || kind > 18) throw DecodeError(\"unknown message kind\");"),
        ("void FrameSplitter::Feed(",
         "std::vector<std::uint8_t> EncodeModelRecord(const ModelRecord& record) {\n"
         "  ByteWriter w;\n  WriteModelRecord(w, record);\n  return w.Take();\n}\n\n"
         "ModelRecord DecodeModelRecord(std::span<const std::uint8_t> bytes) {\n"
         "  ByteReader r(bytes);\n  ModelRecord m = ReadModelRecord(r);\n"
         "  if (r.remaining() != 0) throw DecodeError(\"trailing bytes after model record\");\n"
         "  return m;\n}\n\n"
         "void FrameSplitter::Feed("),
    ])
    patch(f"{ref}/include/tleague/learner/segment_sink.hpp",
          f"{out}/include/tleague/learner/segment_sink.hpp", [
        ('#include "tleague/types.hpp"\n',
         '#include "tleague/learner/segment_batch.hpp"\n#include "tleague/types.hpp"\n'),
        ("  virtual void PushSegment(const TrajectorySegment& segment) = 0;\n",
         "  virtual void PushSegment(const TrajectorySegment& segment) = 0;\n"
         "  // A group of segments of one model key (bulk ingest, message kind 17).  Default:\n"
         "  // one PushSegment per segment, in order.\n"
         "  virtual void PushSegmentBatch(const SegmentBatch& batch) {\n"
         "    for (const TrajectorySegment& s : UnpackSegmentBatch(batch)) PushSegment(s);\n"
         "  }\n"),
    ])
    patch(f"{ref}/include/tleague/learner/learner_service.hpp",
          f"{out}/include/tleague/learner/learner_service.hpp", [
        ("  void PushSegment(const TrajectorySegment& segment) override;\n",
         "  void PushSegment(const TrajectorySegment& segment) override;\n"
         "  void PushSegmentBatch(const SegmentBatch& batch) override;\n"),
    ])
    patch(f"{ref}/src/learner/learner_service.cpp", f"{out}/src/learner/learner_service.cpp", [
        ("  return proto::MakeError(req.correlation_id, proto::kErrBadRequest,",
         "  if (const auto* bulk = std::get_if<proto::SegmentBatchPushBody>(&req.payload)) {\n"
         "    sink_.PushSegmentBatch(bulk->batch);\n"
         "    return proto::MakeAck(req.correlation_id);\n"
         "  }\n"
         "  return proto::MakeError(req.correlation_id, proto::kErrBadRequest,"),
        ("}  // namespace tleague::learner",
         "void LearnerClient::PushSegmentBatch(const SegmentBatch& batch) {\n"
         "  net::Expect<proto::AckBody>(rpc_.Call(proto::SegmentBatchPushBody{batch}));\n"
         "}\n\n"
         "}  // namespace tleague::learner"),
    ])
    patch(f"{ref}/src/pool/model_pool_service.cpp", f"{out}/src/pool/model_pool_service.cpp", [
        ('#include "tleague/pool/model_pool_service.hpp"\n',
         '#include "tleague/pool/model_pool_service.hpp"\n' + EXT),
        ("      auto rec = store_.Get(get->model_key);\n",
         "      auto rec = store_.Get(get->model_key);\n"
         "      if (proto::ext::NeedsChunks(*rec))\n"
         "        return proto::MakeError(corr, proto::kErrTooLarge,\n"
         "                                \"record exceeds one frame: fetch it in ParamChunk slices\");\n"),
        ("    return proto::MakeError(corr, proto::kErrBadRequest,",
         "    if (const auto* chunk = std::get_if<proto::ParamChunkBody>(&req.payload)) {\n"
         "      return proto::ext::HandleParamChunk(store_, *chunk, corr, [this](const ModelRecord& r) {\n"
         "        for (auto& sec : secondaries_) proto::ext::PutChunked(*sec, r);\n"
         "      });\n"
         "    }\n"
         "    return proto::MakeError(corr, proto::kErrBadRequest,"),
        ("  net::Expect<proto::AckBody>(Primary().Call(proto::ParamPutBody{record}));\n",
         "  if (proto::ext::NeedsChunks(record)) return proto::ext::PutChunked(Primary(), record);\n"
         "  net::Expect<proto::AckBody>(Primary().Call(proto::ParamPutBody{record}));\n"),
        ("  auto reply = AnyReplica().Call(proto::ParamGetBody{model_key});\n",
         "  net::RpcClient& rpc = AnyReplica();\n"
         "  auto reply = rpc.Call(proto::ParamGetBody{model_key});\n"
         "  if (proto::ext::IsTooLarge(reply)) return proto::ext::GetChunked(rpc, model_key);\n"),
    ])
    patch(f"{ref}/src/pool/model_store.cpp", f"{out}/src/pool/model_store.cpp", [
        ("  if (record.params.values.size() * sizeof(double) > proto::kMaxFrameBytes / 2)",
         "  if (record.params.values.size() * sizeof(double) > proto::kMaxBlobBytes)"),
    ])
    patch(f"{ref}/src/run/model_io.cpp", f"{out}/src/run/model_io.cpp", [
        ('#include "tleague/proto/codec.hpp"\n', '#include "tleague/proto/codec.hpp"\n' + EXT),
        ("void SaveModel(const std::string& path, const ModelRecord& record) {\n",
         "void SaveModel(const std::string& path, const ModelRecord& record) {\n"
         "  if (proto::ext::SaveChunked(path, record)) return;  // larger than one frame\n"),
        ("  proto::Message msg = proto::Decode(bytes);\n",
         "  if (auto chunked = proto::ext::LoadChunked(bytes)) return *chunked;\n"
         "  proto::Message msg = proto::Decode(bytes);\n"),
    ])


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], base={"src/proto/codec.cpp"})
