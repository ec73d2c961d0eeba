// frames.cc — KV write frames over the B200 pool (the cross-node fallback
// of the reference's TCP fabric, transport.h:6-12).  Header and ack bytes
// come from wire.cc on the host; the payload is gathered from the pool and
// checksummed on the device, so the only host work per frame is the
// header and the one D2H copy a socket needs anyway.
#include <cstring>

#include "wire.h"

using mkv::KVAddr;

namespace {
size_t Align256(size_t x) { return (x + 255) & ~size_t(255); }
}  // namespace

void ss_cache::Crc32(const void* data_dev, int64_t n, uint32_t* crc_dev, cudaStream_t s) {
  RequireDevice("Crc32");
  MKV_CHECK(n >= 0, mkv::kInvalidArgument, "negative length");
  OrderLaunch(s);
  mkv::DevBlock ws = DevAlloc(mkv::crc32_workspace_bytes(n, num_sms_), s);
  mkv::launch_crc32(data_dev, n, crc_dev, ws.ptr, s, num_sms_);
  CountLaunches(1);
  DevFree(ws, s);
  if (s != stream_) NoteUser(s);
}

// EncodeWriteFrame(WriteFrame{tag, layer, dest, GatherRange(seq, [begin, end), layer)})
// (transport.cc:46-62, kv_cache.cc:373-387).  The destination address must
// name exactly the gathered positions (MarkSend's rule, kv_cache.cc:231-243).
int64_t ss_cache::EncodeWriteFrame(SeqId seq, int64_t begin, int64_t end, int32_t layer,
                                   uint64_t tag, const KVAddr& dest, uint8_t* frame, int64_t cap,
                                   bool frame_on_device, cudaStream_t s) {
  RequireDevice("EncodeWriteFrame");
  MKV_CHECK(begin >= 0 && begin <= end, mkv::kInvalidArgument, "bad frame range");
  MKV_CHECK(dest.token_count == end - begin, mkv::kAddrMismatch,
            "destination covers " + std::to_string(dest.token_count) + " tokens, range has " +
                std::to_string(end - begin));
  MKV_CHECK(dest.token_begin == begin, mkv::kAddrMismatch, "destination token_begin mismatch");
  dest.Validate();
  const uint64_t payload = static_cast<uint64_t>(end - begin) * W_ * 8;
  const std::vector<uint8_t> header = mkv::EncodeWriteHeader(tag, layer, dest, payload);
  const int64_t total = static_cast<int64_t>(header.size() + payload + 4);
  if (cap < total) {
    mkv::ThrowStatus(SS_ERR_BUFFER_TOO_SMALL,
                "BufferTooSmall: frame needs " + std::to_string(total) + " bytes");
  }
  const size_t hdr = header.size();
  if (frame_on_device) {
    MKV_CHECK(reinterpret_cast<uintptr_t>(frame + hdr) % 32 == 0, mkv::kInvalidArgument,
              "device frame: payload (frame + header bytes) must be 32-byte aligned");
    // Gather straight into the frame; header and CRC bytes around it.
    GatherRange(seq, begin, end, layer, reinterpret_cast<uint64_t*>(frame + hdr), s);
    OrderLaunch(s);
    mkv::DevBlock tmp = DevAlloc(256, s);
    H2D(frame, header.data(), hdr, s, "H2D frame header");
    mkv::DevBlock ws = DevAlloc(mkv::crc32_workspace_bytes(static_cast<int64_t>(payload), num_sms_), s);
    mkv::launch_crc32(frame + hdr, static_cast<int64_t>(payload), static_cast<uint32_t*>(tmp.ptr),
                      ws.ptr, s, num_sms_);
    CountLaunches(1);
    mkv::CudaCheck(cudaMemcpyAsync(frame + hdr + payload, tmp.ptr, 4, cudaMemcpyDeviceToDevice, s),
              "D2D frame crc");
    DevFree(ws, s);
    DevFree(tmp, s);
    if (s != stream_) NoteUser(s);
    return total;
  }
  // Host frame (what a socket writes): payload + CRC gathered on the device,
  // one D2H of payload||crc straight into the frame.
  cudaStream_t st = stream_;
  const size_t o_crc = Align256(payload);
  mkv::DevBlock stage = DevAlloc(o_crc + 256, st);
  auto* base = static_cast<uint8_t*>(stage.ptr);
  GatherRange(seq, begin, end, layer, reinterpret_cast<uint64_t*>(base), st);
  Crc32(base, static_cast<int64_t>(payload), reinterpret_cast<uint32_t*>(base + o_crc), st);
  std::memcpy(frame, header.data(), hdr);
  if (payload > 0) D2H(frame + hdr, base, payload, st, "D2H frame payload");
  D2H(frame + hdr + payload, base + o_crc, 4, st, "D2H frame crc");
  DevFree(stage, st);
  Sync();
  return total;
}

// One write frame arriving at the transfer agent (tcp_fabric.cc:144-168):
// decode, payload to the device, CRC on the device; a mismatch acks
// ChecksumMismatch without applying, else ApplyRemoteWrite with the frame's
// tag and the ack says UnknownAddress or Ok.
void ss_cache::ReceiveWriteFrame(const uint8_t* frame, int64_t size, uint8_t* ack_out,
                                 int32_t* apply_status) {
  RequireDevice("ReceiveWriteFrame");
  MKV_CHECK(size >= 0, mkv::kInvalidArgument, "negative frame size");
  const mkv::FrameView f = mkv::DecodeFrameHeader(frame, static_cast<size_t>(size));
  MKV_CHECK(f.type == mkv::kFrameWrite, mkv::kInvalidArgument, "not a write frame");
  // The transfer agent's stream (this may run on its own thread).
  cudaStream_t st = recv_stream_;
  const size_t o_crc = Align256(f.payload_bytes);
  mkv::DevBlock stage = DevAlloc(o_crc + 256, st);
  auto* base = static_cast<uint8_t*>(stage.ptr);
  if (f.payload_bytes > 0) H2D(base, frame + f.payload_offset, f.payload_bytes, st, "H2D frame payload");
  mkv::launch_crc32(base, static_cast<int64_t>(f.payload_bytes),
                    reinterpret_cast<uint32_t*>(base + o_crc), nullptr, st, num_sms_);
  CountLaunches(1);
  D2H(h_agent_pinned_, base + o_crc, 4, st, "D2H frame crc");
  mkv::CudaCheck(cudaStreamSynchronize(st), "cudaStreamSynchronize recv");
  const uint32_t crc = *h_agent_pinned_;
  uint8_t ack = mkv::kAckOk;
  int32_t status = -1;
  if (crc != f.wire_crc) {
    ack = mkv::kAckChecksumMismatch;
  } else {
    try {
      status = ApplyRemoteWrite(f.addr, f.layer, reinterpret_cast<const uint64_t*>(base),
                                static_cast<int64_t>(f.payload_bytes / 8), true, f.seq_tag,
                                nullptr, true);
    } catch (...) {
      DevFree(stage, st);
      throw;
    }
    ack = status == SS_APPLY_UNKNOWN_ADDRESS ? mkv::kAckUnknownAddress : mkv::kAckOk;
  }
  DevFree(stage, st);
  const std::vector<uint8_t> a = mkv::EncodeAck(f.seq_tag, f.layer, f.addr.token_begin, ack);
  std::memcpy(ack_out, a.data(), a.size());
  if (apply_status) *apply_status = status;
}
