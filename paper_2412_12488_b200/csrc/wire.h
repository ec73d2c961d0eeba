// wire.h — the reference's wire formats, byte for byte: KVAddrInfo binary
// and JSON encodings (kv_addr.cc:53-118) and the KV transfer frames
// (transport.h:6-12, transport.cc:30-107).  Header and ack bytes are
// encoded on the host (tens of bytes); payload bytes and their CRC-32 stay
// on the device (crc32.cu, cache.cc EncodeWriteFrame / ReceiveWriteFrame).
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "cache.h"

namespace mkv {

constexpr uint32_t kFrameMagic = 0x4B565452u;  // "KVTR" (transport.h:32)
constexpr uint16_t kWireVersion = 1;           // transport.h:33
enum FrameType : uint8_t { kFrameWrite = 0, kFrameAck = 1 };
enum AckStatus : uint8_t { kAckOk = 0, kAckChecksumMismatch = 1, kAckUnknownAddress = 2 };

// KVAddrInfo::EncodeTo / DecodeFrom (kv_addr.cc:90-118): 20 + 8 n bytes.
void EncodeAddr(const KVAddr& a, std::vector<uint8_t>* out);
KVAddr DecodeAddr(const uint8_t* data, size_t size, size_t* pos);
// KVAddrInfo::ToJson / FromJson (kv_addr.cc:53-70), nlohmann's compact dump
// (keys sorted).  Malformed JSON throws JsonError (the reference surfaces a
// non-splitserve exception there).
std::string AddrToJson(const KVAddr& a);
KVAddr AddrFromJson(const std::string& text);
struct JsonError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

// Write frame without payload and CRC: magic, version, type, seq_tag,
// layer, address, payload length (EncodeWriteFrame, transport.cc:46-62).
size_t WriteHeaderSize(size_t n_ranges);
std::vector<uint8_t> EncodeWriteHeader(uint64_t seq_tag, int32_t layer, const KVAddr& addr,
                                       uint64_t payload_bytes);
// EncodeAckFrame (transport.cc:64-74): 26 bytes.
constexpr size_t kAckFrameBytes = 26;
std::vector<uint8_t> EncodeAck(uint64_t seq_tag, int32_t layer, int64_t token_begin,
                               uint8_t status);

// DecodeFrame (transport.cc:76-107) minus the payload CRC, which the device
// computes: the payload stays where it is in `data`.
struct FrameView {
  uint8_t type = 0;
  uint64_t seq_tag = 0;
  int32_t layer = 0;
  KVAddr addr;                // write
  size_t payload_offset = 0;  // write
  size_t payload_bytes = 0;   // write
  uint32_t wire_crc = 0;      // write
  int64_t token_begin = 0;    // ack
  uint8_t ack_status = 0;     // ack
};
FrameView DecodeFrameHeader(const uint8_t* data, size_t size);

}  // namespace mkv
