// wire.cc — host codec of the reference's wire formats (see wire.h).
#include "wire.h"

#include <cctype>
#include <cmath>
#include <cstring>
#include <map>
#include <memory>

namespace mkv {

namespace {

template <typename T>
void PutLE(std::vector<uint8_t>* out, T v) {
  for (size_t i = 0; i < sizeof(T); ++i) {
    out->push_back(static_cast<uint8_t>(static_cast<uint64_t>(v) >> (8 * i)));
  }
}

template <typename T>
T GetLE(const uint8_t* data, size_t size, size_t* pos, const char* what) {
  MKV_CHECK(*pos + sizeof(T) <= size, kInvalidArgument, what);
  uint64_t v = 0;
  for (size_t i = 0; i < sizeof(T); ++i) v |= static_cast<uint64_t>(data[*pos + i]) << (8 * i);
  *pos += sizeof(T);
  return static_cast<T>(v);
}

// ---- a minimal JSON reader (RFC 8259 values), enough for FromJson -------
struct JVal {
  enum Kind { kNull, kBool, kInt, kUInt, kFloat, kString, kArray, kObject } kind = kNull;
  bool b = false;
  int64_t i = 0;
  uint64_t u = 0;
  double f = 0;
  std::string s;
  std::vector<JVal> arr;
  std::map<std::string, JVal> obj;

  bool is_number() const { return kind == kInt || kind == kUInt || kind == kFloat; }
  // nlohmann get<integer>(): numbers convert with static_cast; anything
  // else is a type error.
  template <typename T>
  T as() const {
    if (kind == kInt) return static_cast<T>(i);
    if (kind == kUInt) return static_cast<T>(u);
    if (kind == kFloat) return static_cast<T>(f);
    throw JsonError("type must be number");
  }
  const JVal& at(const std::string& key) const {
    if (kind != kObject) throw JsonError("cannot use at() with a non-object");
    auto it = obj.find(key);
    if (it == obj.end()) throw JsonError("key '" + key + "' not found");
    return it->second;
  }
  const JVal& at(size_t idx) const {
    if (kind != kArray) throw JsonError("cannot use at() with a non-array");
    if (idx >= arr.size()) throw JsonError("array index out of range");
    return arr[idx];
  }
};

class JReader {
 public:
  explicit JReader(const std::string& t) : t_(t) {}
  JVal Parse() {
    JVal v = Value(0);
    Ws();
    if (p_ != t_.size()) Fail("unexpected trailing input");
    return v;
  }

 private:
  [[noreturn]] void Fail(const char* why) {
    throw JsonError(std::string("parse error at byte ") + std::to_string(p_) + ": " + why);
  }
  void Ws() {
    while (p_ < t_.size() && (t_[p_] == ' ' || t_[p_] == '\t' || t_[p_] == '\n' || t_[p_] == '\r'))
      ++p_;
  }
  bool Lit(const char* w) {
    const size_t n = std::strlen(w);
    if (t_.compare(p_, n, w) == 0) {
      p_ += n;
      return true;
    }
    return false;
  }
  JVal Value(int depth) {
    if (depth > 512) Fail("nesting too deep");
    Ws();
    if (p_ >= t_.size()) Fail("unexpected end of input");
    JVal v;
    const char c = t_[p_];
    if (c == '{') {
      ++p_;
      v.kind = JVal::kObject;
      Ws();
      if (p_ < t_.size() && t_[p_] == '}') {
        ++p_;
        return v;
      }
      for (;;) {
        Ws();
        if (p_ >= t_.size() || t_[p_] != '"') Fail("expected object key");
        std::string key = String();
        Ws();
        if (p_ >= t_.size() || t_[p_] != ':') Fail("expected ':'");
        ++p_;
        v.obj[key] = Value(depth + 1);  // last duplicate wins, as in nlohmann
        Ws();
        if (p_ < t_.size() && t_[p_] == ',') {
          ++p_;
          continue;
        }
        if (p_ < t_.size() && t_[p_] == '}') {
          ++p_;
          return v;
        }
        Fail("expected ',' or '}'");
      }
    }
    if (c == '[') {
      ++p_;
      v.kind = JVal::kArray;
      Ws();
      if (p_ < t_.size() && t_[p_] == ']') {
        ++p_;
        return v;
      }
      for (;;) {
        v.arr.push_back(Value(depth + 1));
        Ws();
        if (p_ < t_.size() && t_[p_] == ',') {
          ++p_;
          continue;
        }
        if (p_ < t_.size() && t_[p_] == ']') {
          ++p_;
          return v;
        }
        Fail("expected ',' or ']'");
      }
    }
    if (c == '"') {
      v.kind = JVal::kString;
      v.s = String();
      return v;
    }
    if (Lit("true")) {
      v.kind = JVal::kBool;
      v.b = true;
      return v;
    }
    if (Lit("false")) {
      v.kind = JVal::kBool;
      return v;
    }
    if (Lit("null")) return v;
    return Number();
  }
  std::string String() {
    ++p_;  // opening quote
    std::string out;
    while (p_ < t_.size()) {
      const char c = t_[p_++];
      if (c == '"') return out;
      if (static_cast<unsigned char>(c) < 0x20) Fail("control character in string");
      if (c != '\\') {
        out.push_back(c);
        continue;
      }
      if (p_ >= t_.size()) break;
      const char e = t_[p_++];
      switch (e) {
        case '"': case '\\': case '/': out.push_back(e); break;
        case 'b': out.push_back('\b'); break;
        case 'f': out.push_back('\f'); break;
        case 'n': out.push_back('\n'); break;
        case 'r': out.push_back('\r'); break;
        case 't': out.push_back('\t'); break;
        case 'u': {
          if (p_ + 4 > t_.size()) Fail("bad \\u escape");
          for (int k = 0; k < 4; ++k)
            if (!std::isxdigit(static_cast<unsigned char>(t_[p_ + k]))) Fail("bad \\u escape");
          p_ += 4;  // keys we read are ASCII; the code point itself is not needed
          out.push_back('?');
          break;
        }
        default: Fail("bad escape");
      }
    }
    Fail("unterminated string");
  }
  JVal Number() {
    const size_t b = p_;
    if (p_ < t_.size() && t_[p_] == '-') ++p_;
    if (p_ >= t_.size() || !std::isdigit(static_cast<unsigned char>(t_[p_]))) Fail("syntax error");
    if (t_[p_] == '0') {
      ++p_;
    } else {
      while (p_ < t_.size() && std::isdigit(static_cast<unsigned char>(t_[p_]))) ++p_;
    }
    bool is_float = false;
    if (p_ < t_.size() && t_[p_] == '.') {
      is_float = true;
      ++p_;
      if (p_ >= t_.size() || !std::isdigit(static_cast<unsigned char>(t_[p_]))) Fail("bad fraction");
      while (p_ < t_.size() && std::isdigit(static_cast<unsigned char>(t_[p_]))) ++p_;
    }
    if (p_ < t_.size() && (t_[p_] == 'e' || t_[p_] == 'E')) {
      is_float = true;
      ++p_;
      if (p_ < t_.size() && (t_[p_] == '+' || t_[p_] == '-')) ++p_;
      if (p_ >= t_.size() || !std::isdigit(static_cast<unsigned char>(t_[p_]))) Fail("bad exponent");
      while (p_ < t_.size() && std::isdigit(static_cast<unsigned char>(t_[p_]))) ++p_;
    }
    const std::string lit = t_.substr(b, p_ - b);
    JVal v;
    if (!is_float) {
      errno = 0;
      if (lit[0] == '-') {
        const long long x = std::strtoll(lit.c_str(), nullptr, 10);
        if (errno == 0) {
          v.kind = JVal::kInt;
          v.i = x;
          return v;
        }
      } else {
        const unsigned long long x = std::strtoull(lit.c_str(), nullptr, 10);
        if (errno == 0) {
          v.kind = JVal::kUInt;
          v.u = x;
          return v;
        }
      }
    }
    v.kind = JVal::kFloat;  // out-of-range integers become floats, as in nlohmann
    v.f = std::strtod(lit.c_str(), nullptr);
    return v;
  }

  const std::string& t_;
  size_t p_ = 0;
};

}  // namespace

void EncodeAddr(const KVAddr& a, std::vector<uint8_t>* out) {
  PutLE<uint64_t>(out, static_cast<uint64_t>(a.token_begin));
  PutLE<uint64_t>(out, static_cast<uint64_t>(a.token_count));
  PutLE<uint32_t>(out, static_cast<uint32_t>(a.ranges.size()));
  for (const auto& r : a.ranges) {
    PutLE<uint32_t>(out, static_cast<uint32_t>(r.page_id));
    PutLE<uint16_t>(out, static_cast<uint16_t>(r.slot_begin));
    PutLE<uint16_t>(out, static_cast<uint16_t>(r.slot_count));
  }
}

KVAddr DecodeAddr(const uint8_t* data, size_t size, size_t* consumed) {
  static const char kWhat[] = "truncated address encoding";
  size_t pos = *consumed;
  KVAddr out;
  out.token_begin = static_cast<int64_t>(GetLE<uint64_t>(data, size, &pos, kWhat));
  out.token_count = static_cast<int64_t>(GetLE<uint64_t>(data, size, &pos, kWhat));
  const uint32_t n = GetLE<uint32_t>(data, size, &pos, kWhat);
  // Each range is 8 bytes: refuse counts the buffer cannot hold before
  // reserving (the reference reserves first; same result for valid input).
  MKV_CHECK(static_cast<uint64_t>(n) * 8 <= size - pos, kInvalidArgument, kWhat);
  out.ranges.reserve(n);
  for (uint32_t i = 0; i < n; ++i) {
    SlotRange r;
    r.page_id = GetLE<uint32_t>(data, size, &pos, kWhat);
    r.slot_begin = GetLE<uint16_t>(data, size, &pos, kWhat);
    r.slot_count = GetLE<uint16_t>(data, size, &pos, kWhat);
    out.ranges.push_back(r);
  }
  *consumed = pos;
  out.Validate();
  return out;
}

std::string AddrToJson(const KVAddr& a) {
  std::string s = "{\"ranges\":[";
  for (size_t i = 0; i < a.ranges.size(); ++i) {
    if (i) s += ',';
    s += '[' + std::to_string(a.ranges[i].page_id) + ',' + std::to_string(a.ranges[i].slot_begin) +
         ',' + std::to_string(a.ranges[i].slot_count) + ']';
  }
  s += "],\"token_begin\":" + std::to_string(a.token_begin) +
       ",\"token_count\":" + std::to_string(a.token_count) + '}';
  return s;
}

KVAddr AddrFromJson(const std::string& text) {
  const JVal j = JReader(text).Parse();
  KVAddr out;
  out.token_begin = j.at("token_begin").as<int64_t>();
  out.token_count = j.at("token_count").as<int64_t>();
  const JVal& rs = j.at("ranges");
  // nlohmann iterates an object's values and a primitive as itself.
  std::vector<const JVal*> items;
  if (rs.kind == JVal::kArray) {
    for (const auto& r : rs.arr) items.push_back(&r);
  } else if (rs.kind == JVal::kObject) {
    for (const auto& [k, r] : rs.obj) items.push_back(&r);
  } else if (rs.kind != JVal::kNull) {
    items.push_back(&rs);
  }
  for (const JVal* r : items) {
    out.ranges.push_back({r->at(0).as<int64_t>(), r->at(1).as<int32_t>(), r->at(2).as<int32_t>()});
  }
  out.Validate();
  return out;
}

size_t WriteHeaderSize(size_t n_ranges) { return 4 + 2 + 1 + 8 + 2 + 20 + 8 * n_ranges + 4; }

std::vector<uint8_t> EncodeWriteHeader(uint64_t seq_tag, int32_t layer, const KVAddr& addr,
                                       uint64_t payload_bytes) {
  MKV_CHECK(payload_bytes <= 0xFFFFFFFFull, kInvalidArgument,
            "payload exceeds the frame's u32 length field");
  std::vector<uint8_t> out;
  out.reserve(WriteHeaderSize(addr.ranges.size()));
  PutLE<uint32_t>(&out, kFrameMagic);
  PutLE<uint16_t>(&out, kWireVersion);
  PutLE<uint8_t>(&out, kFrameWrite);
  PutLE<uint64_t>(&out, seq_tag);
  PutLE<uint16_t>(&out, static_cast<uint16_t>(layer));
  EncodeAddr(addr, &out);
  PutLE<uint32_t>(&out, static_cast<uint32_t>(payload_bytes));
  return out;
}

std::vector<uint8_t> EncodeAck(uint64_t seq_tag, int32_t layer, int64_t token_begin,
                               uint8_t status) {
  std::vector<uint8_t> out;
  out.reserve(kAckFrameBytes);
  PutLE<uint32_t>(&out, kFrameMagic);
  PutLE<uint16_t>(&out, kWireVersion);
  PutLE<uint8_t>(&out, kFrameAck);
  PutLE<uint64_t>(&out, seq_tag);
  PutLE<uint16_t>(&out, static_cast<uint16_t>(layer));
  PutLE<uint64_t>(&out, static_cast<uint64_t>(token_begin));
  PutLE<uint8_t>(&out, status);
  return out;
}

FrameView DecodeFrameHeader(const uint8_t* data, size_t size) {
  static const char kWhat[] = "truncated frame";
  size_t pos = 0;
  const uint32_t magic = GetLE<uint32_t>(data, size, &pos, kWhat);
  MKV_CHECK(magic == kFrameMagic, kInvalidArgument, "bad frame magic");
  const uint16_t version = GetLE<uint16_t>(data, size, &pos, kWhat);
  MKV_CHECK(version == kWireVersion, kInvalidArgument, "bad wire version");
  FrameView f;
  f.type = GetLE<uint8_t>(data, size, &pos, kWhat);
  if (f.type == kFrameWrite) {
    f.seq_tag = GetLE<uint64_t>(data, size, &pos, kWhat);
    f.layer = GetLE<uint16_t>(data, size, &pos, kWhat);
    f.addr = DecodeAddr(data, size, &pos);
    const uint32_t payload_bytes = GetLE<uint32_t>(data, size, &pos, kWhat);
    MKV_CHECK(payload_bytes % 8 == 0 && pos + payload_bytes + 4 <= size, kInvalidArgument,
              "bad payload length");
    f.payload_offset = pos;
    f.payload_bytes = payload_bytes;
    pos += payload_bytes;
    f.wire_crc = GetLE<uint32_t>(data, size, &pos, kWhat);
  } else if (f.type == kFrameAck) {
    f.seq_tag = GetLE<uint64_t>(data, size, &pos, kWhat);
    f.layer = GetLE<uint16_t>(data, size, &pos, kWhat);
    f.token_begin = static_cast<int64_t>(GetLE<uint64_t>(data, size, &pos, kWhat));
    f.ack_status = GetLE<uint8_t>(data, size, &pos, kWhat);
  } else {
    Throw(kInvalidArgument, "unknown frame type");
  }
  return f;
}

}  // namespace mkv
