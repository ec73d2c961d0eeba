// hash.cuh — the toy model's hash contract as __host__ __device__ functions.
//
// Contract: /root/reference/proj/core/include/splitserve/hash_model.h:11-20.
// The KV words the cache stores and the entry digests attention folds are
// pure functions of the token prefix (FNV-1a over little-endian bytes, then a
// splitmix-style finaliser); device kernels and host bookkeeping both use
// these definitions so the pool is bit-identical to the reference's.
#pragma once

#include <cstdint>

#if defined(__CUDACC__)
#define MKV_HD __host__ __device__ __forceinline__
#else
#define MKV_HD inline
#endif

namespace mkv {

constexpr uint64_t kFnvBasis = 0xcbf29ce484222325ULL;
constexpr uint64_t kFnvPrime = 0x100000001b3ULL;
// Domain tags (hash_model.cc:13-19).
constexpr uint64_t kTagPrefix = 0x7072656669783031ULL;
constexpr uint64_t kTagKV = 0x6b76656e74727930ULL;
constexpr uint64_t kTagFold = 0x666f6c6430303030ULL;
constexpr uint64_t kTagEmbed = 0x656d626564303030ULL;
constexpr uint64_t kTagQuery = 0x7175657279303030ULL;
constexpr uint64_t kTagHidden = 0x68696464656e3030ULL;
constexpr uint64_t kTagSample = 0x73616d706c653030ULL;

// One FNV-1a byte step.  The prime is 2^40 + 0x1b3, so the product splits
// into a shift and a 9-bit multiply; the compiler does this for us.
MKV_HD uint64_t fnv_step(uint64_t h, uint32_t b) { return (h ^ b) * kFnvPrime; }

MKV_HD uint64_t fnv_u32(uint64_t h, uint32_t w) {
  h = fnv_step(h, w & 0xffu);
  h = fnv_step(h, (w >> 8) & 0xffu);
  h = fnv_step(h, (w >> 16) & 0xffu);
  h = fnv_step(h, w >> 24);
  return h;
}

MKV_HD uint64_t fnv_u64(uint64_t h, uint64_t w) {
  h = fnv_u32(h, static_cast<uint32_t>(w));
  return fnv_u32(h, static_cast<uint32_t>(w >> 32));
}

// Finaliser (hash_model.h:68-75).
MKV_HD uint64_t mix64(uint64_t z) {
  z ^= z >> 30;
  z *= 0xbf58476d1ce4e5b9ULL;
  z ^= z >> 27;
  z *= 0x94d049bb133111ebULL;
  z ^= z >> 31;
  return z;
}

// FNV over the u64 of a small index j < 2^16: bytes 2..7 are zero, and a
// zero byte is a plain multiply, so six steps fold into one multiply by
// prime^6 (mod 2^64).
constexpr uint64_t kFnvPrime6 = []() constexpr {
  uint64_t p = 1;
  for (int i = 0; i < 6; ++i) p *= kFnvPrime;
  return p;
}();

MKV_HD uint64_t fnv_small_index(uint64_t h, uint32_t j) {
  h = fnv_step(h, j & 0xffu);
  h = fnv_step(h, (j >> 8) & 0xffu);
  return h * kFnvPrime6;
}

// Per-(position, layer) base of KvEntryWords (hash_model.cc:42).
MKV_HD uint64_t kv_base(uint64_t prefix_digest, int32_t layer) {
  return fnv_u64(fnv_u64(prefix_digest, kTagKV), static_cast<uint64_t>(static_cast<int64_t>(layer)));
}

// Word j of KvEntryWords (hash_model.cc:43-45).
MKV_HD uint64_t kv_word(uint64_t base, uint32_t j) {
  return mix64(j < 65536u ? fnv_small_index(base, j) : fnv_u64(base, j));
}

MKV_HD uint64_t seed_state(uint64_t hash_seed) { return fnv_u64(kFnvBasis, hash_seed); }

MKV_HD uint64_t entry_digest_init() { return fnv_u64(kFnvBasis, kTagFold); }

MKV_HD uint64_t query(uint64_t hidden) { return mix64(hidden ^ kTagQuery); }

// AttentionOut (hash_model.cc:72-74), wrapping u64.
MKV_HD uint64_t attention_out(uint64_t hidden, int64_t count, uint64_t fold_sum) {
  return static_cast<uint64_t>(count) * query(hidden) + fold_sum;
}

// NextHidden (hash_model.cc:76-81).
MKV_HD uint64_t next_hidden(uint64_t hidden, uint64_t attn_out) {
  uint64_t h = fnv_u64(kFnvBasis, kTagHidden);
  h = fnv_u64(h, hidden);
  h = fnv_u64(h, attn_out);
  return mix64(h);
}

MKV_HD uint64_t embed(uint64_t seed_st, int32_t token, int64_t pos) {
  uint64_t h = fnv_u64(seed_st, kTagEmbed);
  h = fnv_u32(h, static_cast<uint32_t>(token));
  h = fnv_u64(h, static_cast<uint64_t>(pos));
  return mix64(h);
}

MKV_HD int32_t sample_token(uint64_t last_hidden, int32_t vocab) {
  return static_cast<int32_t>(mix64(last_hidden ^ kTagSample) % static_cast<uint64_t>(vocab));
}

}  // namespace mkv
