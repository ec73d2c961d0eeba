/*
 * oracle/hashmodel.c — TEST INFRASTRUCTURE ONLY: CPU restatement of the
 * reference's deterministic toy model (the checker for the device kernels,
 * never the product path).  Pinned against the compiled reference
 * (oracle/_ref) and the golden fixtures in tests/golden/.
 *
 * Restates /root/reference/proj/core/include/splitserve/hash_model.h:11-20
 * (the contract) and /root/reference/proj/core/src/hash_model.cc:
 *   FnvByte/FnvU32/FnvU64      hash_model.h:54-65
 *   Mix64                      hash_model.h:68-75
 *   domain tags                hash_model.cc:13-19
 *   seed state                 hash_model.cc:22-25
 *   InitialPrefixDigest        hash_model.cc:27
 *   ExtendPrefixDigest         hash_model.cc:29-31
 *   KvEntryWords               hash_model.cc:39-46
 *   EntryDigest                hash_model.cc:57-61
 *   Embed                      hash_model.cc:63-68
 *   Query                      hash_model.cc:70
 *   AttentionOut               hash_model.cc:72-74
 *   NextHidden                 hash_model.cc:76-81
 *   SampleToken                hash_model.cc:83-86
 *   Generate                   hash_model.cc:130-166
 * Batch helpers (ho_*_batch) loop the same functions for numpy callers.
 */
#include <stddef.h>
#include <stdint.h>
#include <stdlib.h>

#define FNV_BASIS 0xcbf29ce484222325ULL
#define FNV_PRIME 0x100000001b3ULL
#define TAG_PREFIX 0x7072656669783031ULL
#define TAG_KV 0x6b76656e74727930ULL
#define TAG_FOLD 0x666f6c6430303030ULL
#define TAG_EMBED 0x656d626564303030ULL
#define TAG_QUERY 0x7175657279303030ULL
#define TAG_HIDDEN 0x68696464656e3030ULL
#define TAG_SAMPLE 0x73616d706c653030ULL

static inline uint64_t fnv_byte(uint64_t h, uint8_t b) { return (h ^ b) * FNV_PRIME; }
static inline uint64_t fnv_u32(uint64_t h, uint32_t w) {
  for (int i = 0; i < 4; ++i) h = fnv_byte(h, (uint8_t)(w >> (8 * i)));
  return h;
}
static inline uint64_t fnv_u64(uint64_t h, uint64_t w) {
  for (int i = 0; i < 8; ++i) h = fnv_byte(h, (uint8_t)(w >> (8 * i)));
  return h;
}

uint64_t ho_mix64(uint64_t z) {
  z ^= z >> 30;
  z *= 0xbf58476d1ce4e5b9ULL;
  z ^= z >> 27;
  z *= 0x94d049bb133111ebULL;
  z ^= z >> 31;
  return z;
}

uint64_t ho_fnv_u64(uint64_t h, uint64_t w) { return fnv_u64(h, w); }
uint64_t ho_fnv_u32(uint64_t h, uint32_t w) { return fnv_u32(h, w); }

/* seed_state_ = FnvU64(kFnvBasis, hash_seed)  (hash_model.cc:24) */
uint64_t ho_seed_state(uint64_t hash_seed) { return fnv_u64(FNV_BASIS, hash_seed); }

uint64_t ho_initial_prefix_digest(uint64_t hash_seed) {
  return fnv_u64(ho_seed_state(hash_seed), TAG_PREFIX);
}

uint64_t ho_extend_prefix_digest(uint64_t digest, int32_t token) {
  return fnv_u32(digest, (uint32_t)token);
}

/* out[i] = P(i) for i in [0, n): the digest after token i. */
void ho_prefix_digests(uint64_t hash_seed, const int32_t* tokens, int64_t n, uint64_t* out) {
  uint64_t d = ho_initial_prefix_digest(hash_seed);
  for (int64_t i = 0; i < n; ++i) {
    d = fnv_u32(d, (uint32_t)tokens[i]);
    out[i] = d;
  }
}

void ho_kv_entry_words(uint64_t prefix_digest, int32_t layer, int32_t dim, uint64_t* out) {
  uint64_t base = fnv_u64(fnv_u64(prefix_digest, TAG_KV), (uint64_t)layer);
  for (int32_t j = 0; j < dim; ++j) out[j] = ho_mix64(fnv_u64(base, (uint64_t)j));
}

uint64_t ho_entry_digest(const uint64_t* words, int32_t dim) {
  uint64_t h = fnv_u64(FNV_BASIS, TAG_FOLD);
  for (int32_t j = 0; j < dim; ++j) h = fnv_u64(h, words[j]);
  return ho_mix64(h);
}

uint64_t ho_embed(uint64_t hash_seed, int32_t token, int64_t pos) {
  uint64_t h = fnv_u64(ho_seed_state(hash_seed), TAG_EMBED);
  h = fnv_u32(h, (uint32_t)token);
  h = fnv_u64(h, (uint64_t)pos);
  return ho_mix64(h);
}

uint64_t ho_query(uint64_t hidden) { return ho_mix64(hidden ^ TAG_QUERY); }

uint64_t ho_attention_out(uint64_t hidden, int64_t count, uint64_t fold_sum) {
  return (uint64_t)count * ho_query(hidden) + fold_sum;
}

uint64_t ho_next_hidden(uint64_t hidden, uint64_t attn_out) {
  uint64_t h = fnv_u64(FNV_BASIS, TAG_HIDDEN);
  h = fnv_u64(h, hidden);
  h = fnv_u64(h, attn_out);
  return ho_mix64(h);
}

int32_t ho_sample_token(uint64_t last_hidden, int32_t vocab) {
  return (int32_t)(ho_mix64(last_hidden ^ TAG_SAMPLE) % (uint64_t)vocab);
}

/* KV words for n consecutive positions (digests[n]) at one layer: out[n][dim]. */
void ho_kv_words_batch(const uint64_t* digests, int64_t n, int32_t layer, int32_t dim,
                       uint64_t* out) {
  for (int64_t i = 0; i < n; ++i) ho_kv_entry_words(digests[i], layer, dim, out + i * dim);
}

/* Entry digests of n entries words[n][dim]: out[n]. */
void ho_entry_digest_batch(const uint64_t* words, int64_t n, int32_t dim, uint64_t* out) {
  for (int64_t i = 0; i < n; ++i) out[i] = ho_entry_digest(words + i * dim, dim);
}

/* Generate (hash_model.cc:130-166): whole-prompt greedy generation. */
int ho_generate(uint64_t hash_seed, int32_t layers, int32_t dim, int32_t vocab,
                const int32_t* prompt, int64_t n, int32_t max_tokens, int32_t* out) {
  if (n <= 0 || max_tokens < 1) return -1;
  int64_t cap = n + max_tokens;
  int32_t* toks = (int32_t*)malloc(sizeof(int32_t) * cap);
  uint64_t* fold = (uint64_t*)calloc(layers, sizeof(uint64_t));
  uint64_t* words = (uint64_t*)malloc(sizeof(uint64_t) * dim);
  for (int64_t i = 0; i < n; ++i) toks[i] = prompt[i];
  int64_t len = n, processed = 0;
  int32_t produced = 0;
  uint64_t digest = ho_initial_prefix_digest(hash_seed), last_hidden = 0;
  for (;;) {
    for (; processed < len; ++processed) {
      digest = fnv_u32(digest, (uint32_t)toks[processed]);
      for (int32_t l = 0; l < layers; ++l) {
        ho_kv_entry_words(digest, l, dim, words);
        fold[l] += ho_entry_digest(words, dim);
      }
      uint64_t x = ho_embed(hash_seed, toks[processed], processed);
      for (int32_t l = 0; l < layers; ++l) {
        x = ho_next_hidden(x, ho_attention_out(x, processed + 1, fold[l]));
      }
      last_hidden = x;
    }
    int32_t next = ho_sample_token(last_hidden, vocab);
    out[produced++] = next;
    if (produced >= max_tokens) break;
    toks[len++] = next;
  }
  free(toks);
  free(fold);
  free(words);
  return 0;
}
