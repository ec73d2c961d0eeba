/*
 * oracle/ref_capi.cc — TEST INFRASTRUCTURE ONLY (the checker, never the product).
 *
 * Implements the host entry points of include/microkv.h on top of the
 * UNMODIFIED reference `splitserve::KVCache` / `splitserve::HashModel`,
 * compiled from /root/reference/proj/core/src by oracle/Makefile into
 * oracle/_ref/libmicrokv_ref.so.  Only tests/, __graft_entry__.smoke() and
 * bench.py's reference / cpu_baseline legs load it.
 *
 * Every function is a direct call of the reference member named in
 * microkv.h; this file adds only the POD <-> C++ conversions and the
 * exception -> status mapping.  Device entry points return
 * SS_ERR_UNSUPPORTED.
 *
 * `ssref_bench_migrate` is the reference arm of bench.py: the DirectSend KV
 * migration step (PrepRecv on D, GatherRange -> ApplyRemoteWrite per layer,
 * DrainReceiveCompletions, FreeSequence) run through the reference classes,
 * one engine pair per host thread (the reference's one-executor-per-engine
 * model, kv_cache.h:12-15).
 */
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <deque>
#include <set>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "microkv.h"
#include "splitserve/config.h"
#include "splitserve/errors.h"
#include "splitserve/hash_model.h"
#include "splitserve/kv_cache.h"
#include "splitserve/transport.h"

using namespace splitserve;

struct ss_plan;
struct ss_cache {
  ~ss_cache();
  std::set<ss_plan*> plans;  // released with the cache if still live
  std::unique_ptr<HashModel> model;
  std::unique_ptr<KVCache> cache;
  std::string err;
  int32_t rank = 0;
  ss_config cfg{};
  std::deque<int64_t> drained;  // completions not yet handed out
};

struct ss_plan {
  ForwardPlan plan;
  ss_cache* owner = nullptr;
};

ss_cache::~ss_cache() {
  for (ss_plan* p : plans) delete p;
}

namespace {

int Fail(ss_cache* c, int status, const std::string& msg) {
  if (c) c->err = msg;
  return status;
}

template <typename F>
int Guard(ss_cache* c, F&& f) {
  try {
    return f();
  } catch (const Error& e) {
    return Fail(c, 1 + static_cast<int>(e.code()), e.what());
  } catch (const std::exception& e) {
    return Fail(c, SS_ERR_INTERNAL, e.what());
  }
}

KVAddrInfo ToAddr(const ss_addr* a) {
  KVAddrInfo out;
  out.token_begin = a->token_begin;
  out.token_count = a->token_count;
  out.ranges.reserve(a->n_ranges);
  for (int64_t i = 0; i < a->n_ranges; ++i) {
    out.ranges.push_back({a->ranges[i].page_id, a->ranges[i].slot_begin, a->ranges[i].slot_count});
  }
  return out;
}

int FromAddr(ss_cache* c, const KVAddrInfo& a, ss_addr* out) {
  out->token_begin = a.token_begin;
  out->token_count = a.token_count;
  int64_t n = static_cast<int64_t>(a.ranges.size());
  if (n > out->ranges_cap) {
    out->n_ranges = n;
    return Fail(c, SS_ERR_BUFFER_TOO_SMALL, "address needs " + std::to_string(n) + " ranges");
  }
  for (int64_t i = 0; i < n; ++i) {
    out->ranges[i] = {a.ranges[i].page_id, a.ranges[i].slot_begin, a.ranges[i].slot_count};
  }
  out->n_ranges = n;
  return SS_OK;
}

TokenList ToTokens(const int32_t* t, int64_t n) { return TokenList(t, t + n); }

const char* kNames[] = {"OK",          "OutOfPages",      "DuplicateSequence", "UnknownSequence",
                        "ForkBeyondCommitted", "AddrMismatch", "MissingKV",   "LayerOrderViolation",
                        "CannotEvict", "ChecksumMismatch", "UnknownAddress",  "PeerUnreachable",
                        "NoEngines",   "RoleMissing",     "NoOwner",           "UnknownStrategy",
                        "InvalidArgument", "Aborted",     "Internal"};

}  // namespace

extern "C" {

int ss_abi_version(void) { return SS_ABI_VERSION; }
const char* ss_impl_name(void) { return "splitserve-reference"; }

int ss_cache_create(const ss_config* cfg, ss_cache** out) {
  auto c = std::make_unique<ss_cache>();
  int st = Guard(nullptr, [&]() -> int {
    ModelConfig m;
    m.layers = cfg->layers;
    m.dim = cfg->dim;
    m.vocab = cfg->vocab;
    m.hash_seed = cfg->hash_seed;
    CacheConfig cc;
    cc.num_pages = cfg->num_pages;
    cc.page_size = cfg->page_size;
    c->model = std::make_unique<HashModel>(m);
    c->cache = std::make_unique<KVCache>(cc, c->model.get());
    c->rank = cfg->rank;
    c->cfg = *cfg;
    c->cfg.num_pages = c->cache->cache_config().num_pages;
    c->cfg.page_size = c->cache->cache_config().page_size;
    c->cfg.device = -1;
    return SS_OK;
  });
  if (st != SS_OK) return st;
  *out = c.release();
  return SS_OK;
}

void ss_cache_destroy(ss_cache* c) { delete c; }
const char* ss_last_error(const ss_cache* c) { return c ? c->err.c_str() : ""; }
const char* ss_status_name(int s) {
  if (s >= 0 && s <= 18) return kNames[s];
  switch (s) {
    case SS_ERR_UNSUPPORTED: return "Unsupported";
    case SS_ERR_BUFFER_TOO_SMALL: return "BufferTooSmall";
    case SS_ERR_CUDA: return "Cuda";
    case SS_ERR_NO_DEVICE: return "NoDevice";
  }
  return "Unknown";
}
int ss_status_retryable(int s) {
  if (s >= 1 && s <= 18) return IsRetryable(static_cast<ErrorCode>(s - 1)) ? 1 : 0;
  return 0;
}

uint64_t ss_initial_prefix_digest(const ss_cache* c) { return c->model->InitialPrefixDigest(); }
uint64_t ss_embed(const ss_cache* c, int32_t t, int64_t pos) { return c->model->Embed(t, pos); }
int32_t ss_sample_token(const ss_cache* c, uint64_t h) { return c->model->SampleToken(h); }

int ss_match_prefix(ss_cache* c, const int32_t* tokens, int64_t n, int64_t* match_len,
                    int64_t* seq_out) {
  return Guard(c, [&]() -> int {
    auto r = c->cache->MatchPrefixSeq(std::span<const Token>(tokens, n));
    *match_len = r.match_len;
    if (seq_out) *seq_out = r.seq;
    return SS_OK;
  });
}

int ss_prep_recv(ss_cache* c, int64_t seq, const int32_t* tokens, int64_t n, int64_t end,
                 int64_t* match_len, ss_addr* addr_out) {
  return Guard(c, [&]() -> int {
    auto r = c->cache->PrepRecv(seq, ToTokens(tokens, n), end);
    *match_len = r.match_len;
    return FromAddr(c, r.addr, addr_out);
  });
}

int ss_create_sequence(ss_cache* c, int64_t seq, const int32_t* tokens, int64_t n) {
  return Guard(c, [&]() -> int {
    c->cache->CreateSequence(seq, ToTokens(tokens, n));
    return SS_OK;
  });
}

int ss_fork_sequence(ss_cache* c, int64_t parent, int64_t child, int64_t fork_len,
                     const int32_t* child_tokens, int64_t n) {
  return Guard(c, [&]() -> int {
    c->cache->ForkSequence(parent, child, fork_len, ToTokens(child_tokens, n));
    return SS_OK;
  });
}

int ss_mark_send(ss_cache* c, int64_t seq, int64_t begin, int64_t end, int32_t dest,
                 const ss_addr* dest_addr, uint64_t tag) {
  return Guard(c, [&]() -> int {
    c->cache->MarkSend(seq, {begin, end}, dest, ToAddr(dest_addr), tag);
    return SS_OK;
  });
}

int ss_ensure_allocated(ss_cache* c, int64_t seq, int64_t upto) {
  return Guard(c, [&]() -> int {
    c->cache->EnsureAllocated(seq, upto);
    return SS_OK;
  });
}

int ss_append_token(ss_cache* c, int64_t seq, int32_t token) {
  return Guard(c, [&]() -> int {
    c->cache->AppendToken(seq, token);
    return SS_OK;
  });
}

int ss_begin_forward(ss_cache* c, const ss_batch_entry* batch, int64_t n, ss_plan** plan_out) {
  return Guard(c, [&]() -> int {
    std::vector<BatchEntry> b;
    for (int64_t i = 0; i < n; ++i) {
      b.push_back({batch[i].seq, {batch[i].begin, batch[i].end}, batch[i].is_decode != 0});
    }
    auto p = std::make_unique<ss_plan>();
    p->plan = c->cache->BeginForward(b);
    p->owner = c;
    c->plans.insert(p.get());
    *plan_out = p.release();
    return SS_OK;
  });
}

int64_t ss_plan_total_outputs(const ss_plan* p) { return p->plan.total_outputs; }
int64_t ss_plan_num_sends(const ss_plan* p) { return static_cast<int64_t>(p->plan.sends.size()); }
int32_t ss_plan_next_layer(const ss_plan* p) { return p->plan.next_layer; }
void ss_plan_destroy(ss_plan* p) {
  if (!p) return;
  if (p->owner) p->owner->plans.erase(p);
  delete p;
}

int ss_attention(ss_cache* c, ss_plan* p, int32_t layer, const uint64_t* hidden_in,
                 uint64_t* hidden_out, int64_t n, ss_frame_sink sink, void* user) {
  return Guard(c, [&]() -> int {
    FrameSink fs;
    if (sink) {
      fs = [&](int32_t l, const PlanSend& s, std::vector<uint64_t> payload) {
        std::vector<ss_slot_range> rr;
        for (const auto& r : s.dest_addr.ranges) rr.push_back({r.page_id, r.slot_begin, r.slot_count});
        ss_addr a{s.dest_addr.token_begin, s.dest_addr.token_count,
                  static_cast<int64_t>(rr.size()), rr.data(), static_cast<int64_t>(rr.size())};
        sink(user, l, s.seq, s.range.begin, s.range.end, s.dest, &a, s.user_tag, payload.data(),
             static_cast<int64_t>(payload.size()));
      };
    }
    auto out = c->cache->Attention(layer, &p->plan, std::span<const uint64_t>(hidden_in, n), fs);
    std::copy(out.begin(), out.end(), hidden_out);
    return SS_OK;
  });
}

int ss_gather_range(ss_cache* c, int64_t seq, int64_t begin, int64_t end, int32_t layer,
                    uint64_t* out, int64_t out_words) {
  return Guard(c, [&]() -> int {
    auto v = c->cache->GatherRange(seq, {begin, end}, layer);
    if (static_cast<int64_t>(v.size()) > out_words) {
      return Fail(c, SS_ERR_BUFFER_TOO_SMALL, "gather output too small");
    }
    std::copy(v.begin(), v.end(), out);
    return SS_OK;
  });
}

int ss_build_addr(ss_cache* c, int64_t seq, int64_t begin, int64_t end, ss_addr* addr_out) {
  return Guard(c, [&]() -> int { return FromAddr(c, c->cache->BuildAddr(seq, {begin, end}), addr_out); });
}

int ss_apply_remote_write(ss_cache* c, const ss_addr* addr, int32_t layer, const uint64_t* payload,
                          int64_t n_words, uint64_t tag, int32_t* apply_status) {
  return Guard(c, [&]() -> int {
    auto st = c->cache->ApplyRemoteWrite(ToAddr(addr), layer,
                                         std::span<const uint64_t>(payload, n_words), tag);
    *apply_status = static_cast<int32_t>(st);
    return SS_OK;
  });
}

int ss_drain_receive_completions(ss_cache* c, int64_t* out, int64_t cap, int64_t* n_out) {
  return Guard(c, [&]() -> int {
    for (SeqId s : c->cache->DrainReceiveCompletions()) c->drained.push_back(s);
    int64_t n = 0;
    while (n < cap && !c->drained.empty()) {
      out[n++] = c->drained.front();
      c->drained.pop_front();
    }
    *n_out = n;
    return SS_OK;
  });
}

int ss_set_finished(ss_cache* c, int64_t seq, int32_t f) {
  return Guard(c, [&]() -> int {
    c->cache->SetFinished(seq, f != 0);
    return SS_OK;
  });
}
int ss_commit_to_tree(ss_cache* c, int64_t seq) {
  return Guard(c, [&]() -> int {
    c->cache->CommitToTree(seq);
    return SS_OK;
  });
}
int ss_free_sequence(ss_cache* c, int64_t seq) {
  return Guard(c, [&]() -> int {
    c->cache->FreeSequence(seq);
    return SS_OK;
  });
}
int ss_evict(ss_cache* c, int64_t bytes, int64_t* freed) {
  return Guard(c, [&]() -> int {
    *freed = c->cache->Evict(bytes);
    return SS_OK;
  });
}
int ss_pin(ss_cache* c, const int32_t* prefix, int64_t n, int32_t flag) {
  return Guard(c, [&]() -> int {
    c->cache->Pin(std::span<const Token>(prefix, n), flag != 0);
    return SS_OK;
  });
}

int ss_has_sequence(const ss_cache* c, int64_t seq) { return c->cache->HasSequence(seq) ? 1 : 0; }

int ss_get_record(ss_cache* c, int64_t seq, ss_record_info* info, int64_t* own_pages,
                  int64_t own_cap) {
  return Guard(c, [&]() -> int {
    const SequenceRecord* r = c->cache->GetRecord(seq);
    info->id = r->id;
    info->parent = r->parent;
    info->fork_len = r->fork_len;
    info->refcount = r->refcount;
    info->finished = r->finished ? 1 : 0;
    info->alloc_len = r->alloc_len;
    info->committed_hint = r->committed_hint;
    info->num_tokens = static_cast<int64_t>(r->tokens.size());
    info->num_own_pages = static_cast<int64_t>(r->own_pages.size());
    info->fold_frontier = r->fold_frontier;
    info->digest_len = r->digest_len;
    info->prefix_digest = r->prefix_digest;
    info->has_window = r->window.has_value() ? 1 : 0;
    info->window_complete = r->window ? (r->window->complete ? 1 : 0) : 0;
    info->window_begin = r->window ? r->window->range.begin : 0;
    info->window_end = r->window ? r->window->range.end : 0;
    info->window_expected_writes = r->window ? r->window->expected_writes : 0;
    info->window_received_writes = r->window ? r->window->received_writes : 0;
    if (own_pages) {
      if (own_cap < info->num_own_pages) {
        return Fail(c, SS_ERR_BUFFER_TOO_SMALL, "own_pages buffer too small");
      }
      std::copy(r->own_pages.begin(), r->own_pages.end(), own_pages);
    }
    return SS_OK;
  });
}

int ss_committed(ss_cache* c, int64_t seq, int64_t* out) {
  return Guard(c, [&]() -> int {
    *out = c->cache->Committed(seq);
    return SS_OK;
  });
}

int ss_read_entry_words(ss_cache* c, int64_t seq, int64_t pos, int32_t layer, uint64_t* out,
                        int64_t out_words) {
  return Guard(c, [&]() -> int {
    auto v = c->cache->ReadEntryWords(seq, pos, layer);
    if (static_cast<int64_t>(v.size()) > out_words) {
      return Fail(c, SS_ERR_BUFFER_TOO_SMALL, "entry buffer too small");
    }
    std::copy(v.begin(), v.end(), out);
    return SS_OK;
  });
}

int ss_fill_of(ss_cache* c, int64_t seq, int64_t pos, int32_t layer, int32_t* out) {
  return Guard(c, [&]() -> int {
    *out = static_cast<int32_t>(c->cache->FillOf(seq, pos, layer));
    return SS_OK;
  });
}

int64_t ss_free_pages(const ss_cache* c) { return c->cache->FreePages(); }
int64_t ss_total_pages(const ss_cache* c) { return c->cache->TotalPages(); }
int ss_cache_config(const ss_cache* c, ss_config* out) {  // cache_config(), kv_cache.h:235
  *out = c->cfg;
  return SS_OK;
}
int64_t ss_bytes_per_page(const ss_cache* c) { return c->cache->BytesPerPage(); }
int64_t ss_sequence_count(const ss_cache* c) { return static_cast<int64_t>(c->cache->SequenceCount()); }
int ss_sequence_ids(const ss_cache* c, int64_t* out, int64_t cap, int64_t* n_out) {
  auto ids = c->cache->SequenceIds();
  *n_out = static_cast<int64_t>(ids.size());
  if (static_cast<int64_t>(ids.size()) > cap) return SS_ERR_BUFFER_TOO_SMALL;
  std::copy(ids.begin(), ids.end(), out);
  return SS_OK;
}
int64_t ss_pending_send_count(const ss_cache* c) {
  return static_cast<int64_t>(c->cache->PendingSendCount());
}
int64_t ss_tree_node_count(const ss_cache* c) { return static_cast<int64_t>(c->cache->Tree().NodeCount()); }
int ss_tree_contains(const ss_cache* c, int64_t seq) { return c->cache->Tree().Contains(seq) ? 1 : 0; }
uint64_t ss_tree_last_touch(const ss_cache* c, int64_t seq) { return c->cache->Tree().LastTouch(seq); }
int ss_tree_sequences_by_lru(const ss_cache* c, int64_t* out, int64_t cap, int64_t* n_out) {
  auto ids = c->cache->Tree().SequencesByLru();
  *n_out = static_cast<int64_t>(ids.size());
  if (static_cast<int64_t>(ids.size()) > cap) return SS_ERR_BUFFER_TOO_SMALL;
  std::copy(ids.begin(), ids.end(), out);
  return SS_OK;
}

int ss_addr_validate(const ss_addr* a) {
  return Guard(nullptr, [&]() -> int {
    ToAddr(a).Validate();
    return SS_OK;
  });
}
int ss_addr_slice(const ss_addr* in, int64_t begin, int64_t end, ss_addr* out) {
  return Guard(nullptr, [&]() -> int { return FromAddr(nullptr, ToAddr(in).Slice(begin, end), out); });
}

/* Device entry points: the reference has no device path. */
int ss_device(const ss_cache*) { return -1; }
int ss_attach_peer(ss_cache*, int32_t, ss_cache*) { return SS_ERR_UNSUPPORTED; }
int ss_export_ipc(ss_cache*, ss_ipc_handle*) { return SS_ERR_UNSUPPORTED; }
int ss_import_ipc(ss_cache*, int32_t, const ss_ipc_handle*) { return SS_ERR_UNSUPPORTED; }
int ss_detach_peer(ss_cache*, int32_t) { return SS_ERR_UNSUPPORTED; }
int ss_peer_info(const ss_cache*, int32_t, int32_t*, int32_t*) { return SS_ERR_UNSUPPORTED; }
int ss_set_send_mode(ss_cache*, int32_t, int32_t) { return SS_ERR_UNSUPPORTED; }
int ss_launch_relay_send_async(ss_cache*, ss_plan*, int32_t, int32_t, int64_t, void*) {
  return SS_ERR_UNSUPPORTED;
}
int ss_attention_async(ss_cache*, ss_plan*, int32_t, const uint64_t*, uint64_t*, void*) {
  return SS_ERR_UNSUPPORTED;
}
int ss_direct_send_async(ss_cache*, int64_t, int64_t, int64_t, int32_t, const ss_addr*, uint64_t,
                         int32_t, int32_t, void*) {
  return SS_ERR_UNSUPPORTED;
}
int ss_begin_direct_send(ss_cache*, int64_t, int64_t, int64_t, int32_t, const ss_addr*, uint64_t,
                         ss_plan**) {
  return SS_ERR_UNSUPPORTED;
}
int ss_launch_direct_send_async(ss_cache*, ss_plan*, int32_t, int32_t, void*) {
  return SS_ERR_UNSUPPORTED;
}
int ss_launch_direct_send_after_async(ss_cache*, ss_plan*, int32_t, int32_t, void*, void*) {
  return SS_ERR_UNSUPPORTED;
}
int ss_broadcast_send_async(ss_cache*, int64_t, int64_t, int64_t, int32_t, const int32_t*,
                            const ss_addr*, uint64_t, int32_t, int32_t, void*) {
  return SS_ERR_UNSUPPORTED;
}
int ss_gather_range_async(ss_cache*, int64_t, int64_t, int64_t, int32_t, uint64_t*, void*) {
  return SS_ERR_UNSUPPORTED;
}
int ss_gather_range_layers_async(ss_cache*, int64_t, int64_t, int64_t, int32_t, int32_t, uint64_t*,
                                 void*) {
  return SS_ERR_UNSUPPORTED;
}
int ss_apply_remote_write_async(ss_cache*, const ss_addr*, int32_t, const uint64_t*, int64_t,
                                uint64_t, int32_t*, void*) {
  return SS_ERR_UNSUPPORTED;
}
int ss_append_rows_layers_async(ss_cache*, ss_plan*, int32_t, int32_t, const void*, void*) {
  return SS_ERR_UNSUPPORTED;
}
int ss_append_rows_async(ss_cache*, ss_plan*, int32_t, const void*, void*) {
  return SS_ERR_UNSUPPORTED;
}
int ss_append_rows_send_async(ss_cache*, ss_plan*, ss_plan*, int32_t, int32_t, const void*, void*) {
  return SS_ERR_UNSUPPORTED;
}
int ss_begin_decode(ss_cache*, const int64_t*, const int64_t*, int64_t, ss_plan**) {
  return SS_ERR_UNSUPPORTED;
}
int ss_paged_decode_attention_async(ss_cache*, ss_plan*, int32_t, int32_t, int32_t, int32_t, float,
                                    const void*, void*, void*) {
  return SS_ERR_UNSUPPORTED;
}
int ss_paged_prefill_attention_async(ss_cache*, int64_t, int64_t, int64_t, int32_t, int32_t,
                                     int32_t, int32_t, float, const void*, void*, void*) {
  return SS_ERR_UNSUPPORTED;
}
int ss_pool_layer_ptr(ss_cache*, int32_t, void**) { return SS_ERR_UNSUPPORTED; }
int ss_wait_receive_async(ss_cache*, int64_t, int64_t, void*) { return SS_ERR_UNSUPPORTED; }
int ss_wait_receive_layer_async(ss_cache*, int64_t, int32_t, int64_t, void*) {
  return SS_ERR_UNSUPPORTED;
}
int ss_copy_counters(const ss_cache*, int64_t* h2d, int64_t* d2h) {
  *h2d = 0;
  *d2h = 0;
  return SS_OK;
}
int64_t ss_kernel_launches(const ss_cache*) { return 0; }
int ss_synchronize(ss_cache*) { return SS_OK; }

/* ------------------------------------------------------------------ */
/* Wire formats: the reference codec (kv_addr.cc:53-118,               */
/* transport.cc:14-107) behind the same entry points.                  */
/* ------------------------------------------------------------------ */
int ss_addr_encode(const ss_addr* a, uint8_t* out, int64_t cap, int64_t* len) {
  return Guard(nullptr, [&]() -> int {
    std::vector<uint8_t> b;
    ToAddr(a).EncodeTo(&b);
    *len = static_cast<int64_t>(b.size());
    if (*len > cap) return SS_ERR_BUFFER_TOO_SMALL;
    std::copy(b.begin(), b.end(), out);
    return SS_OK;
  });
}

int ss_addr_decode(const uint8_t* data, int64_t size, int64_t* pos, ss_addr* out) {
  return Guard(nullptr, [&]() -> int {
    size_t p = static_cast<size_t>(*pos);
    KVAddrInfo a = KVAddrInfo::DecodeFrom(data, static_cast<size_t>(size), &p);
    int st = FromAddr(nullptr, a, out);
    if (st == SS_OK) *pos = static_cast<int64_t>(p);
    return st;
  });
}

int ss_addr_to_json(const ss_addr* a, char* out, int64_t cap, int64_t* len) {
  return Guard(nullptr, [&]() -> int {
    std::string j = ToAddr(a).ToJson();
    *len = static_cast<int64_t>(j.size());
    if (*len + 1 > cap) return SS_ERR_BUFFER_TOO_SMALL;
    std::memcpy(out, j.c_str(), j.size() + 1);
    return SS_OK;
  });
}

int ss_addr_from_json(const char* text, int64_t len, ss_addr* out) {
  return Guard(nullptr, [&]() -> int {
    return FromAddr(nullptr, KVAddrInfo::FromJson(std::string(text, static_cast<size_t>(len))), out);
  });
}

int64_t ss_frame_write_header_size(int64_t n_ranges) {
  WriteFrame f;
  f.addr.ranges.resize(static_cast<size_t>(n_ranges));
  return static_cast<int64_t>(EncodeWriteFrame(f).size()) - 4;  // minus the CRC of an empty payload
}

int ss_frame_encode_ack(uint64_t seq_tag, int32_t layer, int64_t token_begin, int32_t status,
                        uint8_t* out, int64_t cap, int64_t* len) {
  return Guard(nullptr, [&]() -> int {
    AckFrame a;
    a.seq_tag = seq_tag;
    a.layer = layer;
    a.token_begin = token_begin;
    a.status = static_cast<AckStatus>(status);
    auto b = EncodeAckFrame(a);
    *len = static_cast<int64_t>(b.size());
    if (*len > cap) return SS_ERR_BUFFER_TOO_SMALL;
    std::copy(b.begin(), b.end(), out);
    return SS_OK;
  });
}

int ss_frame_decode(const uint8_t* frame, int64_t size, ss_frame_info* info) {
  return Guard(nullptr, [&]() -> int {
    DecodedFrame d = DecodeFrame(frame, static_cast<size_t>(size));
    info->type = static_cast<int32_t>(d.type);
    if (d.type == FrameType::kWrite) {
      info->seq_tag = d.write.seq_tag;
      info->layer = d.write.layer;
      info->payload_offset = 41 + 8 * static_cast<int64_t>(d.write.addr.ranges.size());
      info->payload_bytes = static_cast<int64_t>(d.write.payload.size()) * 8;
      const uint8_t* c = frame + info->payload_offset + info->payload_bytes;
      info->wire_crc = c[0] | (c[1] << 8) | (c[2] << 16) | (static_cast<uint32_t>(c[3]) << 24);
      return FromAddr(nullptr, d.write.addr, &info->addr);
    }
    info->seq_tag = d.ack.seq_tag;
    info->layer = d.ack.layer;
    info->token_begin = d.ack.token_begin;
    info->ack_status = static_cast<int32_t>(d.ack.status);
    info->addr.n_ranges = 0;
    return SS_OK;
  });
}

int ss_crc32_async(ss_cache*, const void*, int64_t, uint32_t*, void*) { return SS_ERR_UNSUPPORTED; }

// WriteFrame{tag, layer, dest, GatherRange(seq, range, layer)} with
// MarkSend's address rule (kv_cache.cc:231-243), then EncodeWriteFrame.
int ss_encode_write_frame(ss_cache* c, int64_t seq, int64_t begin, int64_t end, int32_t layer,
                          uint64_t seq_tag, const ss_addr* dest_addr, uint8_t* frame, int64_t cap,
                          int64_t* frame_len) {
  return Guard(c, [&]() -> int {
    WriteFrame f;
    f.seq_tag = seq_tag;
    f.layer = layer;
    f.addr = ToAddr(dest_addr);
    SPLITSERVE_CHECK(f.addr.token_count == end - begin && f.addr.token_begin == begin,
                     ErrorCode::kAddrMismatch, "destination does not cover the range");
    f.addr.Validate();
    f.payload = c->cache->GatherRange(seq, {begin, end}, layer);
    auto b = EncodeWriteFrame(f);
    *frame_len = static_cast<int64_t>(b.size());
    if (*frame_len > cap) return Fail(c, SS_ERR_BUFFER_TOO_SMALL, "frame buffer too small");
    std::copy(b.begin(), b.end(), frame);
    return SS_OK;
  });
}

int ss_encode_write_frame_async(ss_cache*, int64_t, int64_t, int64_t, int32_t, uint64_t,
                                const ss_addr*, void*, int64_t, int64_t*, void*) {
  return SS_ERR_UNSUPPORTED;
}

// The TCP fabric's inbound step (tcp_fabric.cc:144-168) with
// apply = ApplyRemoteWrite(addr, layer, payload, seq_tag).
int ss_receive_write_frame(ss_cache* c, const uint8_t* frame, int64_t size, uint8_t* ack_out,
                           int32_t* apply_status) {
  return Guard(c, [&]() -> int {
    DecodedFrame d = DecodeFrame(frame, static_cast<size_t>(size));
    SPLITSERVE_CHECK(d.type == FrameType::kWrite, ErrorCode::kInvalidArgument, "not a write frame");
    AckFrame ack;
    ack.seq_tag = d.write.seq_tag;
    ack.layer = d.write.layer;
    ack.token_begin = d.write.addr.token_begin;
    *apply_status = -1;
    if (!d.crc_ok) {
      ack.status = AckStatus::kChecksumMismatch;
    } else {
      auto st = c->cache->ApplyRemoteWrite(d.write.addr, d.write.layer, d.write.payload,
                                           d.write.seq_tag);
      *apply_status = static_cast<int32_t>(st);
      ack.status = st == KVCache::ApplyStatus::kUnknownAddress ? AckStatus::kUnknownAddress
                                                                : AckStatus::kOk;
    }
    auto b = EncodeAckFrame(ack);
    std::copy(b.begin(), b.end(), ack_out);
    return SS_OK;
  });
}

/* The reference's calibrated cost model (config.h:40-66, config.cc:36-118),
 * for the parity test of paper_2412_12488_b200/cost_model.py.  out[6] =
 * {alpha, beta, gamma, delta, c0, c1}; fit_* also returns the max relative
 * anchor error.  Anchor arrays: prefill {n_new, n_total, ms} x n_p,
 * transfer {n_tokens, ms} x n_t. */
int ssref_default_cost_model(double* out) {
  const CostModel m = DefaultCostModel();
  const double v[6] = {m.alpha, m.beta, m.gamma, m.delta, m.c0, m.c1};
  std::copy(v, v + 6, out);
  return SS_OK;
}

int ssref_fit_cost_model(const double* prefill, int32_t n_p, const double* transfer, int32_t n_t,
                         double* out, double* max_rel_err) {
  try {
    std::vector<PrefillAnchor> pa;
    for (int32_t i = 0; i < n_p; ++i)
      pa.push_back({static_cast<int64_t>(prefill[3 * i]), static_cast<int64_t>(prefill[3 * i + 1]),
                    prefill[3 * i + 2]});
    std::vector<TransferAnchor> ta;
    for (int32_t i = 0; i < n_t; ++i)
      ta.push_back({static_cast<int64_t>(transfer[2 * i]), transfer[2 * i + 1]});
    const CostFitReport r = FitCostModel(pa, ta);
    const double v[6] = {r.model.alpha, r.model.beta, r.model.gamma, r.model.delta, r.model.c0,
                         r.model.c1};
    std::copy(v, v + 6, out);
    *max_rel_err = r.max_rel_err;
    return SS_OK;
  } catch (const Error& e) {
    return 1 + static_cast<int>(e.code());
  }
}

/* Host CRC-32 of the reference (transport.cc:14-28), for tests. */
uint32_t ssref_crc32(const uint8_t* data, int64_t n) { return Crc32(data, static_cast<size_t>(n)); }

/* ------------------------------------------------------------------ */
/* Reference arm of bench.py: DirectSend KV migration through the      */
/* reference classes.                                                  */
/* ------------------------------------------------------------------ */
typedef struct {
  int32_t layers, dim, page_size, vocab;
  int64_t num_pages;
  uint64_t hash_seed;
  int64_t prompt_len;   /* tokens in the prompt */
  int64_t end;          /* PrepRecv end index (-1 = all but last) */
  int32_t layer_sample; /* layers moved per step (<= layers); 0 = all */
  int32_t threads;      /* independent engine pairs, one host thread each */
  int32_t steps, warmup;
  uint64_t token_seed;
} ssref_migrate_cfg;

typedef struct {
  double seconds;           /* wall time of the timed steps (max over threads) */
  double bytes_moved;       /* KV payload bytes delivered over all threads and steps */
  double prep_recv_s;       /* summed over threads/steps */
  double gather_s;
  double apply_s;
  double drain_free_s;
  int64_t tokens_per_step;  /* per pair */
  int32_t ok;               /* 1 if every step completed its receive window */
} ssref_migrate_result;

int ssref_bench_migrate(const ssref_migrate_cfg* cfg, ssref_migrate_result* res) {
  using clk = std::chrono::steady_clock;
  const int T = std::max(1, cfg->threads);
  std::vector<double> wall(T, 0), prep(T, 0), gath(T, 0), appl(T, 0), drfr(T, 0);
  std::vector<int64_t> moved(T, 0), ntok(T, 0);
  std::atomic<int> ok{1};
  std::atomic<int> ready{0};
  std::string first_err;
  std::atomic<int> failed{0};

  auto body = [&](int t) {
    try {
      ModelConfig m;
      m.layers = cfg->layers;
      m.dim = cfg->dim;
      m.vocab = cfg->vocab;
      m.hash_seed = cfg->hash_seed;
      CacheConfig cc;
      cc.num_pages = cfg->num_pages;
      cc.page_size = cfg->page_size;
      HashModel model(m);
      KVCache P(cc, &model), D(cc, &model);
      // Prompt tokens: splitmix stream, uniform in [0, vocab).
      TokenList tokens(cfg->prompt_len);
      uint64_t s = cfg->token_seed + 0x9e3779b97f4a7c15ULL * (t + 1);
      for (auto& tok : tokens) {
        s += 0x9e3779b97f4a7c15ULL;
        tok = static_cast<Token>(Mix64(s) % static_cast<uint64_t>(cfg->vocab));
      }
      const int64_t e = ResolveEndIndex(cfg->prompt_len, cfg->end);
      // P holds the prefix committed (as after an earlier prefill); its KV
      // bytes arrive through the reference receive path once, untimed.
      auto pr = P.PrepRecv(1, tokens, cfg->prompt_len);
      std::vector<uint64_t> payload(static_cast<size_t>(cfg->prompt_len) * cfg->dim);
      for (int32_t l = 0; l < cfg->layers; ++l) {
        for (size_t i = 0; i < payload.size(); ++i) payload[i] = Mix64((uint64_t(l) << 40) ^ i);
        P.ApplyRemoteWrite(pr.addr, l, payload, 0);
      }
      P.DrainReceiveCompletions();
      const int32_t Ls = cfg->layer_sample > 0 ? std::min(cfg->layer_sample, cfg->layers) : cfg->layers;
      ready.fetch_add(1);
      while (ready.load() < T) std::this_thread::yield();
      clk::time_point t0;
      for (int step = 0; step < cfg->warmup + cfg->steps; ++step) {
        if (step == cfg->warmup) t0 = clk::now();
        const bool timed = step >= cfg->warmup;
        const SeqId seq = 1000 + step;
        auto a0 = clk::now();
        auto r = D.PrepRecv(seq, tokens, cfg->end);
        auto a1 = clk::now();
        double g = 0, ap = 0;
        for (int32_t l = 0; l < Ls; ++l) {
          auto b0 = clk::now();
          auto pl = P.GatherRange(1, {r.match_len, e}, l);
          auto b1 = clk::now();
          auto st = D.ApplyRemoteWrite(r.addr, l, pl, static_cast<uint64_t>(step));
          auto b2 = clk::now();
          if (st != KVCache::ApplyStatus::kOk) ok = 0;
          g += std::chrono::duration<double>(b1 - b0).count();
          ap += std::chrono::duration<double>(b2 - b1).count();
          if (timed) moved[t] += static_cast<int64_t>(pl.size()) * 8;
        }
        auto c0 = clk::now();
        auto done = D.DrainReceiveCompletions();
        if (Ls == cfg->layers && (done.size() != 1 || done[0] != seq)) ok = 0;
        D.FreeSequence(seq);
        auto c1 = clk::now();
        if (timed) {
          prep[t] += std::chrono::duration<double>(a1 - a0).count();
          gath[t] += g;
          appl[t] += ap;
          drfr[t] += std::chrono::duration<double>(c1 - c0).count();
          ntok[t] = e - r.match_len;
        }
      }
      wall[t] = std::chrono::duration<double>(clk::now() - t0).count();
    } catch (const std::exception& ex) {
      if (failed.fetch_add(1) == 0) first_err = ex.what();
      ready.fetch_add(1);
    }
  };
  std::vector<std::thread> th;
  for (int t = 0; t < T; ++t) th.emplace_back(body, t);
  for (auto& x : th) x.join();
  if (failed.load() > 0) {
    fprintf(stderr, "ssref_bench_migrate: %s\n", first_err.c_str());
    return SS_ERR_INTERNAL;
  }
  std::memset(res, 0, sizeof(*res));
  for (int t = 0; t < T; ++t) {
    res->seconds = std::max(res->seconds, wall[t]);
    res->bytes_moved += static_cast<double>(moved[t]);
    res->prep_recv_s += prep[t];
    res->gather_s += gath[t];
    res->apply_s += appl[t];
    res->drain_free_s += drfr[t];
  }
  res->tokens_per_step = ntok[0];
  res->ok = ok.load();
  return SS_OK;
}

}  // extern "C"
