// capi.cc — extern "C" entry points of include/microkv.h for the B200
// product library.  Each one converts POD arguments, calls the engine
// member that mirrors the reference (cache.h), and maps exceptions to the
// status codes of the header.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "../../include/microkv.h"
#include "cache.h"
#include "wire.h"

using mkv::KVAddr;

namespace {

// The cache's device is current for the call and the caller's current
// device is restored afterwards (a multi-GPU host keeps its own device).
struct DeviceScope {
  int prev = -1;
  explicit DeviceScope(const ss_cache* c) {
    if (c == nullptr || c->device() < 0) return;
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    if (prev != c->device()) cudaSetDevice(c->device());
    else prev = -1;
  }
  ~DeviceScope() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

template <typename F>
int Guard(ss_cache* c, F&& f) {
  try {
    DeviceScope scope(c);
    return f();
  } catch (const mkv::Error& e) {
    if (c) c->last_error = e.what();
    return e.status();
  } catch (const std::exception& e) {
    if (c) c->last_error = std::string("Internal: ") + e.what();
    return SS_ERR_INTERNAL;
  }
}

KVAddr ToAddr(const ss_addr* a) {
  KVAddr out;
  out.token_begin = a->token_begin;
  out.token_count = a->token_count;
  out.ranges.reserve(a->n_ranges);
  for (int64_t i = 0; i < a->n_ranges; ++i) {
    out.ranges.push_back({a->ranges[i].page_id, a->ranges[i].slot_begin, a->ranges[i].slot_count});
  }
  return out;
}

int FromAddr(ss_cache* c, const KVAddr& a, ss_addr* out) {
  out->token_begin = a.token_begin;
  out->token_count = a.token_count;
  const int64_t n = static_cast<int64_t>(a.ranges.size());
  if (n > out->ranges_cap) {
    out->n_ranges = n;
    if (c) c->last_error = "BufferTooSmall: address needs " + std::to_string(n) + " ranges";
    return SS_ERR_BUFFER_TOO_SMALL;
  }
  for (int64_t i = 0; i < n; ++i) {
    out->ranges[i] = {a.ranges[i].page_id, a.ranges[i].slot_begin, a.ranges[i].slot_count};
  }
  out->n_ranges = n;
  return SS_OK;
}

std::vector<int32_t> ToTokens(const int32_t* t, int64_t n) {
  return n > 0 ? std::vector<int32_t>(t, t + n) : std::vector<int32_t>();
}

cudaStream_t S(void* s) { return static_cast<cudaStream_t>(s); }

}  // namespace

extern "C" {

int ss_abi_version(void) { return SS_ABI_VERSION; }
const char* ss_impl_name(void) { return "microkv-b200"; }

int ss_cache_create(const ss_config* cfg, ss_cache** out) {
  int prev = -1;
  const bool restore = cfg != nullptr && cfg->device >= 0 && cudaGetDevice(&prev) == cudaSuccess;
  struct Restore {
    bool on;
    int dev;
    ~Restore() {
      if (on) cudaSetDevice(dev);
    }
  } r{restore, prev};
  try {
    *out = new ss_cache(*cfg);
    return SS_OK;
  } catch (const mkv::Error& e) {
    *out = nullptr;
    return e.status();
  } catch (const std::exception&) {
    *out = nullptr;
    return SS_ERR_INTERNAL;
  }
}

void ss_cache_destroy(ss_cache* c) {
  DeviceScope scope(c);
  delete c;
}
const char* ss_last_error(const ss_cache* c) { return c ? c->last_error.c_str() : ""; }
const char* ss_status_name(int s) { return mkv::StatusName(s); }
int ss_status_retryable(int s) {
  return (s == SS_ERR_OUT_OF_PAGES || s == SS_ERR_PEER_UNREACHABLE) ? 1 : 0;
}

uint64_t ss_initial_prefix_digest(const ss_cache* c) { return c->InitialPrefixDigest(); }
uint64_t ss_embed(const ss_cache* c, int32_t t, int64_t pos) { return c->Embed(t, pos); }
int32_t ss_sample_token(const ss_cache* c, uint64_t h) { return c->SampleToken(h); }

int ss_match_prefix(ss_cache* c, const int32_t* tokens, int64_t n, int64_t* match_len,
                    int64_t* seq_out) {
  return Guard(c, [&]() -> int {
    auto r = c->MatchPrefixSeq(std::span<const int32_t>(tokens, n));
    *match_len = r.match_len;
    if (seq_out) *seq_out = r.seq;
    return SS_OK;
  });
}

int ss_prep_recv(ss_cache* c, int64_t seq, const int32_t* tokens, int64_t n, int64_t end,
                 int64_t* match_len, ss_addr* addr_out) {
  return Guard(c, [&]() -> int {
    KVAddr a;
    *match_len = c->PrepRecv(seq, ToTokens(tokens, n), end, &a, addr_out->ranges_cap);
    return FromAddr(c, a, addr_out);
  });
}

int ss_create_sequence(ss_cache* c, int64_t seq, const int32_t* tokens, int64_t n) {
  return Guard(c, [&]() -> int {
    c->CreateSequence(seq, ToTokens(tokens, n));
    return SS_OK;
  });
}

int ss_fork_sequence(ss_cache* c, int64_t parent, int64_t child, int64_t fork_len,
                     const int32_t* child_tokens, int64_t n) {
  return Guard(c, [&]() -> int {
    c->ForkSequence(parent, child, fork_len, ToTokens(child_tokens, n));
    return SS_OK;
  });
}

int ss_mark_send(ss_cache* c, int64_t seq, int64_t begin, int64_t end, int32_t dest,
                 const ss_addr* dest_addr, uint64_t tag) {
  return Guard(c, [&]() -> int {
    c->MarkSend(seq, begin, end, dest, ToAddr(dest_addr), tag);
    return SS_OK;
  });
}

int ss_ensure_allocated(ss_cache* c, int64_t seq, int64_t upto) {
  return Guard(c, [&]() -> int {
    c->EnsureAllocated(seq, upto);
    return SS_OK;
  });
}

int ss_append_token(ss_cache* c, int64_t seq, int32_t token) {
  return Guard(c, [&]() -> int {
    c->AppendToken(seq, token);
    return SS_OK;
  });
}

int ss_begin_forward(ss_cache* c, const ss_batch_entry* batch, int64_t n, ss_plan** plan_out) {
  return Guard(c, [&]() -> int {
    *plan_out = c->BeginForward(batch, n);
    return SS_OK;
  });
}

int64_t ss_plan_total_outputs(const ss_plan* p) { return p->total_outputs; }
int64_t ss_plan_num_sends(const ss_plan* p) { return static_cast<int64_t>(p->sends.size()); }
int32_t ss_plan_next_layer(const ss_plan* p) { return p->next_layer; }
void ss_plan_destroy(ss_plan* p) {
  if (!p) return;
  try {
    p->owner->DestroyPlan(p);
  } catch (...) {
  }
}

int ss_attention(ss_cache* c, ss_plan* p, int32_t layer, const uint64_t* hidden_in,
                 uint64_t* hidden_out, int64_t n, ss_frame_sink sink, void* user) {
  return Guard(c, [&]() -> int {
    c->Attention(p, layer, hidden_in, hidden_out, n, sink, user);
    return SS_OK;
  });
}

int ss_gather_range(ss_cache* c, int64_t seq, int64_t begin, int64_t end, int32_t layer,
                    uint64_t* out, int64_t out_words) {
  return Guard(c, [&]() -> int {
    if (c->device() < 0) mkv::ThrowStatus(SS_ERR_NO_DEVICE, "GatherRange on a host-only cache");
    const int64_t words = std::max<int64_t>(0, end - begin) * c->dim();
    if (words > out_words) mkv::ThrowStatus(SS_ERR_BUFFER_TOO_SMALL, "gather output too small");
    uint64_t* dev = nullptr;
    if (words > 0) mkv::CudaCheck(cudaMalloc(&dev, sizeof(uint64_t) * words), "cudaMalloc");
    try {
      c->GatherRange(seq, begin, end, layer, dev, nullptr);
      if (words > 0) {
        mkv::CudaCheck(cudaMemcpy(out, dev, sizeof(uint64_t) * words, cudaMemcpyDeviceToHost),
                       "D2H gather");
      }
    } catch (...) {
      cudaFree(dev);
      throw;
    }
    cudaFree(dev);
    return SS_OK;
  });
}

int ss_build_addr(ss_cache* c, int64_t seq, int64_t begin, int64_t end, ss_addr* addr_out) {
  return Guard(c, [&]() -> int { return FromAddr(c, c->BuildAddr(seq, begin, end), addr_out); });
}

int ss_apply_remote_write(ss_cache* c, const ss_addr* addr, int32_t layer, const uint64_t* payload,
                          int64_t n_words, uint64_t tag, int32_t* apply_status) {
  return Guard(c, [&]() -> int {
    *apply_status =
        c->ApplyRemoteWrite(ToAddr(addr), layer, payload, n_words, false, tag, nullptr, true);
    return SS_OK;
  });
}

int ss_drain_receive_completions(ss_cache* c, int64_t* out, int64_t cap, int64_t* n_out) {
  return Guard(c, [&]() -> int {
    for (int64_t s : c->DrainReceiveCompletions()) c->drained.push_back(s);
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
    c->SetFinished(seq, f != 0);
    return SS_OK;
  });
}
int ss_commit_to_tree(ss_cache* c, int64_t seq) {
  return Guard(c, [&]() -> int {
    c->CommitToTree(seq);
    return SS_OK;
  });
}
int ss_free_sequence(ss_cache* c, int64_t seq) {
  return Guard(c, [&]() -> int {
    c->FreeSequence(seq);
    return SS_OK;
  });
}
int ss_evict(ss_cache* c, int64_t bytes, int64_t* freed) {
  return Guard(c, [&]() -> int {
    *freed = c->Evict(bytes);
    return SS_OK;
  });
}
int ss_pin(ss_cache* c, const int32_t* prefix, int64_t n, int32_t flag) {
  return Guard(c, [&]() -> int {
    c->Pin(std::span<const int32_t>(prefix, n), flag != 0);
    return SS_OK;
  });
}

int ss_has_sequence(const ss_cache* c, int64_t seq) { return c->HasSequence(seq) ? 1 : 0; }

int ss_get_record(ss_cache* c, int64_t seq, ss_record_info* info, int64_t* own_pages,
                  int64_t own_cap) {
  return Guard(c, [&]() -> int {
    const mkv::Record* r = c->GetRecord(seq);
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
    info->window_begin = r->window ? r->window->begin : 0;
    info->window_end = r->window ? r->window->end : 0;
    info->window_expected_writes = r->window ? r->window->expected : 0;
    info->window_received_writes =
        r->window ? r->window->received + static_cast<int64_t>(r->window->dev_received) : 0;
    if (own_pages) {
      if (own_cap < info->num_own_pages) {
        mkv::ThrowStatus(SS_ERR_BUFFER_TOO_SMALL, "own_pages buffer too small");
      }
      std::copy(r->own_pages.begin(), r->own_pages.end(), own_pages);
    }
    return SS_OK;
  });
}

int ss_committed(ss_cache* c, int64_t seq, int64_t* out) {
  return Guard(c, [&]() -> int {
    *out = c->Committed(seq);
    return SS_OK;
  });
}

int ss_read_entry_words(ss_cache* c, int64_t seq, int64_t pos, int32_t layer, uint64_t* out,
                        int64_t out_words) {
  return Guard(c, [&]() -> int {
    if (out_words < c->dim()) mkv::ThrowStatus(SS_ERR_BUFFER_TOO_SMALL, "entry buffer too small");
    c->ReadEntryWords(seq, pos, layer, out);
    return SS_OK;
  });
}

int ss_fill_of(ss_cache* c, int64_t seq, int64_t pos, int32_t layer, int32_t* out) {
  return Guard(c, [&]() -> int {
    *out = c->FillOf(seq, pos, layer);
    return SS_OK;
  });
}

int64_t ss_free_pages(const ss_cache* c) { return c->FreePages(); }
int64_t ss_total_pages(const ss_cache* c) { return c->TotalPages(); }
int ss_cache_config(const ss_cache* c, ss_config* out) {
  *out = c->config();
  return SS_OK;
}
int64_t ss_bytes_per_page(const ss_cache* c) { return c->BytesPerPage(); }
int64_t ss_sequence_count(const ss_cache* c) { return static_cast<int64_t>(c->SequenceCount()); }
int ss_sequence_ids(const ss_cache* c, int64_t* out, int64_t cap, int64_t* n_out) {
  auto ids = c->SequenceIds();
  *n_out = static_cast<int64_t>(ids.size());
  if (static_cast<int64_t>(ids.size()) > cap) return SS_ERR_BUFFER_TOO_SMALL;
  std::copy(ids.begin(), ids.end(), out);
  return SS_OK;
}
int64_t ss_pending_send_count(const ss_cache* c) { return static_cast<int64_t>(c->PendingSendCount()); }
int64_t ss_tree_node_count(const ss_cache* c) { return static_cast<int64_t>(c->Tree().NodeCount()); }
int ss_tree_contains(const ss_cache* c, int64_t seq) { return c->Tree().Contains(seq) ? 1 : 0; }
uint64_t ss_tree_last_touch(const ss_cache* c, int64_t seq) { return c->Tree().LastTouch(seq); }
int ss_tree_sequences_by_lru(const ss_cache* c, int64_t* out, int64_t cap, int64_t* n_out) {
  auto ids = c->Tree().SequencesByLru();
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

// ---------------------------------------------------------------------------
// Device entry points
// ---------------------------------------------------------------------------
int ss_device(const ss_cache* c) { return c->device(); }

int ss_attach_peer(ss_cache* c, int32_t dest, ss_cache* peer) {
  return Guard(c, [&]() -> int {
    c->AttachPeer(dest, peer);
    return SS_OK;
  });
}

int ss_export_ipc(ss_cache* c, ss_ipc_handle* out) {
  return Guard(c, [&]() -> int {
    c->ExportIpc(out);
    return SS_OK;
  });
}

int ss_import_ipc(ss_cache* c, int32_t dest, const ss_ipc_handle* h) {
  return Guard(c, [&]() -> int {
    c->ImportIpc(dest, h);
    return SS_OK;
  });
}

int ss_peer_info(const ss_cache* c, int32_t dest, int32_t* sys_scope, int32_t* peer_device) {
  return Guard(const_cast<ss_cache*>(c), [&]() -> int {
    c->PeerInfo(dest, sys_scope, peer_device);
    return SS_OK;
  });
}

int ss_detach_peer(ss_cache* c, int32_t dest) {
  return Guard(c, [&]() -> int {
    c->DetachPeer(dest);
    return SS_OK;
  });
}

int ss_attention_async(ss_cache* c, ss_plan* p, int32_t layer, const uint64_t* hin, uint64_t* hout,
                       void* stream) {
  return Guard(c, [&]() -> int {
    c->AttentionAsync(p, layer, hin, hout, S(stream));
    return SS_OK;
  });
}

int ss_direct_send_async(ss_cache* c, int64_t seq, int64_t begin, int64_t end, int32_t dest,
                         const ss_addr* dest_addr, uint64_t tag, int32_t lb, int32_t le,
                         void* stream) {
  return Guard(c, [&]() -> int {
    c->DirectSend(seq, begin, end, dest, ToAddr(dest_addr), tag, lb, le, S(stream));
    return SS_OK;
  });
}

int ss_begin_direct_send(ss_cache* c, int64_t seq, int64_t begin, int64_t end, int32_t dest,
                         const ss_addr* dest_addr, uint64_t tag, ss_plan** plan_out) {
  return Guard(c, [&]() -> int {
    *plan_out = c->BeginDirectSend(seq, begin, end, dest, ToAddr(dest_addr), tag);
    return SS_OK;
  });
}

int ss_launch_direct_send_async(ss_cache* c, ss_plan* p, int32_t lb, int32_t le, void* stream) {
  return Guard(c, [&]() -> int {
    c->LaunchDirectSend(p, lb, le, S(stream));
    return SS_OK;
  });
}

int ss_launch_direct_send_after_async(ss_cache* c, ss_plan* p, int32_t lb, int32_t le, void* event,
                                      void* stream) {
  return Guard(c, [&]() -> int {
    c->LaunchDirectSend(p, lb, le, S(stream), static_cast<cudaEvent_t>(event));
    return SS_OK;
  });
}

int ss_launch_relay_send_async(ss_cache* c, ss_plan* p, int32_t lb, int32_t le, int64_t timeout_ms,
                               void* stream) {
  return Guard(c, [&]() -> int {
    c->LaunchRelaySend(p, lb, le, timeout_ms, S(stream));
    return SS_OK;
  });
}

int ss_set_send_mode(ss_cache* c, int32_t mode, int32_t max_ctas) {
  return Guard(c, [&]() -> int {
    c->SetSendMode(mode, max_ctas);
    return SS_OK;
  });
}

int ss_broadcast_send_async(ss_cache* c, int64_t seq, int64_t begin, int64_t end, int32_t n_dest,
                            const int32_t* dests, const ss_addr* addrs, uint64_t tag, int32_t lb,
                            int32_t le, void* stream) {
  return Guard(c, [&]() -> int {
    if (n_dest < 1 || n_dest > SS_MAX_FANOUT) {
      mkv::Throw(mkv::kInvalidArgument, "n_dest must be 1..SS_MAX_FANOUT");
    }
    std::vector<KVAddr> a;
    for (int32_t d = 0; d < n_dest; ++d) a.push_back(ToAddr(addrs + d));
    c->BroadcastSend(seq, begin, end, n_dest, dests, a.data(), tag, lb, le, S(stream));
    return SS_OK;
  });
}

int ss_gather_range_async(ss_cache* c, int64_t seq, int64_t begin, int64_t end, int32_t layer,
                          uint64_t* out_dev, void* stream) {
  return Guard(c, [&]() -> int {
    c->GatherRange(seq, begin, end, layer, out_dev, S(stream));
    return SS_OK;
  });
}

int ss_gather_range_layers_async(ss_cache* c, int64_t seq, int64_t begin, int64_t end,
                                 int32_t lb, int32_t le, uint64_t* out_dev, void* stream) {
  return Guard(c, [&]() -> int {
    c->GatherRangeLayers(seq, begin, end, lb, le, out_dev, S(stream));
    return SS_OK;
  });
}

int ss_apply_remote_write_async(ss_cache* c, const ss_addr* addr, int32_t layer,
                                const uint64_t* payload_dev, int64_t n_words, uint64_t tag,
                                int32_t* apply_status, void* stream) {
  return Guard(c, [&]() -> int {
    *apply_status =
        c->ApplyRemoteWrite(ToAddr(addr), layer, payload_dev, n_words, true, tag, S(stream));
    return SS_OK;
  });
}

int ss_append_rows_async(ss_cache* c, ss_plan* p, int32_t layer, const void* rows, void* stream) {
  return Guard(c, [&]() -> int {
    c->AppendRows(p, layer, rows, S(stream));
    return SS_OK;
  });
}

int ss_append_rows_layers_async(ss_cache* c, ss_plan* p, int32_t lb, int32_t le, const void* rows,
                                void* stream) {
  return Guard(c, [&]() -> int {
    c->AppendRowsLayers(p, lb, le, rows, S(stream));
    return SS_OK;
  });
}

int ss_append_rows_send_async(ss_cache* c, ss_plan* p, ss_plan* sp, int32_t lb, int32_t le,
                              const void* rows, void* stream) {
  return Guard(c, [&]() -> int {
    c->AppendRowsSend(p, sp, lb, le, rows, S(stream));
    return SS_OK;
  });
}

int ss_begin_decode(ss_cache* c, const int64_t* seqs, const int64_t* ctx_lens, int64_t batch,
                    ss_plan** plan_out) {
  return Guard(c, [&]() -> int {
    *plan_out = c->BeginDecode(seqs, ctx_lens, batch);
    return SS_OK;
  });
}

int ss_paged_decode_attention_async(ss_cache* c, ss_plan* plan, int32_t layer, int32_t hq,
                                    int32_t hkv, int32_t hd, float scale, const void* q, void* out,
                                    void* stream) {
  return Guard(c, [&]() -> int {
    c->DecodeAttention(plan, layer, hq, hkv, hd, scale, q, out, S(stream));
    return SS_OK;
  });
}

int ss_paged_prefill_attention_async(ss_cache* c, int64_t seq, int64_t q_begin, int64_t q_end,
                                     int32_t layer, int32_t hq, int32_t hkv, int32_t hd,
                                     float scale, const void* q, void* out, void* stream) {
  return Guard(c, [&]() -> int {
    c->PrefillAttention(seq, q_begin, q_end, layer, hq, hkv, hd, scale, q, out, S(stream));
    return SS_OK;
  });
}

int ss_pool_layer_ptr(ss_cache* c, int32_t layer, void** dev_ptr) {
  return Guard(c, [&]() -> int {
    if (c->device() < 0) mkv::ThrowStatus(SS_ERR_NO_DEVICE, "pool on a host-only cache");
    if (layer < 0 || layer >= c->layers()) mkv::Throw(mkv::kInvalidArgument, "layer out of range");
    *dev_ptr = c->PoolLayer(layer);
    return SS_OK;
  });
}

int ss_wait_receive_async(ss_cache* c, int64_t seq, int64_t timeout_ms, void* stream) {
  return Guard(c, [&]() -> int {
    c->WaitReceive(seq, timeout_ms, S(stream));
    return SS_OK;
  });
}

int ss_wait_receive_layer_async(ss_cache* c, int64_t seq, int32_t layer, int64_t timeout_ms,
                                void* stream) {
  return Guard(c, [&]() -> int {
    c->WaitReceiveLayer(seq, layer, timeout_ms, S(stream));
    return SS_OK;
  });
}

int ss_copy_counters(const ss_cache* c, int64_t* h2d, int64_t* d2h) {
  *h2d = c->h2d_bytes();
  *d2h = c->d2h_bytes();
  return SS_OK;
}

int64_t ss_kernel_launches(const ss_cache* c) { return c->launches(); }

int ss_synchronize(ss_cache* c) {
  return Guard(c, [&]() -> int {
    c->Synchronize();
    return SS_OK;
  });
}

// ---------------------------------------------------------------------------
// Wire formats (wire.cc, frames.cc)
// ---------------------------------------------------------------------------
int ss_addr_encode(const ss_addr* a, uint8_t* out, int64_t cap, int64_t* len) {
  return Guard(nullptr, [&]() -> int {
    std::vector<uint8_t> b;
    mkv::EncodeAddr(ToAddr(a), &b);
    *len = static_cast<int64_t>(b.size());
    if (*len > cap) return SS_ERR_BUFFER_TOO_SMALL;
    if (!b.empty()) std::memcpy(out, b.data(), b.size());
    return SS_OK;
  });
}

int ss_addr_decode(const uint8_t* data, int64_t size, int64_t* pos, ss_addr* out) {
  return Guard(nullptr, [&]() -> int {
    MKV_CHECK(size >= 0 && *pos >= 0 && *pos <= size, mkv::kInvalidArgument, "bad position");
    size_t p = static_cast<size_t>(*pos);
    const KVAddr a = mkv::DecodeAddr(data, static_cast<size_t>(size), &p);
    const int st = FromAddr(nullptr, a, out);
    if (st == SS_OK) *pos = static_cast<int64_t>(p);
    return st;
  });
}

int ss_addr_to_json(const ss_addr* a, char* out, int64_t cap, int64_t* len) {
  return Guard(nullptr, [&]() -> int {
    const std::string j = mkv::AddrToJson(ToAddr(a));
    *len = static_cast<int64_t>(j.size());
    if (*len + 1 > cap) return SS_ERR_BUFFER_TOO_SMALL;
    std::memcpy(out, j.c_str(), j.size() + 1);
    return SS_OK;
  });
}

int ss_addr_from_json(const char* text, int64_t len, ss_addr* out) {
  return Guard(nullptr, [&]() -> int {
    return FromAddr(nullptr, mkv::AddrFromJson(std::string(text, static_cast<size_t>(len))), out);
  });
}

int64_t ss_frame_write_header_size(int64_t n_ranges) {
  return static_cast<int64_t>(mkv::WriteHeaderSize(static_cast<size_t>(n_ranges)));
}

int ss_frame_encode_ack(uint64_t seq_tag, int32_t layer, int64_t token_begin, int32_t status,
                        uint8_t* out, int64_t cap, int64_t* len) {
  return Guard(nullptr, [&]() -> int {
    const auto b = mkv::EncodeAck(seq_tag, layer, token_begin, static_cast<uint8_t>(status));
    *len = static_cast<int64_t>(b.size());
    if (*len > cap) return SS_ERR_BUFFER_TOO_SMALL;
    std::memcpy(out, b.data(), b.size());
    return SS_OK;
  });
}

int ss_frame_decode(const uint8_t* frame, int64_t size, ss_frame_info* info) {
  return Guard(nullptr, [&]() -> int {
    MKV_CHECK(size >= 0, mkv::kInvalidArgument, "negative frame size");
    const mkv::FrameView f = mkv::DecodeFrameHeader(frame, static_cast<size_t>(size));
    info->type = f.type;
    info->layer = f.layer;
    info->seq_tag = f.seq_tag;
    info->payload_offset = static_cast<int64_t>(f.payload_offset);
    info->payload_bytes = static_cast<int64_t>(f.payload_bytes);
    info->wire_crc = f.wire_crc;
    info->ack_status = f.ack_status;
    info->token_begin = f.token_begin;
    if (f.type == mkv::kFrameWrite) return FromAddr(nullptr, f.addr, &info->addr);
    info->addr.n_ranges = 0;
    return SS_OK;
  });
}

int ss_crc32_async(ss_cache* c, const void* data_dev, int64_t n, uint32_t* crc_dev, void* stream) {
  return Guard(c, [&]() -> int {
    c->Crc32(data_dev, n, crc_dev, S(stream));
    return SS_OK;
  });
}

int ss_encode_write_frame(ss_cache* c, int64_t seq, int64_t begin, int64_t end, int32_t layer,
                          uint64_t seq_tag, const ss_addr* dest_addr, uint8_t* frame, int64_t cap,
                          int64_t* frame_len) {
  return Guard(c, [&]() -> int {
    const KVAddr a = ToAddr(dest_addr);
    *frame_len = static_cast<int64_t>(mkv::WriteHeaderSize(a.ranges.size())) +
                 (end - begin) * c->dim() * 8 + 4;
    *frame_len = c->EncodeWriteFrame(seq, begin, end, layer, seq_tag, a, frame, cap, false, nullptr);
    return SS_OK;
  });
}

int ss_encode_write_frame_async(ss_cache* c, int64_t seq, int64_t begin, int64_t end,
                                int32_t layer, uint64_t seq_tag, const ss_addr* dest_addr,
                                void* frame_dev, int64_t cap, int64_t* frame_len, void* stream) {
  return Guard(c, [&]() -> int {
    const KVAddr a = ToAddr(dest_addr);
    *frame_len = static_cast<int64_t>(mkv::WriteHeaderSize(a.ranges.size())) +
                 (end - begin) * c->dim() * 8 + 4;
    *frame_len = c->EncodeWriteFrame(seq, begin, end, layer, seq_tag, a,
                                     static_cast<uint8_t*>(frame_dev), cap, true, S(stream));
    return SS_OK;
  });
}

int ss_receive_write_frame(ss_cache* c, const uint8_t* frame, int64_t size, uint8_t* ack_out,
                           int32_t* apply_status) {
  return Guard(c, [&]() -> int {
    c->ReceiveWriteFrame(frame, size, ack_out, apply_status);
    return SS_OK;
  });
}

}  // extern "C"
