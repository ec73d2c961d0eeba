/*
 * splitserve_b200.h — C++ drop-in for splitserve::KVCache
 * (/root/reference/proj/core/include/splitserve/kv_cache.h:132-235) over the
 * C ABI in microkv.h (implemented by paper_2412_12488_b200/_lib/libmicrokv.so).
 *
 * Header-only.  It needs the reference's own headers on the include path
 * (splitserve/kv_cache.h and what it includes): every argument and result
 * type is the reference's (TokenRange, KVAddrInfo, BatchEntry, FillState,
 * SequenceRecord, PlanSend, FrameSink, RadixTree::MatchResult, CacheConfig,
 * HashModel, Error), so engine code written against splitserve::KVCache
 * compiles unchanged against splitserve::b200::KVCache — swap the type
 * (a template parameter or a using-declaration) and link libmicrokv.so.
 *
 * Errors: every ABI status is rethrown as splitserve::Error with the same
 * ErrorCode (status = 1 + code, errors.h:14-33); boundary-only statuses
 * (unsupported, buffer too small, CUDA, no device) surface as kInternal with
 * the library's detail string.  The receive path returns ApplyStatus like
 * the reference (kv_cache.h:194).
 *
 * Differences a caller can observe, all at the device boundary:
 *  - ForwardPlan is the facade's own move-only type holding the device plan
 *    (entries/sends live in HBM); next_layer / total_outputs are kept.
 *  - FrameSink receives a PlanSend with seq / range / dest / dest_addr /
 *    user_tag (no PlanSlotRef host pointers: the pages live in HBM).  With
 *    AttachPeer / ImportIpc for the destination rank the rows are stored
 *    device-direct into the peer's pages and the sink is not called.
 *  - GetRecord / ForkSequence / CreateSequence return a snapshot of the
 *    record (valid until the next such call on this cache; tokens and
 *    fold_sums are not copied out).
 *  - Tree() returns a view with the queries RadixTree offers that do not
 *    expose nodes (Contains, LastTouch, SequencesByLru, NodeCount).
 */
#ifndef SPLITSERVE_B200_H_
#define SPLITSERVE_B200_H_

#include <cstdint>
#include <span>
#include <string>
#include <utility>
#include <vector>

#include "microkv.h"
#include "splitserve/errors.h"
#include "splitserve/hash_model.h"
#include "splitserve/kv_cache.h"

namespace splitserve {
namespace b200 {

namespace detail {

inline void Check(const ss_cache* c, int st) {
  if (st == SS_OK) return;
  const std::string msg = c != nullptr ? ss_last_error(c) : ss_status_name(st);
  if (st >= 1 && st <= 18) throw Error(static_cast<ErrorCode>(st - 1), msg);
  throw Error(ErrorCode::kInternal, std::string(ss_status_name(st)) + ": " + msg);
}

// A KVAddrInfo viewed as ss_addr (the ranges copied into `buf`).
inline ss_addr View(const KVAddrInfo& a, std::vector<ss_slot_range>* buf) {
  buf->clear();
  buf->reserve(a.ranges.size());
  for (const auto& r : a.ranges) buf->push_back({r.page_id, r.slot_begin, r.slot_count});
  return ss_addr{a.token_begin, a.token_count, static_cast<int64_t>(buf->size()), buf->data(),
                 static_cast<int64_t>(buf->size())};
}

inline KVAddrInfo FromView(const ss_addr& a) {
  KVAddrInfo out;
  out.token_begin = a.token_begin;
  out.token_count = a.token_count;
  out.ranges.reserve(static_cast<size_t>(a.n_ranges));
  for (int64_t i = 0; i < a.n_ranges; ++i) {
    out.ranges.push_back({a.ranges[i].page_id, a.ranges[i].slot_begin, a.ranges[i].slot_count});
  }
  return out;
}

// Calls an ABI function that fills an ss_addr, growing the range buffer on
// SS_ERR_BUFFER_TOO_SMALL.
template <class F>
KVAddrInfo AddrOut(const ss_cache* c, int64_t first_cap, F&& call) {
  std::vector<ss_slot_range> buf(static_cast<size_t>(first_cap > 0 ? first_cap : 1));
  for (;;) {
    ss_addr out{0, 0, 0, buf.data(), static_cast<int64_t>(buf.size())};
    const int st = call(&out);
    if (st == SS_ERR_BUFFER_TOO_SMALL && out.n_ranges > static_cast<int64_t>(buf.size())) {
      buf.resize(static_cast<size_t>(out.n_ranges));
      continue;
    }
    Check(c, st);
    return FromView(out);
  }
}

}  // namespace detail

/*! \brief The device plan of one BeginForward (kv_cache.h:116-121). */
class ForwardPlan {
 public:
  ForwardPlan() = default;
  explicit ForwardPlan(ss_plan* p) : plan_(p) { Refresh(); }
  ForwardPlan(ForwardPlan&& o) noexcept { *this = std::move(o); }
  ForwardPlan& operator=(ForwardPlan&& o) noexcept {
    if (this != &o) {
      Reset();
      plan_ = std::exchange(o.plan_, nullptr);
      next_layer = o.next_layer;
      total_outputs = o.total_outputs;
    }
    return *this;
  }
  ForwardPlan(const ForwardPlan&) = delete;
  ForwardPlan& operator=(const ForwardPlan&) = delete;
  ~ForwardPlan() { Reset(); }

  int32_t next_layer = 0;
  int64_t total_outputs = 0;
  int64_t num_sends() const { return plan_ ? ss_plan_num_sends(plan_) : 0; }
  ss_plan* native() const { return plan_; }
  void Refresh() {
    if (plan_ != nullptr) {
      next_layer = ss_plan_next_layer(plan_);
      total_outputs = ss_plan_total_outputs(plan_);
    }
  }

 private:
  void Reset() {
    if (plan_ != nullptr) ss_plan_destroy(plan_);
    plan_ = nullptr;
  }
  ss_plan* plan_ = nullptr;
};

/*! \brief Read-only view of the engine's radix tree (radix_tree.h:47-70). */
class TreeView {
 public:
  explicit TreeView(const ss_cache* c) : c_(c) {}
  bool Contains(SeqId seq) const { return ss_tree_contains(c_, seq) != 0; }
  uint64_t LastTouch(SeqId seq) const { return ss_tree_last_touch(c_, seq); }
  size_t NodeCount() const { return static_cast<size_t>(ss_tree_node_count(c_)); }
  std::vector<SeqId> SequencesByLru() const {
    std::vector<int64_t> out(64);
    int64_t n = 0;
    for (;;) {
      const int st = ss_tree_sequences_by_lru(c_, out.data(), static_cast<int64_t>(out.size()), &n);
      if (st == SS_ERR_BUFFER_TOO_SMALL) {
        out.resize(static_cast<size_t>(n));
        continue;
      }
      detail::Check(c_, st);
      return std::vector<SeqId>(out.begin(), out.begin() + n);
    }
  }

 private:
  const ss_cache* c_;
};

/*!
 * \brief splitserve::KVCache with the KV pool, fill states, page tables and
 *        receive windows in one GPU's HBM.  Same members, same semantics.
 */
class KVCache {
 public:
  using PrepRecvResult = ::splitserve::KVCache::PrepRecvResult;
  using ApplyStatus = ::splitserve::KVCache::ApplyStatus;

  /*! \brief kv_cache.h:134; `device` = CUDA ordinal, `rank` = this engine's rank. */
  KVCache(CacheConfig cache_config, const HashModel* model, int device = 0, Rank rank = 0)
      : cache_config_(cache_config) {
    const ModelConfig& m = model->config();
    ss_config cfg{cache_config.num_pages, cache_config.page_size, m.layers, m.dim, m.vocab,
                  m.hash_seed, device, rank};
    detail::Check(nullptr, ss_cache_create(&cfg, &c_));
    layers_ = m.layers;
    dim_ = m.dim;
  }
  KVCache(const KVCache&) = delete;
  KVCache& operator=(const KVCache&) = delete;
  ~KVCache() {
    if (c_ != nullptr) ss_cache_destroy(c_);
  }

  // ---- Declaration stage (kv_cache.h:140-171) ------------------------------
  int64_t MatchPrefix(std::span<const Token> tokens) { return MatchPrefixSeq(tokens).match_len; }
  RadixTree::MatchResult MatchPrefixSeq(std::span<const Token> tokens) {
    RadixTree::MatchResult r;
    int64_t seq = -1;
    detail::Check(c_, ss_match_prefix(c_, tokens.data(), static_cast<int64_t>(tokens.size()),
                                      &r.match_len, &seq));
    r.seq = seq;
    return r;
  }
  PrepRecvResult PrepRecv(SeqId seq_id, TokenList tokens, int64_t end) {
    PrepRecvResult res;
    const int64_t cap = static_cast<int64_t>(tokens.size()) / cache_config_.page_size + 2;
    res.addr = detail::AddrOut(c_, cap, [&](ss_addr* out) {
      return ss_prep_recv(c_, seq_id, tokens.data(), static_cast<int64_t>(tokens.size()), end,
                          &res.match_len, out);
    });
    return res;
  }
  SequenceRecord* ForkSequence(SeqId parent, SeqId child, int64_t fork_len,
                               TokenList child_tokens = {}) {
    detail::Check(c_, ss_fork_sequence(c_, parent, child, fork_len, child_tokens.data(),
                                       static_cast<int64_t>(child_tokens.size())));
    return Snapshot(child);
  }
  SequenceRecord* CreateSequence(SeqId seq_id, TokenList tokens) {
    detail::Check(c_, ss_create_sequence(c_, seq_id, tokens.data(),
                                         static_cast<int64_t>(tokens.size())));
    return Snapshot(seq_id);
  }
  void MarkSend(SeqId seq, TokenRange range, Rank dest, KVAddrInfo dest_addr,
                uint64_t user_tag = 0) {
    std::vector<ss_slot_range> b;
    const ss_addr v = detail::View(dest_addr, &b);
    detail::Check(c_, ss_mark_send(c_, seq, range.begin, range.end, dest, &v, user_tag));
  }
  void EnsureAllocated(SeqId seq, int64_t upto) {
    detail::Check(c_, ss_ensure_allocated(c_, seq, upto));
  }
  void AppendToken(SeqId seq, Token t) { detail::Check(c_, ss_append_token(c_, seq, t)); }
  ForwardPlan BeginForward(const std::vector<BatchEntry>& batch) {
    std::vector<ss_batch_entry> b;
    b.reserve(batch.size());
    for (const auto& e : batch) b.push_back({e.seq, e.range.begin, e.range.end, e.is_decode ? 1 : 0, 0});
    ss_plan* p = nullptr;
    detail::Check(c_, ss_begin_forward(c_, b.data(), static_cast<int64_t>(b.size()), &p));
    return ForwardPlan(p);
  }

  // ---- Computation stage (kv_cache.h:173-189) ------------------------------
  std::vector<uint64_t> Attention(int32_t layer, ForwardPlan* plan,
                                  std::span<const uint64_t> hidden_in, const FrameSink& sink) {
    std::vector<uint64_t> out(hidden_in.size());
    SinkCtx ctx{&sink};
    detail::Check(c_, ss_attention(c_, plan->native(), layer, hidden_in.data(), out.data(),
                                   static_cast<int64_t>(hidden_in.size()),
                                   sink ? &KVCache::SinkTrampoline : nullptr, &ctx));
    plan->Refresh();
    return out;
  }
  std::vector<uint64_t> GatherRange(SeqId seq, TokenRange range, int32_t layer) {
    std::vector<uint64_t> out(static_cast<size_t>(range.size()) * dim_);
    detail::Check(c_, ss_gather_range(c_, seq, range.begin, range.end, layer, out.data(),
                                      static_cast<int64_t>(out.size())));
    return out;
  }
  KVAddrInfo BuildAddr(SeqId seq, TokenRange range) {
    return detail::AddrOut(c_, range.size() / cache_config_.page_size + 2, [&](ss_addr* out) {
      return ss_build_addr(c_, seq, range.begin, range.end, out);
    });
  }

  // ---- Transfer agent (kv_cache.h:191-199) ---------------------------------
  ApplyStatus ApplyRemoteWrite(const KVAddrInfo& addr, int32_t layer,
                               std::span<const uint64_t> payload, uint64_t tag) {
    std::vector<ss_slot_range> b;
    const ss_addr v = detail::View(addr, &b);
    int32_t st = 0;
    detail::Check(c_, ss_apply_remote_write(c_, &v, layer, payload.data(),
                                            static_cast<int64_t>(payload.size()), tag, &st));
    return static_cast<ApplyStatus>(st);
  }
  std::vector<SeqId> DrainReceiveCompletions() {
    // The ABI hands out at most `cap` per call and keeps the rest queued.
    std::vector<SeqId> done;
    int64_t buf[64];
    int64_t n = 0;
    do {
      detail::Check(c_, ss_drain_receive_completions(c_, buf, 64, &n));
      done.insert(done.end(), buf, buf + n);
    } while (n == 64);
    return done;
  }

  // ---- Lifecycle (kv_cache.h:201-217) --------------------------------------
  void SetFinished(SeqId seq, bool finished) {
    detail::Check(c_, ss_set_finished(c_, seq, finished ? 1 : 0));
  }
  void CommitToTree(SeqId seq) { detail::Check(c_, ss_commit_to_tree(c_, seq)); }
  void FreeSequence(SeqId seq) { detail::Check(c_, ss_free_sequence(c_, seq)); }
  int64_t Evict(int64_t bytes_needed) {
    int64_t freed = 0;
    detail::Check(c_, ss_evict(c_, bytes_needed, &freed));
    return freed;
  }
  void Pin(std::span<const Token> prefix, bool flag) {
    detail::Check(c_, ss_pin(c_, prefix.data(), static_cast<int64_t>(prefix.size()), flag ? 1 : 0));
  }

  // ---- Queries (kv_cache.h:219-235) ----------------------------------------
  bool HasSequence(SeqId seq) const { return ss_has_sequence(c_, seq) != 0; }
  const SequenceRecord* GetRecord(SeqId seq) const {
    return const_cast<KVCache*>(this)->Snapshot(seq);
  }
  int64_t Committed(SeqId seq) {
    int64_t v = 0;
    detail::Check(c_, ss_committed(c_, seq, &v));
    return v;
  }
  std::vector<uint64_t> ReadEntryWords(SeqId seq, int64_t pos, int32_t layer) {
    std::vector<uint64_t> out(static_cast<size_t>(dim_));
    detail::Check(c_, ss_read_entry_words(c_, seq, pos, layer, out.data(), dim_));
    return out;
  }
  FillState FillOf(SeqId seq, int64_t pos, int32_t layer) {
    int32_t v = 0;
    detail::Check(c_, ss_fill_of(c_, seq, pos, layer, &v));
    return static_cast<FillState>(v);
  }
  int64_t FreePages() const { return ss_free_pages(c_); }
  int64_t TotalPages() const { return ss_total_pages(c_); }
  int64_t BytesPerPage() const { return ss_bytes_per_page(c_); }
  size_t SequenceCount() const { return static_cast<size_t>(ss_sequence_count(c_)); }
  std::vector<SeqId> SequenceIds() const {
    std::vector<int64_t> out(static_cast<size_t>(ss_sequence_count(c_)) + 1);
    int64_t n = 0;
    detail::Check(c_, ss_sequence_ids(c_, out.data(), static_cast<int64_t>(out.size()), &n));
    return std::vector<SeqId>(out.begin(), out.begin() + n);
  }
  size_t PendingSendCount() const { return static_cast<size_t>(ss_pending_send_count(c_)); }
  TreeView Tree() const { return TreeView(c_); }
  const CacheConfig& cache_config() const { return cache_config_; }

  // ---- B200 additions: peers for device-direct remote_send -----------------
  void AttachPeer(Rank dest, KVCache& peer) { detail::Check(c_, ss_attach_peer(c_, dest, peer.c_)); }
  ss_ipc_handle ExportIpc() {
    ss_ipc_handle h{};
    detail::Check(c_, ss_export_ipc(c_, &h));
    return h;
  }
  void ImportIpc(Rank dest, const ss_ipc_handle& h) { detail::Check(c_, ss_import_ipc(c_, dest, &h)); }
  void DetachPeer(Rank dest) { detail::Check(c_, ss_detach_peer(c_, dest)); }
  /*! \brief Waits for the cache's device work; raises asynchronous errors. */
  void Synchronize() { detail::Check(c_, ss_synchronize(c_)); }
  ss_cache* native() const { return c_; }

 private:
  struct SinkCtx {
    const FrameSink* sink;
  };
  static void SinkTrampoline(void* user, int32_t layer, int64_t seq, int64_t rb, int64_t re,
                             int32_t dest, const ss_addr* addr, uint64_t tag,
                             const uint64_t* payload, int64_t n_words) {
    const auto* ctx = static_cast<const SinkCtx*>(user);
    PlanSend send;
    send.seq = seq;
    send.range = TokenRange{rb, re};
    send.dest = dest;
    send.dest_addr = detail::FromView(*addr);
    send.user_tag = tag;
    (*ctx->sink)(layer, send, std::vector<uint64_t>(payload, payload + n_words));
  }

  SequenceRecord* Snapshot(SeqId seq) {
    ss_record_info info{};
    std::vector<int64_t> pages(16);
    for (;;) {
      const int st = ss_get_record(c_, seq, &info, pages.data(), static_cast<int64_t>(pages.size()));
      if (st == SS_ERR_BUFFER_TOO_SMALL && info.num_own_pages > static_cast<int64_t>(pages.size())) {
        pages.resize(static_cast<size_t>(info.num_own_pages));
        continue;
      }
      detail::Check(c_, st);
      break;
    }
    snap_ = SequenceRecord{};
    snap_.id = info.id;
    snap_.parent = info.parent;
    snap_.fork_len = info.fork_len;
    snap_.refcount = info.refcount;
    snap_.own_pages.assign(pages.begin(), pages.begin() + info.num_own_pages);
    snap_.alloc_len = info.alloc_len;
    snap_.committed_hint = info.committed_hint;
    snap_.finished = info.finished != 0;
    snap_.fold_frontier = info.fold_frontier;
    snap_.prefix_digest = info.prefix_digest;
    snap_.digest_len = info.digest_len;
    if (info.has_window) {
      SequenceRecord::ReceiveWindow w;
      w.range = TokenRange{info.window_begin, info.window_end};
      w.expected_writes = info.window_expected_writes;
      w.received_writes = info.window_received_writes;
      w.complete = info.window_complete != 0;
      snap_.window = std::move(w);
    }
    return &snap_;
  }

  ss_cache* c_ = nullptr;
  CacheConfig cache_config_;
  int32_t layers_ = 0, dim_ = 0;
  SequenceRecord snap_;
};

}  // namespace b200
}  // namespace splitserve

#endif  // SPLITSERVE_B200_H_
