// cache.h — one engine's paged KV cache: host bookkeeping + HBM state.
//
// The host side keeps the reference's bookkeeping semantics bit-for-bit
// (/root/reference/proj/core/src/kv_cache.cc): LIFO page free list,
// fork-relative paging, radix-tree context cache, receive windows, pending
// sends, plans.  Every KV byte, fill state and receive counter lives in HBM
// and is only touched by kernels (kernels.cuh); there is no host copy of
// the pool and no CPU data path.
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <deque>
#include <map>
#include <memory>
#include <mutex>
#include <optional>
#include <set>
#include <span>
#include <stdexcept>
#include <string>
#include <tuple>
#include <vector>

#include "../../include/microkv.h"
#include "kernels.cuh"
#include "radix_tree.h"

namespace mkv {

// splitserve::ErrorCode order (errors.h:14-33); status = 1 + code.
enum ErrorCode : int {
  kOutOfPages = 0,
  kDuplicateSequence,
  kUnknownSequence,
  kForkBeyondCommitted,
  kAddrMismatch,
  kMissingKV,
  kLayerOrderViolation,
  kCannotEvict,
  kChecksumMismatch,
  kUnknownAddress,
  kPeerUnreachable,
  kNoEngines,
  kRoleMissing,
  kNoOwner,
  kUnknownStrategy,
  kInvalidArgument,
  kAborted,
  kInternal,
};

const char* StatusName(int status);

class Error : public std::exception {
 public:
  Error(int status, std::string msg) : status_(status), msg_(std::move(msg)) {}
  int status() const { return status_; }
  const char* what() const noexcept override { return msg_.c_str(); }

 private:
  int status_;
  std::string msg_;
};

[[noreturn]] void Throw(int code, const std::string& detail);
[[noreturn]] void ThrowStatus(int status, const std::string& detail);
#define MKV_CHECK(cond, code, detail) \
  do {                                \
    if (!(cond)) ::mkv::Throw(code, detail); \
  } while (0)
#define MKV_ICHECK(cond, detail) MKV_CHECK(cond, ::mkv::kInternal, detail)
void CudaCheck(cudaError_t e, const char* what);

struct SlotRange {
  int64_t page_id = 0;
  int32_t slot_begin = 0;
  int32_t slot_count = 0;
};

struct KVAddr {
  std::vector<SlotRange> ranges;
  int64_t token_begin = 0;
  int64_t token_count = 0;
  void Validate() const;                         // kv_addr.cc:16-30
  KVAddr Slice(int64_t begin, int64_t end) const;  // kv_addr.cc:32-51
};

struct Window {
  int64_t begin = 0, end = 0;
  int64_t expected = 0;      // (e - m) * L slot writes
  int64_t received = 0;      // host-path writes (ApplyRemoteWrite)
  std::vector<int64_t> received_layer;  // host-path writes per layer
  uint64_t dev_received = 0; // device-direct writes last read from HBM
  bool complete = false;
  std::set<std::tuple<uint64_t, int32_t, int64_t>> applied;  // (tag, layer, token_begin)
  int32_t dev_id = -1;       // row in win_received / win_layer_rows
};

struct Record {
  SeqId id = -1;
  std::vector<Token> tokens;
  SeqId parent = -1;
  int64_t fork_len = 0;
  int32_t refcount = 0;
  std::vector<int64_t> own_pages;
  int64_t alloc_len = 0;
  int64_t committed_hint = 0;
  bool finished = false;
  int64_t fold_frontier = 0;
  uint64_t prefix_digest = 0;
  int64_t digest_len = 0;
  std::optional<Window> window;
  // Resolved slot index (page * P + slot) of every position < alloc_len:
  // the host copy of the page table (the reference walks parents per
  // position, kv_cache.cc:67-77; a child copies its parent's resolved
  // prefix at fork time, which is equivalent since shared prefixes are
  // immutable while referenced).
  std::vector<int32_t> slots;
  // The same page table in HBM (device-resident, grown with the host copy):
  // every kernel that walks a sequence's positions reads it directly.
  int32_t* d_slots = nullptr;
  int64_t d_cap = 0;
  int32_t fold_row = -1;     // row of this sequence in the device fold-sum table
  int64_t touched_end = 0;   // positions >= this were never written by a forward pass
};

struct PlanEntry {
  SeqId seq = -1;
  bool is_decode = false;
  int64_t begin = 0, end = 0;
  int64_t fold_from = 0;
  std::vector<uint64_t> digests;  // prefix digests for [begin, end)
  std::vector<Token> tokens;
  std::vector<int32_t> slots;     // [fold_from, end)
};

struct PlanSend {
  SeqId seq = -1;
  int64_t begin = 0, end = 0;
  Rank dest = -1;
  KVAddr dest_addr;
  uint64_t user_tag = 0;
  std::vector<int32_t> src_slots;  // [begin, end)
};

struct DevBlock {
  void* ptr = nullptr;
  size_t bytes = 0;
};

}  // namespace mkv

struct ss_plan {
  ss_cache* owner = nullptr;
  std::vector<mkv::PlanEntry> entries;
  std::vector<mkv::PlanSend> sends;
  int32_t next_layer = 0;
  int64_t total_outputs = 0;
  // Device copy of the plan, built on first use (BeginForward's "plan once
  // for all layers", kv_cache.h:8-9).
  bool on_device = false;
  mkv::DevBlock dev;
  int64_t n_fold = 0;
  int32_t* d_fold_slots = nullptr;
  int32_t* d_out_slots = nullptr;
  uint64_t* d_digests = nullptr;
  mkv::FoldEntry* d_entries = nullptr;
  uint64_t* d_F = nullptr;
  uint64_t* d_hidden_in = nullptr;
  uint64_t* d_hidden_out = nullptr;
  struct DevSend {
    int32_t* src_slots = nullptr;
    int32_t* dst_slots = nullptr;
    int64_t* range_page = nullptr;
    int32_t* range_begin = nullptr;
    int32_t* range_count = nullptr;
    int32_t* verdict = nullptr;
    uint64_t* staging = nullptr;  // gathered payload for host sinks
    int64_t n_ranges = 0;         // destination ranges validated (0: malformed address)
    // Set by the first launch's validation (a grid or inline): later launches
    // of the plan check the receiver window's generation instead.
    int32_t validated_gen = 0;
    cudaEvent_t validated_ev = nullptr;  // recorded behind that validation
  };
  std::vector<DevSend> dsend;
  bool is_direct_send = false;
  cudaEvent_t upload_ev = nullptr;  // direct-send plans: recorded after the row maps' upload
  // Copy-engine sends: maximal runs of rows consecutive in both the source
  // and the destination slot space (built on the first copy-engine launch).
  struct Run {
    int32_t src, dst, n;
  };
  std::vector<Run> ce_runs;
  int32_t ce_gen = 0;  // launch generation of the plan's (one) copy-engine validation
  // Decode-attention plan (ss_begin_decode): context slot map in CSR form.
  bool is_decode_plan = false;
  int64_t batch = 0;
  int64_t max_ctx = 0;
  int32_t* d_ctx_slots = nullptr;
  int64_t* d_ctx_off = nullptr;
  int32_t* d_ctx_len = nullptr;
  std::vector<int32_t> ctx_lens;
  float* d_partial = nullptr;       // per-piece partial outputs (stream-K)
  float* d_partial_ml = nullptr;    // per-piece (max, sum) per head
  int64_t* d_seg_start = nullptr;   // tile prefix sums over (batch, kv head)
  uint32_t* d_seg_count = nullptr;  // fused-combine arrival counter per segment
  int32_t* d_cta_seg = nullptr;     // first segment of each CTA's tile range
  int64_t total_tiles = 0;
  int32_t decode_hkv = 0, decode_hq = 0, decode_hd = 0;
  int32_t decode_grid = 0;
  // Page-chunk decode (decode_pages.cu): runs of <= 16 consecutive slots
  // {slot0, tok0, n, b} in batch order, built by BeginDecode; uploaded with
  // the per-context piece tables on first use.
  std::vector<int32_t> chunks;  // 4 ints per chunk
  bool pages_ready = false, pages_split = false;
  int32_t pages_grid = 0;
  int32_t* d_chunks = nullptr;  // int4 per chunk, then piece_first[batch], piece_count[batch]
  int32_t* d_piece_first = nullptr;
  int32_t* d_piece_count = nullptr;
  float* d_pages_part = nullptr;
  float* d_pages_ml = nullptr;
};

namespace mkv {

// Destination surface of a peer engine (in-process or CUDA-IPC mapped).
struct PeerTarget {
  uint64_t* pool = nullptr;
  uint8_t* fill = nullptr;
  uint8_t* expecting = nullptr;
  int32_t* page_window = nullptr;
  unsigned long long* win_received = nullptr;
  uint32_t* win_layer_rows = nullptr;
  const unsigned long long* win_gen = nullptr;  // open-generation per window id
  int64_t num_pages = 0;
  int32_t P = 0, L = 0, W = 0;
  int32_t device = -1;
  bool ipc = false;
  std::vector<void*> ipc_ptrs;
  const ss_cache* local = nullptr;  // in-process peer: its window-ready event orders our sends
};

}  // namespace mkv

struct ss_cache {
  explicit ss_cache(const ss_config& cfg);
  ~ss_cache();

  using SeqId = mkv::SeqId;
  using Token = mkv::Token;
  using Rank = mkv::Rank;

  // Declaration stage.
  mkv::RadixTree::MatchResult MatchPrefixSeq(std::span<const Token> tokens);
  int64_t PrepRecv(SeqId seq, std::vector<Token> tokens, int64_t end, mkv::KVAddr* addr,
                   int64_t ranges_cap);
  mkv::Record* ForkSequence(SeqId parent, SeqId child, int64_t fork_len, std::vector<Token> toks);
  mkv::Record* CreateSequence(SeqId seq, std::vector<Token> tokens);
  void MarkSend(SeqId seq, int64_t begin, int64_t end, Rank dest, mkv::KVAddr addr, uint64_t tag);
  void EnsureAllocated(SeqId seq, int64_t upto);
  void AppendToken(SeqId seq, Token t);
  ss_plan* BeginForward(const ss_batch_entry* batch, int64_t n);

  // Computation stage.
  void Attention(ss_plan* plan, int32_t layer, const uint64_t* hidden_in_host,
                 uint64_t* hidden_out_host, int64_t n, ss_frame_sink sink, void* user);
  void AttentionAsync(ss_plan* plan, int32_t layer, const uint64_t* hidden_in_dev,
                      uint64_t* hidden_out_dev, cudaStream_t s);
  void GatherRange(SeqId seq, int64_t begin, int64_t end, int32_t layer, uint64_t* out_dev,
                   cudaStream_t s);
  void GatherRangeLayers(SeqId seq, int64_t begin, int64_t end, int32_t layer_begin,
                         int32_t layer_end, uint64_t* out_dev, cudaStream_t s);
  mkv::KVAddr BuildAddr(SeqId seq, int64_t begin, int64_t end);
  void AppendRows(ss_plan* plan, int32_t layer, const void* rows_dev, cudaStream_t s);
  void AppendRowsSend(ss_plan* fwd, ss_plan* send, int32_t lb, int32_t le, const void* rows,
                      cudaStream_t s);
  void AppendRowsLayers(ss_plan* plan, int32_t layer_begin, int32_t layer_end, const void* rows_dev,
                        cudaStream_t s);

  // Transfer agent.
  // agent = the transfer agent's call (possibly another thread): the
  // receive stream, ordered after the receive windows only.
  int ApplyRemoteWrite(const mkv::KVAddr& addr, int32_t layer, const uint64_t* payload,
                       int64_t n_words, bool payload_on_device, uint64_t tag, cudaStream_t s,
                       bool agent = false);
  std::vector<SeqId> DrainReceiveCompletions();
  void DirectSend(SeqId seq, int64_t begin, int64_t end, Rank dest, const mkv::KVAddr& addr,
                  uint64_t tag, int32_t layer_begin, int32_t layer_end, cudaStream_t s);
  ss_plan* BeginDirectSend(SeqId seq, int64_t begin, int64_t end, Rank dest,
                           const mkv::KVAddr& addr, uint64_t tag);
  // `after` (optional): the event of the producing layer's writes; the
  // validation is enqueued before the stream waits for it, the copy after.
  void LaunchDirectSend(ss_plan* plan, int32_t layer_begin, int32_t layer_end, cudaStream_t s,
                        cudaEvent_t after = nullptr);
  // Relay: forward layers [lb, le) of rows this engine is still receiving
  // to the plan's destination, each layer behind a device-side wait for
  // that layer's receive counter (a relay chain of prefix migration).
  void LaunchRelaySend(ss_plan* plan, int32_t layer_begin, int32_t layer_end, int64_t timeout_ms,
                       cudaStream_t s);
  void BroadcastSend(SeqId seq, int64_t begin, int64_t end, int32_t n_dest, const Rank* dests,
                     const mkv::KVAddr* addrs, uint64_t tag, int32_t layer_begin,
                     int32_t layer_end, cudaStream_t s);

  // Lifecycle.
  void SetFinished(SeqId seq, bool f) { MustGet(seq)->finished = f; }
  void CommitToTree(SeqId seq);
  void FreeSequence(SeqId seq);
  int64_t Evict(int64_t bytes_needed);
  void Pin(std::span<const Token> prefix, bool flag) { tree_.Pin(prefix, flag); }

  // Queries.
  bool HasSequence(SeqId seq) const { return records_.count(seq) > 0; }
  const mkv::Record* GetRecord(SeqId seq) const { return MustGet(seq); }
  int64_t Committed(SeqId seq);
  void ReadEntryWords(SeqId seq, int64_t pos, int32_t layer, uint64_t* out);
  int32_t FillOf(SeqId seq, int64_t pos, int32_t layer);
  int64_t FreePages() const { return static_cast<int64_t>(free_pages_.size()); }
  int64_t TotalPages() const { return num_pages_; }
  int64_t BytesPerPage() const { return static_cast<int64_t>(P_) * L_ * W_ * 8; }
  size_t SequenceCount() const { return records_.size(); }
  std::vector<SeqId> SequenceIds() const;
  size_t PendingSendCount() const { return pending_sends_.size(); }
  const mkv::RadixTree& Tree() const { return tree_; }

  // Device plumbing.
  void AttachPeer(Rank dest, ss_cache* peer);
  void ExportIpc(ss_ipc_handle* out);
  void ImportIpc(Rank dest, const ss_ipc_handle* h);
  void DetachPeer(Rank dest);
  void SetSendMode(int32_t mode, int32_t max_ctas);
  void PeerInfo(Rank dest, int32_t* sys_scope, int32_t* peer_device) const {
    const mkv::PeerTarget& t = PeerFor(dest);
    if (sys_scope) *sys_scope = (t.device != device_ || force_sys_scope_) ? 1 : 0;
    if (peer_device) *peer_device = t.device;
  }
  ss_plan* BeginDecode(const int64_t* seqs, const int64_t* ctx_lens, int64_t batch);
  void PrefillAttention(int64_t seq, int64_t q_begin, int64_t q_end, int32_t layer, int32_t hq,
                        int32_t hkv, int32_t hd, float scale, const void* q, void* out,
                        cudaStream_t s);
  void DecodeAttentionPages(ss_plan* plan, int32_t layer, int32_t hq, int32_t hkv, float scale,
                            const void* q, void* out, cudaStream_t s);
  void DecodeAttention(ss_plan* plan, int32_t layer, int32_t hq, int32_t hkv, int32_t hd,
                       float scale, const void* q, void* out, cudaStream_t s);
  // Wire formats (frames.cc): CRC-32 of device bytes; a KV write frame of
  // GatherRange(seq, [begin, end), layer) encoded byte-identical to the
  // reference's EncodeWriteFrame with gather + CRC on the device; the
  // transfer agent's receive step for one frame (tcp_fabric.cc:144-168).
  void Crc32(const void* data_dev, int64_t n, uint32_t* crc_dev, cudaStream_t s);
  int64_t EncodeWriteFrame(SeqId seq, int64_t begin, int64_t end, int32_t layer, uint64_t tag,
                           const mkv::KVAddr& dest, uint8_t* frame, int64_t cap,
                           bool frame_on_device, cudaStream_t s);
  void ReceiveWriteFrame(const uint8_t* frame, int64_t size, uint8_t* ack_out,
                         int32_t* apply_status);
  void DestroyPlan(ss_plan* plan);
  void FreePlanDevice(ss_plan* plan);
  void Synchronize();
  void WaitReceive(SeqId seq, int64_t timeout_ms, cudaStream_t s);
  void WaitReceiveLayer(SeqId seq, int32_t layer, int64_t timeout_ms, cudaStream_t s);
  int64_t h2d_bytes() const { return h2d_bytes_; }
  int64_t d2h_bytes() const { return d2h_bytes_; }
  uint64_t* PoolLayer(int32_t layer) const;
  bool has_device() const { return device_ >= 0; }
  int32_t dim() const { return W_; }
  int32_t layers() const { return L_; }
  int32_t page_size() const { return P_; }
  ss_config config() const {
    ss_config c{};
    c.num_pages = num_pages_;
    c.page_size = P_;
    c.layers = L_;
    c.dim = W_;
    c.vocab = vocab_;
    c.hash_seed = hash_seed_;
    c.device = device_;
    c.rank = rank_;
    return c;
  }
  int device() const { return device_; }
  int64_t launches() const { return launches_; }
  // Count n kernel launches just enqueued and surface a failed launch
  // (bad configuration, missing image) as SS_ERR_CUDA right away.
  void CountLaunches(int64_t n);

  // Hash model scalars.
  uint64_t InitialPrefixDigest() const;
  uint64_t Embed(Token t, int64_t pos) const;
  Token SampleToken(uint64_t h) const;

  std::string last_error;
  std::deque<SeqId> drained;  // completions not yet handed to the caller

 private:
  mkv::Record* MustGet(SeqId seq);
  const mkv::Record* MustGet(SeqId seq) const;
  int32_t Resolve(const mkv::Record* rec, int64_t pos) const;
  int64_t PagesNeeded(const mkv::Record* rec, int64_t upto) const;
  void AdvanceCommitted(mkv::Record* rec, int64_t known_full_until = -1);
  void TouchLru(mkv::Record* rec);
  void RequireDevice(const char* what) const;
  void Sync();                       // internal stream
  void H2D(void* dst, const void* src, size_t bytes, cudaStream_t s, const char* what);
  void D2H(void* dst, const void* src, size_t bytes, cudaStream_t s, const char* what);
  void OrderAfterUser();             // internal stream waits for async work
  void OrderUser(cudaStream_t s);    // user stream waits for internal work
  void BeginInternal();              // internal work that needs no wait for user streams
  int32_t NextLaunchGen();
  void NoteUser(cudaStream_t s);
  void SyncUserStreams();            // host waits for every caller stream's noted work
  void OrderLaunch(cudaStream_t s);  // user-stream launch: s after internal work
  mkv::DevBlock DevAlloc(size_t bytes, cudaStream_t s);
  void DevFree(mkv::DevBlock& b, cudaStream_t s);
  void PlanToDevice(ss_plan* plan);
  // Device-checked "every slot is non-Empty on `layer`" for positions of a
  // sequence not provably full on the host; throws MissingKV.
  bool CoveredByLivePlan(SeqId seq, int64_t begin, int64_t end) const;
  void CheckFilled(const mkv::Record* rec, int64_t begin, int64_t end, int32_t layer,
                   const char* what, const ss_plan* plan);
  int64_t DeviceFirstNonFull(const mkv::Record* rec, int64_t from, int64_t to);
  const mkv::PeerTarget& PeerFor(Rank dest) const;
  void LaunchRemote(const mkv::PeerTarget& peer, const int32_t* d_src_slots,
                    const int32_t* d_dst_slots, const int64_t* d_rpage, const int32_t* d_rbegin,
                    const int32_t* d_rcount, int64_t n_ranges, int32_t* d_verdict, int64_t n_rows,
                    int32_t layer_begin, int32_t layer_end, cudaStream_t s,
                    cudaEvent_t after = nullptr, ss_plan::DevSend* ds = nullptr);
  void LaunchDirectSendCE(ss_plan* plan, const mkv::PeerTarget& peer, mkv::Record* rec,
                          int32_t lb, int32_t le, cudaStream_t s, cudaEvent_t after);
  void ExpandAddr(const mkv::KVAddr& a, std::vector<int32_t>* slots, std::vector<int64_t>* rp,
                  std::vector<int32_t>* rb, std::vector<int32_t>* rc) const;
  void OpenDeviceWindow(mkv::Record* rec, int64_t m, int64_t e);
  void CloseDeviceWindow(mkv::Record* rec);
  void SyncDeviceTable(mkv::Record* rec, int64_t old_len);
  void PollDeviceWindows();
  void ThrowIfDeviceStatus();

  struct PendingSend {
    SeqId seq;
    int64_t begin, end;
    Rank dest;
    mkv::KVAddr addr;
    uint64_t tag;
  };

  // Geometry.
  int64_t num_pages_;
  int32_t P_, L_, W_, vocab_;
  int32_t page_shift_ = 0;  // log2(P_)
  uint64_t hash_seed_, seed_state_;
  int device_;
  int32_t rank_;
  int num_sms_ = 148;
  bool force_sys_scope_ = false;  // MICROKV_FORCE_SYS_SCOPE=1 (test hook)
  int32_t send_mode_ = SS_SEND_KERNEL;  // ss_set_send_mode
  int32_t send_ctas_ = 0;               // copy-kernel grid cap of sends (0 = none)
  cudaStream_t fused_vstream_ = nullptr;  // AppendRowsSend's validation stream
  cudaEvent_t fused_vev_ = nullptr;
  cudaStream_t verdict_stream_ = nullptr;  // copy-engine sends: validation off the data stream
  cudaEvent_t verdict_ev_ = nullptr;
  cudaStream_t ce_stream_ = nullptr;       // copy-engine sends: the batched copies
  cudaEvent_t ce_ev_ = nullptr;
  std::atomic<int64_t> launches_{0};
  std::atomic<int32_t> launch_gen_{0};  // validated-launch generations (NextLaunchGen)

  // Host bookkeeping.
  std::vector<int64_t> free_pages_;
  std::vector<SeqId> page_owner_;
  std::vector<uint8_t> expecting_;  // [pages][P] (host copy of the reservation bits)
  std::map<SeqId, std::unique_ptr<mkv::Record>> records_;
  std::deque<PendingSend> pending_sends_;
  mkv::RadixTree tree_;
  std::mutex recv_mu_;
  std::vector<SeqId> completed_windows_;
  std::vector<int32_t> free_window_ids_;
  std::vector<int32_t> free_fold_rows_;
  std::map<Rank, mkv::PeerTarget> peers_;
  std::map<Rank, ss_cache*> peer_engines_;  // in-process peers we attached
  std::set<ss_cache*> attached_by_;         // engines that attached us as a peer
  std::set<ss_plan*> live_plans_;           // freed with the cache if still live

  // HBM state.
  cudaStream_t stream_ = nullptr;
  cudaStream_t comm_stream_ = nullptr;  // per-layer sends (overlap with compute)
  cudaEvent_t internal_ev_ = nullptr, comm_ev_ = nullptr, layer_ev_ = nullptr;
  // One event per caller stream that async work was enqueued on: internal
  // work (uploads, frees, resets), plan frees and Synchronize are ordered
  // after the latest work of EVERY such stream, not only the most recently
  // used one (the microkv.h stream contract).
  struct UserStream {
    cudaEvent_t ev = nullptr;
    uint64_t gen = 0, waited = 0;
  };
  std::map<cudaStream_t, UserStream> user_streams_;
  // Recorded after each receive window opens on the device; in-process
  // senders wait on it instead of PrepRecv synchronizing the host.  Once the
  // receive surface is exported to another process PrepRecv synchronizes.
  cudaEvent_t window_ev_ = nullptr;
  bool ipc_exported_ = false;
  // The transfer agent's stream: host-payload ApplyRemoteWrite and
  // ReceiveWriteFrame may run on another thread than the executor
  // (kv_cache.h:12-15), so they use their own stream, ordered after the
  // receive windows (window_ev_), and none of the executor's stream-ordering
  // state.
  cudaStream_t recv_stream_ = nullptr;
  uint32_t* h_agent_pinned_ = nullptr;  // the agent's pinned readback word
  // Pinned staging ring for small host->device uploads (page tables, row
  // maps, window slots): a pageable cudaMemcpyAsync blocks the host while the
  // driver stages it; through the ring the call is a memcpy + an async copy.
  static constexpr int kStageSlots = 16;
  static constexpr size_t kStageBytes = size_t(256) << 10;
  uint8_t* h_stage_ = nullptr;
  cudaEvent_t stage_ev_[kStageSlots] = {};
  bool stage_used_[kStageSlots] = {};
  int stage_next_ = 0;
  std::mutex stage_mu_;
  bool comm_pending_ = false;
  uint64_t comm_gen_ = 0, comm_waited_gen_ = 0;
  uint64_t internal_gen_ = 1, internal_recorded_gen_ = 0;
  std::map<cudaStream_t, uint64_t> user_stream_seen_;
  std::atomic<int64_t> h2d_bytes_{0}, d2h_bytes_{0};
  uint64_t* d_pool_ = nullptr;
  uint8_t* d_fill_ = nullptr;
  uint8_t* d_expecting_ = nullptr;
  int32_t* d_page_window_ = nullptr;
  unsigned long long* d_win_received_ = nullptr;
  uint32_t* d_win_layer_rows_ = nullptr;
  uint64_t* d_fold_sums_ = nullptr;  // [kMaxSeqRows][L]
  uint32_t* d_status_ = nullptr;
  unsigned long long* d_scratch_ = nullptr;
  unsigned long long* h_pinned_ = nullptr;  // small pinned readback area
  // TMA tensor maps of the pool for prefill attention (page box, row box),
  // built on first use (mkv::PoolTensorMap layout).
  alignas(64) unsigned char tmap_page_[128] = {}, tmap_row_[128] = {};
  bool tmaps_ready_ = false;
  alignas(64) unsigned char tmap_chunk_[128] = {};  // {64, 16, 1} boxes for decode chunks
  bool tmap_chunk_ready_ = false;
};
