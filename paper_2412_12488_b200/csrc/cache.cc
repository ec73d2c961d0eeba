// cache.cc — the engine: reference bookkeeping on the host, KV in HBM.
//
// Each member cites the reference function it replaces
// (/root/reference/proj/core/src/kv_cache.cc unless noted).  Bookkeeping
// is kept bit-identical (page ids, page tables, addresses, match lengths,
// window accounting, error codes); the KV bytes move only through the
// kernels of kernels.cu.
#include "cache.h"

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <unordered_map>

#include "hash.cuh"

using namespace mkv;

namespace mkv {

namespace {
constexpr int32_t kMaxWindows = 4096;
constexpr int32_t kMaxSeqRows = 16384;
constexpr uint32_t kIpcMagic = 0x4d4b5631;  // "MKV1"
// Destination addresses up to this many page slots are validated inside the
// copy grid (one launch); MICROKV_INLINE_VALIDATE_SLOTS overrides (0 = never;
// read per launch, like the other A/B switches).
// MICROKV_GEN_CHECK=0: validate every launch (A/B).
bool GenCheckEnabled() {
  const char* e = std::getenv("MICROKV_GEN_CHECK");
  return e == nullptr || std::atoi(e) != 0;
}
int64_t InlineValidateSlots() {
  const char* e = std::getenv("MICROKV_INLINE_VALIDATE_SLOTS");
  return e != nullptr ? std::atoll(e) : int64_t{2048};
}

const char* kCodeNames[] = {"OutOfPages",      "DuplicateSequence", "UnknownSequence",
                            "ForkBeyondCommitted", "AddrMismatch",  "MissingKV",
                            "LayerOrderViolation", "CannotEvict",   "ChecksumMismatch",
                            "UnknownAddress",  "PeerUnreachable",   "NoEngines",
                            "RoleMissing",     "NoOwner",           "UnknownStrategy",
                            "InvalidArgument", "Aborted",           "Internal"};

size_t Align(size_t x) { return (x + 255) & ~size_t(255); }
}  // namespace

const char* StatusName(int status) {
  if (status == 0) return "OK";
  if (status >= 1 && status <= 18) return kCodeNames[status - 1];
  switch (status) {
    case SS_ERR_UNSUPPORTED: return "Unsupported";
    case SS_ERR_BUFFER_TOO_SMALL: return "BufferTooSmall";
    case SS_ERR_CUDA: return "Cuda";
    case SS_ERR_NO_DEVICE: return "NoDevice";
  }
  return "Unknown";
}

void Throw(int code, const std::string& detail) {
  throw Error(1 + code, std::string(kCodeNames[code]) + ": " + detail);
}

void ThrowStatus(int status, const std::string& detail) {
  throw Error(status, std::string(StatusName(status)) + ": " + detail);
}

void CudaCheck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) {
    ThrowStatus(SS_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
  }
}

// kv_addr.cc:16-30.  Same checks and error precedence as the reference (a
// bad range or an overlap is InvalidArgument before the AddrMismatch total
// check).  Overlap needs two ranges on one page: pages are marked in a
// generation-stamped array (O(R)), and only ranges on repeated pages are
// sorted and compared.
void KVAddr::Validate() const {
  int64_t total = 0, max_page = -1;
  for (const auto& r : ranges) {
    MKV_CHECK(r.slot_count > 0 && r.slot_begin >= 0, kInvalidArgument, "bad slot range");
    total += r.slot_count;
    max_page = std::max(max_page, r.page_id);
  }
  std::vector<size_t> repeated;  // indices of ranges on pages seen more than once
  bool negative = false;
  for (const auto& r : ranges) negative |= r.page_id < 0;
  if (!negative && max_page < (int64_t(1) << 26)) {
    thread_local std::vector<uint32_t> stamp;
    thread_local std::vector<int32_t> first;
    thread_local uint32_t gen = 0;
    if (static_cast<int64_t>(stamp.size()) <= max_page) {
      stamp.assign(max_page + 1, 0);
      first.assign(max_page + 1, -1);
      gen = 0;
    }
    if (++gen == 0) {
      std::fill(stamp.begin(), stamp.end(), 0);
      gen = 1;
    }
    for (size_t i = 0; i < ranges.size(); ++i) {
      const int64_t pg = ranges[i].page_id;
      if (stamp[pg] != gen) {
        stamp[pg] = gen;
        first[pg] = static_cast<int32_t>(i);
      } else {
        if (first[pg] >= 0) {
          repeated.push_back(static_cast<size_t>(first[pg]));
          first[pg] = -1;
        }
        repeated.push_back(i);
      }
    }
  } else {
    for (size_t i = 0; i < ranges.size(); ++i) repeated.push_back(i);
  }
  if (!repeated.empty()) {
    std::sort(repeated.begin(), repeated.end(), [&](size_t a, size_t b) {
      const auto& ra = ranges[a];
      const auto& rb = ranges[b];
      return ra.page_id != rb.page_id ? ra.page_id < rb.page_id : ra.slot_begin < rb.slot_begin;
    });
    for (size_t i = 1; i < repeated.size(); ++i) {
      const auto& prev = ranges[repeated[i - 1]];
      const auto& cur = ranges[repeated[i]];
      MKV_CHECK(!(prev.page_id == cur.page_id &&
                  static_cast<int64_t>(prev.slot_begin) + prev.slot_count > cur.slot_begin),
                kInvalidArgument, "overlapping slot ranges");
    }
  }
  MKV_CHECK(total == token_count, kAddrMismatch, "slot counts do not cover token_count");
}

// kv_addr.cc:32-51
KVAddr KVAddr::Slice(int64_t begin, int64_t end) const {
  MKV_CHECK(begin >= token_begin && end <= token_begin + token_count && begin <= end,
            kInvalidArgument, "slice outside address");
  KVAddr out;
  out.token_begin = begin;
  out.token_count = end - begin;
  int64_t pos = token_begin;
  for (const auto& r : ranges) {
    const int64_t lo = std::max(pos, begin), hi = std::min(pos + r.slot_count, end);
    if (lo < hi) {
      out.ranges.push_back({r.page_id, static_cast<int32_t>(r.slot_begin + (lo - pos)),
                            static_cast<int32_t>(hi - lo)});
    }
    pos += r.slot_count;
  }
  return out;
}

namespace {
// kv_cache.cc:13-18
int64_t ResolveEndIndex(int64_t len, int64_t end) {
  const int64_t e = end < 0 ? len + end : end;
  MKV_CHECK(end != 0, kInvalidArgument, "end = 0 is invalid");
  MKV_CHECK(e > 0 && e <= len, kInvalidArgument, "end out of range");
  return e;
}
}  // namespace

}  // namespace mkv

// ---------------------------------------------------------------------------
// Construction (kv_cache.cc:26-47; CacheConfig/ModelConfig::Validate config.cc:17-27)
// ---------------------------------------------------------------------------
ss_cache::ss_cache(const ss_config& cfg)
    : num_pages_(cfg.num_pages),
      P_(cfg.page_size),
      L_(cfg.layers),
      W_(cfg.dim),
      vocab_(cfg.vocab),
      hash_seed_(cfg.hash_seed),
      device_(cfg.device),
      rank_(cfg.rank) {
  MKV_CHECK(cfg.layers >= 1, kInvalidArgument, "layers must be >= 1");
  MKV_CHECK(cfg.dim >= 1, kInvalidArgument, "dim must be >= 1");
  MKV_CHECK(cfg.vocab >= 2, kInvalidArgument, "vocab must be >= 2");
  MKV_CHECK(cfg.num_pages >= 1, kInvalidArgument, "num_pages must be >= 1");
  MKV_CHECK(cfg.page_size >= 1 && (cfg.page_size & (cfg.page_size - 1)) == 0, kInvalidArgument,
            "page_size must be a power of two");
  MKV_CHECK(cfg.num_pages * cfg.page_size < (int64_t(1) << 31), kInvalidArgument,
            "num_pages * page_size must fit int32 slot indices");
  seed_state_ = mkv::seed_state(hash_seed_);
  // Test hook: publish window counters at system scope even to a peer on
  // this GPU, so a one-GPU run executes the cross-GPU (NVLink) branch of
  // the copy kernels: system-scope fence + red.release.sys.
  if (const char* f = std::getenv("MICROKV_FORCE_SYS_SCOPE")) force_sys_scope_ = std::atoi(f) != 0;
  while ((1 << page_shift_) < P_) ++page_shift_;
  // LIFO free list, lowest page first out (kv_cache.cc:45-46).
  free_pages_.reserve(num_pages_);
  for (int64_t i = num_pages_ - 1; i >= 0; --i) free_pages_.push_back(i);
  page_owner_.assign(num_pages_, -1);
  expecting_.assign(static_cast<size_t>(num_pages_) * P_, 0);
  if (device_ < 0) return;

  CudaCheck(cudaSetDevice(device_), "cudaSetDevice");
  int sms = 0;
  CudaCheck(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device_), "sm count");
  num_sms_ = sms;
  {
    // Once per device per process: load every kernel before any receiver
    // can spin on a window counter (mkv::preload_kernels).
    static std::mutex mu;
    static std::vector<bool> loaded;
    std::lock_guard<std::mutex> g(mu);
    if (loaded.size() <= static_cast<size_t>(device_)) loaded.resize(device_ + 1, false);
    if (!loaded[device_]) {
      mkv::preload_kernels();
      loaded[device_] = true;
    }
  }
  {
    // The internal stream at the highest priority: its kernels are the
    // µs-scale device halves of host API calls (open / close a receive
    // window, page resets, fill scans) that the caller waits for, and a long
    // copy grid with more CTAs than are resident (launch_copy_rows) would
    // otherwise hold them until its last CTA is dispatched.
    int lo = 0, hi = 0;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);
    CudaCheck(cudaStreamCreateWithPriority(&stream_, cudaStreamNonBlocking, hi), "stream");
  }
  CudaCheck(cudaEventCreateWithFlags(&internal_ev_, cudaEventDisableTiming), "event");
  CudaCheck(cudaEventCreateWithFlags(&comm_ev_, cudaEventDisableTiming), "event");
  CudaCheck(cudaEventCreateWithFlags(&layer_ev_, cudaEventDisableTiming), "event");
  CudaCheck(cudaEventCreateWithFlags(&window_ev_, cudaEventDisableTiming), "event");
  {
    int lo = 0, hi = 0;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);
    // Transfers get the higher priority so a layer's send is not starved by
    // the next layer's compute (the overlap of PAPER.md:339-344).
    CudaCheck(cudaStreamCreateWithPriority(&comm_stream_, cudaStreamNonBlocking, hi), "stream");
    CudaCheck(cudaStreamCreateWithFlags(&recv_stream_, cudaStreamNonBlocking), "stream");
  }
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, device_) == cudaSuccess) {
    uint64_t thr = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  const size_t slots = static_cast<size_t>(num_pages_) * P_;
  CudaCheck(cudaMalloc(&d_pool_, slots * L_ * W_ * 8), "cudaMalloc pool");
  CudaCheck(cudaMalloc(&d_fill_, slots * L_), "cudaMalloc fill");
  CudaCheck(cudaMalloc(&d_expecting_, slots), "cudaMalloc expecting");
  CudaCheck(cudaMalloc(&d_page_window_, sizeof(int32_t) * num_pages_), "cudaMalloc page_window");
  // [0, kMaxWindows): rows received per window; [kMaxWindows, 2 kMaxWindows):
  // the window id's open-generation (one allocation, so an IPC peer maps both).
  CudaCheck(cudaMalloc(&d_win_received_, sizeof(unsigned long long) * 2 * kMaxWindows),
            "cudaMalloc");
  CudaCheck(cudaMalloc(&d_win_layer_rows_, sizeof(uint32_t) * kMaxWindows * L_), "cudaMalloc");
  CudaCheck(cudaMalloc(&d_fold_sums_, sizeof(uint64_t) * kMaxSeqRows * L_), "cudaMalloc");
  CudaCheck(cudaMalloc(&d_status_, sizeof(uint32_t)), "cudaMalloc");
  CudaCheck(cudaMalloc(&d_scratch_, 256), "cudaMalloc");
  CudaCheck(cudaHostAlloc(&h_pinned_, sizeof(unsigned long long) * kMaxWindows, 0), "pinned");
  CudaCheck(cudaHostAlloc(&h_stage_, kStageSlots * kStageBytes, 0), "pinned staging");
  CudaCheck(cudaHostAlloc(&h_agent_pinned_, sizeof(uint32_t), 0), "pinned agent");
  for (auto& e : stage_ev_) CudaCheck(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
  // A fresh pool is zero-filled like the reference's (kv_cache.cc:37).
  CudaCheck(cudaMemsetAsync(d_pool_, 0, slots * L_ * W_ * 8, stream_), "memset");
  CudaCheck(cudaMemsetAsync(d_fill_, 0, slots * L_, stream_), "memset");
  CudaCheck(cudaMemsetAsync(d_expecting_, 0, slots, stream_), "memset");
  CudaCheck(cudaMemsetAsync(d_page_window_, 0xff, sizeof(int32_t) * num_pages_, stream_), "memset");
  CudaCheck(cudaMemsetAsync(d_win_received_, 0, sizeof(unsigned long long) * 2 * kMaxWindows, stream_),
            "memset");
  CudaCheck(cudaMemsetAsync(d_win_layer_rows_, 0, sizeof(uint32_t) * kMaxWindows * L_, stream_),
            "memset");
  CudaCheck(cudaMemsetAsync(d_status_, 0, sizeof(uint32_t), stream_), "memset");
  CountLaunches(0);  // memsets only: kernels are what the launch counter counts
  for (int32_t i = kMaxWindows - 1; i >= 0; --i) free_window_ids_.push_back(i);
  for (int32_t i = kMaxSeqRows - 1; i >= 0; --i) free_fold_rows_.push_back(i);
  Sync();
}

ss_cache::~ss_cache() {
  // Order-independent teardown: unlink in-process peer relations both ways,
  // then release plans still alive (their handles become invalid).
  for (ss_cache* a : attached_by_) {
    for (auto it = a->peer_engines_.begin(); it != a->peer_engines_.end();) {
      if (it->second == this) {
        a->peers_.erase(it->first);
        it = a->peer_engines_.erase(it);
      } else {
        ++it;
      }
    }
  }
  for (auto& [r, e] : peer_engines_) e->attached_by_.erase(this);
  if (device_ >= 0) {
    cudaSetDevice(device_);
    cudaStreamSynchronize(comm_stream_);
    cudaStreamSynchronize(stream_);
  }
  for (ss_plan* p : live_plans_) {
    if (device_ >= 0) FreePlanDevice(p);
    if (p->upload_ev != nullptr) cudaEventDestroy(p->upload_ev);
    delete p;
  }
  live_plans_.clear();
  if (device_ >= 0) {
    for (auto& [id, rec] : records_) {
      if (rec->d_slots != nullptr) cudaFree(rec->d_slots);
    }
  }
  if (device_ < 0) return;
  cudaSetDevice(device_);
  if (stream_) cudaStreamSynchronize(stream_);
  if (recv_stream_) cudaStreamSynchronize(recv_stream_);
  for (auto& [r, p] : peers_) {
    for (void* ptr : p.ipc_ptrs) cudaIpcCloseMemHandle(ptr);
  }
  cudaFree(d_pool_);
  cudaFree(d_fill_);
  cudaFree(d_expecting_);
  cudaFree(d_page_window_);
  cudaFree(d_win_received_);
  cudaFree(d_win_layer_rows_);
  cudaFree(d_fold_sums_);
  cudaFree(d_status_);
  cudaFree(d_scratch_);
  cudaFreeHost(h_pinned_);
  if (h_agent_pinned_ != nullptr) cudaFreeHost(h_agent_pinned_);
  if (recv_stream_ != nullptr) cudaStreamDestroy(recv_stream_);
  if (h_stage_ != nullptr) {
    for (int i = 0; i < kStageSlots; ++i) {
      if (stage_used_[i]) cudaEventSynchronize(stage_ev_[i]);  // copies on user streams
      cudaEventDestroy(stage_ev_[i]);
    }
    cudaFreeHost(h_stage_);
  }
  if (fused_vstream_ != nullptr) {
    cudaStreamSynchronize(fused_vstream_);
    cudaStreamDestroy(fused_vstream_);
    cudaEventDestroy(fused_vev_);
  }
  if (verdict_stream_ != nullptr) {
    cudaStreamSynchronize(verdict_stream_);
    cudaStreamSynchronize(ce_stream_);
    cudaStreamDestroy(verdict_stream_);
    cudaStreamDestroy(ce_stream_);
    cudaEventDestroy(verdict_ev_);
    cudaEventDestroy(ce_ev_);
  }
  cudaEventDestroy(internal_ev_);
  cudaEventDestroy(window_ev_);
  for (auto& [st, u] : user_streams_) cudaEventDestroy(u.ev);
  cudaStreamSynchronize(comm_stream_);
  cudaEventDestroy(comm_ev_);
  cudaEventDestroy(layer_ev_);
  cudaStreamDestroy(comm_stream_);
  cudaStreamDestroy(stream_);
}

// ---------------------------------------------------------------------------
// Helpers
// ---------------------------------------------------------------------------
Record* ss_cache::MustGet(SeqId seq) {
  auto it = records_.find(seq);
  MKV_CHECK(it != records_.end(), kUnknownSequence, "sequence " + std::to_string(seq));
  return it->second.get();
}

const Record* ss_cache::MustGet(SeqId seq) const {
  auto it = records_.find(seq);
  MKV_CHECK(it != records_.end(), kUnknownSequence, "sequence " + std::to_string(seq));
  return it->second.get();
}

// kv_cache.cc:67-77 (through the resolved host page table).
int32_t ss_cache::Resolve(const Record* rec, int64_t pos) const {
  MKV_ICHECK(pos >= 0 && pos < rec->alloc_len, "position not allocated");
  return rec->slots[pos];
}

// kv_cache.cc:79-84
int64_t ss_cache::PagesNeeded(const Record* rec, int64_t upto) const {
  const int64_t idx = upto - rec->fork_len;
  if (idx <= 0) return 0;
  const int64_t pages = (idx + P_ - 1) / P_;
  return std::max<int64_t>(0, pages - static_cast<int64_t>(rec->own_pages.size()));
}

void ss_cache::RequireDevice(const char* what) const {
  if (device_ < 0) ThrowStatus(SS_ERR_NO_DEVICE, std::string(what) + " on a host-only cache");
}

void ss_cache::Sync() { CudaCheck(cudaStreamSynchronize(stream_), "cudaStreamSynchronize"); }

void ss_cache::H2D(void* dst, const void* src, size_t bytes, cudaStream_t s, const char* what) {
  h2d_bytes_ += static_cast<int64_t>(bytes);
  if (h_stage_ != nullptr && bytes > 0 && bytes <= kStageBytes) {
    std::lock_guard<std::mutex> lock(stage_mu_);
    const int i = stage_next_;
    stage_next_ = (stage_next_ + 1) % kStageSlots;
    if (stage_used_[i]) CudaCheck(cudaEventSynchronize(stage_ev_[i]), "staging slot");
    uint8_t* st = h_stage_ + static_cast<size_t>(i) * kStageBytes;
    std::memcpy(st, src, bytes);
    CudaCheck(cudaMemcpyAsync(dst, st, bytes, cudaMemcpyHostToDevice, s), what);
    CudaCheck(cudaEventRecord(stage_ev_[i], s), "staging event");
    stage_used_[i] = true;
    return;
  }
  CudaCheck(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, s), what);
}

void ss_cache::D2H(void* dst, const void* src, size_t bytes, cudaStream_t s, const char* what) {
  CudaCheck(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, s), what);
  d2h_bytes_ += static_cast<int64_t>(bytes);
}

// Cross-stream ordering between the internal stream (bookkeeping uploads,
// resets) and caller streams (async data path).  Event records and waits
// are skipped when nothing new was enqueued on the other side.
void ss_cache::OrderAfterUser() {
  for (auto& [st, u] : user_streams_) {
    if (u.gen != u.waited) {
      CudaCheck(cudaStreamWaitEvent(stream_, u.ev, 0), "cudaStreamWaitEvent");
      u.waited = u.gen;
    }
  }
  if (comm_pending_ && comm_gen_ != comm_waited_gen_) {
    CudaCheck(cudaStreamWaitEvent(stream_, comm_ev_, 0), "cudaStreamWaitEvent");
    comm_waited_gen_ = comm_gen_;
  }
  ++internal_gen_;  // the caller is about to enqueue internal work
}

void ss_cache::BeginInternal() { ++internal_gen_; }

// Generation of a validated launch (>= 1): a failed validation stores it in
// verdict[1], the copy compares, so verdict words need no reset per launch.
int32_t ss_cache::NextLaunchGen() {
  int32_t g = ++launch_gen_;
  if (g <= 0) {  // wrapped: restart at 1 (a stale failure mark of 2^31 launches ago is moot)
    launch_gen_ = 1;
    g = 1;
  }
  return g;
}

void ss_cache::OrderUser(cudaStream_t s) {
  if (internal_gen_ != internal_recorded_gen_) {
    CudaCheck(cudaEventRecord(internal_ev_, stream_), "cudaEventRecord");
    internal_recorded_gen_ = internal_gen_;
  }
  auto it = user_stream_seen_.find(s);
  if (it != user_stream_seen_.end() && it->second == internal_recorded_gen_) return;
  CudaCheck(cudaStreamWaitEvent(s, internal_ev_, 0), "cudaStreamWaitEvent");
  user_stream_seen_[s] = internal_recorded_gen_;
}

// A launch on user stream s that enqueues nothing on the internal stream:
// s waits only for internal work enqueued since it last waited (nothing, in
// a steady per-layer loop), and NoteUser afterwards orders later internal
// work after it.  No internal-stream round trip per launch: that pair of
// cross-stream dependencies had cost ~10 us of device time per launch.
// Work on two different user streams is not ordered by the library (use
// CUDA events, as with any stream).
void ss_cache::OrderLaunch(cudaStream_t s) {
  if (s == stream_) {
    OrderAfterUser();
    return;
  }
  OrderUser(s);
}

void ss_cache::CountLaunches(int64_t n) {
  launches_ += n;
  CudaCheck(cudaGetLastError(), "kernel launch");
}

void ss_cache::NoteUser(cudaStream_t s) {
  UserStream& u = user_streams_[s];
  if (u.ev == nullptr) CudaCheck(cudaEventCreateWithFlags(&u.ev, cudaEventDisableTiming), "event");
  CudaCheck(cudaEventRecord(u.ev, s), "cudaEventRecord");
  ++u.gen;
}

void ss_cache::SyncUserStreams() {
  for (auto& [st, u] : user_streams_) {
    if (u.gen != 0) CudaCheck(cudaEventSynchronize(u.ev), "cudaEventSynchronize");
  }
}

DevBlock ss_cache::DevAlloc(size_t bytes, cudaStream_t s) {
  DevBlock b;
  b.bytes = bytes;
  if (bytes > 0) CudaCheck(cudaMallocAsync(&b.ptr, bytes, s), "cudaMallocAsync");
  return b;
}

void ss_cache::DevFree(DevBlock& b, cudaStream_t s) {
  if (b.ptr) cudaFreeAsync(b.ptr, s);
  b.ptr = nullptr;
  b.bytes = 0;
}

uint64_t* ss_cache::PoolLayer(int32_t layer) const {
  return d_pool_ + static_cast<int64_t>(layer) * num_pages_ * P_ * W_;
}

// kv_cache.cc:86-102.  Positions proven full on the host (the caller's
// `known_full_until`, or a forward pass that just covered them) are
// skipped; a position that no kernel can have written (beyond every
// forward pass and outside any receive window) stops the walk; anything
// else is decided by a device scan of the fill bytes.
void ss_cache::AdvanceCommitted(Record* rec, int64_t known_full_until) {
  const int64_t limit = std::min<int64_t>(rec->alloc_len, rec->tokens.size());
  int64_t pos = std::max(rec->committed_hint, rec->fork_len);
  if (known_full_until > pos) pos = std::min(known_full_until, limit);
  if (pos < limit && device_ >= 0) {
    const bool in_window = rec->window && pos >= rec->window->begin && pos < rec->window->end;
    if (pos < rec->touched_end || in_window) pos = DeviceFirstNonFull(rec, pos, limit);
  }
  rec->committed_hint = std::max(rec->committed_hint, pos);
}

int64_t ss_cache::DeviceFirstNonFull(const Record* rec, int64_t from, int64_t to) {
  if (from >= to) return to;
  OrderAfterUser();
  const int64_t n = to - from;
  launch_first_nonfull(d_fill_, num_pages_ * P_, L_, rec->d_slots + from, n, d_scratch_, stream_,
                       num_sms_);
  CountLaunches(1);
  D2H(h_pinned_, d_scratch_, sizeof(unsigned long long), stream_, "D2H scan");
  Sync();
  const unsigned long long r = h_pinned_[0];
  return r >= static_cast<unsigned long long>(n) ? to : from + static_cast<int64_t>(r);
}

// Positions [begin, end) of `rec` must be non-Empty at `layer`
// (kv_cache.cc:340-342, 358-361, 379-381).  Positions below the committed
// frontier, or written by `plan` on this layer, are full by construction;
// the rest are checked on the device.
bool ss_cache::CoveredByLivePlan(SeqId seq, int64_t begin, int64_t end) const {
  if (begin >= end) return true;
  for (const ss_plan* p : live_plans_) {
    for (const auto& e : p->entries) {
      if (e.seq == seq && e.begin <= begin && e.end >= end) return true;
    }
  }
  return false;
}

void ss_cache::CheckFilled(const Record* rec, int64_t begin, int64_t end, int32_t layer,
                           const char* what, const ss_plan* plan) {
  std::vector<int32_t> unproven;
  for (int64_t pos = std::max(begin, rec->committed_hint); pos < end; ++pos) {
    bool written = false;
    if (plan) {
      for (const auto& e : plan->entries) {
        if (e.seq == rec->id && pos >= e.begin && pos < e.end) {
          written = true;
          break;
        }
      }
    }
    if (!written) unproven.push_back(Resolve(rec, pos));
  }
  if (unproven.empty()) return;
  RequireDevice(what);
  OrderAfterUser();
  const int64_t n = static_cast<int64_t>(unproven.size());
  DevBlock b = DevAlloc(sizeof(int32_t) * n, stream_);
  // A scratch status word of its own: the sticky d_status_ bits of earlier
  // rejected async sends / timed-out waits must survive until Synchronize.
  uint32_t* d_check = reinterpret_cast<uint32_t*>(d_scratch_ + 1);
  CudaCheck(cudaMemsetAsync(d_check, 0, sizeof(uint32_t), stream_), "memset");
  H2D(b.ptr, unproven.data(), sizeof(int32_t) * n, stream_, "H2D slots");
  launch_check_filled(d_fill_ + static_cast<int64_t>(layer) * num_pages_ * P_,
                      static_cast<int32_t*>(b.ptr), n, d_check, stream_, num_sms_);
  CountLaunches(1);
  uint32_t st = 0;
  D2H(&st, d_check, sizeof(uint32_t), stream_, "D2H status");
  DevFree(b, stream_);
  Sync();
  MKV_CHECK((st & kStatusMissingKV) == 0, kMissingKV, what);
}

// Grows the sequence's HBM page table to alloc_len and uploads the newly
// resolved positions [old_len, alloc_len) (stream-ordered on the internal
// stream; async users are ordered after it by OrderUser).
void ss_cache::SyncDeviceTable(Record* rec, int64_t old_len) {
  if (device_ < 0) return;
  const int64_t need = rec->alloc_len;
  OrderAfterUser();
  if (need > rec->d_cap) {
    const int64_t cap = std::max<int64_t>({need, 2 * rec->d_cap, 256});
    int32_t* nt = nullptr;
    CudaCheck(cudaMallocAsync(&nt, sizeof(int32_t) * cap, stream_), "cudaMallocAsync table");
    if (rec->d_slots != nullptr) {
      if (old_len > 0) {
        CudaCheck(cudaMemcpyAsync(nt, rec->d_slots, sizeof(int32_t) * old_len,
                                  cudaMemcpyDeviceToDevice, stream_),
                  "D2D table");
      }
      cudaFreeAsync(rec->d_slots, stream_);
    }
    rec->d_slots = nt;
    rec->d_cap = cap;
  }
  if (need > old_len) {
    H2D(rec->d_slots + old_len, rec->slots.data() + old_len, sizeof(int32_t) * (need - old_len),
        stream_, "H2D table");
  }
}

// kv_cache.cc:104-110
void ss_cache::TouchLru(Record* rec) {
  if (tree_.Contains(rec->id)) {
    const int64_t n = std::min<int64_t>(rec->committed_hint, rec->tokens.size());
    if (n > 0) tree_.Insert(std::span<const Token>(rec->tokens.data(), n), rec->id);
  }
}

// ---------------------------------------------------------------------------
// Declaration stage
// ---------------------------------------------------------------------------
RadixTree::MatchResult ss_cache::MatchPrefixSeq(std::span<const Token> tokens) {
  return tree_.MatchPrefix(tokens);  // kv_cache.cc:112-118
}

// kv_cache.cc:120-131
Record* ss_cache::CreateSequence(SeqId seq, std::vector<Token> tokens) {
  MKV_CHECK(records_.find(seq) == records_.end(), kDuplicateSequence,
            "sequence " + std::to_string(seq));
  auto rec = std::make_unique<Record>();
  rec->id = seq;
  rec->tokens = std::move(tokens);
  rec->prefix_digest = InitialPrefixDigest();
  if (device_ >= 0) {
    // Retryable like OutOfPages: eviction of finished sequences frees rows.
    MKV_CHECK(!free_fold_rows_.empty(), kOutOfPages,
              "all " + std::to_string(kMaxSeqRows) + " sequence rows in use");
    rec->fold_row = free_fold_rows_.back();
    free_fold_rows_.pop_back();
    OrderAfterUser();
    CudaCheck(cudaMemsetAsync(d_fold_sums_ + static_cast<int64_t>(rec->fold_row) * L_, 0,
                              sizeof(uint64_t) * L_, stream_),
              "memset fold sums");
    CountLaunches(0);
  }
  Record* out = rec.get();
  {
    std::lock_guard<std::mutex> lock(recv_mu_);  // the transfer agent looks records up
    records_[seq] = std::move(rec);
  }
  return out;
}

// kv_cache.cc:133-166
Record* ss_cache::ForkSequence(SeqId parent, SeqId child, int64_t fork_len,
                               std::vector<Token> child_tokens) {
  Record* p = MustGet(parent);
  MKV_CHECK(records_.find(child) == records_.end(), kDuplicateSequence,
            "sequence " + std::to_string(child));
  AdvanceCommitted(p);
  MKV_CHECK(fork_len <= p->committed_hint, kForkBeyondCommitted,
            "fork_len " + std::to_string(fork_len) + " > committed " +
                std::to_string(p->committed_hint));
  MKV_CHECK(fork_len >= 0, kInvalidArgument, "negative fork_len");
  if (child_tokens.empty()) {
    child_tokens.assign(p->tokens.begin(), p->tokens.begin() + fork_len);
  } else {
    MKV_CHECK(static_cast<int64_t>(child_tokens.size()) >= fork_len, kInvalidArgument,
              "child tokens shorter than fork_len");
    for (int64_t i = 0; i < fork_len; ++i) {
      MKV_CHECK(child_tokens[i] == p->tokens[i], kInvalidArgument,
                "child tokens diverge inside the fork prefix");
    }
  }
  Record* rec = CreateSequence(child, std::move(child_tokens));
  rec->parent = fork_len > 0 ? parent : -1;
  rec->fork_len = fork_len;
  rec->alloc_len = fork_len;
  rec->committed_hint = fork_len;
  rec->slots.assign(p->slots.begin(), p->slots.begin() + fork_len);
  SyncDeviceTable(rec, 0);
  if (rec->parent >= 0) ++p->refcount;
  TouchLru(p);
  return rec;
}

// kv_cache.cc:168-183
void ss_cache::EnsureAllocated(SeqId seq, int64_t upto) {
  Record* rec = MustGet(seq);
  MKV_CHECK(upto <= static_cast<int64_t>(rec->tokens.size()), kInvalidArgument,
            "allocation beyond known tokens");
  const int64_t need = PagesNeeded(rec, upto);
  MKV_CHECK(need <= static_cast<int64_t>(free_pages_.size()), kOutOfPages,
            std::to_string(need) + " pages needed, " + std::to_string(free_pages_.size()) +
                " free");
  const int64_t old_len = rec->alloc_len;
  if (need > 0) {
    std::lock_guard<std::mutex> lock(recv_mu_);  // page_owner_ is read by the transfer agent
    rec->own_pages.reserve(rec->own_pages.size() + need);
    size_t at = rec->slots.size();
    rec->slots.resize(at + static_cast<size_t>(need) * P_);
    int32_t* sl = rec->slots.data() + at;
    for (int64_t i = 0; i < need; ++i) {
      const int64_t page = free_pages_.back();
      free_pages_.pop_back();
      page_owner_[page] = seq;
      rec->own_pages.push_back(page);
      const int32_t base = static_cast<int32_t>(page * P_);
      for (int32_t s = 0; s < P_; ++s) sl[s] = base + s;
      sl += P_;
    }
  }
  rec->alloc_len = rec->fork_len + static_cast<int64_t>(rec->own_pages.size()) * P_;
  if (need > 0) SyncDeviceTable(rec, old_len);
}

void ss_cache::AppendToken(SeqId seq, Token t) { MustGet(seq)->tokens.push_back(t); }

// kv_cache.cc:187-229
int64_t ss_cache::PrepRecv(SeqId seq, std::vector<Token> tokens, int64_t end, KVAddr* addr,
                           int64_t ranges_cap) {
  MKV_CHECK(!tokens.empty(), kInvalidArgument, "empty prompt");
  MKV_CHECK(records_.find(seq) == records_.end(), kDuplicateSequence,
            "sequence " + std::to_string(seq));
  const int64_t e = ResolveEndIndex(static_cast<int64_t>(tokens.size()), end);
  const auto match = tree_.MatchPrefix(std::span<const Token>(tokens.data(), e));
  const int64_t m = match.match_len;
  // All-or-nothing: fail before any state change when capacity is short.
  const int64_t pages_needed = (e - m + P_ - 1) / P_;
  MKV_CHECK(pages_needed <= static_cast<int64_t>(free_pages_.size()), kOutOfPages,
            std::to_string(pages_needed) + " pages needed, " +
                std::to_string(free_pages_.size()) + " free");
  // Device rows a new receive needs, checked before any state change like
  // the pages (a window per open receive, recycled once it completes and is
  // drained; a fold-sum row per live sequence).
  if (device_ >= 0) {
    MKV_CHECK(e == m || !free_window_ids_.empty(), kOutOfPages,
              "all " + std::to_string(kMaxWindows) + " receive windows are open");
    MKV_CHECK(!free_fold_rows_.empty(), kOutOfPages,
              "all " + std::to_string(kMaxSeqRows) + " sequence rows in use");
  }
  if (pages_needed > ranges_cap) {
    ThrowStatus(SS_ERR_BUFFER_TOO_SMALL,
                "address needs " + std::to_string(pages_needed) + " ranges");
  }
  Record* rec = m > 0 ? ForkSequence(match.seq, seq, m, std::move(tokens))
                      : CreateSequence(seq, std::move(tokens));
  EnsureAllocated(seq, e);
  *addr = BuildAddr(seq, m, e);
  {
    std::lock_guard<std::mutex> lock(recv_mu_);
    for (int64_t pos = m; pos < e; ++pos) expecting_[rec->slots[pos]] = 1;
    if (e > m) {
      Window w;
      w.begin = m;
      w.end = e;
      w.expected = (e - m) * L_;
      w.received_layer.assign(L_, 0);
      rec->window = std::move(w);
    }
    if (device_ >= 0) OpenDeviceWindow(rec, m, e);
  }
  return m;
}

// Device half of PrepRecv: reservation bits, page -> window map, counters.
// Synchronous, so a peer that receives the address sees a ready receiver.
void ss_cache::OpenDeviceWindow(Record* rec, int64_t m, int64_t e) {
  if (e <= m) return;
  MKV_CHECK(!free_window_ids_.empty(), kOutOfPages, "all receive windows are open");
  const int32_t wid = free_window_ids_.back();
  free_window_ids_.pop_back();
  rec->window->dev_id = wid;
  const int64_t n = e - m, np = static_cast<int64_t>(rec->own_pages.size());
  const size_t off_pages = Align(sizeof(int32_t) * n);
  std::vector<uint8_t> host(off_pages + sizeof(int64_t) * np);
  std::memcpy(host.data(), rec->slots.data() + m, sizeof(int32_t) * n);
  std::memcpy(host.data() + off_pages, rec->own_pages.data(), sizeof(int64_t) * np);
  OrderAfterUser();
  DevBlock b = DevAlloc(host.size(), stream_);
  H2D(b.ptr, host.data(), host.size(), stream_, "H2D window");
  launch_open_window(d_expecting_, static_cast<int32_t*>(b.ptr), n, d_page_window_,
                     reinterpret_cast<int64_t*>(static_cast<uint8_t*>(b.ptr) + off_pages), np, wid,
                     d_win_received_, d_win_layer_rows_, d_win_received_ + kMaxWindows, L_, stream_);
  CountLaunches(1);
  DevFree(b, stream_);
  if (ipc_exported_) {
    Sync();  // a peer process sees a ready receiver once it holds the address
  } else {
    CudaCheck(cudaEventRecord(window_ev_, stream_), "cudaEventRecord window");
  }
}

// A completed and drained window gives its device row back: its pages stop
// mapping to it first (a stale device-direct sender is then rejected, as a
// write into a freed window, instead of counting into the row's next window).
// The reset is on the internal stream, after every caller stream's queued
// work (a receive wait still reading the row's counters).
void ss_cache::CloseDeviceWindow(Record* rec) {
  if (device_ < 0 || !rec->window || rec->window->dev_id < 0) return;
  const int32_t wid = rec->window->dev_id;
  const int64_t np = static_cast<int64_t>(rec->own_pages.size());
  if (np > 0) {
    OrderAfterUser();
    DevBlock b = DevAlloc(sizeof(int64_t) * np, stream_);
    H2D(b.ptr, rec->own_pages.data(), sizeof(int64_t) * np, stream_, "H2D window pages");
    launch_close_window(d_page_window_, static_cast<int64_t*>(b.ptr), np, wid, stream_);
    CountLaunches(1);
    DevFree(b, stream_);
    if (ipc_exported_) Sync();  // another process's sender validates against it
  }
  std::lock_guard<std::mutex> lock(recv_mu_);
  free_window_ids_.push_back(wid);
  rec->window->dev_id = -1;
}

// kv_cache.cc:231-243
void ss_cache::MarkSend(SeqId seq, int64_t begin, int64_t end, Rank dest, KVAddr addr,
                        uint64_t tag) {
  Record* rec = MustGet(seq);
  MKV_CHECK(begin >= 0 && end <= static_cast<int64_t>(rec->tokens.size()) && begin <= end,
            kInvalidArgument, "send range outside sequence");
  MKV_CHECK(addr.token_count == end - begin, kAddrMismatch,
            "destination covers " + std::to_string(addr.token_count) + " tokens, range has " +
                std::to_string(end - begin));
  MKV_CHECK(addr.token_begin == begin, kAddrMismatch, "destination token_begin mismatch");
  pending_sends_.push_back({seq, begin, end, dest, std::move(addr), tag});
}

// kv_cache.cc:245-306
ss_plan* ss_cache::BeginForward(const ss_batch_entry* batch, int64_t n) {
  auto plan = std::make_unique<ss_plan>();
  plan->owner = this;
  std::set<SeqId> seen;
  for (int64_t i = 0; i < n; ++i) {
    const ss_batch_entry& be = batch[i];
    Record* rec = MustGet(be.seq);
    MKV_ICHECK(seen.insert(be.seq).second, "sequence batched twice");
    const int64_t nt = static_cast<int64_t>(rec->tokens.size());
    MKV_CHECK(be.begin >= 0 && be.begin < be.end && be.end <= nt, kInvalidArgument,
              "bad forward range");
    AdvanceCommitted(rec);
    MKV_CHECK(rec->committed_hint >= be.begin, kMissingKV,
              "position " + std::to_string(rec->committed_hint) +
                  " is empty before prefill begin " + std::to_string(be.begin));
    MKV_ICHECK(rec->alloc_len >= be.end, "forward range not allocated");
    MKV_ICHECK(rec->fold_frontier <= be.begin, "fold frontier beyond range");
    MKV_ICHECK(rec->digest_len <= be.begin, "digest beyond range");
    PlanEntry pe;
    pe.seq = be.seq;
    pe.is_decode = be.is_decode != 0;
    pe.begin = be.begin;
    pe.end = be.end;
    pe.fold_from = rec->fold_frontier;
    pe.slots.assign(rec->slots.begin() + pe.fold_from, rec->slots.begin() + be.end);
    while (rec->digest_len < be.end) {
      rec->prefix_digest = fnv_u32(rec->prefix_digest,
                                   static_cast<uint32_t>(rec->tokens[rec->digest_len]));
      ++rec->digest_len;
      if (rec->digest_len > be.begin) pe.digests.push_back(rec->prefix_digest);
    }
    pe.tokens.assign(rec->tokens.begin() + be.begin, rec->tokens.begin() + be.end);
    plan->total_outputs += be.end - be.begin;
    plan->entries.push_back(std::move(pe));
  }
  for (auto it = pending_sends_.begin(); it != pending_sends_.end();) {
    if (!seen.count(it->seq)) {
      ++it;
      continue;
    }
    PlanSend ps;
    ps.seq = it->seq;
    ps.begin = it->begin;
    ps.end = it->end;
    ps.dest = it->dest;
    ps.dest_addr = std::move(it->addr);
    ps.user_tag = it->tag;
    const Record* rec = MustGet(ps.seq);
    ps.src_slots.reserve(ps.end - ps.begin);
    for (int64_t pos = ps.begin; pos < ps.end; ++pos) ps.src_slots.push_back(Resolve(rec, pos));
    plan->sends.push_back(std::move(ps));
    it = pending_sends_.erase(it);
  }
  live_plans_.insert(plan.get());
  return plan.release();
}

void ss_cache::ExpandAddr(const KVAddr& a, std::vector<int32_t>* slots, std::vector<int64_t>* rp,
                          std::vector<int32_t>* rb, std::vector<int32_t>* rc) const {
  for (const auto& r : a.ranges) {
    if (rp) {
      rp->push_back(r.page_id);
      rb->push_back(r.slot_begin);
      rc->push_back(r.slot_count);
    }
    for (int32_t s = 0; s < r.slot_count; ++s) {
      slots->push_back(static_cast<int32_t>(r.page_id * P_ + r.slot_begin + s));
    }
  }
}

// Lays the plan out in one device block: everything all L layers share is
// uploaded once (kv_cache.h:8-9, "plan once for all layers").
void ss_cache::PlanToDevice(ss_plan* plan) {
  if (plan->on_device) return;
  plan->n_fold = 0;
  for (const auto& e : plan->entries) plan->n_fold += e.end - e.fold_from;
  const int64_t nf = plan->n_fold, no = plan->total_outputs;
  const int64_t ne = static_cast<int64_t>(plan->entries.size());
  struct SendLayout {
    size_t src, dst, rpage, rbegin, rcount, verdict, staging;
    bool ok = true;
    std::vector<int32_t> dst_slots, rb, rc;
    std::vector<int64_t> rp;
  };
  std::vector<SendLayout> sl(plan->sends.size());
  size_t off = 0;
  auto take = [&](size_t bytes) {
    size_t o = off;
    off += Align(bytes);
    return o;
  };
  const size_t o_fold = take(sizeof(int32_t) * nf);
  const size_t o_out = take(sizeof(int32_t) * no);
  const size_t o_dig = take(sizeof(uint64_t) * no);
  const size_t o_ent = take(sizeof(FoldEntry) * ne);
  const size_t upload_end_core = off;
  for (size_t i = 0; i < plan->sends.size(); ++i) {
    const PlanSend& s = plan->sends[i];
    const int64_t n = s.end - s.begin;
    // MarkSend keeps the reference's checks only (kv_cache.cc:231-243); a
    // malformed destination (overlaps, slot counts not covering the rows)
    // is rejected where the reference's receiver would reject its frame:
    // the send's validation sees no ranges, marks the verdict failed and
    // raises UnknownAddress, and the copy never reads a destination slot.
    bool addr_ok = true;
    try {
      s.dest_addr.Validate();
    } catch (const Error&) {
      addr_ok = false;
    }
    if (addr_ok) ExpandAddr(s.dest_addr, &sl[i].dst_slots, &sl[i].rp, &sl[i].rb, &sl[i].rc);
    if (static_cast<int64_t>(sl[i].dst_slots.size()) != n) {
      addr_ok = false;
      sl[i].dst_slots.clear();
      sl[i].rp.clear();
      sl[i].rb.clear();
      sl[i].rc.clear();
    }
    sl[i].ok = addr_ok;
    const int64_t nr = static_cast<int64_t>(sl[i].rp.size());
    sl[i].src = take(sizeof(int32_t) * n);
    sl[i].dst = take(sizeof(int32_t) * sl[i].dst_slots.size());
    sl[i].rpage = take(sizeof(int64_t) * nr);
    sl[i].rbegin = take(sizeof(int32_t) * nr);
    sl[i].rcount = take(sizeof(int32_t) * nr);
    sl[i].verdict = take(4 * sizeof(int32_t));
  }
  const size_t upload_end = off;
  const size_t o_F = take(sizeof(uint64_t) * nf);
  const size_t o_hin = take(sizeof(uint64_t) * no);
  const size_t o_hout = take(sizeof(uint64_t) * no);
  for (size_t i = 0; i < plan->sends.size(); ++i) {
    const PlanSend& s = plan->sends[i];
    sl[i].staging = peers_.count(s.dest) ? SIZE_MAX : take(sizeof(uint64_t) * (s.end - s.begin) * W_);
  }
  std::vector<uint8_t> host(upload_end, 0);
  {
    int32_t* fold = reinterpret_cast<int32_t*>(host.data() + o_fold);
    int32_t* outs = reinterpret_cast<int32_t*>(host.data() + o_out);
    uint64_t* dig = reinterpret_cast<uint64_t*>(host.data() + o_dig);
    FoldEntry* ent = reinterpret_cast<FoldEntry*>(host.data() + o_ent);
    int64_t fo = 0, oo = 0;
    for (int64_t i = 0; i < ne; ++i) {
      const PlanEntry& e = plan->entries[i];
      const Record* rec = MustGet(e.seq);
      const int64_t nfe = e.end - e.fold_from, noe = e.end - e.begin;
      std::memcpy(fold + fo, e.slots.data(), sizeof(int32_t) * nfe);
      std::memcpy(outs + oo, e.slots.data() + (e.begin - e.fold_from), sizeof(int32_t) * noe);
      std::memcpy(dig + oo, e.digests.data(), sizeof(uint64_t) * noe);
      ent[i] = FoldEntry{fo, nfe, e.begin - e.fold_from, oo, e.fold_from,
                         d_fold_sums_ + static_cast<int64_t>(rec->fold_row) * L_};
      fo += nfe;
      oo += noe;
    }
    for (size_t i = 0; i < plan->sends.size(); ++i) {
      const PlanSend& s = plan->sends[i];
      std::memcpy(host.data() + sl[i].src, s.src_slots.data(), sizeof(int32_t) * s.src_slots.size());
      std::memcpy(host.data() + sl[i].dst, sl[i].dst_slots.data(),
                  sizeof(int32_t) * sl[i].dst_slots.size());
      std::memcpy(host.data() + sl[i].rpage, sl[i].rp.data(), sizeof(int64_t) * sl[i].rp.size());
      std::memcpy(host.data() + sl[i].rbegin, sl[i].rb.data(), sizeof(int32_t) * sl[i].rb.size());
      std::memcpy(host.data() + sl[i].rcount, sl[i].rc.data(), sizeof(int32_t) * sl[i].rc.size());
    }
  }
  (void)upload_end_core;
  plan->dev = DevAlloc(off, stream_);
  uint8_t* base = static_cast<uint8_t*>(plan->dev.ptr);
  if (upload_end > 0) {
    H2D(base, host.data(), upload_end, stream_, "H2D plan");
  }
  plan->d_fold_slots = reinterpret_cast<int32_t*>(base + o_fold);
  plan->d_out_slots = reinterpret_cast<int32_t*>(base + o_out);
  plan->d_digests = reinterpret_cast<uint64_t*>(base + o_dig);
  plan->d_entries = reinterpret_cast<FoldEntry*>(base + o_ent);
  plan->d_F = reinterpret_cast<uint64_t*>(base + o_F);
  plan->d_hidden_in = reinterpret_cast<uint64_t*>(base + o_hin);
  plan->d_hidden_out = reinterpret_cast<uint64_t*>(base + o_hout);
  plan->dsend.resize(plan->sends.size());
  for (size_t i = 0; i < plan->sends.size(); ++i) {
    auto& d = plan->dsend[i];
    d.src_slots = reinterpret_cast<int32_t*>(base + sl[i].src);
    d.dst_slots = reinterpret_cast<int32_t*>(base + sl[i].dst);
    d.range_page = reinterpret_cast<int64_t*>(base + sl[i].rpage);
    d.range_begin = reinterpret_cast<int32_t*>(base + sl[i].rbegin);
    d.range_count = reinterpret_cast<int32_t*>(base + sl[i].rcount);
    d.verdict = reinterpret_cast<int32_t*>(base + sl[i].verdict);
    d.staging = sl[i].staging == SIZE_MAX ? nullptr : reinterpret_cast<uint64_t*>(base + sl[i].staging);
    d.n_ranges = static_cast<int64_t>(sl[i].rp.size());  // 0 when the address is malformed
  }
  plan->on_device = true;
}

void ss_cache::FreePlanDevice(ss_plan* plan) {
  if (plan->dev.ptr) {
    cudaStreamSynchronize(comm_stream_);
    for (auto& [st, u] : user_streams_) {
      if (u.gen != 0) cudaEventSynchronize(u.ev);
    }
    cudaStreamSynchronize(stream_);
    cudaFree(plan->dev.ptr);
    plan->dev = DevBlock{};
  }
  if (plan->d_partial || plan->d_chunks) {
    cudaDeviceSynchronize();
    if (plan->d_partial) cudaFree(plan->d_partial);
    if (plan->d_chunks) cudaFree(plan->d_chunks);
    plan->d_partial = nullptr;
    plan->d_chunks = nullptr;
    plan->pages_ready = false;
  }
}

void ss_cache::DestroyPlan(ss_plan* plan) {
  live_plans_.erase(plan);
  if (plan->upload_ev != nullptr) cudaEventDestroy(plan->upload_ev);
  for (auto& d : plan->dsend)
    if (d.validated_ev != nullptr) cudaEventDestroy(d.validated_ev);
  if (device_ >= 0 && (plan->dev.ptr || plan->d_partial || plan->d_chunks)) {
    cudaSetDevice(device_);
    OrderAfterUser();
    DevFree(plan->dev, stream_);
    if (plan->d_partial || plan->d_chunks) {
      Sync();
      if (plan->d_partial) cudaFree(plan->d_partial);
      if (plan->d_chunks) cudaFree(plan->d_chunks);
    }
  }
  delete plan;
}

// ---------------------------------------------------------------------------
// Computation stage
// ---------------------------------------------------------------------------
const PeerTarget& ss_cache::PeerFor(Rank dest) const {
  auto it = peers_.find(dest);
  if (it == peers_.end()) Throw(kPeerUnreachable, "no peer attached for rank " + std::to_string(dest));
  return it->second;
}

void ss_cache::LaunchRemote(const PeerTarget& peer, const int32_t* d_src_slots,
                            const int32_t* d_dst_slots, const int64_t* d_rpage,
                            const int32_t* d_rbegin, const int32_t* d_rcount, int64_t n_ranges,
                            int32_t* d_verdict, int64_t n_rows, int32_t lb, int32_t le,
                            cudaStream_t s, cudaEvent_t after, ss_plan::DevSend* ds) {
  // A plan whose address an earlier launch validated: no validation grid,
  // the copy checks that the receiver's window is the one validated (first
  // page still maps to it, open-generation unchanged).  Per-layer sends of
  // one plan pay the validation once.
  const bool gen_check = ds != nullptr && ds->validated_gen != 0 && peer.win_gen != nullptr &&
                         GenCheckEnabled();
  if (gen_check) {
    CudaCheck(cudaStreamWaitEvent(s, ds->validated_ev, 0), "wait validation");
  } else if (peer.local != nullptr) {
    // The receiver's window must be open on its device before validation.
    CudaCheck(cudaStreamWaitEvent(s, peer.local->window_ev_, 0), "wait window");
  }
  ValidateParams v{};
  v.range_page = d_rpage;
  v.range_begin = d_rbegin;
  v.range_count = d_rcount;
  v.n_ranges = n_ranges;
  v.page_window = peer.page_window;
  v.expecting = peer.expecting;
  v.num_pages = peer.num_pages;
  v.P = peer.P;
  v.verdict = d_verdict;
  v.status = d_status_;
  v.win_gen = peer.win_gen;
  v.gen = gen_check ? ds->validated_gen : NextLaunchGen();
  // Small addresses (a few pages): each copy CTA validates the address
  // itself, one launch instead of validation + copy (a 16-token migration
  // is launch-bound).  Larger ones: a validation grid ahead of the producer,
  // the copy a programmatic dependent of it.
  const bool inline_validate = !gen_check && n_ranges * peer.P <= InlineValidateSlots();
  const bool grid_validate = !gen_check && !inline_validate;
  if (grid_validate) launch_validate_remote(v, s);
  // Validation ahead of the producer: only the copy waits for its writes.
  if (after != nullptr) CudaCheck(cudaStreamWaitEvent(s, after, 0), "wait producer");
  CopyParams c{};
  const int64_t src_lw = num_pages_ * P_ * W_, dst_lw = peer.num_pages * peer.P * W_;
  c.src = d_pool_ + lb * src_lw;
  c.src_layer_words = src_lw;
  c.src_idx = d_src_slots;
  c.dst = peer.pool + lb * dst_lw;
  c.dst_layer_words = dst_lw;
  c.dst_idx = d_dst_slots;
  c.dst_fill = peer.fill + lb * peer.num_pages * peer.P;
  c.dst_fill_layer = peer.num_pages * peer.P;
  c.fill_value = 2;  // FillState::kReceivedRemote
  c.n_rows = n_rows;
  c.layer0 = lb;
  c.n_layers = le - lb;
  c.W = W_;
  c.win_received = peer.win_received;
  c.win_layer_rows = peer.win_layer_rows;
  c.win_layers = peer.L;
  c.verdict = d_verdict;
  c.status = d_status_;
  c.sys_scope = (peer.device != device_ || force_sys_scope_) ? 1 : 0;
  c.pdl = after == nullptr ? 1 : 0;  // overlaps the copy grid's launch with its predecessor
  c.gen = v.gen;
  c.max_ctas = send_ctas_;
  c.inline_validate = inline_validate ? 1 : 0;
  c.val = v;
  c.gen_check = gen_check ? 1 : 0;
  c.win_gen = peer.win_gen;
  c.page_window = peer.page_window;
  c.first_page = d_rpage;
  // Right behind its validation grid (no producer event between them): the
  // first rows may be read before the grid dependency wait.
  c.prefetch_src = (grid_validate && after == nullptr) ? 1 : 0;
  launch_copy_rows(c, s, num_sms_);
  CountLaunches(grid_validate ? 2 : 1);
  if (ds != nullptr && !gen_check && n_ranges > 0) {
    // This launch validated the plan's address: later launches may check
    // the window's generation instead (ordered behind this validation).
    if (ds->validated_ev == nullptr)
      CudaCheck(cudaEventCreateWithFlags(&ds->validated_ev, cudaEventDisableTiming), "event");
    CudaCheck(cudaEventRecord(ds->validated_ev, s), "cudaEventRecord");
    ds->validated_gen = v.gen;
  }
}

// kv_cache.cc:308-371 on device.  Hidden buffers are device pointers; the
// host wrapper (Attention) stages them.
void ss_cache::AttentionAsync(ss_plan* plan, int32_t layer, const uint64_t* hin, uint64_t* hout,
                              cudaStream_t s) {
  RequireDevice("Attention");
  MKV_CHECK(layer == plan->next_layer && layer < L_, kLayerOrderViolation,
            "expected layer " + std::to_string(plan->next_layer) + ", got " +
                std::to_string(layer));
  if (!plan->on_device) OrderAfterUser();  // the upload follows earlier user work
  PlanToDevice(plan);
  OrderLaunch(s);
  uint64_t* pool_l = PoolLayer(layer);
  uint8_t* fill_l = d_fill_ + static_cast<int64_t>(layer) * num_pages_ * P_;
  // Hot loop A: KV write for Empty output slots, entry digests, fold + hidden.
  launch_attn_write_hash(pool_l, fill_l, plan->d_out_slots, plan->d_digests, plan->total_outputs,
                         layer, W_, s, num_sms_);
  launch_entry_digest(pool_l, plan->d_fold_slots, plan->n_fold, W_, plan->d_F, s, num_sms_);
  launch_fold_scan(plan->d_entries, static_cast<int64_t>(plan->entries.size()), plan->d_F, hin,
                   hout, layer, s);
  CountLaunches(3);
  for (const auto& e : plan->entries) {
    Record* rec = MustGet(e.seq);
    rec->touched_end = std::max(rec->touched_end, e.end);
    CheckFilled(rec, e.fold_from, e.begin, layer, "fold over empty slot", nullptr);
    if (layer == L_ - 1) {
      rec->fold_frontier = e.end;
      AdvanceCommitted(rec, e.end);
    }
  }
  // Hot loop B: stream this layer's KV of every marked send, on the
  // communication stream, ordered after this layer's writes only.
  if (!plan->sends.empty()) {
    for (size_t i = 0; i < plan->sends.size(); ++i) {
      const PlanSend& snd = plan->sends[i];
      CheckFilled(MustGet(snd.seq), snd.begin, snd.end, layer, "sending empty slot", plan);
      PeerFor(snd.dest);
    }
    CudaCheck(cudaEventRecord(layer_ev_, s), "cudaEventRecord");
    CudaCheck(cudaStreamWaitEvent(comm_stream_, layer_ev_, 0), "cudaStreamWaitEvent");
    for (size_t i = 0; i < plan->sends.size(); ++i) {
      const PlanSend& snd = plan->sends[i];
      auto& d = plan->dsend[i];
      LaunchRemote(PeerFor(snd.dest), d.src_slots, d.dst_slots, d.range_page, d.range_begin,
                   d.range_count, d.n_ranges, d.verdict, snd.end - snd.begin, layer, layer + 1,
                   comm_stream_, nullptr, &d);
    }
    CudaCheck(cudaEventRecord(comm_ev_, comm_stream_), "cudaEventRecord");
    comm_pending_ = true;
    ++comm_gen_;
  }
  if (s != stream_) NoteUser(s);
  ++plan->next_layer;
}

// Host-buffer Attention: stages hidden states, sends to attached peers
// device-direct and everything else through the host sink (the
// reference's FrameSink path).
void ss_cache::Attention(ss_plan* plan, int32_t layer, const uint64_t* hidden_in,
                         uint64_t* hidden_out, int64_t n, ss_frame_sink sink, void* user) {
  RequireDevice("Attention");
  MKV_CHECK(layer == plan->next_layer && layer < L_, kLayerOrderViolation,
            "expected layer " + std::to_string(plan->next_layer) + ", got " +
                std::to_string(layer));
  MKV_ICHECK(n == plan->total_outputs, "hidden input size mismatch");
  OrderAfterUser();
  PlanToDevice(plan);
  if (n > 0) {
    H2D(plan->d_hidden_in, hidden_in, sizeof(uint64_t) * n, stream_, "H2D hidden");
  }
  uint64_t* pool_l = PoolLayer(layer);
  uint8_t* fill_l = d_fill_ + static_cast<int64_t>(layer) * num_pages_ * P_;
  launch_attn_write_hash(pool_l, fill_l, plan->d_out_slots, plan->d_digests, plan->total_outputs,
                         layer, W_, stream_, num_sms_);
  launch_entry_digest(pool_l, plan->d_fold_slots, plan->n_fold, W_, plan->d_F, stream_, num_sms_);
  launch_fold_scan(plan->d_entries, static_cast<int64_t>(plan->entries.size()), plan->d_F,
                   plan->d_hidden_in, plan->d_hidden_out, layer, stream_);
  CountLaunches(3);
  if (n > 0) {
    D2H(hidden_out, plan->d_hidden_out, sizeof(uint64_t) * n, stream_, "D2H hidden");
  }
  for (const auto& e : plan->entries) {
    Record* rec = MustGet(e.seq);
    rec->touched_end = std::max(rec->touched_end, e.end);
    CheckFilled(rec, e.fold_from, e.begin, layer, "fold over empty slot", nullptr);
    if (layer == L_ - 1) {
      rec->fold_frontier = e.end;
      AdvanceCommitted(rec, e.end);
    }
  }
  std::vector<uint64_t> payload;
  for (size_t i = 0; i < plan->sends.size(); ++i) {
    const PlanSend& snd = plan->sends[i];
    CheckFilled(MustGet(snd.seq), snd.begin, snd.end, layer, "sending empty slot", plan);
    auto& d = plan->dsend[i];
    const int64_t rows = snd.end - snd.begin;
    auto pit = peers_.find(snd.dest);
    if (pit != peers_.end()) {
      LaunchRemote(pit->second, d.src_slots, d.dst_slots, d.range_page, d.range_begin,
                   d.range_count, d.n_ranges, d.verdict, rows, layer, layer + 1, stream_,
                   nullptr, &d);
      continue;
    }
    if (!sink) continue;
    // Gather this layer's rows in token order, then hand them to the sink.
    CopyParams c{};
    c.src = pool_l;
    c.src_idx = d.src_slots;
    c.dst = d.staging;
    c.n_rows = rows;
    c.layer0 = layer;
    c.n_layers = 1;
    c.W = W_;
    launch_copy_rows(c, stream_, num_sms_);
    CountLaunches(1);
    payload.resize(static_cast<size_t>(rows) * W_);
    if (rows > 0) {
      D2H(payload.data(), d.staging, sizeof(uint64_t) * rows * W_, stream_, "D2H payload");
    }
    Sync();
    std::vector<ss_slot_range> rr;
    for (const auto& r : snd.dest_addr.ranges) rr.push_back({r.page_id, r.slot_begin, r.slot_count});
    ss_addr a{snd.dest_addr.token_begin, snd.dest_addr.token_count,
              static_cast<int64_t>(rr.size()), rr.data(), static_cast<int64_t>(rr.size())};
    sink(user, layer, snd.seq, snd.begin, snd.end, snd.dest, &a, snd.user_tag, payload.data(),
         static_cast<int64_t>(payload.size()));
  }
  Sync();
  ++plan->next_layer;
}

// kv_cache.cc:373-387 into device memory.
void ss_cache::GatherRange(SeqId seq, int64_t begin, int64_t end, int32_t layer, uint64_t* out,
                           cudaStream_t s) {
  MKV_CHECK(layer >= 0 && layer < L_, kInvalidArgument, "layer out of range");
  GatherRangeLayers(seq, begin, end, layer, layer + 1, out, s);
}

// GatherRange of layers [lb, le) in one launch: out[le - lb][end - begin][W].
void ss_cache::GatherRangeLayers(SeqId seq, int64_t begin, int64_t end, int32_t lb, int32_t le,
                                 uint64_t* out, cudaStream_t s) {
  RequireDevice("GatherRange");
  const Record* rec = MustGet(seq);
  MKV_CHECK(lb >= 0 && lb < le && le <= L_, kInvalidArgument, "layer out of range");
  MKV_CHECK(begin >= 0 && begin <= end, kInvalidArgument, "bad gather range");
  MKV_ICHECK(end <= rec->alloc_len, "position not allocated");
  // As in LaunchDirectSend: a live forward plan covering the range proves it
  // (frames encoded layer by layer during a prefill need no host sync).
  if (end > rec->committed_hint &&
      !CoveredByLivePlan(seq, std::max(begin, rec->committed_hint), end)) {
    AdvanceCommitted(MustGet(seq));
    for (int32_t l = lb; l < le && end > rec->committed_hint; ++l) {
      CheckFilled(rec, begin, end, l, "gather over empty slot", nullptr);
    }
  }
  const int64_t n = end - begin;
  if (n == 0) return;
  OrderLaunch(s);
  CopyParams c{};
  c.src = PoolLayer(lb);
  c.src_layer_words = num_pages_ * P_ * W_;
  c.src_idx = rec->d_slots + begin;
  c.dst = out;
  c.dst_layer_words = n * W_;
  c.n_rows = n;
  c.layer0 = lb;
  c.n_layers = le - lb;
  c.W = W_;
  c.pdl = 1;  // launch overlaps the previous kernel's tail; waits for it before reading
  launch_copy_rows(c, s, num_sms_);
  CountLaunches(1);
  if (s != stream_) NoteUser(s);
}

// kv_cache.cc:389-407
KVAddr ss_cache::BuildAddr(SeqId seq, int64_t begin, int64_t end) {
  const Record* rec = MustGet(seq);
  MKV_CHECK(begin >= rec->fork_len, kInvalidArgument, "address must cover own slots only");
  KVAddr addr;
  addr.token_begin = begin;
  addr.token_count = end - begin;
  if (end > begin) {
    MKV_ICHECK(begin >= 0 && end <= rec->alloc_len, "position not allocated");
    addr.ranges.reserve((end - begin) / P_ + 2);
  }
  const int32_t* table = rec->slots.data();
  for (int64_t pos = begin; pos < end;) {
    const int32_t slot = table[pos];
    const int64_t page = slot >> page_shift_;  // page_size is a power of two
    const int32_t s = slot & (P_ - 1);
    // Own pages are filled slot 0..P-1 in position order, so a run usually
    // spans to the page end; confirm the run end, else step one position.
    int64_t run = std::min<int64_t>(P_ - s, end - pos);
    if (run > 1 && table[pos + run - 1] != slot + run - 1) run = 1;
    if (!addr.ranges.empty() && addr.ranges.back().page_id == page &&
        addr.ranges.back().slot_begin + addr.ranges.back().slot_count == s) {
      addr.ranges.back().slot_count += static_cast<int32_t>(run);
    } else {
      addr.ranges.push_back({page, s, static_cast<int32_t>(run)});
    }
    pos += run;
  }
  addr.Validate();
  return addr;
}

// KV append from the producing layer's dense K||V rows (write rule of
// kv_cache.cc:328-334).
void ss_cache::AppendRows(ss_plan* plan, int32_t layer, const void* rows, cudaStream_t s) {
  AppendRowsLayers(plan, layer, layer + 1, rows, s);
}

void ss_cache::AppendRowsLayers(ss_plan* plan, int32_t lb, int32_t le, const void* rows,
                                cudaStream_t s) {
  RequireDevice("AppendRows");
  MKV_CHECK(lb >= 0 && lb < le && le <= L_, kInvalidArgument, "layer out of range");
  if (!plan->on_device) OrderAfterUser();  // the upload follows earlier user work
  PlanToDevice(plan);
  OrderLaunch(s);
  CopyParams c{};
  c.src = static_cast<const uint64_t*>(rows);
  c.src_layer_words = plan->total_outputs * W_;
  c.dst = PoolLayer(lb);
  c.dst_layer_words = num_pages_ * P_ * W_;
  c.dst_idx = plan->d_out_slots;
  c.dst_fill = d_fill_ + static_cast<int64_t>(lb) * num_pages_ * P_;
  c.dst_fill_layer = num_pages_ * P_;
  c.fill_value = 1;  // FillState::kComputedLocal
  c.n_rows = plan->total_outputs;
  c.layer0 = lb;
  c.n_layers = le - lb;
  c.W = W_;
  c.pdl = 1;  // launch overlaps the previous kernel's tail; waits for it before reading
  launch_copy_rows(c, s, num_sms_);
  CountLaunches(1);
  for (const auto& e : plan->entries) {
    Record* rec = MustGet(e.seq);
    rec->touched_end = std::max(rec->touched_end, e.end);
  }
  if (s != stream_) NoteUser(s);
}

// KV append fused with remote_send ("write-through"): the producing
// layer's dense K||V rows are read once and stored both into this engine's
// output slots (the Attention write rule, kv_cache.cc:328-334) and into the
// peer's reserved pages for the send plan's range (the send loop,
// kv_cache.cc:353-367, + ApplyRemoteWrite's Empty-only rule), with the
// peer's per-layer window counters published by the same kernel.  A row
// whose local slot was already non-Empty is sent from that slot, as the
// reference sends the pool contents after the write.  The receiver's
// address is validated by a kernel ahead of it on `s` (the fused kernel is
// its programmatic dependent), so a rejected address writes nothing remote
// while the local append still happens.
void ss_cache::AppendRowsSend(ss_plan* fwd, ss_plan* send, int32_t lb, int32_t le,
                              const void* rows, cudaStream_t s) {
  RequireDevice("AppendRowsSend");
  MKV_CHECK(lb >= 0 && lb < le && le <= L_, kInvalidArgument, "layer out of range");
  MKV_CHECK(send->is_direct_send, kInvalidArgument, "not a direct-send plan");
  MKV_CHECK(!fwd->is_direct_send && !fwd->is_decode_plan, kInvalidArgument, "not a forward plan");
  const PlanSend& snd = send->sends[0];
  int64_t off = 0;
  bool covered = false;
  for (const auto& e : fwd->entries) {
    if (e.seq == snd.seq && e.begin <= snd.begin && snd.end <= e.end) {
      off += snd.begin - e.begin;
      covered = true;
      break;
    }
    off += e.end - e.begin;
  }
  MKV_CHECK(covered, kInvalidArgument, "the send range is not output by the forward plan");
  if ((W_ != 512 && W_ != 128) || send_mode_ == SS_SEND_COPY_ENGINE) {
    // Rows the fan-out kernel is not specialised for, or a copy-engine
    // mover: the append, then the send behind it on the same stream.
    AppendRowsLayers(fwd, lb, le, rows, s);
    LaunchDirectSend(send, lb, le, s);
    return;
  }
  if (!fwd->on_device) OrderAfterUser();
  PlanToDevice(fwd);
  const PeerTarget& peer = PeerFor(snd.dest);
  OrderLaunch(s);
  const auto& d = send->dsend[0];
  // Validation off the producer's critical path: on a high-priority side
  // stream (behind the plan's upload and the receiver's window open), so it
  // runs while the producing layer still computes; `s` only waits for its
  // event.  A validation of a later layer may rewrite the verdict while
  // this layer's copy reads it: on success with the same window, on failure
  // with -1, which makes this copy fail closed too.
  const bool side = [] {
    const char* e = std::getenv("MICROKV_FUSED_VALIDATE");
    return e == nullptr || std::strcmp(e, "inline") != 0;
  }();
  cudaStream_t vs = s;
  if (side) {
    if (fused_vstream_ == nullptr) {
      int lo = 0, hi = 0;
      CudaCheck(cudaDeviceGetStreamPriorityRange(&lo, &hi), "priority range");
      CudaCheck(cudaStreamCreateWithPriority(&fused_vstream_, cudaStreamNonBlocking, hi), "stream");
      CudaCheck(cudaEventCreateWithFlags(&fused_vev_, cudaEventDisableTiming), "event");
    }
    vs = fused_vstream_;
    // Behind the send plan's row-map upload only — not behind `s`, where the
    // producing layer's compute is queued.
    CudaCheck(cudaStreamWaitEvent(vs, send->upload_ev, 0), "wait plan");
  }
  if (peer.local != nullptr) CudaCheck(cudaStreamWaitEvent(vs, peer.local->window_ev_, 0), "wait window");
  ValidateParams v{};
  v.range_page = d.range_page;
  v.range_begin = d.range_begin;
  v.range_count = d.range_count;
  v.n_ranges = d.n_ranges;
  v.page_window = peer.page_window;
  v.expecting = peer.expecting;
  v.num_pages = peer.num_pages;
  v.P = peer.P;
  v.verdict = d.verdict;
  v.status = d_status_;
  v.gen = NextLaunchGen();
  launch_validate_remote(v, vs);
  if (side) {
    CudaCheck(cudaEventRecord(fused_vev_, vs), "cudaEventRecord");
    CudaCheck(cudaStreamWaitEvent(s, fused_vev_, 0), "wait validation");
  }
  FanoutParams f{};
  f.src = static_cast<const uint64_t*>(rows);
  f.src_layer_words = fwd->total_outputs * W_;
  f.src_idx = nullptr;
  f.n_rows = fwd->total_outputs;
  f.layer0 = lb;
  f.n_layers = le - lb;
  f.W = W_;
  f.n_dest = 2;
  f.gen = v.gen;
  f.pdl = 1;
  f.truth = 0;
  // 0: this engine's output slots (no validation, no counters)
  f.dst[0] = PoolLayer(lb);
  f.dst_layer_words[0] = num_pages_ * P_ * W_;
  f.dst_idx[0] = fwd->d_out_slots;
  f.dst_fill[0] = d_fill_ + static_cast<int64_t>(lb) * num_pages_ * P_;
  f.dst_fill_layer[0] = num_pages_ * P_;
  f.fill_value[0] = 1;  // FillState::kComputedLocal
  f.row_off[0] = 0;
  f.row_cnt[0] = fwd->total_outputs;
  // 1: the peer's reserved pages for the send range
  const int64_t dst_lw = peer.num_pages * peer.P * W_;
  f.dst[1] = peer.pool + lb * dst_lw;
  f.dst_layer_words[1] = dst_lw;
  f.dst_idx[1] = d.dst_slots;
  f.dst_fill[1] = peer.fill + lb * peer.num_pages * peer.P;
  f.dst_fill_layer[1] = peer.num_pages * peer.P;
  f.fill_value[1] = 2;  // FillState::kReceivedRemote
  f.row_off[1] = off;
  f.row_cnt[1] = snd.end - snd.begin;
  f.win_received[1] = peer.win_received;
  f.win_layer_rows[1] = peer.win_layer_rows;
  f.win_layers[1] = peer.L;
  f.verdict[1] = d.verdict;
  f.sys_scope = (peer.device != device_ || force_sys_scope_) ? 1 : 0;
  launch_copy_rows_fanout(f, s, num_sms_);
  CountLaunches(2);
  for (const auto& e : fwd->entries) {
    Record* rec = MustGet(e.seq);
    rec->touched_end = std::max(rec->touched_end, e.end);
  }
  if (s != stream_) NoteUser(s);
}

// ---------------------------------------------------------------------------
// Transfer agent
// ---------------------------------------------------------------------------
// kv_cache.cc:409-463.  Validation, dedupe and window accounting are the
// reference's, on the host; the scatter of Empty slots runs on the device.
int ss_cache::ApplyRemoteWrite(const KVAddr& addr, int32_t layer, const uint64_t* payload,
                               int64_t n_words, bool on_device, uint64_t tag, cudaStream_t s,
                               bool agent) {
  MKV_CHECK(n_words == addr.token_count * W_, kInvalidArgument, "payload size mismatch");
  RequireDevice("ApplyRemoteWrite");
  MKV_CHECK(layer >= 0 && layer < L_, kInvalidArgument, "layer out of range");
  std::lock_guard<std::mutex> lock(recv_mu_);
  SeqId owner = -1;
  for (const auto& r : addr.ranges) {
    if (r.page_id < 0 || r.page_id >= num_pages_) return SS_APPLY_UNKNOWN_ADDRESS;
    const SeqId po = page_owner_[r.page_id];
    if (po < 0) return SS_APPLY_UNKNOWN_ADDRESS;
    if (owner == -1) owner = po;
    if (po != owner) return SS_APPLY_UNKNOWN_ADDRESS;
    for (int32_t sl = r.slot_begin; sl < r.slot_begin + r.slot_count; ++sl) {
      if (sl < 0 || sl >= P_ || !expecting_[r.page_id * P_ + sl]) return SS_APPLY_UNKNOWN_ADDRESS;
    }
  }
  auto it = records_.find(owner);
  if (it == records_.end() || !it->second->window.has_value()) return SS_APPLY_UNKNOWN_ADDRESS;
  Record* rec = it->second.get();
  Window& win = *rec->window;
  if (!win.applied.insert({tag, layer, addr.token_begin}).second) return SS_APPLY_DUPLICATE;

  std::vector<int32_t> dst;
  ExpandAddr(addr, &dst, nullptr, nullptr, nullptr);
  const int64_t n = static_cast<int64_t>(dst.size());
  if (n > 0) {
    // Host payload (the transfer agent, possibly on its own thread): the
    // receive stream, after the windows opened so far; a device payload on a
    // caller stream (executor thread): ordered with the executor's streams.
    cudaStream_t st = agent ? recv_stream_ : (s ? s : stream_);
    if (agent) {
      CudaCheck(cudaStreamWaitEvent(st, window_ev_, 0), "wait window");
    } else {
      OrderLaunch(st);
    }
    const size_t o_pay = Align(sizeof(int32_t) * n);
    DevBlock b = DevAlloc(o_pay + (on_device ? 0 : sizeof(uint64_t) * n_words), st);
    uint8_t* base = static_cast<uint8_t*>(b.ptr);
    H2D(base, dst.data(), sizeof(int32_t) * n, st, "H2D slots");
    const uint64_t* src = payload;
    if (!on_device) {
      H2D(base + o_pay, payload, sizeof(uint64_t) * n_words, st, "H2D payload");
      src = reinterpret_cast<const uint64_t*>(base + o_pay);
    }
    CopyParams c{};
    c.src = src;
    c.dst = PoolLayer(layer);
    c.dst_idx = reinterpret_cast<int32_t*>(base);
    c.dst_fill = d_fill_ + static_cast<int64_t>(layer) * num_pages_ * P_;
    c.fill_value = 2;  // FillState::kReceivedRemote
    c.n_rows = n;
    c.layer0 = layer;
    c.n_layers = 1;
    c.W = W_;
    launch_copy_rows(c, st, num_sms_);
    CountLaunches(1);
    DevFree(b, st);
    if (agent) {
      CudaCheck(cudaStreamSynchronize(st), "cudaStreamSynchronize recv");
    } else if (st == stream_) {
      Sync();
    } else {
      NoteUser(st);
    }
  }
  // Every addressed slot counts, filled or not (kv_cache.cc:452-456).
  win.received += n;
  if (static_cast<int32_t>(win.received_layer.size()) == L_) win.received_layer[layer] += n;
  if (!win.complete && win.received + static_cast<int64_t>(win.dev_received) >= win.expected) {
    win.complete = true;
    completed_windows_.push_back(owner);
  }
  return SS_APPLY_OK;
}

// Reads the device counters of windows that peers fill device-direct.
void ss_cache::PollDeviceWindows() {
  if (device_ < 0) return;
  std::vector<Record*> open;
  {
    std::lock_guard<std::mutex> lock(recv_mu_);
    for (auto& [id, rec] : records_) {
      if (rec->window && !rec->window->complete && rec->window->dev_id >= 0) open.push_back(rec.get());
    }
  }
  if (open.empty()) return;
  for (size_t i = 0; i < open.size(); ++i) {
    D2H(h_pinned_ + i, d_win_received_ + open[i]->window->dev_id,
                              sizeof(unsigned long long), stream_, "D2H window");
  }
  Sync();
  std::lock_guard<std::mutex> lock(recv_mu_);
  for (size_t i = 0; i < open.size(); ++i) {
    Window& w = *open[i]->window;
    w.dev_received = h_pinned_[i];
    if (!w.complete && w.received + static_cast<int64_t>(w.dev_received) >= w.expected) {
      w.complete = true;
      completed_windows_.push_back(open[i]->id);
    }
  }
}

// kv_cache.cc:465-480
std::vector<SeqId> ss_cache::DrainReceiveCompletions() {
  PollDeviceWindows();
  std::vector<SeqId> done;
  {
    std::lock_guard<std::mutex> lock(recv_mu_);
    done.swap(completed_windows_);
  }
  for (SeqId seq : done) {
    auto it = records_.find(seq);
    if (it == records_.end()) continue;
    Record* rec = it->second.get();
    AdvanceCommitted(rec);
    rec->finished = true;
    CommitToTree(seq);
    CloseDeviceWindow(rec);
  }
  return done;
}

// DirectSend: GatherRange + ApplyRemoteWrite per layer, fused into one
// launch that stores the sender's rows straight into the receiver's pages.
// Declaration: resolve the source page table and expand the destination
// address once, upload both row maps with the range table in one copy.
ss_plan* ss_cache::BeginDirectSend(SeqId seq, int64_t begin, int64_t end, Rank dest,
                                   const KVAddr& addr, uint64_t tag) {
  RequireDevice("DirectSend");
  Record* rec = MustGet(seq);
  MKV_CHECK(begin >= 0 && end <= static_cast<int64_t>(rec->tokens.size()) && begin <= end,
            kInvalidArgument, "send range outside sequence");
  MKV_CHECK(addr.token_count == end - begin, kAddrMismatch,
            "destination covers " + std::to_string(addr.token_count) + " tokens, range has " +
                std::to_string(end - begin));
  MKV_CHECK(addr.token_begin == begin, kAddrMismatch, "destination token_begin mismatch");
  // The address may come from another process (decoded, not built here):
  // the same checks as the reference's frame decode (kv_addr.cc:16-30), so
  // the expanded slot list has exactly one destination slot per row.
  addr.Validate();
  PeerFor(dest);
  MKV_ICHECK(end <= rec->alloc_len, "position not allocated");
  auto plan = std::make_unique<ss_plan>();
  plan->owner = this;
  PlanSend ps;
  ps.seq = seq;
  ps.begin = begin;
  ps.end = end;
  ps.dest = dest;
  ps.dest_addr = addr;
  ps.user_tag = tag;
  plan->sends.push_back(std::move(ps));
  std::vector<int32_t> dst;
  std::vector<int64_t> rp;
  std::vector<int32_t> rb, rc;
  ExpandAddr(addr, &dst, &rp, &rb, &rc);
  MKV_CHECK(static_cast<int64_t>(dst.size()) == end - begin, kAddrMismatch,
            "destination slots do not cover the send range");
  const int64_t nr = static_cast<int64_t>(rp.size());
  const size_t o_dst = 0;
  const size_t o_rp = o_dst + Align(sizeof(int32_t) * dst.size());
  const size_t o_rb = o_rp + Align(sizeof(int64_t) * nr);
  const size_t o_rc = o_rb + Align(sizeof(int32_t) * nr);
  const size_t o_v = o_rc + Align(sizeof(int32_t) * nr);
  const size_t total = o_v + Align(4 * sizeof(int32_t));
  std::vector<uint8_t> host(total, 0);
  std::memcpy(host.data() + o_dst, dst.data(), sizeof(int32_t) * dst.size());
  std::memcpy(host.data() + o_rp, rp.data(), sizeof(int64_t) * nr);
  std::memcpy(host.data() + o_rb, rb.data(), sizeof(int32_t) * nr);
  std::memcpy(host.data() + o_rc, rc.data(), sizeof(int32_t) * nr);
  // A fresh block and a host upload: nothing earlier user work may still be
  // reading (plan blocks are freed on the internal stream after the user
  // work that read them), so no wait for the user streams here — the copy
  // of the previous request keeps running while this plan uploads.
  BeginInternal();
  plan->dev = DevAlloc(total, stream_);
  uint8_t* base = static_cast<uint8_t*>(plan->dev.ptr);
  H2D(base, host.data(), total, stream_, "H2D send");
  plan->dsend.resize(1);
  auto& d = plan->dsend[0];
  d.src_slots = nullptr;  // read from the sender's HBM page table at launch
  d.dst_slots = reinterpret_cast<int32_t*>(base + o_dst);
  d.range_page = reinterpret_cast<int64_t*>(base + o_rp);
  d.range_begin = reinterpret_cast<int32_t*>(base + o_rb);
  d.range_count = reinterpret_cast<int32_t*>(base + o_rc);
  d.verdict = reinterpret_cast<int32_t*>(base + o_v);
  d.n_ranges = nr;
  plan->on_device = true;
  plan->is_direct_send = true;
  CudaCheck(cudaEventRecord(internal_ev_, stream_), "cudaEventRecord");
  CudaCheck(cudaEventCreateWithFlags(&plan->upload_ev, cudaEventDisableTiming), "event");
  CudaCheck(cudaEventRecord(plan->upload_ev, stream_), "cudaEventRecord");
  live_plans_.insert(plan.get());
  return plan.release();
}

// Computation: validation + one copy launch over rows x [lb, le).  The
// source rows must be non-Empty (GatherRange's MissingKV, kv_cache.cc:379).
void ss_cache::LaunchDirectSend(ss_plan* plan, int32_t lb, int32_t le, cudaStream_t s,
                                cudaEvent_t after) {
  RequireDevice("DirectSend");
  MKV_CHECK(plan->is_direct_send, kInvalidArgument, "not a direct-send plan");
  MKV_CHECK(lb >= 0 && lb <= le && le <= L_, kInvalidArgument, "bad layer range");
  const PlanSend& snd = plan->sends[0];
  Record* rec = MustGet(snd.seq);
  // Positions past the committed prefix must be filled: proven by a live
  // forward plan whose outputs cover them (PrefillThenSend: the caller sends
  // layer l after the plan's layer-l writes on its streams), else by a
  // device scan.  The scan synchronises with the caller's queued work, so
  // the live-plan proof keeps a layer-by-layer send loop free of host syncs.
  if (snd.end > rec->committed_hint &&
      !CoveredByLivePlan(rec->id, std::max(snd.begin, rec->committed_hint), snd.end)) {
    AdvanceCommitted(rec);
    for (int32_t l = lb; l < le && snd.end > rec->committed_hint; ++l) {
      CheckFilled(rec, snd.begin, snd.end, l, "gather over empty slot", nullptr);
    }
  }
  if (lb == le) return;
  const PeerTarget& peer = PeerFor(snd.dest);
  OrderLaunch(s);
  if (send_mode_ == SS_SEND_COPY_ENGINE) {
    LaunchDirectSendCE(plan, peer, rec, lb, le, s, after);
    if (s != stream_) NoteUser(s);
    return;
  }
  auto& d = plan->dsend[0];
  LaunchRemote(peer, rec->d_slots + snd.begin, d.dst_slots, d.range_page, d.range_begin,
               d.range_count, d.n_ranges, d.verdict, snd.end - snd.begin, lb, le, s, after, &d);
  if (s != stream_) NoteUser(s);
}

// Relay chain (context-cache migration to several engines):
// engine i receives a prefix from engine i-1 and forwards each layer to
// engine i+1 as soon as that layer has fully landed here, so every link
// carries the prefix once and the owner's egress is not multiplied by the
// number of targets (a fan-out from the owner pushes k copies through its
// one NVLink port).  The rows being forwarded are proven by this engine's
// own receive counters — a device-side wait per layer, no host sync —
// instead of a fill scan; a wait that times out marks the layer's launch
// rejected (nothing is forwarded) and raises Aborted at Synchronize.
void ss_cache::LaunchRelaySend(ss_plan* plan, int32_t lb, int32_t le, int64_t timeout_ms,
                               cudaStream_t s) {
  RequireDevice("RelaySend");
  MKV_CHECK(plan->is_direct_send, kInvalidArgument, "not a direct-send plan");
  MKV_CHECK(lb >= 0 && lb <= le && le <= L_, kInvalidArgument, "bad layer range");
  MKV_CHECK(timeout_ms > 0, kInvalidArgument, "relay needs a positive timeout");
  const PlanSend& snd = plan->sends[0];
  Record* rec = MustGet(snd.seq);
  const bool receiving = rec->window && rec->window->dev_id >= 0 && !rec->window->complete &&
                         rec->window->begin <= std::max(snd.begin, rec->committed_hint) &&
                         snd.end <= rec->window->end;
  if (!receiving) {  // already landed (or never received): an ordinary DirectSend
    LaunchDirectSend(plan, lb, le, s);
    return;
  }
  if (lb == le || snd.end == snd.begin) return;
  const PeerTarget& peer = PeerFor(snd.dest);
  OrderLaunch(s);
  const auto& d = plan->dsend[0];
  const Window& w = *rec->window;
  // Rows per layer the window still expects from device-direct senders
  // (host-path frames counted on the host are already in place).
  int64_t host_min = INT64_MAX;
  {
    std::lock_guard<std::mutex> lock(recv_mu_);
    for (int32_t l = lb; l < le; ++l) {
      host_min = std::min<int64_t>(host_min, static_cast<int32_t>(w.received_layer.size()) == L_
                                                 ? w.received_layer[l] : 0);
    }
  }
  const int64_t target = std::max<int64_t>(0, (w.end - w.begin) - host_min);
  if (peer.local != nullptr) CudaCheck(cudaStreamWaitEvent(s, peer.local->window_ev_, 0), "wait window");
  ValidateParams v{};
  v.range_page = d.range_page;
  v.range_begin = d.range_begin;
  v.range_count = d.range_count;
  v.n_ranges = d.n_ranges;
  v.page_window = peer.page_window;
  v.expecting = peer.expecting;
  v.num_pages = peer.num_pages;
  v.P = peer.P;
  v.verdict = d.verdict;
  v.status = d_status_;
  v.gen = NextLaunchGen();
  launch_validate_remote(v, s);
  CopyParams c{};
  const int64_t src_lw = num_pages_ * P_ * W_, dst_lw = peer.num_pages * peer.P * W_;
  c.src = d_pool_ + lb * src_lw;
  c.src_layer_words = src_lw;
  c.src_idx = rec->d_slots + snd.begin;
  c.dst = peer.pool + lb * dst_lw;
  c.dst_layer_words = dst_lw;
  c.dst_idx = d.dst_slots;
  c.dst_fill = peer.fill + lb * peer.num_pages * peer.P;
  c.dst_fill_layer = peer.num_pages * peer.P;
  c.fill_value = 2;  // FillState::kReceivedRemote
  c.n_rows = snd.end - snd.begin;
  c.layer0 = lb;
  c.n_layers = le - lb;
  c.W = W_;
  c.win_received = peer.win_received;
  c.win_layer_rows = peer.win_layer_rows;
  c.win_layers = peer.L;
  c.verdict = d.verdict;
  c.status = d_status_;
  c.sys_scope = (peer.device != device_ || force_sys_scope_) ? 1 : 0;
  c.gen = v.gen;
  c.pdl = 1;
  c.max_ctas = send_ctas_;
  launch_relay_rows(c, d_win_layer_rows_ + static_cast<int64_t>(w.dev_id) * L_,
                    static_cast<uint32_t>(target), timeout_ms * 1000000LL, s, num_sms_);
  CountLaunches(2);
  if (s != stream_) NoteUser(s);
}

void ss_cache::SetSendMode(int32_t mode, int32_t max_ctas) {
  MKV_CHECK(mode == SS_SEND_KERNEL || mode == SS_SEND_COPY_ENGINE, kInvalidArgument,
            "unknown send mode");
  MKV_CHECK(max_ctas >= 0, kInvalidArgument, "negative CTA budget");
  RequireDevice("SetSendMode");
  send_mode_ = mode;
  send_ctas_ = max_ctas;
}

// Copy-engine DirectSend.  Validation runs on a side stream (not behind the
// data stream's earlier copies) and the host takes the verdict, so a
// rejected address writes nothing; the rows then move as 2-D copies on the
// copy-engine stream — one per row run, its height the layer range, the
// pools' layer stride as the pitch — and k_copy_rows in no-data mode marks
// the fill states and publishes the window counters behind them.
void ss_cache::LaunchDirectSendCE(ss_plan* plan, const PeerTarget& peer, Record* rec, int32_t lb,
                                  int32_t le, cudaStream_t s, cudaEvent_t after) {
  const PlanSend& snd = plan->sends[0];
  const auto& d = plan->dsend[0];
  if (plan->ce_runs.empty() && snd.end > snd.begin) {
    std::vector<int32_t> dst;
    ExpandAddr(snd.dest_addr, &dst, nullptr, nullptr, nullptr);
    const int32_t* src = rec->slots.data() + snd.begin;
    const int64_t n = snd.end - snd.begin;
    for (int64_t i = 0; i < n; ++i) {
      auto& runs = plan->ce_runs;
      if (!runs.empty() && runs.back().src + runs.back().n == src[i] &&
          runs.back().dst + runs.back().n == dst[i]) {
        ++runs.back().n;
      } else {
        runs.push_back({src[i], dst[i], 1});
      }
    }
  }
  if (verdict_stream_ == nullptr) {
    CudaCheck(cudaStreamCreateWithFlags(&verdict_stream_, cudaStreamNonBlocking), "stream");
    CudaCheck(cudaStreamCreateWithFlags(&ce_stream_, cudaStreamNonBlocking), "stream");
    CudaCheck(cudaEventCreateWithFlags(&verdict_ev_, cudaEventDisableTiming), "event");
    CudaCheck(cudaEventCreateWithFlags(&ce_ev_, cudaEventDisableTiming), "event");
  }
  // The address is validated once per plan, at its first copy-engine launch
  // (the host takes the verdict: copies cannot be cancelled on the device).
  // Later launches of the plan reuse the verdict — a per-launch host wait
  // for a validation kernel would queue behind the compute occupying the
  // SMs and stall the host's layer loop — so the receiver must keep the
  // window open while the send is in flight (its counters still gate
  // completion).
  if (plan->ce_gen == 0) {
    // The plan's upload and the receiver's window open first (the plan's
    // own upload event: the internal stream itself may be queued behind
    // caller streams' compute by now).
    CudaCheck(cudaStreamWaitEvent(verdict_stream_, plan->upload_ev, 0), "wait plan");
    if (peer.local != nullptr) {
      CudaCheck(cudaStreamWaitEvent(verdict_stream_, peer.local->window_ev_, 0), "wait window");
    }
    ValidateParams v{};
    v.range_page = d.range_page;
    v.range_begin = d.range_begin;
    v.range_count = d.range_count;
    v.n_ranges = d.n_ranges;
    v.page_window = peer.page_window;
    v.expecting = peer.expecting;
    v.num_pages = peer.num_pages;
    v.P = peer.P;
    v.verdict = d.verdict;
    v.status = nullptr;  // reported synchronously below
    v.gen = NextLaunchGen();
    launch_validate_remote(v, verdict_stream_);
    D2H(h_pinned_, d.verdict, 2 * sizeof(int32_t), verdict_stream_, "D2H verdict");
    CountLaunches(1);
    CudaCheck(cudaStreamSynchronize(verdict_stream_), "verdict");
    const int32_t* vh = reinterpret_cast<const int32_t*>(h_pinned_);
    if (vh[1] == v.gen || vh[0] < 0) {
      Throw(kUnknownAddress, "the receiver rejected the destination address");
    }
    plan->ce_gen = v.gen;
  }
  // The copies run on ce_stream_ (the copy-engine stream),
  // after `s`'s earlier work and the producer's event, and `s` continues
  // after them.
  CudaCheck(cudaEventRecord(verdict_ev_, s), "cudaEventRecord");
  CudaCheck(cudaStreamWaitEvent(ce_stream_, verdict_ev_, 0), "wait caller stream");
  if (after != nullptr) CudaCheck(cudaStreamWaitEvent(ce_stream_, after, 0), "wait producer");
  const int32_t nl = le - lb;
  const size_t row_b = static_cast<size_t>(W_) * 8;
  const size_t src_lb = static_cast<size_t>(num_pages_) * P_ * row_b;
  const size_t dst_lb = static_cast<size_t>(peer.num_pages) * peer.P * row_b;
  // One strided copy per row run: the run's bytes in every layer of
  // [lb, le), layer pitch on both sides (a 2-D copy the copy engines take
  // as one descriptor).
  for (const auto& r : plan->ce_runs) {
    CudaCheck(cudaMemcpy2DAsync(reinterpret_cast<uint8_t*>(peer.pool) + lb * dst_lb + r.dst * row_b,
                                dst_lb,
                                reinterpret_cast<const uint8_t*>(d_pool_) + lb * src_lb + r.src * row_b,
                                src_lb, r.n * row_b, nl, cudaMemcpyDeviceToDevice, ce_stream_),
              "cudaMemcpy2DAsync");
  }
  CudaCheck(cudaEventRecord(ce_ev_, ce_stream_), "cudaEventRecord");
  CudaCheck(cudaStreamWaitEvent(s, ce_ev_, 0), "wait copies");
  CopyParams c{};
  const int64_t src_lw = num_pages_ * P_ * W_, dst_lw = peer.num_pages * peer.P * W_;
  c.src = d_pool_ + lb * src_lw;
  c.src_layer_words = src_lw;
  c.src_idx = rec->d_slots + snd.begin;
  c.dst = peer.pool + lb * dst_lw;
  c.dst_layer_words = dst_lw;
  c.dst_idx = d.dst_slots;
  c.dst_fill = peer.fill + lb * peer.num_pages * peer.P;
  c.dst_fill_layer = peer.num_pages * peer.P;
  c.fill_value = 2;  // FillState::kReceivedRemote
  c.n_rows = snd.end - snd.begin;
  c.layer0 = lb;
  c.n_layers = nl;
  c.W = W_;
  c.win_received = peer.win_received;
  c.win_layer_rows = peer.win_layer_rows;
  c.win_layers = peer.L;
  c.verdict = d.verdict;
  c.status = d_status_;
  c.sys_scope = (peer.device != device_ || force_sys_scope_) ? 1 : 0;
  c.gen = plan->ce_gen;
  c.no_data = 1;
  launch_copy_rows(c, s, num_sms_);
  CountLaunches(1);
}

// Fan-out DirectSend: n_dest DirectSends of one source range, each source
// row read once (context-cache migration to several engines).
void ss_cache::BroadcastSend(SeqId seq, int64_t begin, int64_t end, int32_t n_dest,
                             const Rank* dests, const KVAddr* addrs, uint64_t tag, int32_t lb,
                             int32_t le, cudaStream_t s) {
  RequireDevice("BroadcastSend");
  MKV_CHECK(n_dest >= 1 && n_dest <= kMaxFanout, kInvalidArgument, "1..8 destinations");
  Record* rec = MustGet(seq);
  MKV_CHECK(begin >= 0 && end <= static_cast<int64_t>(rec->tokens.size()) && begin <= end,
            kInvalidArgument, "send range outside sequence");
  MKV_CHECK(lb >= 0 && lb <= le && le <= L_, kInvalidArgument, "bad layer range");
  MKV_ICHECK(end <= rec->alloc_len, "position not allocated");
  for (int32_t d = 0; d < n_dest; ++d) {
    MKV_CHECK(addrs[d].token_count == end - begin, kAddrMismatch,
              "destination covers " + std::to_string(addrs[d].token_count) +
                  " tokens, range has " + std::to_string(end - begin));
    MKV_CHECK(addrs[d].token_begin == begin, kAddrMismatch, "destination token_begin mismatch");
    addrs[d].Validate();  // one destination slot per row (kv_addr.cc:16-30)
    PeerFor(dests[d]);
  }
  if (W_ != 512 && W_ != 128) {  // the fan-out kernel is specialised for these rows
    for (int32_t d = 0; d < n_dest; ++d) DirectSend(seq, begin, end, dests[d], addrs[d], tag, lb, le, s);
    return;
  }
  if (end > rec->committed_hint &&
      !CoveredByLivePlan(seq, std::max(begin, rec->committed_hint), end)) {
    AdvanceCommitted(rec);
    for (int32_t l = lb; l < le && end > rec->committed_hint; ++l) {
      CheckFilled(rec, begin, end, l, "gather over empty slot", nullptr);
    }
  }
  if (lb == le) return;
  const int64_t n = end - begin;
  struct Lay {
    size_t dst, rp, rb, rc, v;
    std::vector<int32_t> slots, rb_, rc_;
    std::vector<int64_t> rp_;
  };
  std::vector<Lay> lay(n_dest);
  size_t off = 0;
  auto take = [&](size_t bytes) {
    const size_t o = off;
    off += Align(bytes);
    return o;
  };
  for (int32_t d = 0; d < n_dest; ++d) {
    ExpandAddr(addrs[d], &lay[d].slots, &lay[d].rp_, &lay[d].rb_, &lay[d].rc_);
    MKV_CHECK(static_cast<int64_t>(lay[d].slots.size()) == n, kAddrMismatch,
              "destination slots do not cover the send range");
    const size_t nr = lay[d].rp_.size();
    lay[d].dst = take(sizeof(int32_t) * lay[d].slots.size());
    lay[d].rp = take(sizeof(int64_t) * nr);
    lay[d].rb = take(sizeof(int32_t) * nr);
    lay[d].rc = take(sizeof(int32_t) * nr);
    lay[d].v = take(4 * sizeof(int32_t));
  }
  std::vector<uint8_t> host(off, 0);
  for (int32_t d = 0; d < n_dest; ++d) {
    std::memcpy(host.data() + lay[d].dst, lay[d].slots.data(), sizeof(int32_t) * lay[d].slots.size());
    std::memcpy(host.data() + lay[d].rp, lay[d].rp_.data(), sizeof(int64_t) * lay[d].rp_.size());
    std::memcpy(host.data() + lay[d].rb, lay[d].rb_.data(), sizeof(int32_t) * lay[d].rb_.size());
    std::memcpy(host.data() + lay[d].rc, lay[d].rc_.data(), sizeof(int32_t) * lay[d].rc_.size());
  }
  OrderLaunch(s);
  DevBlock b = DevAlloc(off, s);
  uint8_t* base = static_cast<uint8_t*>(b.ptr);
  H2D(base, host.data(), off, s, "H2D broadcast");
  FanoutParams f{};
  const int64_t src_lw = num_pages_ * P_ * W_;
  f.src = d_pool_ + lb * src_lw;
  f.src_layer_words = src_lw;
  f.src_idx = rec->d_slots + begin;
  f.n_rows = n;
  f.layer0 = lb;
  f.n_layers = le - lb;
  f.W = W_;
  f.n_dest = n_dest;
  f.gen = NextLaunchGen();
  f.truth = -1;
  for (int32_t d = 0; d < n_dest; ++d) {
    const PeerTarget& peer = PeerFor(dests[d]);
    if (peer.local != nullptr) CudaCheck(cudaStreamWaitEvent(s, peer.local->window_ev_, 0), "wait window");
    ValidateParams v{};
    v.range_page = reinterpret_cast<int64_t*>(base + lay[d].rp);
    v.range_begin = reinterpret_cast<int32_t*>(base + lay[d].rb);
    v.range_count = reinterpret_cast<int32_t*>(base + lay[d].rc);
    v.n_ranges = static_cast<int64_t>(lay[d].rp_.size());
    v.page_window = peer.page_window;
    v.expecting = peer.expecting;
    v.num_pages = peer.num_pages;
    v.P = peer.P;
    v.verdict = reinterpret_cast<int32_t*>(base + lay[d].v);
    v.status = d_status_;
    v.gen = f.gen;
    launch_validate_remote(v, s);
    const int64_t dst_lw = peer.num_pages * peer.P * W_;
    f.dst[d] = peer.pool + lb * dst_lw;
    f.dst_layer_words[d] = dst_lw;
    f.dst_idx[d] = reinterpret_cast<int32_t*>(base + lay[d].dst);
    f.dst_fill[d] = peer.fill + lb * peer.num_pages * peer.P;
    f.dst_fill_layer[d] = peer.num_pages * peer.P;
    f.win_received[d] = peer.win_received;
    f.win_layer_rows[d] = peer.win_layer_rows;
    f.win_layers[d] = peer.L;
    f.verdict[d] = v.verdict;
    f.fill_value[d] = 2;  // FillState::kReceivedRemote
    f.row_off[d] = 0;
    f.row_cnt[d] = n;
    if (peer.device != device_ || force_sys_scope_) f.sys_scope = 1;
  }
  launch_copy_rows_fanout(f, s, num_sms_);
  CountLaunches(1 + n_dest);
  DevFree(b, s);
  if (s != stream_) NoteUser(s);
  (void)tag;
}

void ss_cache::DirectSend(SeqId seq, int64_t begin, int64_t end, Rank dest, const KVAddr& addr,
                          uint64_t tag, int32_t lb, int32_t le, cudaStream_t s) {
  ss_plan* plan = BeginDirectSend(seq, begin, end, dest, addr, tag);
  try {
    LaunchDirectSend(plan, lb, le, s);
  } catch (...) {
    DestroyPlan(plan);
    throw;
  }
  DestroyPlan(plan);  // stream-ordered free after the launch
}

// ---------------------------------------------------------------------------
// Lifecycle
// ---------------------------------------------------------------------------
// kv_cache.cc:484-490
void ss_cache::CommitToTree(SeqId seq) {
  Record* rec = MustGet(seq);
  AdvanceCommitted(rec);
  const int64_t n = std::min<int64_t>(rec->committed_hint, rec->tokens.size());
  if (n <= 0) return;
  tree_.Insert(std::span<const Token>(rec->tokens.data(), n), seq);
}

// kv_cache.cc:492-518
void ss_cache::FreeSequence(SeqId seq) {
  Record* rec = MustGet(seq);
  MKV_CHECK(rec->refcount == 0, kInternal, "freeing a sequence with live children");
  {
    std::lock_guard<std::mutex> lock(recv_mu_);
    if (rec->window && rec->window->dev_id >= 0) free_window_ids_.push_back(rec->window->dev_id);
    rec->window.reset();
    for (int64_t page : rec->own_pages) {
      page_owner_[page] = -1;
      std::fill(expecting_.begin() + page * P_, expecting_.begin() + (page + 1) * P_, 0);
      free_pages_.push_back(page);
    }
  }
  if (device_ >= 0) {
    if (!rec->own_pages.empty()) {
      OrderAfterUser();
      const int64_t np = static_cast<int64_t>(rec->own_pages.size());
      DevBlock b = DevAlloc(sizeof(int64_t) * np, stream_);
      H2D(b.ptr, rec->own_pages.data(), sizeof(int64_t) * np, stream_, "H2D pages");
      launch_reset_pages(d_fill_, d_expecting_, d_page_window_, static_cast<int64_t*>(b.ptr), np,
                         L_, num_pages_, P_, stream_);
      CountLaunches(1);
      DevFree(b, stream_);
      Sync();
    }
    if (rec->fold_row >= 0) free_fold_rows_.push_back(rec->fold_row);
    if (rec->d_slots != nullptr) {
      OrderAfterUser();
      cudaFreeAsync(rec->d_slots, stream_);
      rec->d_slots = nullptr;
    }
  }
  if (rec->parent >= 0) {
    auto it = records_.find(rec->parent);
    if (it != records_.end()) --it->second->refcount;
  }
  for (auto it = pending_sends_.begin(); it != pending_sends_.end();) {
    it = it->seq == seq ? pending_sends_.erase(it) : std::next(it);
  }
  tree_.Remove(seq);
  std::lock_guard<std::mutex> lock(recv_mu_);
  records_.erase(seq);
}

// kv_cache.cc:520-546
int64_t ss_cache::Evict(int64_t bytes_needed) {
  if (bytes_needed <= 0) return 0;
  int64_t freed_tokens = 0;
  auto satisfied = [&] {
    return static_cast<int64_t>(free_pages_.size()) * BytesPerPage() >= bytes_needed;
  };
  while (!satisfied()) {
    SeqId victim = -1;
    for (SeqId seq : tree_.SequencesByLru()) {
      auto it = records_.find(seq);
      if (it == records_.end()) continue;
      const Record* rec = it->second.get();
      if (!rec->finished || rec->refcount != 0) continue;
      if (rec->own_pages.empty()) continue;
      if (tree_.HasPinnedNode(seq)) continue;
      victim = seq;
      break;
    }
    MKV_CHECK(victim >= 0, kCannotEvict, "all remaining sequences are pinned or live");
    const Record* rec = records_.at(victim).get();
    freed_tokens += std::max<int64_t>(
        0, std::min<int64_t>(rec->tokens.size(), rec->alloc_len) - rec->fork_len);
    FreeSequence(victim);
  }
  return freed_tokens;
}

// ---------------------------------------------------------------------------
// Queries
// ---------------------------------------------------------------------------
int64_t ss_cache::Committed(SeqId seq) {
  Record* rec = MustGet(seq);
  AdvanceCommitted(rec);
  return rec->committed_hint;
}

void ss_cache::ReadEntryWords(SeqId seq, int64_t pos, int32_t layer, uint64_t* out) {
  RequireDevice("ReadEntryWords");
  const Record* rec = MustGet(seq);
  MKV_CHECK(layer >= 0 && layer < L_, kInvalidArgument, "layer out of range");
  const int32_t slot = Resolve(rec, pos);
  OrderAfterUser();
  D2H(out, PoolLayer(layer) + static_cast<int64_t>(slot) * W_,
                            sizeof(uint64_t) * W_, stream_, "D2H entry");
  Sync();
}

int32_t ss_cache::FillOf(SeqId seq, int64_t pos, int32_t layer) {
  RequireDevice("FillOf");
  const Record* rec = MustGet(seq);
  MKV_CHECK(layer >= 0 && layer < L_, kInvalidArgument, "layer out of range");
  const int32_t slot = Resolve(rec, pos);
  uint8_t v = 0;
  OrderAfterUser();
  D2H(&v, d_fill_ + static_cast<int64_t>(layer) * num_pages_ * P_ + slot, 1, stream_, "D2H fill");
  Sync();
  return v;
}

std::vector<SeqId> ss_cache::SequenceIds() const {
  std::vector<SeqId> out;
  out.reserve(records_.size());
  for (const auto& [id, rec] : records_) out.push_back(id);
  return out;
}

// ---------------------------------------------------------------------------
// Peers
// ---------------------------------------------------------------------------
void ss_cache::AttachPeer(Rank dest, ss_cache* peer) {
  RequireDevice("AttachPeer");
  MKV_CHECK(peer != nullptr && peer->device_ >= 0, kInvalidArgument, "peer has no device");
  MKV_CHECK(peer->L_ == L_ && peer->W_ == W_, kInvalidArgument, "peer geometry mismatch");
  if (peer->device_ != device_) {
    int ok = 0;
    CudaCheck(cudaDeviceCanAccessPeer(&ok, device_, peer->device_), "cudaDeviceCanAccessPeer");
    MKV_CHECK(ok, kPeerUnreachable, "no peer access between devices");
    cudaSetDevice(device_);
    cudaError_t e = cudaDeviceEnablePeerAccess(peer->device_, 0);
    if (e != cudaErrorPeerAccessAlreadyEnabled) CudaCheck(e, "cudaDeviceEnablePeerAccess");
    cudaGetLastError();
  }
  PeerTarget t;
  t.pool = peer->d_pool_;
  t.fill = peer->d_fill_;
  t.expecting = peer->d_expecting_;
  t.page_window = peer->d_page_window_;
  t.win_received = peer->d_win_received_;
  t.win_gen = peer->d_win_received_ + kMaxWindows;
  t.win_layer_rows = peer->d_win_layer_rows_;
  t.num_pages = peer->num_pages_;
  t.P = peer->P_;
  t.L = peer->L_;
  t.W = peer->W_;
  t.device = peer->device_;
  t.local = peer;
  DetachPeer(dest);
  peers_[dest] = t;
  peer_engines_[dest] = peer;
  peer->attached_by_.insert(this);
}

namespace {
struct IpcBlob {
  uint32_t magic;
  uint32_t version;
  int64_t num_pages;
  int32_t P, L, W, device;
  cudaIpcMemHandle_t h[6];
  unsigned char uuid[16];  // exporter's GPU: ordinals differ across processes
};
static_assert(sizeof(IpcBlob) <= SS_IPC_HANDLE_BYTES, "ipc blob too large");
}  // namespace

void ss_cache::ExportIpc(ss_ipc_handle* out) {
  RequireDevice("ExportIpc");
  ipc_exported_ = true;
  Sync();  // windows opened so far are visible to the peer process
  IpcBlob b{};
  b.magic = kIpcMagic;
  b.version = SS_ABI_VERSION;
  b.num_pages = num_pages_;
  b.P = P_;
  b.L = L_;
  b.W = W_;
  b.device = device_;
  cudaDeviceProp prop{};
  CudaCheck(cudaGetDeviceProperties(&prop, device_), "cudaGetDeviceProperties");
  std::memcpy(b.uuid, prop.uuid.bytes, sizeof(b.uuid));
  void* ptrs[6] = {d_pool_, d_fill_, d_expecting_, d_page_window_, d_win_received_,
                   d_win_layer_rows_};
  for (int i = 0; i < 6; ++i) CudaCheck(cudaIpcGetMemHandle(&b.h[i], ptrs[i]), "cudaIpcGetMemHandle");
  std::memset(out->bytes, 0, sizeof(out->bytes));
  std::memcpy(out->bytes, &b, sizeof(b));
}

void ss_cache::ImportIpc(Rank dest, const ss_ipc_handle* h) {
  RequireDevice("ImportIpc");
  IpcBlob b;
  std::memcpy(&b, h->bytes, sizeof(b));
  MKV_CHECK(b.magic == kIpcMagic && b.version == SS_ABI_VERSION, kInvalidArgument,
            "not a microkv IPC handle");
  MKV_CHECK(b.L == L_ && b.W == W_, kInvalidArgument, "peer geometry mismatch");
  PeerTarget t;
  void* ptrs[6] = {};
  CudaCheck(cudaSetDevice(device_), "cudaSetDevice");
  for (int i = 0; i < 6; ++i) {
    cudaError_t e = cudaIpcOpenMemHandle(&ptrs[i], b.h[i], cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) {
      for (int j = 0; j < i; ++j) cudaIpcCloseMemHandle(ptrs[j]);
      CudaCheck(e, "cudaIpcOpenMemHandle");
    }
    t.ipc_ptrs.push_back(ptrs[i]);
  }
  t.pool = static_cast<uint64_t*>(ptrs[0]);
  t.fill = static_cast<uint8_t*>(ptrs[1]);
  t.expecting = static_cast<uint8_t*>(ptrs[2]);
  t.page_window = static_cast<int32_t*>(ptrs[3]);
  t.win_received = static_cast<unsigned long long*>(ptrs[4]);
  t.win_gen = t.win_received + kMaxWindows;
  t.win_layer_rows = static_cast<uint32_t*>(ptrs[5]);
  t.num_pages = b.num_pages;
  t.P = b.P;
  t.L = b.L;
  t.W = b.W;
  // Same physical GPU (another process on it) -> device-scope publication
  // suffices; any other GPU -> system scope.
  cudaDeviceProp prop{};
  CudaCheck(cudaGetDeviceProperties(&prop, device_), "cudaGetDeviceProperties");
  t.device = std::memcmp(prop.uuid.bytes, b.uuid, sizeof(b.uuid)) == 0 ? device_ : -2;
  t.ipc = true;
  DetachPeer(dest);
  peers_[dest] = t;
}

void ss_cache::DetachPeer(Rank dest) {
  auto it = peers_.find(dest);
  if (it == peers_.end()) return;
  if (device_ >= 0) {
    Sync();
    CudaCheck(cudaStreamSynchronize(comm_stream_), "cudaStreamSynchronize");
  }
  for (void* p : it->second.ipc_ptrs) cudaIpcCloseMemHandle(p);
  peers_.erase(it);
  auto e = peer_engines_.find(dest);
  if (e != peer_engines_.end()) {
    e->second->attached_by_.erase(this);
    peer_engines_.erase(e);
  }
}

void ss_cache::Synchronize() {
  if (device_ < 0) return;
  Sync();
  SyncUserStreams();
  CudaCheck(cudaStreamSynchronize(comm_stream_), "cudaStreamSynchronize");
  uint32_t st = 0;
  CudaCheck(cudaMemcpy(&st, d_status_, sizeof(uint32_t), cudaMemcpyDeviceToHost), "D2H status");
  d2h_bytes_ += sizeof(uint32_t);
  if (st & (kStatusUnknownAddress | kStatusWaitTimeout)) {
    CudaCheck(cudaMemset(d_status_, 0, sizeof(uint32_t)), "memset");
    if (st & kStatusUnknownAddress) {
      Throw(kUnknownAddress, "a device-direct remote write was rejected by the receiver");
    }
    Throw(kAborted, "device-side receive wait timed out");
  }
}

void ss_cache::WaitReceive(SeqId seq, int64_t timeout_ms, cudaStream_t s) {
  RequireDevice("WaitReceive");
  Record* rec = MustGet(seq);
  MKV_CHECK(rec->window.has_value(), kInvalidArgument,
            "sequence " + std::to_string(seq) + " has no receive window");
  if (rec->window->complete && rec->window->dev_id < 0) return;  // drained: every row landed
  MKV_CHECK(rec->window->dev_id >= 0, kInvalidArgument,
            "sequence " + std::to_string(seq) + " has no device receive window");
  const Window& w = *rec->window;
  const int64_t target = std::max<int64_t>(0, w.expected - w.received);
  OrderLaunch(s);
  launch_wait_counter(d_win_received_ + w.dev_id, static_cast<unsigned long long>(target),
                      timeout_ms * 1000000LL, d_status_, s);
  CountLaunches(1);
  if (s != stream_) NoteUser(s);
}

void ss_cache::WaitReceiveLayer(SeqId seq, int32_t layer, int64_t timeout_ms, cudaStream_t s) {
  RequireDevice("WaitReceive");
  MKV_CHECK(layer >= 0 && layer < L_, kInvalidArgument, "layer out of range");
  Record* rec = MustGet(seq);
  MKV_CHECK(rec->window.has_value(), kInvalidArgument,
            "sequence " + std::to_string(seq) + " has no receive window");
  if (rec->window->complete && rec->window->dev_id < 0) return;  // drained: every row landed
  MKV_CHECK(rec->window->dev_id >= 0, kInvalidArgument,
            "sequence " + std::to_string(seq) + " has no device receive window");
  const Window& w = *rec->window;
  int64_t host_rows = 0;
  {
    std::lock_guard<std::mutex> lock(recv_mu_);
    if (static_cast<int32_t>(w.received_layer.size()) == L_) host_rows = w.received_layer[layer];
  }
  const int64_t target = std::max<int64_t>(0, (w.end - w.begin) - host_rows);
  OrderLaunch(s);
  launch_wait_counter32(d_win_layer_rows_ + static_cast<int64_t>(w.dev_id) * L_ + layer,
                        static_cast<uint32_t>(target), timeout_ms * 1000000LL, d_status_, s);
  CountLaunches(1);
  if (s != stream_) NoteUser(s);
}

// ---------------------------------------------------------------------------
// Hash model scalars (hash_model.cc:27, 63-68, 83-86)
// ---------------------------------------------------------------------------
uint64_t ss_cache::InitialPrefixDigest() const { return fnv_u64(seed_state_, kTagPrefix); }
uint64_t ss_cache::Embed(Token t, int64_t pos) const { return embed(seed_state_, t, pos); }
mkv::Token ss_cache::SampleToken(uint64_t h) const { return sample_token(h, vocab_); }

// ---------------------------------------------------------------------------
// Decode attention plan: per-position slot map of each context, uploaded
// once and read by every layer's launch.
// ---------------------------------------------------------------------------
ss_plan* ss_cache::BeginDecode(const int64_t* seqs, const int64_t* ctx_lens, int64_t batch) {
  RequireDevice("BeginDecode");
  MKV_CHECK(batch >= 1, kInvalidArgument, "empty decode batch");
  std::vector<int64_t> off(batch + 1, 0);
  std::vector<int32_t> len(batch);
  int64_t max_ctx = 0;
  for (int64_t b = 0; b < batch; ++b) {
    Record* rec = MustGet(seqs[b]);
    const int64_t n = ctx_lens[b];
    MKV_CHECK(n >= 1 && n <= rec->alloc_len, kInvalidArgument, "bad decode context length");
    if (n > rec->committed_hint) AdvanceCommitted(rec);
    MKV_CHECK(rec->committed_hint >= n, kMissingKV,
              "decode context " + std::to_string(n) + " beyond committed " +
                  std::to_string(rec->committed_hint));
    len[b] = static_cast<int32_t>(n);
    off[b + 1] = off[b] + n;
    max_ctx = std::max(max_ctx, n);
  }
  const size_t o_off = 0;
  const size_t o_len = o_off + Align(sizeof(int64_t) * (batch + 1));
  const size_t o_tab = o_len + Align(sizeof(int32_t) * batch);
  const size_t o_slots = o_tab + Align(sizeof(int32_t*) * batch);
  const size_t upload = o_slots;
  const size_t total = o_slots + Align(sizeof(int32_t) * off[batch]);
  std::vector<uint8_t> host(upload, 0);
  std::memcpy(host.data() + o_off, off.data(), sizeof(int64_t) * (batch + 1));
  std::memcpy(host.data() + o_len, len.data(), sizeof(int32_t) * batch);
  for (int64_t b = 0; b < batch; ++b) {
    const int32_t* t = MustGet(seqs[b])->d_slots;
    std::memcpy(host.data() + o_tab + sizeof(int32_t*) * b, &t, sizeof(t));
  }
  auto plan = std::make_unique<ss_plan>();
  plan->owner = this;
  plan->is_decode_plan = true;
  plan->batch = batch;
  plan->max_ctx = max_ctx;
  plan->ctx_lens = len;
  // Page chunks for decode_pages.cu: maximal runs of consecutive slots, at
  // most 16 positions.  A page's positions are consecutive slots, so the
  // run check is one comparison per page, not per position.
  for (int64_t b = 0; b < batch; ++b) {
    const std::vector<int32_t>& sl = MustGet(seqs[b])->slots;
    const int64_t n = len[b];
    for (int64_t pos = 0; pos < n;) {
      const int32_t s0 = sl[pos];
      int64_t k = std::min<int64_t>({16, n - pos, static_cast<int64_t>(P_) - s0 % P_});
      if (sl[pos + k - 1] != s0 + k - 1) {  // not one run (never for a fresh page): per position
        k = 1;
        while (k < 16 && pos + k < n && sl[pos + k] == s0 + k) ++k;
      } else {  // extend into the next page when it is the next slot block
        while (k < 16 && pos + k < n && sl[pos + k] == s0 + k) ++k;
      }
      plan->chunks.insert(plan->chunks.end(),
                          {s0, static_cast<int32_t>(pos), static_cast<int32_t>(k),
                           static_cast<int32_t>(b)});
      pos += k;
    }
  }
  OrderAfterUser();
  plan->dev = DevAlloc(total, stream_);
  uint8_t* base = static_cast<uint8_t*>(plan->dev.ptr);
  H2D(base, host.data(), upload, stream_, "H2D ctx");
  launch_gather_tables(reinterpret_cast<const int32_t* const*>(base + o_tab),
                       reinterpret_cast<const int64_t*>(base + o_off),
                       reinterpret_cast<const int32_t*>(base + o_len), batch, off[batch],
                       reinterpret_cast<int32_t*>(base + o_slots), stream_, num_sms_);
  CountLaunches(1);
  plan->d_ctx_slots = reinterpret_cast<int32_t*>(base + o_slots);
  plan->d_ctx_off = reinterpret_cast<int64_t*>(base + o_off);
  plan->d_ctx_len = reinterpret_cast<int32_t*>(base + o_len);
  plan->on_device = true;
  Sync();
  live_plans_.insert(plan.get());
  return plan.release();
}

// Where split segments are merged.  Few pieces per segment (large batch:
// most segments whole, none split more than a few ways): in the attention
// kernel's last arriving CTA, which saves the second launch (B=32 8K 0.97
// -> 1.0 of HBM, B=128 +2%).  Many pieces (small batch, up to 32 per
// segment): a separate programmatic-dependent combine kernel, whose 64+
// CTAs merge faster than one CTA per segment (B=1 8K: 16.6 vs 20.6 us).
// MICROKV_DECODE_COMBINE=kernel|fused overrides (A/B).
static bool DecodeCombineKernel(int64_t max_pieces) {
  if (const char* e = std::getenv("MICROKV_DECODE_COMBINE")) return std::string(e) == "kernel";
  return max_pieces > 4;
}

void ss_cache::DecodeAttention(ss_plan* plan, int32_t layer, int32_t hq, int32_t hkv, int32_t hd,
                               float scale, const void* q, void* out, cudaStream_t s) {
  RequireDevice("DecodeAttention");
  MKV_CHECK(plan->is_decode_plan, kInvalidArgument, "not a decode plan");
  MKV_CHECK(layer >= 0 && layer < L_, kInvalidArgument, "layer out of range");
  MKV_CHECK(hkv >= 1 && hq % hkv == 0 && hq / hkv <= 16, kInvalidArgument,
            "num_q_heads must be a multiple of num_kv_heads with group <= 16");
  MKV_CHECK(hd == 64 || hd == 128, kInvalidArgument, "head_dim must be 64 or 128");
  MKV_CHECK(static_cast<int64_t>(W_) * 8 == 4LL * hkv * hd, kInvalidArgument,
            "entry width must equal K||V bf16 bytes (dim * 8 == 4 * num_kv_heads * head_dim)");
  if (decode_pages_supported(hq, hkv, hd, W_) && [] {
        const char* e = std::getenv("MICROKV_DECODE_KERNEL");
        return e == nullptr || std::strcmp(e, "v1") != 0;
      }()) {
    DecodeAttentionPages(plan, layer, hq, hkv, scale, q, out, s);
    return;
  }
  if (plan->decode_grid == 0 || plan->decode_hkv != hkv || plan->decode_hq != hq ||
      plan->decode_hd != hd) {
    // Tile prefix sums over segments (batch, kv head) for the stream-K split,
    // and partial storage for at most grid + segments pieces.
    plan->decode_grid = decode_attn_resident_ctas(hd, num_sms_);
    const int64_t n_seg = plan->batch * hkv;
    // Segment-aligned grid: k CTAs per (batch, kv head) segment, so with
    // equal contexts no CTA straddles two segments (one prologue/epilogue and
    // one partial per CTA), at most 32 pieces per segment.  Measured on B200
    // (profiles/r01/decode_grid_sweep.txt): B=8 ctx 8K 0.69 -> 0.74 of HBM,
    // B=32 0.93 -> 0.97, B=8 ctx 32K 0.97 -> 1.0, B=1 0.21 -> 0.27.
    if (n_seg <= plan->decode_grid) {
      // At most 32 pieces per segment (measured: B=1 ctx 8K 16.4 us at 32
      // pieces, 21.7 at 48; ctx 32K 32.8 us at 32, 44.2 at 55 — more, shorter
      // pieces only add prologues, epilogues and partials) and at least 16
      // tiles per piece.
      int64_t min_tiles = INT64_MAX;
      for (int64_t b = 0; b < plan->batch; ++b) {
        min_tiles = std::min<int64_t>(min_tiles, (plan->ctx_lens[b] + 15) / 16);
      }
      int64_t cap = std::clamp<int64_t>(min_tiles / 16, 1, 32);
      if (const char* c = std::getenv("MICROKV_DECODE_MAX_PIECES")) cap = std::max(1, std::atoi(c));
      const int64_t k = std::min<int64_t>(plan->decode_grid / n_seg, cap);
      plan->decode_grid = static_cast<int32_t>(n_seg * k);
    }
    if (const char* g = std::getenv("MICROKV_DECODE_GRID")) {  // tuning experiments
      const int v = std::atoi(g);
      if (v > 0 && v < plan->decode_grid) plan->decode_grid = v;
    }
    std::vector<int64_t> seg(n_seg + 1, 0);
    for (int64_t b = 0; b < plan->batch; ++b) {
      const int64_t tiles = (plan->ctx_lens[b] + 15) / 16;
      for (int32_t h = 0; h < hkv; ++h) seg[b * hkv + h + 1] = seg[b * hkv + h] + tiles;
    }
    plan->total_tiles = seg[n_seg];
    OrderAfterUser();  // internal upload below; OrderLaunch then orders s after it
    Sync();
    if (plan->d_partial) cudaFree(plan->d_partial);
    const int64_t pieces = plan->decode_grid + n_seg;
    const int64_t G = hq / hkv;
    const size_t bytes_o = sizeof(float) * pieces * G * hd, bytes_ml = sizeof(float) * pieces * G * 2;
    uint8_t* buf = nullptr;
    const size_t bytes_seg = sizeof(int64_t) * (n_seg + 1);
    // First segment of each CTA's tile range (see k_decode_attn), uploaded
    // right behind the prefix sums.
    const int64_t grid = std::min<int64_t>(plan->decode_grid, std::max<int64_t>(1, plan->total_tiles));
    std::vector<int32_t> cta_seg(grid);
    for (int64_t c = 0, sgi = 0; c < grid; ++c) {
      const int64_t t0 = c * plan->total_tiles / grid;
      while (sgi + 1 < n_seg && seg[sgi + 1] <= t0) ++sgi;
      cta_seg[c] = static_cast<int32_t>(sgi);
    }
    const size_t bytes_cta = sizeof(int32_t) * grid;
    CudaCheck(cudaMalloc(&buf, bytes_o + bytes_ml + bytes_seg + bytes_cta + sizeof(uint32_t) * n_seg),
              "cudaMalloc partials");
    plan->d_partial = reinterpret_cast<float*>(buf);
    plan->d_partial_ml = reinterpret_cast<float*>(buf + bytes_o);
    plan->d_seg_start = reinterpret_cast<int64_t*>(buf + bytes_o + bytes_ml);
    plan->d_cta_seg = reinterpret_cast<int32_t*>(buf + bytes_o + bytes_ml + bytes_seg);
    plan->d_seg_count = reinterpret_cast<uint32_t*>(buf + bytes_o + bytes_ml + bytes_seg + bytes_cta);
    H2D(plan->d_seg_start, seg.data(), bytes_seg, stream_, "H2D segments");
    H2D(plan->d_cta_seg, cta_seg.data(), bytes_cta, stream_, "H2D cta segments");
    // Arrival counters of the fused combine (each launch leaves them at 0).
    CudaCheck(cudaMemsetAsync(plan->d_seg_count, 0, sizeof(uint32_t) * n_seg, stream_), "memset");
    plan->decode_hkv = hkv;
    plan->decode_hq = hq;
    plan->decode_hd = hd;
  }
  // Pieces per segment: k with the segment-aligned grid, at most 3 when
  // segments outnumber CTAs.
  const int64_t n_seg = plan->batch * hkv;
  const bool use_kernel =
      DecodeCombineKernel(n_seg >= plan->decode_grid ? 3 : plan->decode_grid / n_seg);
  OrderLaunch(s);
  const bool ok = launch_decode_attn(PoolLayer(layer), static_cast<int64_t>(W_) * 4,
                                     plan->d_ctx_slots, plan->d_ctx_off, plan->d_ctx_len,
                                     plan->d_seg_start, plan->batch * hkv, plan->total_tiles, q,
                                     static_cast<int>(plan->batch), hq, hkv, hd, scale,
                                     plan->d_partial, plan->d_partial_ml, out, plan->decode_grid,
                                     use_kernel ? nullptr : plan->d_seg_count, plan->d_cta_seg, s);
  MKV_CHECK(ok, kInvalidArgument, "unsupported head_dim");
  CountLaunches(use_kernel ? 2 : 1);
  if (s != stream_) NoteUser(s);
}

// Page-chunk decode attention (decode_pages.cu) for 4 KiB K||V rows of 8 KV
// heads x 128: the chunks' equal split over one CTA per SM, per-context
// piece tables and partial storage built once per plan.
void ss_cache::DecodeAttentionPages(ss_plan* plan, int32_t layer, int32_t hq, int32_t hkv,
                                    float scale, const void* q, void* out, cudaStream_t s) {
  if (!tmap_chunk_ready_) {
    if (!make_pool_tensor_map(d_pool_, L_, num_pages_ * P_, W_, 16,
                              reinterpret_cast<PoolTensorMap*>(tmap_chunk_)))
      mkv::ThrowStatus(SS_ERR_CUDA, "cuTensorMapEncodeTiled failed for the pool");
    tmap_chunk_ready_ = true;
  }
  const int64_t T = static_cast<int64_t>(plan->chunks.size() / 4);
  if (!plan->pages_ready || plan->decode_hq != hq) {
    const int grid = decode_pages_grid(num_sms_, T);
    const int64_t B = plan->batch;
    std::vector<int32_t> first(B, -1), count(B, 0);
    for (int64_t c = 0; c < grid; ++c) {
      const int64_t j0 = c * T / grid, j1 = (c + 1) * T / grid;
      int32_t last_b = -1;
      for (int64_t j = j0; j < j1; ++j) {
        const int32_t b = plan->chunks[4 * j + 3];
        if (b == last_b) continue;
        last_b = b;
        if (first[b] < 0) first[b] = static_cast<int32_t>(c);
        ++count[b];
      }
    }
    bool split = false;
    for (int64_t b = 0; b < B; ++b) split |= count[b] > 1;
    const int64_t G = hq / hkv;
    const int64_t pieces = grid + B;
    const size_t b_ch = Align(sizeof(int32_t) * plan->chunks.size());
    const size_t b_tab = Align(sizeof(int32_t) * B);
    const size_t b_o = Align(sizeof(float) * pieces * hkv * G * 128);
    const size_t b_ml = Align(sizeof(float) * pieces * hkv * G * 2);
    OrderAfterUser();
    Sync();
    if (plan->d_chunks) cudaFree(plan->d_chunks);
    uint8_t* buf = nullptr;
    CudaCheck(cudaMalloc(&buf, b_ch + 2 * b_tab + b_o + b_ml), "cudaMalloc decode chunks");
    plan->d_chunks = reinterpret_cast<int32_t*>(buf);
    plan->d_piece_first = reinterpret_cast<int32_t*>(buf + b_ch);
    plan->d_piece_count = reinterpret_cast<int32_t*>(buf + b_ch + b_tab);
    plan->d_pages_part = reinterpret_cast<float*>(buf + b_ch + 2 * b_tab);
    plan->d_pages_ml = reinterpret_cast<float*>(buf + b_ch + 2 * b_tab + b_o);
    H2D(plan->d_chunks, plan->chunks.data(), sizeof(int32_t) * plan->chunks.size(), stream_,
        "H2D decode chunks");
    H2D(plan->d_piece_first, first.data(), sizeof(int32_t) * B, stream_, "H2D pieces");
    H2D(plan->d_piece_count, count.data(), sizeof(int32_t) * B, stream_, "H2D pieces");
    plan->pages_grid = grid;
    plan->pages_split = split;
    plan->pages_ready = true;
    plan->decode_hq = hq;
  }
  OrderLaunch(s);
  const int nl = launch_decode_pages(
      *reinterpret_cast<const PoolTensorMap*>(tmap_chunk_), layer,
      reinterpret_cast<const int4*>(plan->d_chunks), T, plan->d_piece_first, plan->d_piece_count,
      plan->pages_split, q, static_cast<int>(plan->batch), hq, hkv, scale, plan->d_pages_part,
      plan->d_pages_ml, out, plan->pages_grid, s);
  CountLaunches(nl);
  if (s != stream_) NoteUser(s);
}

// Causal prefill attention of queries [q_begin, q_end) of `seq` over keys
// [0, q_end) of this layer, read through the sequence's HBM page table
// (balanced-PD tail prefill on the decode engine).  The
// caller has written this layer's K||V rows for [0, q_end) (the queries' own
// rows through ss_append_rows_async, the prefix by a receive or earlier
// prefill); per-layer fill is not re-checked here.
void ss_cache::PrefillAttention(int64_t seq, int64_t q_begin, int64_t q_end, int32_t layer,
                                int32_t hq, int32_t hkv, int32_t hd, float scale, const void* q,
                                void* out, cudaStream_t s) {
  RequireDevice("PrefillAttention");
  Record* rec = MustGet(seq);
  MKV_CHECK(layer >= 0 && layer < L_, kInvalidArgument, "layer out of range");
  MKV_CHECK(0 <= q_begin && q_begin < q_end && q_end <= rec->alloc_len, kInvalidArgument,
            "query range must be non-empty and allocated");
  MKV_CHECK(q_end <= INT32_MAX, kInvalidArgument, "context too long");
  MKV_CHECK(prefill_attn_supported(P_, hq, hkv, hd), kInvalidArgument,
            "prefill attention supports head_dim 128, a query-head group (num_q_heads / "
            "num_kv_heads) dividing 128 and a power-of-two page size >= 8");
  MKV_CHECK(static_cast<int64_t>(W_) * 8 == 4LL * hkv * hd, kInvalidArgument,
            "entry width must equal K||V bf16 bytes (dim * 8 == 4 * num_kv_heads * head_dim)");
  if (!tmaps_ready_) {
    const int64_t rows = num_pages_ * P_;
    auto* pm = reinterpret_cast<PoolTensorMap*>(tmap_page_);
    auto* rm = reinterpret_cast<PoolTensorMap*>(tmap_row_);
    if (!make_pool_tensor_map(d_pool_, L_, rows, W_, prefill_attn_box_rows(P_), pm) ||
        !make_pool_tensor_map(d_pool_, L_, rows, W_, 1, rm))
      mkv::ThrowStatus(SS_ERR_CUDA, "cuTensorMapEncodeTiled failed for the pool");
    tmaps_ready_ = true;
  }
  OrderLaunch(s);
  const int nl = launch_prefill_attn(*reinterpret_cast<const PoolTensorMap*>(tmap_page_),
                                      *reinterpret_cast<const PoolTensorMap*>(tmap_row_), layer, P_,
                                      num_pages_ * P_, rec->d_slots, q, static_cast<int>(q_begin),
                                      static_cast<int>(q_end - q_begin), hq, hkv, hd, scale, out, s);
  MKV_CHECK(nl > 0, kInvalidArgument, "unsupported prefill attention shape");
  CountLaunches(nl);
  if (s != stream_) NoteUser(s);
}
