/*
 * microkv.h — C ABI of the B200-native paged-KV hot path behind the
 * microserving sub-request APIs (arXiv 2412.12488, "A System for
 * Microserving of LLMs").
 *
 * Drop-in boundary for `splitserve::KVCache`
 * (/root/reference/proj/core/include/splitserve/kv_cache.h:132-266): every
 * entry point below mirrors one reference member function with plain
 * pointers and sizes (no C++ or torch types).  A C++ engine keeps calling
 * the reference's class API through a thin facade that rethrows
 * `splitserve::Error` from the returned status.
 *
 * Two libraries implement this header:
 *   paper_2412_12488_b200/_lib/libmicrokv.so   B200 product: host bookkeeping in C++,
 *                                              KV pool, page tables and all data
 *                                              movement on the GPU (sm_100a kernels).
 *   oracle/_ref/libmicrokv_ref.so              test oracle only: the UNMODIFIED reference
 *                                              KVCache compiled from /root/reference
 *                                              behind the same ABI (host entry points only).
 *
 * Conventions
 *  - Every function returning `int` returns SS_OK (0) or a status: 1 + the
 *    reference `ErrorCode` value (errors.h:14-33), or one of the SS_ERR_*
 *    codes >= 100 that exist only at this boundary.  `ss_last_error()` holds
 *    the detail string of the last failure (the reference's `Error::what()`).
 *  - Tokens are int32 (common.h:15), sequence ids int64 (common.h:19), ranks
 *    int32 (common.h:22).  Token ranges are half-open [begin, end).
 *  - "Host" entry points take host buffers and complete synchronously, like
 *    the reference.  `*_async` entry points take device pointers and a
 *    `cudaStream_t` passed as `void*` (NULL = legacy default stream) and
 *    only enqueue work.  Work enqueued on a stream is ordered after the
 *    cache's earlier device work (uploads, window opens, resets), and the
 *    cache's later device work is ordered after it; two different caller
 *    streams are not ordered against each other by the library (use CUDA
 *    events, as with any stream).  The cache's own device work (window
 *    opens / closes, page resets, receive polls) runs on an internal stream
 *    of the highest priority: those kernels are microseconds long and host
 *    calls wait for them, so they are not held behind a caller's long copy
 *    grid; transfers launched by the library on its comm stream are high
 *    priority too (a layer's send is not starved by the next layer's
 *    compute).
 *  - A cache created with `device = -1` is host-only: bookkeeping calls
 *    (match, prep_recv page reservation, fork, allocate, build_addr, free,
 *    evict, pin, queries on metadata) work; any call that touches KV bytes
 *    returns SS_ERR_NO_DEVICE.  There is no CPU data path.
 */
#ifndef MICROKV_H_
#define MICROKV_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SS_ABI_VERSION 1

/* ------------------------------------------------------------------ */
/* Status codes                                                        */
/* ------------------------------------------------------------------ */
enum ss_status {
  SS_OK = 0,
  /* 1 + splitserve::ErrorCode (errors.h:14-33), same order. */
  SS_ERR_OUT_OF_PAGES = 1,
  SS_ERR_DUPLICATE_SEQUENCE = 2,
  SS_ERR_UNKNOWN_SEQUENCE = 3,
  SS_ERR_FORK_BEYOND_COMMITTED = 4,
  SS_ERR_ADDR_MISMATCH = 5,
  SS_ERR_MISSING_KV = 6,
  SS_ERR_LAYER_ORDER_VIOLATION = 7,
  SS_ERR_CANNOT_EVICT = 8,
  SS_ERR_CHECKSUM_MISMATCH = 9,
  SS_ERR_UNKNOWN_ADDRESS = 10,
  SS_ERR_PEER_UNREACHABLE = 11,
  SS_ERR_NO_ENGINES = 12,
  SS_ERR_ROLE_MISSING = 13,
  SS_ERR_NO_OWNER = 14,
  SS_ERR_UNKNOWN_STRATEGY = 15,
  SS_ERR_INVALID_ARGUMENT = 16,
  SS_ERR_ABORTED = 17,
  SS_ERR_INTERNAL = 18,
  /* Boundary-only codes. */
  SS_ERR_UNSUPPORTED = 100,      /* entry point not provided by this library */
  SS_ERR_BUFFER_TOO_SMALL = 101, /* output capacity short; *_n outputs hold the need */
  SS_ERR_CUDA = 102,             /* CUDA runtime failure; detail in ss_last_error */
  SS_ERR_NO_DEVICE = 103         /* data-path call on a host-only cache */
};

/* KVCache::ApplyStatus (kv_cache.h:194). */
enum ss_apply_status { SS_APPLY_OK = 0, SS_APPLY_DUPLICATE = 1, SS_APPLY_UNKNOWN_ADDRESS = 2 };

/* FillState (kv_cache.h:40-44). */
enum ss_fill_state { SS_FILL_EMPTY = 0, SS_FILL_COMPUTED_LOCAL = 1, SS_FILL_RECEIVED_REMOTE = 2 };

typedef struct ss_cache ss_cache; /* one engine's KVCache */
typedef struct ss_plan ss_plan;   /* ForwardPlan (kv_cache.h:116-121) */

/* ------------------------------------------------------------------ */
/* Plain-data mirrors of the reference types                           */
/* ------------------------------------------------------------------ */

/* CacheConfig (config.h:101-108) + ModelConfig (config.h:22-30). */
typedef struct {
  int64_t num_pages;  /* CacheConfig::num_pages (default 4096) */
  int32_t page_size;  /* CacheConfig::page_size, power of two (default 16) */
  int32_t layers;     /* ModelConfig::layers L */
  int32_t dim;        /* ModelConfig::dim = u64 words W per (token, layer) entry */
  int32_t vocab;      /* ModelConfig::vocab */
  uint64_t hash_seed; /* ModelConfig::hash_seed (default 0x5eed5eed5eed5eed) */
  int32_t device;     /* CUDA device ordinal; -1 = host-only bookkeeping */
  int32_t rank;       /* this engine's rank (EngineConfig::rank, config.h:112) */
} ss_config;

/* SlotRange (kv_addr.h:19-24). */
typedef struct {
  int64_t page_id;
  int32_t slot_begin;
  int32_t slot_count;
} ss_slot_range;

/* KVAddrInfo (kv_addr.h:30-48).  As an output, `ranges` is caller storage
 * of `ranges_cap` entries; `n_ranges` is set to the count written (or the
 * count needed, with SS_ERR_BUFFER_TOO_SMALL). */
typedef struct {
  int64_t token_begin;
  int64_t token_count;
  int64_t n_ranges;
  ss_slot_range* ranges;
  int64_t ranges_cap;
} ss_addr;

/* BatchEntry (kv_cache.h:85-89). */
typedef struct {
  int64_t seq;
  int64_t begin;
  int64_t end;
  int32_t is_decode;
  int32_t _pad;
} ss_batch_entry;

/* Scalar fields of SequenceRecord (kv_cache.h:56-82). */
typedef struct {
  int64_t id;
  int64_t parent;
  int64_t fork_len;
  int32_t refcount;
  int32_t finished;
  int64_t alloc_len;
  int64_t committed_hint;
  int64_t num_tokens;
  int64_t num_own_pages;
  int64_t fold_frontier;
  int64_t digest_len;
  uint64_t prefix_digest;
  int32_t has_window;
  int32_t window_complete;
  int64_t window_begin;
  int64_t window_end;
  int64_t window_expected_writes;
  int64_t window_received_writes;
} ss_record_info;

/* FrameSink (kv_cache.h:124-125): called once per (send, layer) by
 * ss_attention with the gathered host payload (send.range.size() * dim
 * words, token order).  The payload is borrowed for the duration of the
 * call (the reference moves a std::vector into the sink). */
typedef void (*ss_frame_sink)(void* user, int32_t layer, int64_t seq, int64_t range_begin,
                              int64_t range_end, int32_t dest, const ss_addr* dest_addr,
                              uint64_t user_tag, const uint64_t* payload, int64_t n_words);

/* Opaque CUDA IPC export of an engine's receive surface (KV pool, fill
 * bytes, page->window map, window counters) for a peer process. */
#define SS_IPC_HANDLE_BYTES 512
typedef struct {
  uint8_t bytes[SS_IPC_HANDLE_BYTES];
} ss_ipc_handle;

/* ------------------------------------------------------------------ */
/* Construction, errors, hash model                                    */
/* ------------------------------------------------------------------ */
/* KVCache(CacheConfig, const HashModel*) kv_cache.cc:26-47 with the
 * HashModel(ModelConfig) ctor hash_model.cc:22-25 folded in.  Validation:
 * CacheConfig::Validate / ModelConfig::Validate (config.cc:17-27). */
int ss_cache_create(const ss_config* config, ss_cache** out);
void ss_cache_destroy(ss_cache* cache);
int ss_abi_version(void);
const char* ss_last_error(const ss_cache* cache);
/* ErrorCodeName (event_log.cc:11-33) for 1..18; boundary names otherwise. */
const char* ss_status_name(int status);
/* IsRetryable (event_log.cc:35-43). */
int ss_status_retryable(int status);
/* Which implementation is behind the ABI: "microkv-b200" or "splitserve-reference". */
const char* ss_impl_name(void);

/* HashModel entry points an engine needs around the cache
 * (hash_model.cc:27-37,63-86). */
uint64_t ss_initial_prefix_digest(const ss_cache* cache);
uint64_t ss_embed(const ss_cache* cache, int32_t token, int64_t pos);
int32_t ss_sample_token(const ss_cache* cache, uint64_t last_hidden);

/* ------------------------------------------------------------------ */
/* Declaration stage (kv_cache.h:136-171)                              */
/* ------------------------------------------------------------------ */
/* MatchPrefixSeq (kv_cache.cc:116-118 -> radix_tree.cc:28-53). `seq_out` may be NULL. */
int ss_match_prefix(ss_cache* cache, const int32_t* tokens, int64_t n, int64_t* match_len,
                    int64_t* seq_out);
/* PrepRecv (kv_cache.cc:187-229).  addr_out->ranges_cap must cover
 * ceil((e - m) / page_size) ranges, else SS_ERR_BUFFER_TOO_SMALL with no
 * allocation (the radix LRU touch of the match has happened, as on the
 * reference's OutOfPages path). */
int ss_prep_recv(ss_cache* cache, int64_t seq, const int32_t* tokens, int64_t n, int64_t end,
                 int64_t* match_len, ss_addr* addr_out);
/* CreateSequence (kv_cache.cc:120-131). */
int ss_create_sequence(ss_cache* cache, int64_t seq, const int32_t* tokens, int64_t n);
/* ForkSequence (kv_cache.cc:133-166); n = 0 copies the parent's prefix tokens. */
int ss_fork_sequence(ss_cache* cache, int64_t parent, int64_t child, int64_t fork_len,
                     const int32_t* child_tokens, int64_t n);
/* MarkSend (kv_cache.cc:231-243). */
int ss_mark_send(ss_cache* cache, int64_t seq, int64_t begin, int64_t end, int32_t dest,
                 const ss_addr* dest_addr, uint64_t user_tag);
/* EnsureAllocated (kv_cache.cc:168-183). */
int ss_ensure_allocated(ss_cache* cache, int64_t seq, int64_t upto);
/* AppendToken (kv_cache.cc:185). */
int ss_append_token(ss_cache* cache, int64_t seq, int32_t token);
/* BeginForward (kv_cache.cc:245-306).  The plan lives until ss_plan_destroy. */
int ss_begin_forward(ss_cache* cache, const ss_batch_entry* batch, int64_t n, ss_plan** plan_out);
int64_t ss_plan_total_outputs(const ss_plan* plan);
int64_t ss_plan_num_sends(const ss_plan* plan);
int32_t ss_plan_next_layer(const ss_plan* plan);
void ss_plan_destroy(ss_plan* plan);

/* ------------------------------------------------------------------ */
/* Computation stage (kv_cache.h:173-189)                              */
/* ------------------------------------------------------------------ */
/* Attention (kv_cache.cc:308-371): KV write for Empty output slots, fold,
 * hidden outputs, then one sink call per marked send.  Sends whose `dest`
 * has an attached peer (ss_attach_peer / ss_import_ipc) are stored straight
 * into the peer's reserved pages instead of going through `sink`. */
int ss_attention(ss_cache* cache, ss_plan* plan, int32_t layer, const uint64_t* hidden_in,
                 uint64_t* hidden_out, int64_t n, ss_frame_sink sink, void* user);
/* GatherRange (kv_cache.cc:373-387) into caller storage of out_words. */
int ss_gather_range(ss_cache* cache, int64_t seq, int64_t begin, int64_t end, int32_t layer,
                    uint64_t* out, int64_t out_words);
/* BuildAddr (kv_cache.cc:389-407). */
int ss_build_addr(ss_cache* cache, int64_t seq, int64_t begin, int64_t end, ss_addr* addr_out);

/* ------------------------------------------------------------------ */
/* Transfer agent (kv_cache.h:191-199)                                 */
/* ------------------------------------------------------------------ */
/* ApplyRemoteWrite (kv_cache.cc:409-463); *apply_status = ss_apply_status.
 * Payload-size mismatch returns SS_ERR_INVALID_ARGUMENT (kv_cache.cc:411). */
int ss_apply_remote_write(ss_cache* cache, const ss_addr* addr, int32_t layer,
                          const uint64_t* payload, int64_t n_words, uint64_t tag,
                          int32_t* apply_status);
/* DrainReceiveCompletions (kv_cache.cc:465-480).  Also completes windows
 * filled by device-direct peer sends. */
int ss_drain_receive_completions(ss_cache* cache, int64_t* seqs_out, int64_t cap, int64_t* n_out);

/* ------------------------------------------------------------------ */
/* Lifecycle (kv_cache.h:201-217)                                      */
/* ------------------------------------------------------------------ */
int ss_set_finished(ss_cache* cache, int64_t seq, int32_t finished);   /* kv_cache.cc:482 */
int ss_commit_to_tree(ss_cache* cache, int64_t seq);                   /* kv_cache.cc:484-490 */
int ss_free_sequence(ss_cache* cache, int64_t seq);                    /* kv_cache.cc:492-518 */
int ss_evict(ss_cache* cache, int64_t bytes_needed, int64_t* freed_tokens); /* :520-546 */
int ss_pin(ss_cache* cache, const int32_t* prefix, int64_t n, int32_t flag); /* :548 */

/* ------------------------------------------------------------------ */
/* Queries (kv_cache.h:219-235)                                        */
/* ------------------------------------------------------------------ */
int ss_has_sequence(const ss_cache* cache, int64_t seq);
/* GetRecord (kv_cache.cc:552); own_pages may be NULL. */
int ss_get_record(ss_cache* cache, int64_t seq, ss_record_info* info, int64_t* own_pages,
                  int64_t own_cap);
/* Committed (kv_cache.cc:554-558). */
int ss_committed(ss_cache* cache, int64_t seq, int64_t* out);
/* ReadEntryWords (kv_cache.cc:560-566) into out[dim]. */
int ss_read_entry_words(ss_cache* cache, int64_t seq, int64_t pos, int32_t layer, uint64_t* out,
                        int64_t out_words);
/* FillOf (kv_cache.cc:568-574). */
int ss_fill_of(ss_cache* cache, int64_t seq, int64_t pos, int32_t layer, int32_t* out);
int64_t ss_free_pages(const ss_cache* cache);
int64_t ss_total_pages(const ss_cache* cache);
/* cache_config() (kv_cache.h:235) together with the model geometry the
 * cache was created with (the ss_config it was created from). */
int ss_cache_config(const ss_cache* cache, ss_config* out);
int64_t ss_bytes_per_page(const ss_cache* cache);
int64_t ss_sequence_count(const ss_cache* cache);
int ss_sequence_ids(const ss_cache* cache, int64_t* out, int64_t cap, int64_t* n_out);
int64_t ss_pending_send_count(const ss_cache* cache);
/* Radix tree probes (radix_tree.h:49-56), for parity tests of its quirks. */
int64_t ss_tree_node_count(const ss_cache* cache);
int ss_tree_contains(const ss_cache* cache, int64_t seq);
uint64_t ss_tree_last_touch(const ss_cache* cache, int64_t seq);
int ss_tree_sequences_by_lru(const ss_cache* cache, int64_t* out, int64_t cap, int64_t* n_out);

/* KVAddrInfo helpers (kv_addr.cc:16-51). */
int ss_addr_validate(const ss_addr* addr);
int ss_addr_slice(const ss_addr* in, int64_t begin, int64_t end, ss_addr* out);

/* ------------------------------------------------------------------ */
/* B200 device entry points (no reference counterpart; the reference   */
/* moves KV with host memcpy + TCP frames, transport.h:78-88)          */
/* ------------------------------------------------------------------ */
/* Device the cache lives on (-1 for host-only). */
int ss_device(const ss_cache* cache);
/* Attach an in-process peer engine as the destination for `dest` ranks'
 * sends (same GPU or a peer-accessible GPU). */
int ss_attach_peer(ss_cache* cache, int32_t dest, ss_cache* peer);
/* Export this engine's receive surface for another process. */
int ss_export_ipc(ss_cache* cache, ss_ipc_handle* out);
/* Map a peer process's receive surface as the destination for `dest`. */
int ss_import_ipc(ss_cache* cache, int32_t dest, const ss_ipc_handle* handle);
int ss_detach_peer(ss_cache* cache, int32_t dest);
/* How sends to `dest` publish (evidence / tests): *sys_scope = 1 when the
 * window counters are released at system scope (the peer is another GPU,
 * or MICROKV_FORCE_SYS_SCOPE=1), *peer_device = the peer's device ordinal
 * in this process (-2: another physical GPU mapped through CUDA IPC). */
int ss_peer_info(const ss_cache* cache, int32_t dest, int32_t* sys_scope, int32_t* peer_device);

/* Attention with device hidden buffers, enqueued on `stream`.  Marked
 * sends must target attached peers (device-direct); otherwise
 * SS_ERR_PEER_UNREACHABLE.  Each layer's sends run on the engine's
 * communication stream, ordered after that layer's KV writes, so layer l's
 * transfer overlaps layer l+1's compute;
 * ss_synchronize waits for them. */
int ss_attention_async(ss_cache* cache, ss_plan* plan, int32_t layer, const uint64_t* hidden_in_dev,
                       uint64_t* hidden_out_dev, void* stream);
/* DirectSend (SPEC.md:292-299 Case 1; GatherRange + ApplyRemoteWrite per
 * layer): stores layers [layer_begin, layer_end) of positions [begin, end)
 * of `seq` straight into `dest`'s pages named by `dest_addr`.  Receiver
 * semantics are ApplyRemoteWrite's: Empty slots only, every slot counts
 * toward the window, completion seen by the receiver's drain. */
int ss_direct_send_async(ss_cache* cache, int64_t seq, int64_t begin, int64_t end, int32_t dest,
                         const ss_addr* dest_addr, uint64_t user_tag, int32_t layer_begin,
                         int32_t layer_end, void* stream);
/* The same DirectSend split into the reference's two stages
 * (kv_cache.h:6-10): ss_begin_direct_send resolves both page tables and
 * uploads the row maps once (declaration); ss_launch_direct_send_async
 * enqueues only the validation + copy kernels for a layer range
 * (computation) and may be called repeatedly, e.g. once per layer as the
 * producing layer finishes.  The plan is freed with ss_plan_destroy. */
int ss_begin_direct_send(ss_cache* cache, int64_t seq, int64_t begin, int64_t end, int32_t dest,
                         const ss_addr* dest_addr, uint64_t user_tag, ss_plan** plan_out);
int ss_launch_direct_send_async(ss_cache* cache, ss_plan* plan, int32_t layer_begin,
                                int32_t layer_end, void* stream);
/* As ss_launch_direct_send_async, for a send that follows the producer's
 * writes of these layers recorded in `event` (a cudaEvent_t): the address
 * validation is enqueued on `stream` first, then the stream waits for
 * `event`, then the copy — the validation's latency leaves the
 * compute -> transfer handoff. */
int ss_launch_direct_send_after_async(ss_cache* cache, ss_plan* plan, int32_t layer_begin,
                                      int32_t layer_end, void* event, void* stream);
/* Relay chain for prefix migration to several engines:
 * `plan` is an ss_begin_direct_send plan on an engine that is itself still
 * RECEIVING [begin, end) of `seq` (an open receive window).  Each layer in
 * [layer_begin, layer_end) is forwarded to the plan's destination as soon
 * as that layer has fully landed here (the forwarding kernel's warps wait
 * on this engine's per-layer receive counters, at most timeout_ms; on
 * timeout the rest is not forwarded and ss_synchronize raises Aborted).
 * The kernel runs at most one CTA per SM (max_ctas of ss_set_send_mode
 * caps it further) so an upstream copy on the same GPU keeps SMs.  As with
 * any device-side wait: a kernel that is lazily loaded (CUDA 12's default
 * module loading) while relay warps wait may stall until they time out —
 * load such kernels first, or run with CUDA_MODULE_LOADING=EAGER (every
 * kernel of this library is loaded when a cache is created).
 * Owner -> T1 -> T2 ... puts each prefix byte on every link once, instead
 * of k times on the owner's egress.  A range that has already landed is
 * sent as a plain DirectSend. */
int ss_launch_relay_send_async(ss_cache* cache, ss_plan* plan, int32_t layer_begin,
                               int32_t layer_end, int64_t timeout_ms, void* stream);
/* How this engine's device-direct sends (DirectSend launches) move rows:
 *   SS_SEND_KERNEL       the copy kernel (default); max_ctas > 0 caps its
 *                        grid (an SM budget, so a send overlapping the next
 *                        layer's prefill takes at most max_ctas SMs' worth
 *                        of CTAs from it); 0 = the whole machine.
 *   SS_SEND_COPY_ENGINE  the GPU's copy engines (zero SMs for the rows):
 *                        at a plan's first launch the address is validated
 *                        on the device and the host waits for the verdict
 *                        (a rejected address raises UnknownAddress there,
 *                        nothing is written); every launch then moves its
 *                        (row run, layer) blocks as one batch of 3-D copies
 *                        and a small kernel marks fill states and bumps the
 *                        window counters.  Reserved receive slots are Empty
 *                        (prep_recv hands out fresh pages, re-prefill is
 *                        forbidden), so the write-Empty-only rule holds
 *                        without a per-row check; the receiver must keep
 *                        the window open while the send is in flight. */
#define SS_SEND_KERNEL 0
#define SS_SEND_COPY_ENGINE 1
int ss_set_send_mode(ss_cache* cache, int32_t mode, int32_t max_ctas);
/* Fan-out DirectSend (context-cache migration to several engines,
 * SPEC.md:434-441): the same positions [begin, end) of `seq` stored into
 * n_dest receivers at once, each through its own KVAddrInfo covering
 * [begin, end).  Semantically n_dest DirectSends; each source row is read
 * once.  n_dest <= SS_MAX_FANOUT. */
#define SS_MAX_FANOUT 8
int ss_broadcast_send_async(ss_cache* cache, int64_t seq, int64_t begin, int64_t end,
                            int32_t n_dest, const int32_t* dests, const ss_addr* dest_addrs,
                            uint64_t user_tag, int32_t layer_begin, int32_t layer_end,
                            void* stream);
/* GatherRange for layers [layer_begin, layer_end) in one launch, into
 * out_dev[layer_end - layer_begin][end - begin][dim] (a migration or a
 * prefix export that takes every layer at once). */
int ss_gather_range_layers_async(ss_cache* cache, int64_t seq, int64_t begin, int64_t end,
                                 int32_t layer_begin, int32_t layer_end, uint64_t* out_dev,
                                 void* stream);
/* GatherRange into device memory out_dev[(end-begin) * dim] on `stream`. */
int ss_gather_range_async(ss_cache* cache, int64_t seq, int64_t begin, int64_t end, int32_t layer,
                          uint64_t* out_dev, void* stream);
/* ApplyRemoteWrite with a device-resident payload. */
int ss_apply_remote_write_async(ss_cache* cache, const ss_addr* addr, int32_t layer,
                                const uint64_t* payload_dev, int64_t n_words, uint64_t tag,
                                int32_t* apply_status, void* stream);
/* KV append from a dense device row buffer rows_dev[total_outputs][dim]
 * (the producing layer's K||V rows, plan output order): Empty output slots
 * are written and marked ComputedLocal (kv_cache.cc:328-334 write rule). */
int ss_append_rows_async(ss_cache* cache, ss_plan* plan, int32_t layer, const void* rows_dev,
                         void* stream);
/* The same append for layers [layer_begin, layer_end) in one launch, from
 * rows_dev[layer_end - layer_begin][total_outputs][dim] (a producer that
 * has every layer's rows at once, e.g. a batched prefill or a KV import). */
int ss_append_rows_layers_async(ss_cache* cache, ss_plan* plan, int32_t layer_begin,
                                int32_t layer_end, const void* rows_dev, void* stream);

/* KV append fused with remote_send (write-through): one launch reads the
 * producing layer's dense rows rows_dev[layer_end - layer_begin]
 * [total_outputs][dim] once and stores them into this engine's output
 * slots (as ss_append_rows_layers_async) AND into the destination pages of
 * `send_plan` (an ss_begin_direct_send plan whose [begin, end) lies inside
 * one entry of `plan`), bumping the receiver's per-layer window counters
 * like ss_launch_direct_send_async.  Replaces the append -> send pair of a
 * PrefillThenSend layer (kv_cache.cc:328-367): the send's re-read of the
 * rows and its second launch disappear, so the P->D handoff after the last
 * layer is the append itself.  The address is validated on `stream` ahead
 * of the copy (a rejected address writes nothing remote; the local append
 * still happens).  Rows of 128 or 512 words; other dims (and the
 * copy-engine send mode) run the append and the send as two launches. */
int ss_append_rows_send_async(ss_cache* cache, ss_plan* plan, ss_plan* send_plan,
                              int32_t layer_begin, int32_t layer_end, const void* rows_dev,
                              void* stream);

/* Paged GQA decode attention over the pool, reading K||V rows through the
 * device page table: each (token, layer) entry of dim u64 words holds
 * K[num_kv_heads][head_dim] then V[num_kv_heads][head_dim] in bf16
 * (dim * 8 == 4 * num_kv_heads * head_dim).  q_dev/out_dev are bf16
 * [batch][num_q_heads][head_dim]; context of batch b = positions
 * [0, ctx_lens[b]) of seqs[b]. */
int ss_begin_decode(ss_cache* cache, const int64_t* seqs, const int64_t* ctx_lens, int64_t batch,
                    ss_plan** plan_out);
int ss_paged_decode_attention_async(ss_cache* cache, ss_plan* decode_plan, int32_t layer,
                                    int32_t num_q_heads, int32_t num_kv_heads, int32_t head_dim,
                                    float softmax_scale, const void* q_dev, void* out_dev,
                                    void* stream);
/* Paged causal GQA prefill attention (the decode engine's tail prefill in
 * balanced PD): queries at positions [q_begin, q_end) of
 * `seq` attend to keys [0, pos] of layer `layer`, read through the
 * sequence's device page table; tcgen05 tensor cores.  q_dev/out_dev are
 * bf16 [q_end - q_begin][num_q_heads][head_dim].  The caller has written
 * this layer's K||V rows for [0, q_end).  Supports head_dim 128 with a
 * group num_q_heads / num_kv_heads that divides 128 (Llama 70B: 8, Llama
 * 8B: 4, MHA: 1); SS_ERR (InvalidArgument) otherwise. */
int ss_paged_prefill_attention_async(ss_cache* cache, int64_t seq, int64_t q_begin, int64_t q_end,
                                     int32_t layer, int32_t num_q_heads, int32_t num_kv_heads,
                                     int32_t head_dim, float softmax_scale, const void* q_dev,
                                     void* out_dev, void* stream);

/* Device pointer of layer `layer`'s pool slab ([num_pages][page_size][dim]
 * u64 words) — for filling synthetic KV in tests and benchmarks. */
int ss_pool_layer_ptr(ss_cache* cache, int32_t layer, void** dev_ptr);
/* Enqueue on `stream` a device-side wait until the receive window of
 * `seq` has counted all its expected slot writes (device-direct sends from
 * peers), so receiver work queued behind it starts without a host round
 * trip.  Gives up after timeout_ms (sets the sticky status reported by
 * ss_synchronize as SS_ERR_ABORTED) so a lost sender cannot hang the GPU. */
int ss_wait_receive_async(ss_cache* cache, int64_t seq, int64_t timeout_ms, void* stream);
/* The same for one layer: the wait ends when every position of the window
 * has landed for `layer` (the per-layer ready flag peers bump after each
 * layer's rows), so the receiver can start layer-l work while later layers
 * are still in flight (PAPER.md:339-344 on the receiving side). */
int ss_wait_receive_layer_async(ss_cache* cache, int64_t seq, int32_t layer, int64_t timeout_ms,
                                void* stream);
/* Host<->device bytes this cache has copied (evidence counters). */
int ss_copy_counters(const ss_cache* cache, int64_t* h2d_bytes, int64_t* d2h_bytes);
/* Number of kernel launches this cache has issued (evidence counter). */
int64_t ss_kernel_launches(const ss_cache* cache);
/* Sync the cache's internal stream. */
int ss_synchronize(ss_cache* cache);

/* ------------------------------------------------------------------ */
/* Wire formats (transport.h:6-12; kv_addr.cc:53-118;                   */
/* transport.cc:14-107) — byte-identical to the reference's encodings   */
/* ------------------------------------------------------------------ */
#define SS_FRAME_MAGIC 0x4B565452u /* "KVTR", transport.h:32 */
#define SS_WIRE_VERSION 1          /* transport.h:33 */
#define SS_ACK_FRAME_BYTES 26
enum ss_frame_type { SS_FRAME_WRITE = 0, SS_FRAME_ACK = 1 };       /* FrameType */
enum ss_ack_status {                                                /* AckStatus */
  SS_ACK_OK = 0,
  SS_ACK_CHECKSUM_MISMATCH = 1,
  SS_ACK_UNKNOWN_ADDRESS = 2
};

/* DecodeFrame (transport.cc:76-107) without the payload copy: the payload
 * stays in the frame at payload_offset; its CRC is the device's job
 * (ss_crc32_async / ss_receive_write_frame).  For a write frame `addr`
 * receives the address (caller sets addr.ranges / addr.ranges_cap). */
typedef struct {
  int32_t type;           /* ss_frame_type */
  int32_t layer;
  uint64_t seq_tag;
  ss_addr addr;           /* write */
  int64_t payload_offset; /* write: byte offset of the payload in the frame */
  int64_t payload_bytes;  /* write */
  uint32_t wire_crc;      /* write: the frame's CRC-32 field */
  int32_t ack_status;     /* ack: ss_ack_status */
  int64_t token_begin;    /* ack */
} ss_frame_info;

/* KVAddrInfo::EncodeTo / DecodeFrom (kv_addr.cc:90-118): 20 + 8 n bytes,
 * little-endian.  Decode starts at *pos and advances it; it validates the
 * address (kv_addr.cc:16-30) like the reference. */
int ss_addr_encode(const ss_addr* addr, uint8_t* out, int64_t cap, int64_t* len);
int ss_addr_decode(const uint8_t* data, int64_t size, int64_t* pos, ss_addr* out);
/* KVAddrInfo::ToJson / FromJson (kv_addr.cc:53-70); `len` excludes the NUL
 * written after the text when it fits.  Malformed JSON returns
 * SS_ERR_INTERNAL, as the reference's nlohmann exception does at this ABI. */
int ss_addr_to_json(const ss_addr* addr, char* out, int64_t cap, int64_t* len);
int ss_addr_from_json(const char* text, int64_t len, ss_addr* out);
/* Bytes of a write frame before its payload: 41 + 8 * n_ranges. */
int64_t ss_frame_write_header_size(int64_t n_ranges);
/* EncodeAckFrame (transport.cc:64-74) into out[SS_ACK_FRAME_BYTES]. */
int ss_frame_encode_ack(uint64_t seq_tag, int32_t layer, int64_t token_begin, int32_t status,
                        uint8_t* out, int64_t cap, int64_t* len);
int ss_frame_decode(const uint8_t* frame, int64_t size, ss_frame_info* info);
/* CRC-32 (Crc32, transport.cc:14-28: IEEE 802.3, reflected, 0xEDB88320)
 * of n_bytes of device memory (any alignment), written as a uint32 to
 * crc_dev, enqueued on `stream`.  One sm_100a launch. */
int ss_crc32_async(ss_cache* cache, const void* data_dev, int64_t n_bytes, uint32_t* crc_dev,
                   void* stream);
/* EncodeWriteFrame(WriteFrame{seq_tag, layer, dest_addr,
 * GatherRange(seq, [begin, end), layer)}) (transport.cc:46-62): the layer's
 * rows are gathered through the page table and checksummed on the GPU.
 * dest_addr must cover exactly [begin, end) (SS_ERR_ADDR_MISMATCH, as
 * MarkSend).  Host variant: `frame` is host memory, returns when the frame
 * is complete.  Device variant: `frame_dev` is device memory with
 * frame_dev + ss_frame_write_header_size(n_ranges) 32-byte aligned;
 * enqueued on `stream`.  Either way *frame_len = the frame's size
 * (header + payload + 4); short `cap` returns SS_ERR_BUFFER_TOO_SMALL with
 * *frame_len = the size needed. */
int ss_encode_write_frame(ss_cache* cache, int64_t seq, int64_t begin, int64_t end, int32_t layer,
                          uint64_t seq_tag, const ss_addr* dest_addr, uint8_t* frame, int64_t cap,
                          int64_t* frame_len);
int ss_encode_write_frame_async(ss_cache* cache, int64_t seq, int64_t begin, int64_t end,
                                int32_t layer, uint64_t seq_tag, const ss_addr* dest_addr,
                                void* frame_dev, int64_t cap, int64_t* frame_len, void* stream);
/* The transfer agent's step for one received write frame in host memory
 * (TCP fabric inbound loop, tcp_fabric.cc:144-168): decode, payload to the
 * device, CRC-32 on the device; on a mismatch the ack is ChecksumMismatch
 * and nothing is applied (*apply_status = -1); otherwise ApplyRemoteWrite
 * (addr, layer, payload, seq_tag) runs and the ack is UnknownAddress or Ok
 * (*apply_status = ss_apply_status).  ack_out receives the 26-byte ack
 * frame to send back.  Framing errors return SS_ERR_INVALID_ARGUMENT. */
int ss_receive_write_frame(ss_cache* cache, const uint8_t* frame, int64_t size, uint8_t* ack_out,
                           int32_t* apply_status);

#ifdef __cplusplus
} /* extern "C" */
#endif

#endif /* MICROKV_H_ */
