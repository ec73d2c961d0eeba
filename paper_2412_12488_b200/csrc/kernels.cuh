// kernels.cuh — launch interfaces of the sm_100a page-operation kernels.
//
// HBM layout of one engine:
//   pool  u64 [L][num_pages][P][W]   a (layer, page) block is P*W*8 bytes
//                                    contiguous (64 KiB at Llama shapes), a
//                                    (layer, slot) row is W*8 bytes (4 KiB)
//   fill  u8  [L][num_pages][P]      FillState per (layer, slot)
//   expecting u8 [num_pages][P]      receive reservation (kv_cache.h:52)
//   page_window i32 [num_pages]      open receive window of the page's owner
//   win_received u64 [max_windows]   slot writes counted per window
//   win_layer_rows u32 [max_windows][L]  rows landed per (window, layer)
// A "slot index" is page * P + slot.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace mkv {

// Device status bits (sticky, per engine).
enum : uint32_t {
  kStatusUnknownAddress = 1u << 0,  // a remote write failed receiver validation
  kStatusMissingKV = 1u << 1,       // a read hit an Empty slot
  kStatusWaitTimeout = 1u << 2,     // a device-side receive wait gave up
};

// Device-side wait: spin (acquire, system scope) until *counter >= target
// or timeout_ns elapses; on timeout set kStatusWaitTimeout.
// Load every kernel of the library into the current context (see kernels.cu).
void preload_kernels();
void preload_decode_attn_kernels();
void preload_prefill_attn_kernels();
void preload_crc32_kernels();

void launch_wait_counter32(const uint32_t* counter, uint32_t target, long long timeout_ns,
                           uint32_t* status, cudaStream_t s);
void launch_wait_counter(const unsigned long long* counter, unsigned long long target,
                         long long timeout_ns, uint32_t* status, cudaStream_t s);

// Row copy between slot-addressed (or dense) row arrays, over
// rows x layers items.  All row copies of the hot path go through it:
//   remote_send / DirectSend   slots -> peer slots (fill check, window counters)
//   send gather, GatherRange   slots -> dense staging
//   ApplyRemoteWrite           dense staging -> slots (fill check)
//   KV append                  dense rows -> slots (fill check)
struct ValidateParams {
  const int64_t* range_page;   // per range
  const int32_t* range_begin;
  const int32_t* range_count;
  int64_t n_ranges;
  const int32_t* page_window;  // destination engine
  const uint8_t* expecting;    // destination engine [pages][P]
  int64_t num_pages;
  int32_t P;
  int32_t* verdict;            // [0] window id, [1] = gen of the last failed validation,
                               // [2] the window's open-generation when it validated
  const unsigned long long* win_gen;  // destination: generation per window id (bumped at open)
  uint32_t* status;            // sender-side sticky status (kStatusUnknownAddress)
  int32_t gen;                 // launch generation (>= 1): no reset of verdict[1] needed
};

struct CopyParams {
  const uint64_t* src;        // layer-0 base
  int64_t src_layer_words;    // words between layers
  const int32_t* src_idx;     // slot per row, or null = dense row r
  uint64_t* dst;
  int64_t dst_layer_words;
  const int32_t* dst_idx;
  uint8_t* dst_fill;          // layer-0 base of dst fill, or null = no fill rule
  int64_t dst_fill_layer;     // bytes between layers
  uint8_t fill_value;         // state written into Empty dst slots
  int64_t n_rows;
  int32_t layer0;             // first layer (absolute)
  int32_t n_layers;
  int32_t W;                  // u64 words per row
  // Receive-window accounting on the destination engine (remote sends).
  unsigned long long* win_received;  // null = none
  uint32_t* win_layer_rows;
  int32_t win_layers;         // L of the destination (row stride of win_layer_rows)
  const int32_t* verdict;     // validation result: >= 0 window id, < 0 reject
  uint32_t* status;           // sender-side sticky status
  int32_t group;              // rows per warp item (set by the launcher)
  int32_t sys_scope;          // 1: the counters' observer is another GPU (fence/reds at
                              // system scope); 0: same GPU (device scope is enough)
  int32_t gen;                // launch generation: verdict[1] == gen means rejected
  int32_t pdl;                // 1: launched as a programmatic dependent of the
                              // validation kernel (griddepcontrol.wait before
                              // the verdict is read)
  int32_t max_ctas;           // > 0: grid cap (SM budget of a send); 0 = whole machine
  int32_t no_data;            // 1: the rows were moved by the copy engines; only
                              // mark fill states and publish the window counters
  // 1: every CTA validates the destination address itself (`val`) before
  // copying, instead of reading a separate validation grid's verdict — one
  // launch per small send (all CTAs read the same receiver state, so the
  // verdict is the same in every CTA: all rows land or none does).
  int32_t inline_validate;
  ValidateParams val;
  // 1: the grid's predecessor on the stream is the validation kernel, which
  // itself started after the rows' producer completed, so each warp's first
  // source row is loaded before griddepcontrol.wait (overlapping the
  // validation); the stores still wait for the verdict.
  int32_t prefetch_src;
  // 1: no validation grid for this launch: the plan's address was validated
  // by an earlier launch (verdict words, gen = that launch's generation) and
  // is still good iff its first page still maps to the window and the
  // window's open-generation is unchanged (a close, free or re-open changes
  // one of them).
  int32_t gen_check;
  const unsigned long long* win_gen;  // destination window generations
  const int32_t* page_window;         // destination page -> window
  const int64_t* first_page;          // the address's first page (plan data)
};
void launch_copy_rows(const CopyParams& p, cudaStream_t s, int num_sms);

// Relay hop: copy rows layer by layer as this engine's own receive
// counters wait[layer0 + l] reach `target` (see k_relay_rows).
void launch_relay_rows(const CopyParams& p, const uint32_t* wait, uint32_t target,
                       long long timeout_ns, cudaStream_t s, int num_sms);

// Fan-out row copy: one source row set stored into up to kMaxFanout
// destinations (each with its own slots, fill rule and window counters).
// Destination d takes source rows [row_off[d], row_off[d] + row_cnt[d])
// (its dst_idx indexed from row_off[d]); a null verdict means no
// validation (the engine's own pages), a null win_received no counters.
// truth >= 0 names the destination whose existing non-Empty rows take
// precedence over the source row for every other destination: the fused
// KV append + remote_send sends what the sender's page holds, as the
// reference's send loop reads the pool after the write (kv_cache.cc:328-367).
constexpr int kMaxFanout = 8;
struct FanoutParams {
  const uint64_t* src;
  int64_t src_layer_words;
  const int32_t* src_idx;     // slot per row, or null = dense row r
  int64_t n_rows;
  int32_t layer0, n_layers, W, n_dest;
  uint64_t* dst[kMaxFanout];
  int64_t dst_layer_words[kMaxFanout];
  const int32_t* dst_idx[kMaxFanout];
  uint8_t* dst_fill[kMaxFanout];
  int64_t dst_fill_layer[kMaxFanout];
  uint8_t fill_value[kMaxFanout];
  int64_t row_off[kMaxFanout];
  int64_t row_cnt[kMaxFanout];
  unsigned long long* win_received[kMaxFanout];
  uint32_t* win_layer_rows[kMaxFanout];
  int32_t win_layers[kMaxFanout];
  const int32_t* verdict[kMaxFanout];
  int32_t truth;              // -1: none
  int32_t group;              // rows per warp item (set by the launcher)
  int32_t sys_scope;          // as CopyParams::sys_scope, for any destination
  int32_t gen;                // launch generation, as CopyParams::gen
  int32_t pdl;                // as CopyParams::pdl
};
void launch_copy_rows_fanout(const FanoutParams& p, cudaStream_t s, int num_sms);

// Receiver-side validation of a remote write (ApplyRemoteWrite's checks,
// kv_cache.cc:415-436): every addressed page maps to the same open window
// and every slot is expecting-remote.  Writes the window id or -1 to *verdict.
void launch_validate_remote(const ValidateParams& p, cudaStream_t s);

// Attention write (kv_cache.cc:328-334 + KvEntryWords hash_model.cc:39-46):
// for each output row, if its fill is Empty write the W hash words of
// (digest, layer) and set ComputedLocal.
void launch_attn_write_hash(uint64_t* pool_l, uint8_t* fill_l, const int32_t* slots,
                            const uint64_t* digests, int64_t n, int32_t layer, int32_t W,
                            cudaStream_t s, int num_sms);

// EntryDigest of each slot row (hash_model.cc:57-61) -> F[n].
void launch_entry_digest(const uint64_t* pool_l, const int32_t* slots, int64_t n, int32_t W,
                         uint64_t* F, cudaStream_t s, int num_sms);

// Per-entry inclusive fold + hidden update (kv_cache.cc:319-351).
struct FoldEntry {
  int64_t fold_off;    // first fold row of the entry in F
  int64_t n_fold;      // end - fold_from
  int64_t first_out;   // begin - fold_from
  int64_t out_off;     // first output row in hidden arrays
  int64_t pos0;        // fold_from
  uint64_t* fold_sums; // device [L] running sums of the sequence
};
void launch_fold_scan(const FoldEntry* entries, int64_t n_entries, const uint64_t* F,
                      const uint64_t* hidden_in, uint64_t* hidden_out, int32_t layer,
                      cudaStream_t s);

// Zero fill/expecting bytes and page_window of freed pages (kv_cache.cc:499-507).
void launch_reset_pages(uint8_t* fill, uint8_t* expecting, int32_t* page_window,
                        const int64_t* pages, int64_t n_pages, int32_t L, int64_t num_pages,
                        int32_t P, cudaStream_t s);

// prep_recv's device half (kv_cache.cc:215-227): mark reserved slots
// expecting-remote, point the sequence's pages at receive window `window`,
// zero that window's counters.
void launch_open_window(uint8_t* expecting, const int32_t* slots, int64_t n_slots,
                        int32_t* page_window, const int64_t* pages, int64_t n_pages,
                        int32_t window, unsigned long long* win_received,
                        uint32_t* win_layer_rows, unsigned long long* win_gen, int32_t L,
                        cudaStream_t s);

// A drained receive window's pages stop mapping to it (page_window = -1
// where it still equals `window`).
void launch_close_window(int32_t* page_window, const int64_t* pages, int64_t n_pages,
                         int32_t window, cudaStream_t s);

// First position in [0, n) whose slot has an Empty fill on any layer (n if none).
void launch_first_nonfull(const uint8_t* fill, int64_t fill_layer_bytes, int32_t L,
                          const int32_t* slots, int64_t n, unsigned long long* out,
                          cudaStream_t s, int num_sms);

// Concatenate per-sequence device page tables into a CSR slot map:
// out[off[b] + t] = tables[b][t] for t < len[b].
void launch_gather_tables(const int32_t* const* tables, const int64_t* off, const int32_t* len,
                          int64_t batch, int64_t total, int32_t* out, cudaStream_t s, int num_sms);

// Any Empty fill on `layer` among the slot rows -> status |= kStatusMissingKV.
void launch_check_filled(const uint8_t* fill_l, const int32_t* slots, int64_t n, uint32_t* status,
                         cudaStream_t s, int num_sms);

// Paged GQA decode attention (decode_attn.cu): stream-K split over the
// (batch, kv head, 16-token tile) space, partials + combine.
size_t decode_attn_smem(int head_dim);
int decode_attn_resident_ctas(int head_dim, int num_sms);
bool launch_decode_attn(const void* pool_l, int64_t row_elems, const int32_t* slots,
                        const int64_t* ctx_off, const int32_t* ctx_len, const int64_t* seg_start,
                        int64_t n_seg, int64_t total_tiles, const void* q, int batch, int Hq,
                        int Hkv, int D, float scale, float* part_o, float* part_ml, void* out,
                        int grid, uint32_t* seg_count, const int32_t* cta_seg,
                        cudaStream_t s);

// Paged GQA decode attention with TMA page-chunk loads (decode_pages.cu):
// 8 KV heads x head_dim 128 (4 KiB rows), up to 8 query heads per KV head.
// chunks: int4 {slot0, tok0, n, b} runs of <= 16 consecutive slots in batch
// order; the grid (decode_pages_grid) splits them into equal ranges;
// piece_first / piece_count per context: the CTAs its chunks span.
struct PoolTensorMap;
bool decode_pages_supported(int Hq, int Hkv, int D, int64_t row_u64);
int decode_pages_grid(int num_sms, int64_t n_chunks);
int launch_decode_pages(const PoolTensorMap& map, int layer, const int4* chunks, int64_t n_chunks,
                        const int32_t* piece_first, const int32_t* piece_count, bool any_split,
                        const void* q, int batch, int Hq, int Hkv, float scale, float* part_o,
                        float* part_ml, void* out, int grid, cudaStream_t s);
void preload_decode_pages_kernels();

// Paged causal GQA prefill attention on tcgen05 (prefill_attn.cu): queries
// [q_pos0, q_pos0 + n_q) of one sequence over keys [0, q_pos0 + n_q).  K/V
// come by TMA through two tensor maps of the whole pool viewed as bf16
// [layers][rows][row_u64 * 4]: boxes of {64, prefill_attn_box_rows(P), 1} (a page chunk)
// and {64, 1, 1} (one row, for chunks whose slots are not consecutive).
struct alignas(64) PoolTensorMap {
  unsigned char bytes[128];
};
bool make_pool_tensor_map(void* pool, int64_t layers, int64_t rows, int64_t row_u64,
                          int box_rows, PoolTensorMap* out);
bool prefill_attn_supported(int page_size, int Hq, int Hkv, int D);
int prefill_attn_box_rows(int page_size);  // rows of the page-chunk box
// Returns the number of kernels launched (0: unsupported shape).
int launch_prefill_attn(const PoolTensorMap& page_map, const PoolTensorMap& row_map, int layer,
                         int page_size, int64_t pool_rows, const int32_t* slots, const void* q,
                         int q_pos0, int n_q, int Hq, int Hkv, int D, float scale, void* out,
                         cudaStream_t s);

// CRC-32 (IEEE, reflected) of n device bytes (crc32.cu): one launch, any
// alignment and length; workspace of crc32_workspace_bytes(n) device bytes
// (its first word is reset by the launch).  crc32_x8n(n) = x^(8n) mod P.
size_t crc32_workspace_bytes(int64_t n, int num_sms);
void launch_crc32(const void* data, int64_t n, uint32_t* out, void* workspace, cudaStream_t s,
                  int num_sms);
uint32_t crc32_x8n(uint64_t n);

}  // namespace mkv
