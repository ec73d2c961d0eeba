// kernels.cu — sm_100a kernels of the paged-KV page operations.
//
// All of them are HBM- (or, across engines, NVLink-) bound byte movers or
// integer hash loops; none is GEMM-shaped, so there is no tensor-core work
// here ("Kernels and their rooflines").  Rows are 16-byte
// vectorised, one warp per (row, layer) item, grids sized to a multiple of
// the SM count with every warp striding over items.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>

#include "hash.cuh"
#include "kernels.cuh"

namespace mkv {

namespace {

constexpr int kCopyThreads = 256;

__device__ __forceinline__ ulonglong2 ld_stream(const ulonglong2* p) {
  ulonglong2 v;
  asm volatile("ld.global.nc.L1::no_allocate.v2.u64 {%0, %1}, [%2];"
               : "=l"(v.x), "=l"(v.y)
               : "l"(p));
  return v;
}

__device__ __forceinline__ void st_vec(ulonglong2* p, ulonglong2 v) {
  asm volatile("st.global.v2.u64 [%0], {%1, %2};" ::"l"(p), "l"(v.x), "l"(v.y) : "memory");
}

struct alignas(32) u256 {
  unsigned long long a, b, c, d;
};

// Coherent (not .nc) 32-byte load: ptxas may not sink it below a store that
// could alias, so a row's loads stay grouped ahead of its stores and each
// lane keeps 4 requests in flight (with .nc, ptxas interleaved them 1:1 and
// the copy lost ~12%; profiles/micro/lib_kernel.cu).
__device__ __forceinline__ u256 ld256(const void* p) {
  u256 v;
#ifndef MKV_LD_NO_EF  // rows are read once: L2 evict-first leaves L2 to the writes (+1%)
  asm volatile("ld.global.L1::no_allocate.L2::evict_first.v4.u64 {%0, %1, %2, %3}, [%4];"
#else
  asm volatile("ld.global.L1::no_allocate.v4.u64 {%0, %1, %2, %3}, [%4];"
#endif
               : "=l"(v.a), "=l"(v.b), "=l"(v.c), "=l"(v.d)
               : "l"(p)
               : "memory");
  return v;
}

__device__ __forceinline__ void st256(void* p, const u256& v) {
#ifdef MKV_ST_CS  // A/B: streaming (evict-first) row stores
  asm volatile("st.global.cs.v4.u64 [%0], {%1, %2, %3, %4};" ::"l"(p), "l"(v.a), "l"(v.b), "l"(v.c),
#else
  asm volatile("st.global.v4.u64 [%0], {%1, %2, %3, %4};" ::"l"(p), "l"(v.a), "l"(v.b), "l"(v.c),
#endif
               "l"(v.d)
               : "memory");
}

// Fire-and-forget system-scope reductions for the window counters (a
// returning atomicAdd_system is one full round trip per call; thread 0
// looping over 80 layers of them cost ~25 us per launch).
// Scope: system when the counters' observer is another GPU, device when it
// is this GPU (another engine or process on it): a system-scope fence per
// launch cost ~20 us even for a 5 MB transfer.
__device__ __forceinline__ void red_sys_add(uint32_t* p, uint32_t v, bool sys) {
  if (sys) asm volatile("red.release.sys.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
  else asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void red_sys_add(unsigned long long* p, unsigned long long v, bool sys) {
  if (sys) asm volatile("red.release.sys.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
  else asm volatile("red.release.gpu.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void fence_publish(bool sys) {
  if (sys) asm volatile("fence.acq_rel.sys;" ::: "memory");
  else asm volatile("fence.acq_rel.gpu;" ::: "memory");
}

__device__ __forceinline__ uint8_t ld_cg_u8(const uint8_t* p) {
  unsigned short v;
  asm volatile("ld.global.cg.u8 %0, [%1];" : "=h"(v) : "l"(p));
  return static_cast<uint8_t>(v);
}

// One warp moves one W-word row: 32-byte vectors when the row allows it
// (4 per lane in flight for a 4 KiB row), else 16-byte, else words.
__device__ __forceinline__ void warp_copy_row(const uint64_t* __restrict__ src,
                                              uint64_t* __restrict__ dst, int32_t W, int lane) {
  if ((W & 3) == 0) {
    const u256* s4 = reinterpret_cast<const u256*>(src);
    u256* d4 = reinterpret_cast<u256*>(dst);
    const int nv = W >> 2;
    int v = lane;
    for (; v + 32 * 3 < nv; v += 32 * 4) {
      u256 t[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) t[u] = ld256(s4 + v + 32 * u);
#pragma unroll
      for (int u = 0; u < 4; ++u) st256(d4 + v + 32 * u, t[u]);
    }
    for (; v < nv; v += 32) st256(d4 + v, ld256(s4 + v));
  } else if ((W & 1) == 0) {
    const ulonglong2* s2 = reinterpret_cast<const ulonglong2*>(src);
    ulonglong2* d2 = reinterpret_cast<ulonglong2*>(dst);
    for (int v = lane; v < (W >> 1); v += 32) st_vec(d2 + v, ld_stream(s2 + v));
  } else {
    for (int j = lane; j < W; j += 32) dst[j] = __ldg(src + j);
  }
}

// Items are groups of kGroup consecutive rows of one layer.  Lanes
// 0..kGroup-1 fetch the group's slot indices and destination fill bytes in
// one coalesced access each, so no row waits on a dependent load; rows are
// then copied back to back and the fill marks stored lane-parallel.  (A
// per-row fill check serialised a fill load before every store and cost
// ~15% of bandwidth; profiles/micro/copy_variants.cu.)
#ifndef MKV_GROUP
#define MKV_GROUP 4
#endif
constexpr int kGroup = MKV_GROUP;
#ifndef MKV_SMALL_SEND_ROWS
#define MKV_SMALL_SEND_ROWS 2048
#endif
constexpr int64_t kSmallSendRows = MKV_SMALL_SEND_ROWS;  // rows per item for long launches (1 for launches within one wave)

// kVec > 0: rows are exactly kVec 32-byte vectors per lane (W = 128*kVec
// words), fully unrolled; kVec == 0: any W.
template <int kVec>
__device__ __forceinline__ void copy_row(const uint64_t* __restrict__ src, uint64_t* __restrict__ dst,
                                         int32_t W, int lane) {
  if constexpr (kVec > 0) {
    const u256* s4 = reinterpret_cast<const u256*>(src) + lane;
    u256* d4 = reinterpret_cast<u256*>(dst) + lane;
    u256 t[kVec];
#pragma unroll
    for (int u = 0; u < kVec; ++u) t[u] = ld256(s4 + 32 * u);
#pragma unroll
    for (int u = 0; u < kVec; ++u) st256(d4 + 32 * u, t[u]);
  } else {
    warp_copy_row(src, dst, W, lane);
  }
}

// The checks of k_validate_remote by one CTA over the whole address (small
// sends): returns the window id, or -1 when the address is rejected; CTA 0
// records the verdict / status as the validation grid would.  Every thread
// of the CTA must call it (CTA barrier inside).
__device__ int32_t validate_in_cta(const ValidateParams& p) {
  int32_t w0 = -1;
  bool bad = p.n_ranges <= 0;
  if (p.n_ranges > 0) {
    const int64_t pg0 = p.range_page[0];
    if (pg0 < 0 || pg0 >= p.num_pages) {
      bad = true;
    } else {
      w0 = *reinterpret_cast<const volatile int32_t*>(p.page_window + pg0);
      if (w0 < 0) bad = true;
    }
  }
  const int64_t work = p.n_ranges * p.P;
  for (int64_t i = threadIdx.x; !bad && i < work; i += blockDim.x) {
    const int64_t r = i / p.P;
    const int32_t k = static_cast<int32_t>(i % p.P);
    const int64_t pg = p.range_page[r];
    const int32_t b = p.range_begin[r], c = p.range_count[r];
    if (pg < 0 || pg >= p.num_pages || b < 0 || c < 0 || b + c > p.P) {
      bad = true;
    } else if (k < c) {
      if (k == 0 && *reinterpret_cast<const volatile int32_t*>(p.page_window + pg) != w0) bad = true;
      if (reinterpret_cast<const volatile uint8_t*>(p.expecting)[pg * p.P + b + k] == 0) bad = true;
    }
  }
  bad = __syncthreads_or(bad) != 0;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    p.verdict[0] = w0;
    if (w0 >= 0 && p.win_gen != nullptr)
      p.verdict[2] = static_cast<int32_t>(*reinterpret_cast<const volatile unsigned long long*>(p.win_gen + w0));
    if (bad) {
      *reinterpret_cast<volatile int32_t*>(p.verdict + 1) = p.gen;
      if (p.status != nullptr) atomicOr(p.status, kStatusUnknownAddress);
    }
  }
  return bad ? -1 : w0;
}

template <int kVec, bool kPrefetch = false>
__global__ void __launch_bounds__(kCopyThreads) k_copy_rows(CopyParams p) {
  extern __shared__ uint32_t s_rows[];  // per relative layer (accounting only)
  const int lane = threadIdx.x & 31;
  const int64_t warp = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t n_warps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  const int group = p.group > 0 ? p.group : kGroup;
  const int64_t groups = (p.n_rows + group - 1) / group;
  const int64_t items = groups * p.n_layers;
  // The first item's slot indices before waiting for the previous kernel:
  // slot maps and page tables are host uploads ordered by stream events,
  // never written by a kernel, so they may be read while the predecessor
  // drains (fill bytes and row data are read after the wait).
  int32_t pre_s = 0, pre_d = 0;
  // kVec > 0 and p.prefetch_src: the first item's first row, loaded before
  // the grid dependency wait (see CopyParams::prefetch_src).
  u256 pre_row[kVec > 0 && kPrefetch ? kVec : 1];
  bool have_pre_row = false;
  if (warp < items) {
    const int32_t lrel = static_cast<int32_t>(warp / groups);
    const int64_t r0 = (warp - static_cast<int64_t>(lrel) * groups) * group;
    if (lane < p.n_rows - r0 && lane < group) {
      pre_s = p.src_idx ? __ldg(p.src_idx + r0 + lane) : static_cast<int32_t>(r0 + lane);
      pre_d = p.dst_idx ? __ldg(p.dst_idx + r0 + lane) : static_cast<int32_t>(r0 + lane);
    }
    if constexpr (kVec > 0 && kPrefetch) {
      if (!p.no_data) {
        const int64_t si = __shfl_sync(0xffffffffu, pre_s, 0);
        const u256* s4 = reinterpret_cast<const u256*>(p.src + lrel * p.src_layer_words + si * p.W) + lane;
#pragma unroll
        for (int u = 0; u < kVec; ++u) pre_row[u] = ld256(s4 + 32 * u);
        have_pre_row = true;
      }
    }
  }
  // Programmatic dependent of the previous kernel on the stream (the
  // validation kernel, or the previous copy): this grid's launch overlaps
  // it; nothing it may have written is read before it completed.
  if (p.pdl) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    // The next PDL launch on the stream (another copy) may start its CTAs as
    // ours drain; it waits for our completion before touching memory.
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  }
  int32_t window = -1;
  if (p.inline_validate) {
    window = validate_in_cta(p.val);
    if (window < 0) return;  // rejected: no writes, no counts (uniform over the CTA)
  } else if (p.gen_check) {
    const volatile int32_t* v = reinterpret_cast<const volatile int32_t*>(p.verdict);
    window = v[1] == p.gen ? -1 : v[0];
    if (window >= 0) {
      const int64_t pg = *p.first_page;
      const bool same_window = reinterpret_cast<const volatile int32_t*>(p.page_window)[pg] == window;
      const bool same_open = static_cast<int32_t>(
          reinterpret_cast<const volatile unsigned long long*>(p.win_gen)[window]) == v[2];
      if (!same_window || !same_open) window = -1;
    }
    if (window < 0) {
      if (blockIdx.x == 0 && threadIdx.x == 0 && p.status != nullptr)
        atomicOr(p.status, kStatusUnknownAddress);
      return;  // the receiver's window changed since validation: nothing written
    }
  } else if (p.verdict != nullptr) {
    window = reinterpret_cast<const volatile int32_t*>(p.verdict)[1] == p.gen
                 ? -1
                 : reinterpret_cast<const volatile int32_t*>(p.verdict)[0];
    if (window < 0) return;  // rejected by validation: no writes, no counts
  }
  const bool account = p.win_received != nullptr;
  if (account) {
    for (int i = threadIdx.x; i < p.n_layers; i += blockDim.x) s_rows[i] = 0;
    __syncthreads();
  }
  for (int64_t it = warp; it < items; it += n_warps) {
    const int32_t lrel = static_cast<int32_t>(it / groups);
    const int64_t r0 = (it - static_cast<int64_t>(lrel) * groups) * group;
    const int nr = static_cast<int>(p.n_rows - r0 < group ? p.n_rows - r0 : group);
    int32_t my_s = 0, my_d = 0;  // slot indices fit int32 (checked at cache creation)
    uint8_t my_f = 0;
#ifdef MKV_NO_FILL  // measurement only: no destination fill read / mark on remote sends
    uint8_t* fill_l = p.verdict != nullptr ? nullptr
                      : (p.dst_fill != nullptr ? p.dst_fill + lrel * p.dst_fill_layer : nullptr);
#else
    uint8_t* fill_l = p.dst_fill != nullptr ? p.dst_fill + lrel * p.dst_fill_layer : nullptr;
#endif
    const uint64_t* src_l = p.src + lrel * p.src_layer_words;
    uint64_t* dst_l = p.dst + lrel * p.dst_layer_words;
    if (lane < nr) {
#ifndef MKV_NO_PREFETCH
      if (it == warp) {
#else
      if (false) {
#endif
        my_s = pre_s;
        my_d = pre_d;
      } else {
        my_s = p.src_idx ? __ldg(p.src_idx + r0 + lane) : static_cast<int32_t>(r0 + lane);
        my_d = p.dst_idx ? __ldg(p.dst_idx + r0 + lane) : static_cast<int32_t>(r0 + lane);
      }
      if (fill_l != nullptr) my_f = ld_cg_u8(fill_l + my_d);
    }
    // Empty destination slots only (kv_cache.cc:447); every row counts.
    const unsigned todo = __ballot_sync(0xffffffffu, lane < nr && my_f == 0);
    // One row's loads in flight per lane before its stores: two rows
    // (-DMKV_PAIR_ROWS in round 2) measured 1% slower on the 80-layer send
    // and 15% slower on per-layer appends (registers: fewer resident CTAs).
#pragma unroll 1
    for (int k = 0; k < nr; ++k) {
      const int64_t si = __shfl_sync(0xffffffffu, my_s, k);
      const int64_t di = __shfl_sync(0xffffffffu, my_d, k);  // int32 shuffles, widened
      if constexpr (kVec > 0 && kPrefetch) {
        if (have_pre_row && it == warp && k == 0) {
          if ((todo & 1u) && !p.no_data) {
            u256* d4 = reinterpret_cast<u256*>(dst_l + di * p.W) + lane;
#pragma unroll
            for (int u = 0; u < kVec; ++u) st256(d4 + 32 * u, pre_row[u]);
          }
          continue;
        }
      }
      if (((todo >> k) & 1u) && !p.no_data) copy_row<kVec>(src_l + si * p.W, dst_l + di * p.W, p.W, lane);
    }
    if (fill_l != nullptr) {
      __syncwarp();
      if ((todo >> lane) & 1u) fill_l[my_d] = p.fill_value;
    }
    if (account && lane == 0) atomicAdd(&s_rows[lrel], static_cast<uint32_t>(nr));
  }
  if (account) {
    // Publish: every thread's row stores, then the counters.  The CTA
    // barrier puts every thread's stores before each counter update in
    // causality order and the updates are release reductions (cumulative),
    // so a peer engine that acquires a counter also observes the rows — the
    // barrier + red.release pattern of CUTLASS's semaphores; no per-thread
    // fence (-DMKV_FENCE_ALL restores one per thread for A/B).
#ifdef MKV_FENCE_ALL
    fence_publish(p.sys_scope != 0);
#endif
    __syncthreads();
    // Per-layer counters in parallel, one thread per layer; the total by
    // thread 0.
    for (int i = threadIdx.x; i < p.n_layers; i += blockDim.x) {
      if (s_rows[i] != 0) {
        red_sys_add(p.win_layer_rows + static_cast<int64_t>(window) * p.win_layers + p.layer0 + i,
                    s_rows[i], p.sys_scope != 0);
      }
    }
    // The window total last: once a receiver's drain sees the window
    // complete, no per-layer counter update of it is still in flight (the
    // window row is recycled after the drain).
    __syncthreads();
    if (threadIdx.x == 0) {
      unsigned long long total = 0;
      for (int i = 0; i < p.n_layers; ++i) total += s_rows[i];
      if (total != 0) red_sys_add(p.win_received + window, total, p.sys_scope != 0);
    }
  }
}

// Relay forward (a hop of a prefix-migration chain): like k_copy_rows from
// this engine's slots into a peer's, but layer lrel of the source is only
// read once this engine's own receive counter for it reached `target`
// rows (lane 0 of a warp polls it with acquire loads when the warp first
// reaches the layer), and each warp publishes its rows per layer as it
// leaves the layer (release reductions), so the next hop can start on a
// layer while this one is still receiving later layers.  The grid is
// bounded (it spins while upstream layers are in flight) so the upstream
// copy keeps SMs on a shared GPU.  A wait past timeout_ns sets
// kStatusWaitTimeout and the warp stops (nothing more is forwarded).
template <int kVec>
__global__ void __launch_bounds__(kCopyThreads) k_relay_rows(CopyParams p, const uint32_t* wait,
                                                             uint32_t target, long long timeout_ns) {
  if (p.pdl) asm volatile("griddepcontrol.wait;" ::: "memory");
  const int32_t window = reinterpret_cast<const volatile int32_t*>(p.verdict)[1] == p.gen
                             ? -1
                             : reinterpret_cast<const volatile int32_t*>(p.verdict)[0];
  if (window < 0) return;  // rejected by validation
  const bool sys = p.sys_scope != 0;
  const int lane = threadIdx.x & 31;
  const int64_t warp = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t n_warps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  const int group = kGroup;
  const int64_t groups = (p.n_rows + group - 1) / group;
  const int64_t items = groups * p.n_layers;
  int32_t ready = -1, cur = -1;
  uint32_t cur_rows = 0;
  unsigned long long t0 = 0;
  auto publish = [&](int32_t l, uint32_t rows) {
    __syncwarp();
    if (lane == 0 && rows != 0) {
      red_sys_add(p.win_layer_rows + static_cast<int64_t>(window) * p.win_layers + p.layer0 + l,
                  rows, sys);
      red_sys_add(p.win_received + window, static_cast<unsigned long long>(rows), sys);
    }
  };
  for (int64_t it = warp; it < items; it += n_warps) {
    const int32_t lrel = static_cast<int32_t>(it / groups);
    const int64_t r0 = (it - static_cast<int64_t>(lrel) * groups) * group;
    const int nr = static_cast<int>(p.n_rows - r0 < group ? p.n_rows - r0 : group);
    if (lrel != cur) {
      if (cur >= 0) publish(cur, cur_rows);
      cur = lrel;
      cur_rows = 0;
    }
    if (lrel > ready) {
      int ok = 1;
      if (lane == 0) {
        if (t0 == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
        for (;;) {
          uint32_t v;
          asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(wait + p.layer0 + lrel)
                       : "memory");
          if (v >= target) break;
          unsigned long long now;
          asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
          if (static_cast<long long>(now - t0) > timeout_ns) {
            atomicOr(p.status, kStatusWaitTimeout);
            ok = 0;
            break;
          }
          __nanosleep(256);
        }
      }
      if (!__shfl_sync(0xffffffffu, ok, 0)) return;
      ready = lrel;
    }
    int32_t my_s = 0, my_d = 0;
    uint8_t my_f = 0;
    uint8_t* fill_l = p.dst_fill + lrel * p.dst_fill_layer;
    if (lane < nr) {
      my_s = __ldg(p.src_idx + r0 + lane);
      my_d = __ldg(p.dst_idx + r0 + lane);
      my_f = ld_cg_u8(fill_l + my_d);
    }
    const unsigned todo = __ballot_sync(0xffffffffu, lane < nr && my_f == 0);
    const uint64_t* src_l = p.src + lrel * p.src_layer_words;
    uint64_t* dst_l = p.dst + lrel * p.dst_layer_words;
#pragma unroll 1
    for (int k = 0; k < nr; ++k) {
      const int64_t si = __shfl_sync(0xffffffffu, my_s, k);
      const int64_t di = __shfl_sync(0xffffffffu, my_d, k);
      if ((todo >> k) & 1u) copy_row<kVec>(src_l + si * p.W, dst_l + di * p.W, p.W, lane);
    }
    __syncwarp();
    if ((todo >> lane) & 1u) fill_l[my_d] = p.fill_value;
    cur_rows += static_cast<uint32_t>(nr);
  }
  if (cur >= 0) publish(cur, cur_rows);
}

// One thread per (range, slot) across as many CTAs as needed: every check
// is an independent (possibly peer) load, so the address validates in about
// one memory latency.  verdict[0] = window of the first page (block 0),
// verdict[1] = any failure (zeroed by the launcher).
// Fan-out DirectSend: like k_copy_rows, but each source row is loaded once
// and stored to every destination whose slot is Empty.
template <int kVec>
#ifndef MKV_FANOUT_MIN_BLOCKS
#define MKV_FANOUT_MIN_BLOCKS 1
#endif
__global__ void __launch_bounds__(kCopyThreads, MKV_FANOUT_MIN_BLOCKS) k_copy_rows_fanout(FanoutParams p) {
  extern __shared__ uint32_t s_rows[];  // [n_dest][n_layers]
  if (p.pdl) asm volatile("griddepcontrol.wait;" ::: "memory");
  int32_t window[kMaxFanout];
  bool live_any = false;
#pragma unroll
  for (int d = 0; d < kMaxFanout; ++d) {
    window[d] = -1;
    if (d < p.n_dest) {
      const volatile int32_t* v = p.verdict[d];
      window[d] = v == nullptr ? 0 : (v[1] == p.gen ? -1 : v[0]);
      live_any |= window[d] >= 0;
    }
  }
  if (!live_any) return;
  for (int i = threadIdx.x; i < p.n_dest * p.n_layers; i += blockDim.x) s_rows[i] = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int64_t warp = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t n_warps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  const int group = p.group > 0 ? p.group : kGroup;
  const int64_t groups = (p.n_rows + group - 1) / group;
  const int64_t items = groups * p.n_layers;
  for (int64_t it = warp; it < items; it += n_warps) {
    const int32_t lrel = static_cast<int32_t>(it / groups);
    const int64_t r0 = (it - static_cast<int64_t>(lrel) * groups) * group;
    const int nr = static_cast<int>(p.n_rows - r0 < group ? p.n_rows - r0 : group);
    const int32_t my_s =
        lane < nr ? (p.src_idx ? __ldg(p.src_idx + r0 + lane) : static_cast<int32_t>(r0 + lane)) : 0;
    int32_t my_d[kMaxFanout];
    unsigned todo[kMaxFanout];  // rows to store (in range, slot Empty)
    unsigned inm[kMaxFanout];   // rows addressed (in range): what the counters count
    unsigned any = 0;
#pragma unroll
    for (int d = 0; d < kMaxFanout; ++d) {
      my_d[d] = 0;
      todo[d] = 0;
      inm[d] = 0;
      if (d < p.n_dest && window[d] >= 0) {
        const int64_t rr = r0 + lane - p.row_off[d];
        const bool in = lane < nr && rr >= 0 && rr < p.row_cnt[d];
        uint8_t f = 1;
        if (in) {
          my_d[d] = __ldg(p.dst_idx[d] + rr);
          f = ld_cg_u8(p.dst_fill[d] + lrel * p.dst_fill_layer[d] + my_d[d]);
        }
        todo[d] = __ballot_sync(0xffffffffu, in && f == 0);
        inm[d] = __ballot_sync(0xffffffffu, in);
        any |= todo[d];
      }
    }
    // Rows the truth destination already holds are sent from its page.
    unsigned from_truth = 0;
    int32_t truth_slot = 0;
    uint64_t* truth_l = nullptr;
#pragma unroll
    for (int d = 0; d < kMaxFanout; ++d) {
      if (d == p.truth) {
        from_truth = inm[d] & ~todo[d];
        truth_slot = my_d[d];
        truth_l = p.dst[d] + lrel * p.dst_layer_words[d];
      }
    }
    const uint64_t* src_l = p.src + lrel * p.src_layer_words;
#pragma unroll 1
    for (int k = 0; k < nr; ++k) {
      const int64_t si = __shfl_sync(0xffffffffu, my_s, k);
      const int64_t ti = __shfl_sync(0xffffffffu, truth_slot, k);
      if (!((any >> k) & 1u)) continue;
      const uint64_t* row = (from_truth >> k) & 1u ? truth_l + ti * p.W : src_l + si * p.W;
      const u256* s4 = reinterpret_cast<const u256*>(row) + lane;
      u256 t[kVec];
#pragma unroll
      for (int u = 0; u < kVec; ++u) t[u] = ld256(s4 + 32 * u);
#pragma unroll
      for (int d = 0; d < kMaxFanout; ++d) {
        const int64_t di = __shfl_sync(0xffffffffu, my_d[d], k);
        if (d < p.n_dest && ((todo[d] >> k) & 1u)) {
          u256* d4 = reinterpret_cast<u256*>(p.dst[d] + lrel * p.dst_layer_words[d] + di * p.W) + lane;
#pragma unroll
          for (int u = 0; u < kVec; ++u) st256(d4 + 32 * u, t[u]);
        }
      }
    }
    __syncwarp();
#pragma unroll
    for (int d = 0; d < kMaxFanout; ++d) {
      if (d < p.n_dest && window[d] >= 0) {
        if ((todo[d] >> lane) & 1u) p.dst_fill[d][lrel * p.dst_fill_layer[d] + my_d[d]] = p.fill_value[d];
        if (lane == 0 && inm[d] != 0 && p.win_received[d] != nullptr) {
          atomicAdd(&s_rows[d * p.n_layers + lrel], static_cast<uint32_t>(__popc(inm[d])));
        }
      }
    }
  }
#ifdef MKV_FENCE_ALL
  fence_publish(p.sys_scope != 0);
#endif
  __syncthreads();  // rows before counters (barrier + release reductions, see k_copy_rows)
  for (int d = 0; d < p.n_dest; ++d) {
    if (window[d] < 0 || p.win_received[d] == nullptr) continue;
    for (int i = threadIdx.x; i < p.n_layers; i += blockDim.x) {
      const uint32_t c = s_rows[d * p.n_layers + i];
      if (c != 0) {
        red_sys_add(p.win_layer_rows[d] + static_cast<int64_t>(window[d]) * p.win_layers[d] +
                        p.layer0 + i,
                    c, p.sys_scope != 0);
      }
    }
    __syncthreads();  // the window total after its layer counters (see k_copy_rows)
    if (threadIdx.x == 0) {
      unsigned long long total = 0;
      for (int i = 0; i < p.n_layers; ++i) total += s_rows[d * p.n_layers + i];
      if (total != 0) red_sys_add(p.win_received[d] + window[d], total, p.sys_scope != 0);
    }
  }
}

__global__ void k_validate_remote(ValidateParams p) {
  // Let the dependent copy grid launch now (it waits for this grid's
  // completion before reading the verdict).
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int64_t work = p.n_ranges * p.P;
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  int32_t w0 = -1;
  bool bad = p.n_ranges <= 0;
  if (p.n_ranges > 0) {
    const int64_t pg0 = p.range_page[0];
    if (pg0 < 0 || pg0 >= p.num_pages) {
      bad = true;
    } else {
      w0 = *reinterpret_cast<const volatile int32_t*>(p.page_window + pg0);
      if (w0 < 0) bad = true;
    }
  }
  if (i == 0) {
    p.verdict[0] = w0;
    if (w0 >= 0 && p.win_gen != nullptr)
      p.verdict[2] = static_cast<int32_t>(*reinterpret_cast<const volatile unsigned long long*>(p.win_gen + w0));
  }
  if (!bad && i < work) {
    const int64_t r = i / p.P;
    const int32_t k = static_cast<int32_t>(i % p.P);
    const int64_t pg = p.range_page[r];
    const int32_t b = p.range_begin[r], c = p.range_count[r];
    if (pg < 0 || pg >= p.num_pages || b < 0 || c < 0 || b + c > p.P) {
      bad = true;
    } else if (k < c) {
      if (k == 0 && *reinterpret_cast<const volatile int32_t*>(p.page_window + pg) != w0) bad = true;
      if (reinterpret_cast<const volatile uint8_t*>(p.expecting)[pg * p.P + b + k] == 0) bad = true;
    }
  }
  if (bad && (i < work || i == 0)) {
    *reinterpret_cast<volatile int32_t*>(p.verdict + 1) = p.gen;
    if (p.status != nullptr) atomicOr(p.status, kStatusUnknownAddress);
  }
}

__global__ void __launch_bounds__(256) k_attn_write_hash(uint64_t* __restrict__ pool_l,
                                                         uint8_t* __restrict__ fill_l,
                                                         const int32_t* __restrict__ slots,
                                                         const uint64_t* __restrict__ digests,
                                                         int64_t n, int32_t layer, int32_t W) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t n_warps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  for (int64_t r = warp; r < n; r += n_warps) {
    const int64_t slot = __ldg(slots + r);
    uint8_t* f = fill_l + slot;
    if (*reinterpret_cast<volatile uint8_t*>(f) != 0) continue;  // re-prefill is skipped
    const uint64_t base = kv_base(__ldg(digests + r), layer);
    uint64_t* row = pool_l + slot * W;
    if ((W & 1) == 0) {
      ulonglong2* row2 = reinterpret_cast<ulonglong2*>(row);
      for (int v = lane; v < (W >> 1); v += 32) {
        ulonglong2 w;
        w.x = kv_word(base, 2u * v);
        w.y = kv_word(base, 2u * v + 1u);
        st_vec(row2 + v, w);
      }
    } else {
      for (int j = lane; j < W; j += 32) row[j] = kv_word(base, static_cast<uint32_t>(j));
    }
    __syncwarp();
    if (lane == 0) *f = 1;  // FillState::kComputedLocal
  }
}

// One thread folds one row serially (FNV-1a is a byte-serial chain); 8
// words are prefetched ahead of the chain.
__global__ void __launch_bounds__(128) k_entry_digest(const uint64_t* __restrict__ pool_l,
                                                      const int32_t* __restrict__ slots, int64_t n,
                                                      int32_t W, uint64_t* __restrict__ F) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t r = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; r < n;
       r += stride) {
    const uint64_t* row = pool_l + static_cast<int64_t>(__ldg(slots + r)) * W;
    uint64_t h = entry_digest_init();
    if ((W & 7) == 0) {
      const ulonglong2* r2 = reinterpret_cast<const ulonglong2*>(row);
      ulonglong2 cur[4], nxt[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) cur[u] = __ldg(r2 + u);
      const int nb = W >> 3;  // blocks of 8 words
      for (int b = 0; b < nb; ++b) {
        if (b + 1 < nb) {
#pragma unroll
          for (int u = 0; u < 4; ++u) nxt[u] = __ldg(r2 + 4 * (b + 1) + u);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          h = fnv_u64(h, cur[u].x);
          h = fnv_u64(h, cur[u].y);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) cur[u] = nxt[u];
      }
    } else {
      for (int j = 0; j < W; ++j) h = fnv_u64(h, __ldg(row + j));
    }
    F[r] = mix64(h);
  }
}

constexpr int kScanThreads = 1024;

__global__ void __launch_bounds__(kScanThreads) k_fold_scan(const FoldEntry* __restrict__ entries,
                                                            const uint64_t* __restrict__ F,
                                                            const uint64_t* __restrict__ hidden_in,
                                                            uint64_t* __restrict__ hidden_out,
                                                            int32_t layer) {
  __shared__ uint64_t s_warp[kScanThreads / 32];
  const FoldEntry e = entries[blockIdx.x];
  const uint64_t base = e.fold_sums[layer];
  const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
  const int64_t chunk = (e.n_fold + kScanThreads - 1) / kScanThreads;
  const int64_t lo = e.n_fold < t * chunk ? e.n_fold : t * chunk;
  const int64_t hi = e.n_fold < lo + chunk ? e.n_fold : lo + chunk;
  const uint64_t* f = F + e.fold_off;
  uint64_t local = 0;
  for (int64_t i = lo; i < hi; ++i) local += f[i];
  // Exclusive scan of the per-thread sums (wrapping u64 adds).
  uint64_t incl = local;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    uint64_t v = __shfl_up_sync(0xffffffffu, incl, d);
    if (lane >= d) incl += v;
  }
  if (lane == 31) s_warp[wid] = incl;
  __syncthreads();
  if (wid == 0) {
    uint64_t w = s_warp[lane];
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      uint64_t v = __shfl_up_sync(0xffffffffu, w, d);
      if (lane >= d) w += v;
    }
    s_warp[lane] = w;  // inclusive over warps
  }
  __syncthreads();
  uint64_t sum = base + (wid > 0 ? s_warp[wid - 1] : 0) + (incl - local);
  for (int64_t i = lo; i < hi; ++i) {
    sum += f[i];
    if (i >= e.first_out) {
      const int64_t o = e.out_off + (i - e.first_out);
      const uint64_t x = hidden_in[o];
      hidden_out[o] = next_hidden(x, attention_out(x, e.pos0 + i + 1, sum));
    }
  }
  __syncthreads();
  if (t == 0) e.fold_sums[layer] = base + s_warp[31];
}

__global__ void k_reset_pages(uint8_t* fill, uint8_t* expecting, int32_t* page_window,
                              const int64_t* __restrict__ pages, int64_t n_pages, int32_t L,
                              int64_t num_pages, int32_t P) {
  const int64_t total = n_pages * P;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
       i += stride) {
    const int64_t pg = pages[i / P];
    const int64_t slot = pg * P + (i % P);
    for (int32_t l = 0; l < L; ++l) fill[static_cast<int64_t>(l) * num_pages * P + slot] = 0;
    expecting[slot] = 0;
    if (i % P == 0) page_window[pg] = -1;
  }
}

__global__ void k_open_window(uint8_t* expecting, const int32_t* __restrict__ slots,
                              int64_t n_slots, int32_t* page_window,
                              const int64_t* __restrict__ pages, int64_t n_pages, int32_t window,
                              unsigned long long* win_received, uint32_t* win_layer_rows,
                              unsigned long long* win_gen, int32_t L) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  const int64_t t0 = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  for (int64_t i = t0; i < n_slots; i += stride) expecting[slots[i]] = 1;
  for (int64_t i = t0; i < n_pages; i += stride) page_window[pages[i]] = window;
  if (window >= 0) {
    for (int64_t i = t0; i < L; i += stride) win_layer_rows[static_cast<int64_t>(window) * L + i] = 0;
    if (t0 == 0) {
      win_received[window] = 0;
      win_gen[window] += 1;  // senders validated against an earlier opening re-validate
    }
  }
}

__global__ void k_close_window(int32_t* page_window, const int64_t* __restrict__ pages,
                               int64_t n_pages, int32_t window) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n_pages;
       i += stride) {
    const int64_t pg = pages[i];
    if (page_window[pg] == window) page_window[pg] = -1;
  }
}

// One thread per (layer, position), positions fastest: a warp reads 32
// adjacent fill bytes of one layer (a page's slots are consecutive), so the
// scan is one coalesced pass over n * L bytes instead of L dependent byte
// loads per position.
__global__ void k_first_nonfull(const uint8_t* __restrict__ fill, int64_t fill_layer_bytes,
                                int32_t L, const int32_t* __restrict__ slots, int64_t n,
                                unsigned long long* out) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  const int64_t total = n * L;
  for (int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; k < total;
       k += stride) {
    const int64_t l = k / n, i = k - l * n;
    if (fill[l * fill_layer_bytes + __ldg(slots + i)] == 0)
      atomicMin(out, static_cast<unsigned long long>(i));
  }
}

__global__ void k_gather_tables(const int32_t* const* __restrict__ tables,
                                const int64_t* __restrict__ off, const int32_t* __restrict__ len,
                                int64_t batch, int32_t* __restrict__ out) {
  for (int64_t b = blockIdx.y; b < batch; b += gridDim.y) {
    const int32_t* t = tables[b];
    const int64_t o = off[b];
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < len[b];
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
      out[o + i] = t[i];
    }
  }
}

__global__ void k_check_filled(const uint8_t* __restrict__ fill_l, const int32_t* __restrict__ slots,
                               int64_t n, uint32_t* status) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += stride) {
    if (fill_l[slots[i]] == 0) atomicOr(status, kStatusMissingKV);
  }
}

__global__ void k_wait_counter(const unsigned long long* counter, unsigned long long target,
                               long long timeout_ns, uint32_t* status) {
  unsigned long long t0, now;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (;;) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(counter) : "memory");
    if (v >= target) return;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
    if (static_cast<long long>(now - t0) > timeout_ns) {
      atomicOr(status, kStatusWaitTimeout);
      return;
    }
    __nanosleep(200);
  }
}

__global__ void k_wait_counter32(const uint32_t* counter, uint32_t target, long long timeout_ns,
                                 uint32_t* status) {
  unsigned long long t0, now;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (;;) {
    uint32_t v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(counter) : "memory");
    if (v >= target) return;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
    if (static_cast<long long>(now - t0) > timeout_ns) {
      atomicOr(status, kStatusWaitTimeout);
      return;
    }
    __nanosleep(200);
  }
}

inline int grid_for(int64_t work, int per_block, int num_sms, int max_per_sm) {
  int64_t blocks = (work + per_block - 1) / per_block;
  int64_t cap = static_cast<int64_t>(num_sms) * max_per_sm;
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  return static_cast<int>(blocks);
}

// Resident CTAs per SM of a k_copy_rows instantiation (its occupancy at the
// largest per-layer accounting array), queried once per process.
// Launches of at least this many items (4-row groups x layers) use 11 CTAs
// per SM instead of 7 (profiles/r02/copy_grid_ab.txt: 6144 tokens x 80
// layers 0.982 -> 0.989, 8192: 0.982 -> 0.993; 4096 and below equal or worse).
constexpr int64_t kHugeItems = 96 * 1024;

int copy_rows_ctas_per_sm(int32_t W, bool prefetch) {
  static int cache[3][2] = {{0, 0}, {0, 0}, {0, 0}};
  const int wi = W == 512 ? 0 : W == 128 ? 1 : 2;
  int& c = cache[wi][prefetch ? 1 : 0];
  if (c == 0) {
    void (*k)(CopyParams) = W == 512 ? (prefetch ? k_copy_rows<4, true> : k_copy_rows<4>)
                            : W == 128 ? (prefetch ? k_copy_rows<1, true> : k_copy_rows<1>)
                                       : k_copy_rows<0>;
    int n = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k, kCopyThreads, 1024) != cudaSuccess ||
        n < 1)
      n = 1;
    c = n;
  }
  return c;
}

}  // namespace

void launch_copy_rows(const CopyParams& p, cudaStream_t s, int num_sms) {
  const int64_t items = p.n_rows * p.n_layers;
  if (items <= 0) return;
  const int warps_per_block = kCopyThreads / 32;
  // Long launches: 4-row groups on a grid of 7 CTAs per SM -- more CTAs than
  // are resident (2 for the prefetching send kernel at 95 registers, 4 for
  // the plain copy at 64), so CTAs retire and are replaced through the
  // launch instead of one resident wave striding over all items.  Measured
  // (profiles/r02/copy_grid_ab.txt, behind a sleep gate): the 80-layer
  // DirectSend 0.94 -> 0.98 of the HBM copy peak, all-layer append / gather
  // in one launch 0.93 -> 0.99; 2, 4, 6 and 8 per SM all slower than 7.
  // The largest launches (>= kHugeItems) on 11 per SM: another ~1% at 6K-32K
  // tokens x 80 layers, but 2-6% slower at 512-4K tokens, so only there.
  // Launches that fit one wave of resident warps (per-layer append /
  // gather): one row per warp, 8 CTAs per SM, so no warp chains several
  // rows' load latencies.
  CopyParams q = p;
#ifndef MKV_SHORT_GROUP
#define MKV_SHORT_GROUP 1
#endif
#ifndef MKV_SHORT_PER_SM
#define MKV_SHORT_PER_SM 8
#endif
  const int64_t one_wave = static_cast<int64_t>(num_sms) * 8 * warps_per_block;
  // Short launches (a wave or less of resident warps): one row per warp for
  // plain copies (append / gather: +10%), 4-row items for sends that publish
  // window counters (a quarter of the CTAs pay the publication: one 70B
  // layer 25.6 -> 19.5 us).
  int short_group = p.win_received != nullptr ? 4 : MKV_SHORT_GROUP;
  // A small send (a few pages x layers): one row per warp, every row's loads
  // in flight at once; its few CTAs' publication is cheap.
  if (p.win_received != nullptr && p.n_rows * p.n_layers <= kSmallSendRows) short_group = 1;
  const bool short_launch = items <= one_wave * short_group;
  q.group = short_launch ? short_group : kGroup;
  // Publishing sends that fit one wave: rows per item chosen so the items
  // fill the warps actually resident (the kernel's occupancy) exactly once,
  // instead of a wave plus a small tail (256 tokens x 80 layers: 43 -> 35 us).
  if (short_launch && p.win_received != nullptr && short_group > 1) {
    const int64_t resident = static_cast<int64_t>(num_sms) *
                             copy_rows_ctas_per_sm(q.W, q.prefetch_src != 0) * warps_per_block;
    const int64_t per_layer = resident / q.n_layers > 0 ? resident / q.n_layers : 1;
    const int64_t g = (q.n_rows + per_layer - 1) / per_layer;
    q.group = static_cast<int32_t>(g < 2 ? 2 : (g > 32 ? 32 : g));  // (1-row items: publication per CTA)
  }
  const int64_t groups = (q.n_rows + q.group - 1) / q.group * q.n_layers;
#ifndef MKV_LONG_PER_SM
#define MKV_LONG_PER_SM 7
#endif
#ifndef MKV_MID_PER_SM
#define MKV_MID_PER_SM 7  // 512-768 tokens x 80 layers: 2-3% over 8 (copy_grid_ab.txt)
#endif
#ifndef MKV_HUGE_PER_SM
#define MKV_HUGE_PER_SM 11  // >= 96K items (e.g. 6K-32K tokens x 80 layers): +1% over 7
#endif
  const int per_sm = short_launch ? MKV_SHORT_PER_SM
                     : groups >= kHugeItems ? MKV_HUGE_PER_SM
                     : (groups >= static_cast<int64_t>(num_sms) * 2 * warps_per_block * 8 ? MKV_LONG_PER_SM : MKV_MID_PER_SM);
  int grid = grid_for(groups, warps_per_block, num_sms, per_sm);
  if (q.max_ctas > 0 && grid > q.max_ctas) grid = q.max_ctas;
  const size_t smem = q.win_received ? sizeof(uint32_t) * q.n_layers : 0;
  // (The prefetching instantiation, for sends right behind their validation
  // grid, holds a row in registers across the wait: its own kernel, so the
  // plain copies keep their register count and occupancy.)
  void (*kern)(CopyParams) =
      q.W == 512 ? (q.prefetch_src ? k_copy_rows<4, true> : k_copy_rows<4>)  // 8B/70B rows: 4 KiB
      : q.W == 128 ? (q.prefetch_src ? k_copy_rows<1, true> : k_copy_rows<1>)  // tiny: 1 KiB
                   : k_copy_rows<0>;
  if (q.pdl) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(static_cast<unsigned>(grid));
    cfg.blockDim = dim3(kCopyThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, kern, q);
  } else {
    kern<<<grid, kCopyThreads, smem, s>>>(q);
  }
}

void launch_relay_rows(const CopyParams& p, const uint32_t* wait, uint32_t target,
                       long long timeout_ns, cudaStream_t s, int num_sms) {
  const int64_t groups = (p.n_rows + kGroup - 1) / kGroup * p.n_layers;
  if (groups <= 0) return;
  const int warps_per_block = kCopyThreads / 32;
  // One CTA per SM at most (its warps spin while upstream layers are in
  // flight; the upstream copy must keep the rest of the machine).
  int grid = grid_for(groups, warps_per_block, num_sms, 1);
  if (p.max_ctas > 0 && grid > p.max_ctas) grid = p.max_ctas;
  void (*kern)(CopyParams, const uint32_t*, uint32_t, long long) =
      p.W == 512 ? k_relay_rows<4> : p.W == 128 ? k_relay_rows<1> : k_relay_rows<0>;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(static_cast<unsigned>(grid));
  cfg.blockDim = dim3(kCopyThreads);
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = p.pdl ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kern, p, wait, target, timeout_ns);
}

#ifndef MKV_FANOUT_SHORT_GROUP_MAX
#define MKV_FANOUT_SHORT_GROUP_MAX 32
#endif
void launch_copy_rows_fanout(const FanoutParams& p, cudaStream_t s, int num_sms) {
  const int64_t groups = (p.n_rows + kGroup - 1) / kGroup * p.n_layers;
  if (groups <= 0) return;
  const int warps_per_block = kCopyThreads / 32;
  // As k_copy_rows: launches that fit one wave at 8 CTAs per SM (a layer of
  // a fused append + send) spread over 8 CTAs per SM, long ones over a grid
  // of 7 per SM (3-target prefix fan-out: 0.78 of HBM at 2, 4, 6 or 8 per
  // SM, 0.85 at 7; profiles/r02/copy_grid_ab.txt).
  FanoutParams q = p;
  const int64_t rows = p.n_rows * p.n_layers;
  const bool short_launch = rows <= static_cast<int64_t>(num_sms) * 8 * warps_per_block * kGroup;
  q.group = kGroup;
  if (short_launch) {
    // Rows per item fitted to the warps actually resident (the kernel's
    // occupancy), as for publishing copies: one wave of items, no tail.
    // A fused 8B layer (4095 rows) gets 2-row items, a 70B one (8191) 4:
    // 8B 20.5 -> 19.4 us per layer, 70B unchanged (profiles/r02/copy_grid_ab.txt).
    static int occ[2] = {0, 0};
    int& o = occ[p.W == 512 ? 0 : 1];
    if (o == 0) {
      int n = 0;
      void (*k)(FanoutParams) = p.W == 512 ? k_copy_rows_fanout<4> : k_copy_rows_fanout<1>;
      if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k, kCopyThreads, 1024) != cudaSuccess ||
          n < 1)
        n = 1;
      o = n;
    }
    const int64_t resident = static_cast<int64_t>(num_sms) * o * warps_per_block;
    const int64_t per_layer = resident / p.n_layers > 0 ? resident / p.n_layers : 1;
    const int64_t g = (p.n_rows + per_layer - 1) / per_layer;
    q.group = static_cast<int32_t>(g < 2 ? 2 : (g > MKV_FANOUT_SHORT_GROUP_MAX ? MKV_FANOUT_SHORT_GROUP_MAX : g));
  }
  if (const char* e = std::getenv("MICROKV_FANOUT_GROUP")) q.group = std::atoi(e) > 0 ? std::atoi(e) : q.group;
  const int64_t items = (q.n_rows + q.group - 1) / q.group * q.n_layers;
  int per_sm = short_launch ? 8 : (items >= kHugeItems ? 11 : 7);
  if (const char* e = std::getenv("MICROKV_FANOUT_PER_SM")) per_sm = std::atoi(e) > 0 ? std::atoi(e) : per_sm;
  const int grid = grid_for(items, warps_per_block, num_sms, per_sm);
  const size_t smem = sizeof(uint32_t) * p.n_dest * p.n_layers;
  // Rows that are not 128 or 512 words use the single-destination kernel
  // once per destination (the callers split); not reached here.
  void (*kern)(FanoutParams) = p.W == 512 ? k_copy_rows_fanout<4> : k_copy_rows_fanout<1>;
  if (p.W != 512 && p.W != 128) return;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(static_cast<unsigned>(grid));
  cfg.blockDim = dim3(kCopyThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = p.pdl ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kern, q);
}

void launch_validate_remote(const ValidateParams& p, cudaStream_t s) {
  int64_t work = p.n_ranges * p.P;
  int64_t grid = (work + 255) / 256;
  if (grid < 1) grid = 1;
  if (grid > 0x7fffffff) grid = 0x7fffffff;
  k_validate_remote<<<static_cast<unsigned>(grid), 256, 0, s>>>(p);
}

void launch_attn_write_hash(uint64_t* pool_l, uint8_t* fill_l, const int32_t* slots,
                            const uint64_t* digests, int64_t n, int32_t layer, int32_t W,
                            cudaStream_t s, int num_sms) {
  if (n <= 0) return;
  k_attn_write_hash<<<grid_for(n, 8, num_sms, 8), 256, 0, s>>>(pool_l, fill_l, slots, digests, n,
                                                                layer, W);
}

void launch_entry_digest(const uint64_t* pool_l, const int32_t* slots, int64_t n, int32_t W,
                         uint64_t* F, cudaStream_t s, int num_sms) {
  if (n <= 0) return;
  k_entry_digest<<<grid_for(n, 128, num_sms, 16), 128, 0, s>>>(pool_l, slots, n, W, F);
}

void launch_fold_scan(const FoldEntry* entries, int64_t n_entries, const uint64_t* F,
                      const uint64_t* hidden_in, uint64_t* hidden_out, int32_t layer,
                      cudaStream_t s) {
  if (n_entries <= 0) return;
  k_fold_scan<<<static_cast<unsigned>(n_entries), kScanThreads, 0, s>>>(entries, F, hidden_in,
                                                                         hidden_out, layer);
}

void launch_reset_pages(uint8_t* fill, uint8_t* expecting, int32_t* page_window,
                        const int64_t* pages, int64_t n_pages, int32_t L, int64_t num_pages,
                        int32_t P, cudaStream_t s) {
  if (n_pages <= 0) return;
  int64_t total = n_pages * P;
  int grid = static_cast<int>((total + 255) / 256);
  if (grid > 4096) grid = 4096;
  k_reset_pages<<<grid, 256, 0, s>>>(fill, expecting, page_window, pages, n_pages, L, num_pages, P);
}

void launch_open_window(uint8_t* expecting, const int32_t* slots, int64_t n_slots,
                        int32_t* page_window, const int64_t* pages, int64_t n_pages,
                        int32_t window, unsigned long long* win_received,
                        uint32_t* win_layer_rows, unsigned long long* win_gen, int32_t L,
                        cudaStream_t s) {
  int64_t work = n_slots > n_pages ? n_slots : n_pages;
  if (work < L) work = L;
  int grid = static_cast<int>((work + 255) / 256);
  if (grid > 1024) grid = 1024;
  if (grid < 1) grid = 1;
  k_open_window<<<grid, 256, 0, s>>>(expecting, slots, n_slots, page_window, pages, n_pages, window,
                                     win_received, win_layer_rows, win_gen, L);
}

void launch_close_window(int32_t* page_window, const int64_t* pages, int64_t n_pages,
                         int32_t window, cudaStream_t s) {
  if (n_pages <= 0) return;
  int grid = static_cast<int>((n_pages + 255) / 256);
  if (grid > 1024) grid = 1024;
  k_close_window<<<grid, 256, 0, s>>>(page_window, pages, n_pages, window);
}

void launch_first_nonfull(const uint8_t* fill, int64_t fill_layer_bytes, int32_t L,
                          const int32_t* slots, int64_t n, unsigned long long* out,
                          cudaStream_t s, int num_sms) {
  cudaMemsetAsync(out, 0xff, sizeof(unsigned long long), s);
  if (n <= 0) return;
  k_first_nonfull<<<grid_for(n * L, 256, num_sms, 8), 256, 0, s>>>(fill, fill_layer_bytes, L,
                                                                    slots, n, out);
}

void launch_wait_counter(const unsigned long long* counter, unsigned long long target,
                         long long timeout_ns, uint32_t* status, cudaStream_t s) {
  k_wait_counter<<<1, 1, 0, s>>>(counter, target, timeout_ns, status);
}

void launch_wait_counter32(const uint32_t* counter, uint32_t target, long long timeout_ns,
                           uint32_t* status, cudaStream_t s) {
  k_wait_counter32<<<1, 1, 0, s>>>(counter, target, timeout_ns, status);
}

void launch_gather_tables(const int32_t* const* tables, const int64_t* off, const int32_t* len,
                          int64_t batch, int64_t total, int32_t* out, cudaStream_t s, int num_sms) {
  if (batch <= 0 || total <= 0) return;
  const int64_t per = (total / batch + 255) / 256;
  dim3 grid(static_cast<unsigned>(per < 64 ? (per < 1 ? 1 : per) : 64),
            static_cast<unsigned>(batch < 1024 ? batch : 1024));
  (void)num_sms;
  k_gather_tables<<<grid, 256, 0, s>>>(tables, off, len, batch, out);
}

void launch_check_filled(const uint8_t* fill_l, const int32_t* slots, int64_t n, uint32_t* status,
                         cudaStream_t s, int num_sms) {
  if (n <= 0) return;
  k_check_filled<<<grid_for(n, 256, num_sms, 4), 256, 0, s>>>(fill_l, slots, n, status);
}


// Lazy module loading (the CUDA 12 default) loads a kernel at its first
// launch, and a load can wait for the device to go idle.  A receiver that
// spins in k_wait_counter32 until a sender's first-ever k_copy_rows lands
// would then hang until its timeout, so every kernel of the library is
// loaded up front when a device cache is created.
void preload_kernels() {
  cudaFuncAttributes a;
  cudaFuncGetAttributes(&a, k_copy_rows<4>);
  cudaFuncGetAttributes(&a, k_copy_rows<4, true>);
  cudaFuncGetAttributes(&a, k_copy_rows<1>);
  cudaFuncGetAttributes(&a, k_copy_rows<1, true>);
  cudaFuncGetAttributes(&a, k_copy_rows<0>);
  cudaFuncGetAttributes(&a, k_copy_rows_fanout<4>);
  cudaFuncGetAttributes(&a, k_relay_rows<4>);
  cudaFuncGetAttributes(&a, k_relay_rows<1>);
  cudaFuncGetAttributes(&a, k_relay_rows<0>);
  cudaFuncGetAttributes(&a, k_copy_rows_fanout<1>);
  cudaFuncGetAttributes(&a, k_validate_remote);
  cudaFuncGetAttributes(&a, k_attn_write_hash);
  cudaFuncGetAttributes(&a, k_entry_digest);
  cudaFuncGetAttributes(&a, k_fold_scan);
  cudaFuncGetAttributes(&a, k_reset_pages);
  cudaFuncGetAttributes(&a, k_open_window);
  cudaFuncGetAttributes(&a, k_close_window);
  cudaFuncGetAttributes(&a, k_first_nonfull);
  cudaFuncGetAttributes(&a, k_gather_tables);
  cudaFuncGetAttributes(&a, k_check_filled);
  cudaFuncGetAttributes(&a, k_wait_counter);
  cudaFuncGetAttributes(&a, k_wait_counter32);
  preload_decode_attn_kernels();
  preload_decode_pages_kernels();
  preload_prefill_attn_kernels();
  preload_crc32_kernels();
  cudaGetLastError();
}

}  // namespace mkv
