// decode_pages.cu — paged GQA decode attention with TMA page-chunk loads
// (sm_100a), for K||V rows of 8 KV heads x head_dim 128 (4 KiB per token
// and layer: the Llama-3.1-8B / 70B KV shape) and up to 8 query heads per
// KV head.  Other shapes use k_decode_attn (decode_attn.cu).
//
// No reference analogue (the reference's "attention" is the integer fold,
// kv_cache.cc:319-351); numerics are checked against fp32 PyTorch
// (tests/test_decode_attention_gpu.py, test_attention_bench_shapes_gpu.py).
//
// Work unit = a chunk: a run of at most 16 positions of one context whose
// slots are consecutive (normally one 16-token page).  Its rows are one
// contiguous 16 x 4 KiB block of the layer's pool, loaded by 32 TMA boxes
// of {64 bf16, 16 rows} (one per 128-byte column block of the row: K of
// head h = blocks 2h, 2h+1; V = blocks 16+2h, 17+2h) into a SWIZZLE_128B
// stage — 64 KiB per TMA stage, no per-thread load instructions, the DRAM
// stream sequential per page.  Chunks are flattened over the batch and the
// grid (one CTA per SM) splits them into equal ranges (stream-K); a CTA's
// range cut by a context boundary gives one piece per context.
//
// CTA: warp 8 produces (its lanes issue the 32 boxes of a chunk: lanes 0-15
// the K column blocks into one 32 KiB stage, lanes 16-31 the V blocks into
// the next, each onto its own full barrier), warps 0..7 consume, warp h = KV
// head h; a chunk's K stage is released as soon as S^T is computed, its V
// stage after PV (3 chunks = 6 half-stages in flight).  Per chunk
// the warp computes S^T = K Q^T (M = 16 tokens, N = 8 query heads, K = 128)
// and O^T += V^T P^T (M = 128 dims in 8 tiles, N = 8 query heads, K = 16
// tokens) with bf16 mma.sync m16n8k16 — the query heads of the GQA group
// are the N side, so no MMA row is padding (the M = 16 query-head layout
// of k_decode_attn wastes half of every MMA and every O register at G = 8).
// P^T goes from the S^T accumulators to the PV B operand by movmatrix.trans.
// Online softmax per query head over the token axis; O^T lives in 32 fp32
// registers per lane.  A piece that is a whole context writes bf16 output;
// the others write (O, m, l) partials merged by k_decode_pages_combine.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <cstring>

#include "kernels.cuh"

namespace mkv {

namespace {

constexpr int kHkv = 8;                  // KV heads (consumer warps)
constexpr int kD = 128;                  // head dim
constexpr int kChunk = 16;               // rows per chunk / TMA box
constexpr int kBlocks = 4 * kHkv * kD * 2 / 128 / 2;  // 128-byte column blocks per row: 32
constexpr int kBlockBytes = kChunk * 128;             // 2 KiB
constexpr int kStageBytes = kBlocks * kBlockBytes;    // 64 KiB
constexpr int kStages = 3;                       // chunks in flight
constexpr int kHalfBytes = kStageBytes / 2;      // the K (or V) column blocks of a chunk: 32 KiB
constexpr int kRing = 2 * kStages;               // K and V half-stages (one barrier pair each)
constexpr int kConsumers = kHkv;  // one consumer warp per KV head
constexpr int kThreads = (kConsumers + 1) * 32;
constexpr size_t kSmem = static_cast<size_t>(kStages) * kStageBytes + 1024 + 256;
static_assert(2 * 8 * 2 * kStages <= 256, "barrier area");
static_assert(kBlocks == 32, "4 KiB rows");

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(bar),
               "r"(bytes)
               : "memory");
}
// Bounded wait: a completion that never arrives traps instead of hanging.
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t phase) {
  uint32_t done = 0;
  const long long t0 = clock64();
  for (;;) {
    asm volatile(
        "{\n\t.reg .pred P;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, P;\n\t}\n"
        : "=r"(done)
        : "r"(bar), "r"(phase)
        : "memory");
    if (done) return;
    if (clock64() - t0 > (4ll << 30)) __trap();
  }
}
__device__ __forceinline__ void tma_load_3d(uint32_t dst, const CUtensorMap* map, int c0, int c1,
                                            int c2, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
      "%3, %4}], [%5];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t (&r)[4]) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0, %1, %2, %3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t (&r)[4]) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0, %1, %2, %3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(addr));
}
__device__ __forceinline__ uint32_t movm_t(uint32_t x) {
  uint32_t y;
  asm volatile("movmatrix.sync.aligned.m8n8.trans.b16 %0, %1;" : "=r"(y) : "r"(x));
  return y;
}
__device__ __forceinline__ void mma(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, "
      "{%8, %9}, {%0, %1, %2, %3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}
__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// Byte offset of 16-byte chunk c (0..7) of row r in a SWIZZLE_128B column
// block of 16 rows x 128 bytes (1024-byte aligned).
__device__ __forceinline__ uint32_t sw(int r, int c) {
  return static_cast<uint32_t>(r * 128 + ((c ^ (r & 7)) << 4));
}

struct PagesArgs {
  const int4* chunks;          // {slot0, tok0, n, b} per chunk, batch order
  int64_t n_chunks;
  const int32_t* piece_first;  // [batch]: CTA holding the context's first chunk
  const int32_t* piece_count;  // [batch]: CTAs (pieces) the context spans
  const __nv_bfloat16* q;      // [batch][Hq][128]
  __nv_bfloat16* out;          // [batch][Hq][128]
  float* part_o;               // [(piece * Hkv + h) * G + g][128], piece = cta + b
  float* part_ml;              // [(piece * Hkv + h) * G + g][2]
  int layer, Hq, G;
  float scale_log2;
};

// 112 registers (no spills): with the combine kernel's 121 x 256 a combine
// CTA fits beside a main CTA, so the programmatic-dependent combine is
// resident and waiting when the main grid drains (118 registers left no room).
__global__ void __maxnreg__(112)
    k_decode_pages(const __grid_constant__ CUtensorMap map, const PagesArgs a) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kStages * kStageBytes);  // full, empty
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t T = a.n_chunks;
  const int64_t c0 = static_cast<int64_t>(blockIdx.x) * T / gridDim.x;
  const int64_t c1 = static_cast<int64_t>(blockIdx.x + 1) * T / gridDim.x;
  const uint32_t full0 = smem_u32(bars), empty0 = smem_u32(bars + kRing);
  if (threadIdx.x == 0) {
    for (int s = 0; s < kRing; ++s) {
      mbar_init(full0 + 8 * s, 1);
      mbar_init(empty0 + 8 * s, kHkv);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  // The first chunk descriptors (plan data, uploaded before any predecessor
  // ran) are requested before the grid dependency wait.
  int4 first = make_int4(0, 0, 0, 0);
  if (warp == kConsumers && c0 + lane < c1) first = __ldg(a.chunks + c0 + lane);
  __syncthreads();
  // Programmatic dependent of the previous kernel: everything above (plan
  // reads, barrier setup) overlapped its tail; the pool (the new token's
  // K||V row) and the queries are read only after it completed.
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (c0 >= c1) return;

  if (warp == kConsumers) {
    // Producer: chunk descriptors 32 at a time (one coalesced load), then
    // per chunk lane 0 arms the stage and each lane issues one column block.
    const uint32_t base = smem_u32(smem);
    for (int64_t j0 = c0; j0 < c1; j0 += 32) {
      const int4 mine = j0 == c0 ? first
                        : (j0 + lane < c1 ? __ldg(a.chunks + j0 + lane) : make_int4(0, 0, 0, 0));
      const int cnt = static_cast<int>(c1 - j0 < 32 ? c1 - j0 : 32);
      for (int k = 0; k < cnt; ++k) {
        const int64_t i = j0 + k - c0;
        const int slot0 = __shfl_sync(0xffffffffu, mine.x, k);
        // K half (blocks 0-15) into slot (2 i) % 6, V half into (2 i + 1) % 6.
        const int64_t qk = 2 * i, qv = 2 * i + 1;
        const int sk = static_cast<int>(qk % kRing), sv = static_cast<int>(qv % kRing);
        if (qk >= kRing) mbar_wait(empty0 + 8 * sk, (static_cast<uint32_t>(qk / kRing) & 1u) ^ 1u);
        if (qv >= kRing) mbar_wait(empty0 + 8 * sv, (static_cast<uint32_t>(qv / kRing) & 1u) ^ 1u);
        if (lane == 0) {
          mbar_expect_tx(full0 + 8 * sk, kHalfBytes);
          mbar_expect_tx(full0 + 8 * sv, kHalfBytes);
        }
        __syncwarp();
        const int hs = lane < 16 ? sk : sv;
        tma_load_3d(base + hs * kHalfBytes + (lane & 15) * kBlockBytes, &map, lane * 64, slot0,
                    a.layer, full0 + 8 * hs);
      }
    }
    return;
  }

  // Consumer warp h = KV head h.
  const int h = warp, G = a.G, Hq = a.Hq;
  const int r4 = lane >> 2, c4 = lane & 3;  // fragment row / column-pair of the lane
  float o[8][4];                            // O^T: dims mt*16 + r4 (+8) x heads 2*c4 (+1)
  float m[2], l[2];                         // per query head 2*c4, 2*c4+1 (l: this lane's share)
  uint32_t qb[8][2];                        // Q^T B fragments, K = 128 dims in 8 steps
  int cur_b = -1;
  bool whole = false;
  auto flush = [&]() {
    // l: sum the lanes' shares (same query head = same c4).
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      l[e] += __shfl_xor_sync(0xffffffffu, l[e], 4);
      l[e] += __shfl_xor_sync(0xffffffffu, l[e], 8);
      l[e] += __shfl_xor_sync(0xffffffffu, l[e], 16);
    }
    const int64_t piece = static_cast<int64_t>(blockIdx.x) + cur_b;
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int g = 2 * c4 + e;
      if (g >= G) continue;
      const float inv = l[e] > 0.f ? 1.f / l[e] : 0.f;
      if (whole) {
        __nv_bfloat16* ob = a.out + (static_cast<int64_t>(cur_b) * Hq + h * G + g) * kD;
#pragma unroll
        for (int mt = 0; mt < 8; ++mt) {
          ob[mt * 16 + r4] = __float2bfloat16_rn(o[mt][e] * inv);
          ob[mt * 16 + r4 + 8] = __float2bfloat16_rn(o[mt][2 + e] * inv);
        }
      } else {
        const int64_t row = (piece * kHkv + h) * G + g;
        float* po = a.part_o + row * kD;
#pragma unroll
        for (int mt = 0; mt < 8; ++mt) {
          po[mt * 16 + r4] = o[mt][e] * inv;
          po[mt * 16 + r4 + 8] = o[mt][2 + e] * inv;
        }
        if (r4 == 0) {
          a.part_ml[2 * row] = m[e];
          a.part_ml[2 * row + 1] = l[e];
        }
      }
    }
  };
  const uint32_t base = smem_u32(smem);
  int4 desc = make_int4(0, 0, 0, 0);  // descriptors 32 at a time (piece boundaries of every chunk)
  for (int64_t j = c0; j < c1; ++j) {
    const int64_t i = j - c0;
    if ((i & 31) == 0) desc = j + lane < c1 ? __ldg(a.chunks + j + lane) : make_int4(0, 0, 0, 0);
    const int n = __shfl_sync(0xffffffffu, desc.z, static_cast<int>(i & 31));
    const int b = __shfl_sync(0xffffffffu, desc.w, static_cast<int>(i & 31));
    if (b != cur_b) {
      if (cur_b >= 0) flush();
      cur_b = b;
      whole = a.piece_count[b] == 1;
#pragma unroll
      for (int mt = 0; mt < 8; ++mt) o[mt][0] = o[mt][1] = o[mt][2] = o[mt][3] = 0.f;
      m[0] = m[1] = -INFINITY;
      l[0] = l[1] = 0.f;
      // B[k][n] = Q[head n][dim k]: lane holds dims 2*c4 (+1) and +8 of head r4.
      const bool valid = r4 < G;
      const __nv_bfloat16* qh = a.q + (static_cast<int64_t>(b) * Hq + h * G + (valid ? r4 : 0)) * kD;
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        qb[kk][0] = valid ? *reinterpret_cast<const uint32_t*>(qh + kk * 16 + 2 * c4) : 0u;
        qb[kk][1] = valid ? *reinterpret_cast<const uint32_t*>(qh + kk * 16 + 8 + 2 * c4) : 0u;
      }
    }
    const int64_t qk = 2 * i, qv = 2 * i + 1;
    const int sk = static_cast<int>(qk % kRing), sv = static_cast<int>(qv % kRing);
    mbar_wait(full0 + 8 * sk, static_cast<uint32_t>(qk / kRing) & 1u);
    const uint32_t kb = base + sk * kHalfBytes + (2 * h) * kBlockBytes;  // K dims 0..63, 64..127
    const uint32_t vb = base + sv * kHalfBytes + (2 * h) * kBlockBytes;  // V likewise
    uint8_t* const v0 = smem + sv * kHalfBytes + (2 * h) * kBlockBytes;
    // S^T = K Q^T: A = K (16 tokens x 16 dims per step) by ldmatrix.
    float s[4] = {0.f, 0.f, 0.f, 0.f};
    {
      const int mi = lane >> 3;
      const int row = (lane & 7) + ((mi & 1) << 3);
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        const int c = 2 * kk + (mi >> 1);  // 16-byte chunk of the head's 256 bytes
        uint32_t ka[4];
        ldsm_x4(kb + (c >> 3) * kBlockBytes + sw(row, c & 7), ka);
        mma(s, ka, qb[kk][0], qb[kk][1]);
      }
    }
    // Mask, scale; per query head the max over the 16 tokens.
    const bool t0v = r4 < n, t1v = r4 + 8 < n;
    s[0] = t0v ? s[0] * a.scale_log2 : -INFINITY;
    s[1] = t0v ? s[1] * a.scale_log2 : -INFINITY;
    s[2] = t1v ? s[2] * a.scale_log2 : -INFINITY;
    s[3] = t1v ? s[3] * a.scale_log2 : -INFINITY;
    float mx[2] = {fmaxf(s[0], s[2]), fmaxf(s[1], s[3])};
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      mx[e] = fmaxf(mx[e], __shfl_xor_sync(0xffffffffu, mx[e], 4));
      mx[e] = fmaxf(mx[e], __shfl_xor_sync(0xffffffffu, mx[e], 8));
      mx[e] = fmaxf(mx[e], __shfl_xor_sync(0xffffffffu, mx[e], 16));
    }
    float alpha[2];
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const float nm = fmaxf(m[e], mx[e]);
      alpha[e] = nm == -INFINITY ? 1.f : ex2(m[e] - nm);
      m[e] = nm;
    }
    float p[4];
    p[0] = m[0] == -INFINITY ? 0.f : ex2(s[0] - m[0]);
    p[1] = m[1] == -INFINITY ? 0.f : ex2(s[1] - m[1]);
    p[2] = m[0] == -INFINITY ? 0.f : ex2(s[2] - m[0]);
    p[3] = m[1] == -INFINITY ? 0.f : ex2(s[3] - m[1]);
    l[0] = l[0] * alpha[0] + p[0] + p[2];
    l[1] = l[1] * alpha[1] + p[1] + p[3];
#pragma unroll
    for (int mt = 0; mt < 8; ++mt) {
      o[mt][0] *= alpha[0];
      o[mt][1] *= alpha[1];
      o[mt][2] *= alpha[0];
      o[mt][3] *= alpha[1];
    }
    // P^T (16 tokens x 8 heads) -> the PV B fragments (tokens x head r4).
    const uint32_t pb0 = movm_t(pack_bf16(p[0], p[1]));
    const uint32_t pb1 = movm_t(pack_bf16(p[2], p[3]));
    __syncwarp();
    if (lane == 0) mbar_arrive(empty0 + 8 * sk);  // K half consumed: the producer may refill it
    mbar_wait(full0 + 8 * sv, static_cast<uint32_t>(qv / kRing) & 1u);
    if (n < kChunk) {
      // Rows past the chunk hold other slots' words (any bit pattern): zero
      // this head's V rows so P = 0 there cannot meet a NaN.
      for (int e = lane; e < 2 * (kChunk - n) * 8; e += 32) {
        const int blk = e / ((kChunk - n) * 8), rem = e % ((kChunk - n) * 8);
        *reinterpret_cast<uint4*>(v0 + blk * kBlockBytes + (n + rem / 8) * 128 + (rem % 8) * 16) =
            make_uint4(0u, 0u, 0u, 0u);
      }
      __syncwarp();
    }
    // O^T += V^T P^T: A = V^T (16 dims x 16 tokens) by ldmatrix.trans.
    {
      const int mi = lane >> 3;
      const int row = (lane & 7) + ((mi >> 1) << 3);  // token row
#pragma unroll
      for (int mt = 0; mt < 8; ++mt) {
        const int c = 2 * mt + (mi & 1);
        uint32_t va[4];
        ldsm_x4_t(vb + (c >> 3) * kBlockBytes + sw(row, c & 7), va);
        mma(o[mt], va, pb0, pb1);
      }
    }
    if (n < kChunk) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // our V zeros
    __syncwarp();
    if (lane == 0) mbar_arrive(empty0 + 8 * sv);
  }
  if (cur_b >= 0) flush();
}

// Merge each (context, KV head, query head)'s pieces: out = sum_p w_p O_p /
// sum_p w_p, w_p = l_p 2^(m_p - M).  One CTA per (context, KV head, query
// head); its 8 warps take every 8th piece with 4 pieces' loads in flight
// per lane (a float4 of the 128 dims), then the warps' sums are added in
// shared memory — at batch 1 a context has a piece per SM, and one thread
// walking them would be ~150 dependent L2 round trips.
constexpr int kCombineWarps = 8;
constexpr int kCombinePer = 20;  // pieces per warp with loads in flight together (160 pieces)
constexpr int kMlPer = 5;        // (m, l) pairs per lane of warp 0 requested together (160 pieces)
__global__ void __launch_bounds__(kCombineWarps * 32) k_decode_pages_combine(const PagesArgs a, int Hkv) {
  extern __shared__ float cw[];  // [n] weights (padded to 4), then [kCombineWarps][128] sums
  const int G = a.G;
  const int b = blockIdx.x / (Hkv * G), h = (blockIdx.x / G) % Hkv, g = blockIdx.x % G;
  const int n = a.piece_count[b];
  if (n <= 1) return;
  const int first = a.piece_first[b];
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int64_t row0 = ((static_cast<int64_t>(first) + b) * Hkv + h) * G + g;
  const int64_t step = static_cast<int64_t>(Hkv) * G;  // rows between consecutive pieces
  float* red = cw + ((n + 3) & ~3);
  __shared__ float s_sum;
  // One round trip: this warp's pieces' partial rows and (warp 0) every
  // piece's (m, l) are all requested before any is used.
  const float4* po = reinterpret_cast<const float4*>(a.part_o + row0 * kD) + lane;
  const int64_t step4 = step * kD / 4;
  float4 v[kCombinePer];
#pragma unroll
  for (int k = 0; k < kCombinePer; ++k) {
    const int p = wid + k * kCombineWarps;
    v[k] = p < n ? __ldcg(po + p * step4) : make_float4(0.f, 0.f, 0.f, 0.f);
  }
  if (wid == 0) {
    // Every piece's (m, l) requested at once (kMlPer per lane, registers),
    // then the max and the weights from registers: one L2 round trip where
    // a loop over the pieces would chain ~2 n / 32 of them (B = 1: the
    // combine 6.3 -> ~3 us).
    const float2* ml2 = reinterpret_cast<const float2*>(a.part_ml) + row0;
    float2 mlr[kMlPer];
#pragma unroll
    for (int k = 0; k < kMlPer; ++k) {
      const int p = lane + 32 * k;
      mlr[k] = p < n ? __ldcg(ml2 + p * step) : make_float2(-INFINITY, 0.f);
    }
    float mx = -INFINITY;
#pragma unroll
    for (int k = 0; k < kMlPer; ++k) mx = fmaxf(mx, mlr[k].x);
    for (int p = lane + 32 * kMlPer; p < n; p += 32) mx = fmaxf(mx, __ldcg(ml2 + p * step).x);
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, off));
    float wl = 0.f;
#pragma unroll
    for (int k = 0; k < kMlPer; ++k) {
      const int p = lane + 32 * k;
      if (p < n) {
        const float2 ml = mlr[k];
        const float w = (mx == -INFINITY || ml.x == -INFINITY || ml.y <= 0.f) ? 0.f : ml.y * ex2(ml.x - mx);
        cw[p] = w;
        wl += w;
      }
    }
    for (int p = lane + 32 * kMlPer; p < n; p += 32) {  // more pieces than kMlPer * 32 (not at 148 SMs)
      const float2 ml = __ldcg(ml2 + p * step);
      const float w = (mx == -INFINITY || ml.x == -INFINITY || ml.y <= 0.f) ? 0.f : ml.y * ex2(ml.x - mx);
      cw[p] = w;
      wl += w;
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) wl += __shfl_xor_sync(0xffffffffu, wl, off);
    if (lane == 0) s_sum = wl;
  }
  __syncthreads();
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
  for (int k = 0; k < kCombinePer; ++k) {
    const int p = wid + k * kCombineWarps;
    const float w = p < n ? cw[p] : 0.f;
    acc.x += w * v[k].x;
    acc.y += w * v[k].y;
    acc.z += w * v[k].z;
    acc.w += w * v[k].w;
  }
  for (int p = wid + kCombinePer * kCombineWarps; p < n; p += kCombineWarps) {  // > 160 pieces
    const float4 x = __ldcg(po + p * step4);
    const float w = cw[p];
    acc.x += w * x.x;
    acc.y += w * x.y;
    acc.z += w * x.z;
    acc.w += w * x.w;
  }
  reinterpret_cast<float4*>(red + wid * kD)[lane] = acc;
  __syncthreads();
  if (threadIdx.x < kD) {
    float t = 0.f;
#pragma unroll
    for (int w = 0; w < kCombineWarps; ++w) t += red[w * kD + threadIdx.x];
    const float inv = s_sum > 0.f ? 1.f / s_sum : 0.f;
    a.out[(static_cast<int64_t>(b) * a.Hq + h * G + g) * kD + threadIdx.x] = __float2bfloat16_rn(t * inv);
  }
}

// Large batches (a context spans few CTAs): one CTA per (context, KV
// head), warp g = query head g, lanes over the 128 dims (a float4 each);
// the (m, l) pairs and the pieces' rows requested together.
__global__ void __launch_bounds__(kCombineWarps * 32) k_decode_pages_combine_heads(const PagesArgs a,
                                                                                 int Hkv) {
  const int G = a.G;
  const int b = blockIdx.x / Hkv, h = blockIdx.x % Hkv;
  const int n = a.piece_count[b];
  if (n <= 1) return;
  const int first = a.piece_first[b];
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const int lane = threadIdx.x & 31, g = threadIdx.x >> 5;
  if (g >= G) return;
  const int64_t row0 = ((static_cast<int64_t>(first) + b) * Hkv + h) * G + g;
  const int64_t step = static_cast<int64_t>(Hkv) * G;
  const float2* ml2 = reinterpret_cast<const float2*>(a.part_ml) + row0;
  const float4* po = reinterpret_cast<const float4*>(a.part_o + row0 * kD) + lane;
  const int64_t step4 = step * kD / 4;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  float mx = -INFINITY, wl = 0.f;
  for (int p0 = 0; p0 < n; p0 += 8) {
    float2 ml[8];
    float4 v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const bool ok = p0 + k < n;
      ml[k] = ok ? __ldcg(ml2 + (p0 + k) * step) : make_float2(-INFINITY, 0.f);
      v[k] = ok ? __ldcg(po + (p0 + k) * step4) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      if (ml[k].x == -INFINITY || ml[k].y <= 0.f) continue;
      // Running rescale as in the attention kernel: merge piece k into (mx, wl, acc).
      const float nm = fmaxf(mx, ml[k].x);
      const float sa = mx == -INFINITY ? 0.f : ex2(mx - nm), sb = ml[k].y * ex2(ml[k].x - nm);
      acc.x = acc.x * sa + sb * v[k].x;
      acc.y = acc.y * sa + sb * v[k].y;
      acc.z = acc.z * sa + sb * v[k].z;
      acc.w = acc.w * sa + sb * v[k].w;
      wl = wl * sa + sb;
      mx = nm;
    }
  }
  const float inv = wl > 0.f ? 1.f / wl : 0.f;
  __nv_bfloat16* ob = a.out + (static_cast<int64_t>(b) * a.Hq + h * G + g) * kD + 4 * lane;
  reinterpret_cast<uint2*>(ob)[0] =
      make_uint2(pack_bf16(acc.x * inv, acc.y * inv), pack_bf16(acc.z * inv, acc.w * inv));
}

}  // namespace

bool decode_pages_supported(int Hq, int Hkv, int D, int64_t row_u64) {
  return D == kD && Hkv == kHkv && Hq % Hkv == 0 && Hq / Hkv >= 1 && Hq / Hkv <= 8 &&
         row_u64 * 8 == 4LL * Hkv * D;
}

int decode_pages_grid(int num_sms, int64_t n_chunks) {
  return static_cast<int>(n_chunks < num_sms ? (n_chunks < 1 ? 1 : n_chunks) : num_sms);
}

int launch_decode_pages(const PoolTensorMap& map, int layer, const int4* chunks, int64_t n_chunks,
                        const int32_t* piece_first, const int32_t* piece_count, bool any_split,
                        const void* q, int batch, int Hq, int Hkv, float scale, float* part_o,
                        float* part_ml, void* out, int grid, cudaStream_t s) {
  PagesArgs a;
  a.chunks = chunks;
  a.n_chunks = n_chunks;
  a.piece_first = piece_first;
  a.piece_count = piece_count;
  a.q = static_cast<const __nv_bfloat16*>(q);
  a.out = static_cast<__nv_bfloat16*>(out);
  a.part_o = part_o;
  a.part_ml = part_ml;
  a.layer = layer;
  a.Hq = Hq;
  a.G = Hq / Hkv;
  a.scale_log2 = scale * 1.4426950408889634f;
  CUtensorMap m;
  std::memcpy(&m, map.bytes, sizeof(m));
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(static_cast<unsigned>(grid));
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = kSmem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, k_decode_pages, m, a);
  if (!any_split) return 1;
  const int max_pieces = grid;  // a context spans at most every CTA
  // Few contexts, many pieces each: a CTA per (context, KV head, query
  // head) spreads the pieces over its warps.  Many contexts (at most a few
  // pieces each): a CTA per (context, KV head).
  const bool per_row = static_cast<int64_t>(batch) * Hkv * a.G <= 8LL * grid;
  cfg.gridDim = dim3(static_cast<unsigned>(batch * Hkv * (per_row ? a.G : 1)));
  cfg.blockDim = dim3(kCombineWarps * 32);
  cfg.dynamicSmemBytes =
      per_row ? sizeof(float) * (static_cast<size_t>(max_pieces + 3) + kCombineWarps * kD) : 0;
  if (per_row) cudaLaunchKernelEx(&cfg, k_decode_pages_combine, a, Hkv);
  else cudaLaunchKernelEx(&cfg, k_decode_pages_combine_heads, a, Hkv);
  return 2;
}

void preload_decode_pages_kernels() {
  cudaFuncSetAttribute(k_decode_pages, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       static_cast<int>(kSmem));
  cudaFuncAttributes fa;
  cudaFuncGetAttributes(&fa, k_decode_pages);
  cudaFuncGetAttributes(&fa, k_decode_pages_combine);
  cudaFuncGetAttributes(&fa, k_decode_pages_combine_heads);
}

}  // namespace mkv
