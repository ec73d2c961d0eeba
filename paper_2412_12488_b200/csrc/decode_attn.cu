// decode_attn.cu — paged GQA decode attention over the KV pool (sm_100a).
//
// No reference analogue (the reference's "attention" is the integer fold,
// kv_cache.cc:319-351); numerics are checked against a plain fp32 PyTorch
// reference (tests/test_decode_attention_gpu.py, tolerance stated there).
//
// Each (token, layer) entry of the pool is one row of dim u64 words holding
// K[Hkv][D] then V[Hkv][D] in bf16, addressed through the decode plan's
// per-position slot map (gathered from the device page tables).
//
// Work split (stream-K): segment s = (batch b, kv head h) owns
// ceil(ctx_b / 16) tiles of 16 tokens; seg_start[] is their prefix sum (T
// tiles in all).  A resident-sized grid gives CTA c the equal share
// [c*T/grid, (c+1)*T/grid), which may finish one segment and start the
// next.  Each (CTA, segment) piece folds its tiles for the G = Hq/Hkv query
// heads of that KV head (4 warps, 16-token tiles, double-buffered cp.async)
// and writes one normalised partial (O, m, l) at index c + s — unique,
// because pieces are ordered by both c and s.  A combine kernel merges each
// segment's pieces.  Equal shares remove the wave-quantisation loss of
// per-(split, head, batch) work items.
//
// Why tensor cores: per 4 KiB token row the group does 2*G*D*Hkv = 16 K
// FMAs at the 70B shape (G = 8), i.e. 26 T FMA/s at the 6.5 TB/s HBM
// roofline — 72% of the FP32 CUDA-core peak before any softmax or
// conversion work — so QK^T and PV run as bf16 mma.sync m16n8k16 with fp32
// accumulation (M = query heads of the group, padded to 16).  The kernel is
// HBM-bound; the MMA pipe is far from saturated.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <type_traits>

namespace mkv {

namespace {

constexpr int kWarps = 4;
constexpr int kTile = 16;  // tokens per warp tile

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, bool valid) {
  const int n = valid ? 16 : 0;  // zero-fill rows past the context
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(n)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

__device__ __forceinline__ void ldmatrix_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2,
                                            uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0, %1, %2, %3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
__device__ __forceinline__ void ldmatrix_x4_trans(uint32_t addr, uint32_t& r0, uint32_t& r1,
                                                  uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0, %1, %2, %3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}

__device__ __forceinline__ void mma_bf16(float (&c)[4], const uint32_t (&a)[4], uint32_t b0,
                                         uint32_t b1) {
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

// Swizzled byte offset of 16-byte chunk `c` of token row `r` in a
// [16][D] bf16 tile (row = D*2 bytes): XOR with r%8 removes the 8-way bank
// conflict of ldmatrix on 256-byte rows.
template <int D>
__device__ __forceinline__ uint32_t tile_off(int r, int c) {
  return static_cast<uint32_t>(r * (D * 2) + ((c ^ (r & 7)) * 16));
}

__host__ __device__ __forceinline__ int64_t cta_tile_start(int64_t c, int64_t T, int64_t grid) {
  return c * T / grid;
}

// CTA whose tile range [cta_tile_start(c), cta_tile_start(c + 1)) holds tile x.
__device__ __forceinline__ int64_t cta_of_tile(int64_t x, int64_t T, int64_t grid) {
  int64_t c = x * grid / T;
  while (c + 1 < grid && cta_tile_start(c + 1, T, grid) <= x) ++c;
  while (c > 0 && cta_tile_start(c, T, grid) > x) --c;
  return c;
}

// Shared memory per CTA: [warp][stage][K|V][16][D] tiles, then Q [16][D]
// (swizzled like the tiles; rows >= G zero).  The end-of-piece warp merge
// reuses the tile area.
#ifndef DA_STAGES
#define DA_STAGES 2  // 2 measured best (3: -2..4%, 4: fewer resident CTAs, -25%)
#endif
constexpr int kStages = DA_STAGES;  // cp.async ring depth per warp (tiles in flight)

template <int D>
__host__ __device__ constexpr size_t tiles_bytes() {
  return static_cast<size_t>(kWarps) * 2 * kStages * kTile * D * 2;
}

template <int D>
__global__ void __launch_bounds__(kWarps * 32, 3) k_decode_attn(
    const __nv_bfloat16* __restrict__ pool_l, int64_t row_elems, const int32_t* __restrict__ slots,
    const int64_t* __restrict__ ctx_off, const int32_t* __restrict__ ctx_len,
    const int64_t* __restrict__ seg_start, int64_t n_seg, const __nv_bfloat16* __restrict__ q,
    int Hq, int Hkv, float scale_log2, float* __restrict__ part_o, float* __restrict__ part_ml,
    __nv_bfloat16* __restrict__ out, uint32_t* __restrict__ seg_count,
    const int32_t* __restrict__ cta_seg) {
  static_assert(D % 16 == 0 && D <= 256, "head_dim");
  __shared__ int merge_here;
  constexpr int kChunks = D / 8;             // 16-byte chunks per row
  constexpr int kTileBytes = kTile * D * 2;  // one K or V tile
  extern __shared__ __align__(128) uint8_t smem[];
  uint8_t* q_sm = smem + tiles_bytes<D>();
  const int G = Hq / Hkv;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t T = seg_start[n_seg];
  int64_t t0 = cta_tile_start(blockIdx.x, T, gridDim.x);
  const int64_t t1 = cta_tile_start(blockIdx.x + 1, T, gridDim.x);
  if (t0 >= t1) return;
  // Last segment whose first tile is <= t0, precomputed per CTA by the host
  // (a device binary search here chained ~log2(segments) dependent loads
  // before the first KV byte could be requested).
  const int64_t lo = cta_seg[blockIdx.x];
  // Launched as a programmatic dependent of the previous kernel on the
  // stream: the plan reads above and the first piece's slot fetch overlap
  // its tail; Q and the pool (which it may have written: the new token's
  // K||V row, the query) are read only after griddepcontrol.wait.
  bool waited = false;
  for (int64_t sgi = lo; t0 < t1 && sgi < n_seg; ++sgi) {
    const int64_t s_begin = seg_start[sgi], s_end = seg_start[sgi + 1];
    if (s_end <= t0) continue;  // empty segment
    const int64_t pe = s_end < t1 ? s_end : t1;
    const int b = static_cast<int>(sgi / Hkv), h = static_cast<int>(sgi % Hkv);
    const int len = ctx_len[b];
    const int first_tile = static_cast<int>(t0 - s_begin);
    const int n_tiles = static_cast<int>(pe - t0);
    const int tok0 = first_tile * kTile;
    const int tok_end = min(len, (first_tile + n_tiles) * kTile);
    const int32_t* sl = slots + ctx_off[b];
    __syncthreads();  // the previous piece's merge used the tile area

    float o[D / 8][4];
#pragma unroll
    for (int j = 0; j < D / 8; ++j) o[j][0] = o[j][1] = o[j][2] = o[j][3] = 0.f;
    float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;

    uint8_t* wsm = smem + warp * (2 * kStages * kTileBytes);  // [stage][K|V][16][D]
    const int64_t k_off = static_cast<int64_t>(h) * D, v_off = static_cast<int64_t>(Hkv + h) * D;
    const uint32_t q_base = smem_u32(q_sm);
    // Lanes 0..15 hold the slot of row `lane` of a tile (fetched a tile ahead).
    auto fetch_slot = [&](int tile) -> int32_t {
      const int t = tok0 + tile * kTile + (lane & 15);
      return (tile < n_tiles && t < tok_end) ? __ldg(sl + t) : 0;
    };
    auto load_tile = [&](int tile, int stage, int32_t my_slot) {
      const int r0 = tok0 + tile * kTile;
      const uint32_t kbase = smem_u32(wsm + stage * 2 * kTileBytes);
      const uint32_t vbase = kbase + kTileBytes;
#pragma unroll
      for (int i = lane; i < kTile * kChunks; i += 32) {
        const int r = i / kChunks, c = i % kChunks;
        const int64_t slot = __shfl_sync(0xffffffffu, my_slot, r);
        const bool valid = r0 + r < tok_end;
        const __nv_bfloat16* row = pool_l + slot * row_elems;
        cp_async16(kbase + tile_off<D>(r, c), row + k_off + c * 8, valid);
        cp_async16(vbase + tile_off<D>(r, c), row + v_off + c * 8, valid);
      }
    };

    int my = 0;  // tiles of this piece handled by this warp: warp, warp + 4, ...
    // The first K/V loads go out before Q is staged (one memory round trip
    // less per piece: short pieces, e.g. batch 1, are latency-bound).
    // Prologue: the first kStages - 1 tiles in flight.
    int32_t nxt = fetch_slot(warp);
    if (!waited) {
      asm volatile("griddepcontrol.wait;" ::: "memory");
      // The combine kernel (a programmatic dependent) may launch now; it
      // waits for this grid's completion before reading partials.  Not with
      // the fused merge (large batches): the next call's CTAs would then be
      // placed early, on whichever SMs have room, and run unbalanced
      // (B=32 ctx 8K: 0.99 -> 0.88 of HBM).
      if (seg_count == nullptr) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
      waited = true;
    }
#pragma unroll
    for (int pre = 0; pre < kStages - 1; ++pre) {
      const int t = warp + pre * kWarps;
      if (t < n_tiles) load_tile(t, pre, nxt);
      cp_async_commit();
      nxt = fetch_slot(t + kWarps);
    }
    {  // Stage the group's Q rows (coalesced 16-byte loads).
      const __nv_bfloat16* qb =
          q + (static_cast<int64_t>(b) * Hq + static_cast<int64_t>(h) * G) * D;
      for (int i = threadIdx.x; i < kTile * kChunks; i += blockDim.x) {
        const int r = i / kChunks, c = i % kChunks;
        uint4 v = make_uint4(0u, 0u, 0u, 0u);
        if (r < G) v = *reinterpret_cast<const uint4*>(qb + static_cast<int64_t>(r) * D + c * 8);
        *reinterpret_cast<uint4*>(q_sm + tile_off<D>(r, c)) = v;
      }
    }
    __syncthreads();
    for (int tile = warp; tile < n_tiles; tile += kWarps, ++my) {
      const int stage = my % kStages;
      const int ahead = tile + (kStages - 1) * kWarps;
      if (ahead < n_tiles) load_tile(ahead, (my + kStages - 1) % kStages, nxt);
      cp_async_commit();
      nxt = fetch_slot(ahead + kWarps);
      cp_async_wait<kStages - 1>();
      __syncwarp();
      const uint32_t kbase = smem_u32(wsm + stage * 2 * kTileBytes);
      const uint32_t vbase = kbase + kTileBytes;

      // S = Q K^T over 16 tokens (two n8 tiles); Q fragments via ldmatrix.
      float sc[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
#pragma unroll
      for (int kk = 0; kk < D / 16; ++kk) {
        uint32_t qa[4];
        {
          const int mi = lane >> 3, r = (lane & 7) + ((mi & 1) << 3);
          const int c = 2 * kk + (mi >> 1);
          ldmatrix_x4(q_base + tile_off<D>(r, c), qa[0], qa[1], qa[2], qa[3]);
        }
        const int mi = lane >> 3, r = (lane & 7) + ((mi >> 1) << 3);
        const int c = 2 * kk + (mi & 1);
        uint32_t b0, b1, b2, b3;
        ldmatrix_x4(kbase + tile_off<D>(r, c), b0, b1, b2, b3);
        mma_bf16(sc[0], qa, b0, b1);
        mma_bf16(sc[1], qa, b2, b3);
      }
      // Mask tokens past the piece, scale, online softmax per query row.
      const int tt = tok0 + tile * kTile;
#pragma unroll
      for (int j = 0; j < 2; ++j) {
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int t = tt + 8 * j + 2 * (lane & 3) + (e & 1);
          sc[j][e] = t < tok_end ? sc[j][e] * scale_log2 : -INFINITY;
        }
      }
      float mx0 = fmaxf(fmaxf(sc[0][0], sc[0][1]), fmaxf(sc[1][0], sc[1][1]));
      float mx1 = fmaxf(fmaxf(sc[0][2], sc[0][3]), fmaxf(sc[1][2], sc[1][3]));
      mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 1));
      mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 2));
      mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 1));
      mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 2));
      const float nm0 = fmaxf(m0, mx0), nm1 = fmaxf(m1, mx1);
      const float a0 = exp2f(m0 - nm0), a1 = exp2f(m1 - nm1);
      m0 = nm0;
      m1 = nm1;
      float p[2][4];
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        p[j][0] = exp2f(sc[j][0] - m0);
        p[j][1] = exp2f(sc[j][1] - m0);
        p[j][2] = exp2f(sc[j][2] - m1);
        p[j][3] = exp2f(sc[j][3] - m1);
      }
      float rs0 = p[0][0] + p[0][1] + p[1][0] + p[1][1];
      float rs1 = p[0][2] + p[0][3] + p[1][2] + p[1][3];
      rs0 += __shfl_xor_sync(0xffffffffu, rs0, 1);
      rs0 += __shfl_xor_sync(0xffffffffu, rs0, 2);
      rs1 += __shfl_xor_sync(0xffffffffu, rs1, 1);
      rs1 += __shfl_xor_sync(0xffffffffu, rs1, 2);
      l0 = l0 * a0 + rs0;
      l1 = l1 * a1 + rs1;
#pragma unroll
      for (int j = 0; j < D / 8; ++j) {
        o[j][0] *= a0;
        o[j][1] *= a0;
        o[j][2] *= a1;
        o[j][3] *= a1;
      }
      // O += P V (P: A operand from the S accumulators; V via ldmatrix.trans).
      uint32_t pa[4];
      pa[0] = pack_bf16(p[0][0], p[0][1]);
      pa[1] = pack_bf16(p[0][2], p[0][3]);
      pa[2] = pack_bf16(p[1][0], p[1][1]);
      pa[3] = pack_bf16(p[1][2], p[1][3]);
#pragma unroll
      for (int j = 0; j < D / 8; j += 2) {
        const int mi = lane >> 3, r = (lane & 7) + ((mi & 1) << 3);
        const int c = j + (mi >> 1);
        uint32_t b0, b1, b2, b3;
        ldmatrix_x4_trans(vbase + tile_off<D>(r, c), b0, b1, b2, b3);
        mma_bf16(o[j], pa, b0, b1);
        mma_bf16(o[j + 1], pa, b2, b3);
      }
      __syncwarp();
    }
    cp_async_wait<0>();
    __syncthreads();

    // Merge the 4 warps' (m, l, O) in shared memory, rows < G only.
    float* red = reinterpret_cast<float*>(smem);  // [warp][16][D] then m,l [warp][16][2]
    float* red_ml = red + kWarps * 16 * D;
    {
      const int r0 = lane >> 2, r1 = r0 + 8;
#pragma unroll
      for (int j = 0; j < D / 8; ++j) {
        const int c = 8 * j + 2 * (lane & 3);
        *reinterpret_cast<float2*>(&red[(warp * 16 + r0) * D + c]) = make_float2(o[j][0], o[j][1]);
        *reinterpret_cast<float2*>(&red[(warp * 16 + r1) * D + c]) = make_float2(o[j][2], o[j][3]);
      }
      if ((lane & 3) == 0) {
        red_ml[(warp * 16 + r0) * 2] = m0;
        red_ml[(warp * 16 + r0) * 2 + 1] = l0;
        red_ml[(warp * 16 + r1) * 2] = m1;
        red_ml[(warp * 16 + r1) * 2 + 1] = l1;
      }
    }
    __syncthreads();
    const int64_t piece = static_cast<int64_t>(blockIdx.x) + sgi;
    // A piece that is the whole segment is final: write the bf16 output.
    const bool whole = t0 == s_begin && pe == s_end;
    for (int i = threadIdx.x; i < G * D; i += blockDim.x) {
      const int r = i / D, c = i % D;
      float M = -INFINITY;
#pragma unroll
      for (int w = 0; w < kWarps; ++w) M = fmaxf(M, red_ml[(w * 16 + r) * 2]);
      float acc = 0.f, lsum = 0.f;
      if (M != -INFINITY) {
#pragma unroll
        for (int w = 0; w < kWarps; ++w) {
          const float mw = red_ml[(w * 16 + r) * 2];
          if (mw == -INFINITY) continue;
          const float scl = exp2f(mw - M);
          acc += scl * red[(w * 16 + r) * D + c];
          lsum += scl * red_ml[(w * 16 + r) * 2 + 1];
        }
      }
      if (whole) {
        out[((static_cast<int64_t>(b) * Hq + static_cast<int64_t>(h) * G + r) * D) + c] =
            __float2bfloat16_rn(lsum > 0.f ? acc / lsum : 0.f);
        continue;
      }
      part_o[(piece * G + r) * D + c] = lsum > 0.f ? acc / lsum : 0.f;
      if (c == 0) {
        part_ml[(piece * G + r) * 2] = M;
        part_ml[(piece * G + r) * 2 + 1] = lsum;
      }
    }
    if (!whole && seg_count != nullptr) {
      // Fused combine: the last CTA to finish a piece of this segment
      // merges all of its pieces (threadfence-reduction pattern: partials,
      // fence, counter; the last arriver fences and reads them from L2),
      // so no second kernel and no launch gap.
      const int64_t c_first = cta_of_tile(s_begin, T, gridDim.x);
      const int n = static_cast<int>(cta_of_tile(s_end - 1, T, gridDim.x) - c_first + 1);
      // One fence per CTA: bar.sync makes the CTA's partial stores visible
      // to thread 0, whose (cumulative) gpu-scope fence orders them before
      // the counter update; the last arriver fences again before reading.
      __syncthreads();
      if (threadIdx.x == 0) {
        __threadfence();
        const unsigned prev = atomicAdd(seg_count + sgi, 1u);
        merge_here = prev == static_cast<unsigned>(n - 1);
        if (merge_here) {
          seg_count[sgi] = 0;  // ready for the next launch
          __threadfence();
        }
      }
      __syncthreads();
      if (merge_here) {
        float* wts = reinterpret_cast<float*>(smem);  // [G][n] weights, then [G] sums
        float* wsum = wts + G * n;
        const float2* ml2 = reinterpret_cast<const float2*>(part_ml);
        for (int r = warp; r < G; r += kWarps) {
          // (m, l) of pieces lane, lane + 32 in registers: one round trip.
          float2 v2[2];
#pragma unroll
          for (int k = 0; k < 2; ++k)
            v2[k] = lane + 32 * k < n ? __ldcg(ml2 + (c_first + lane + 32 * k + sgi) * G + r)
                                      : make_float2(-INFINITY, 0.f);
          float m = fmaxf(v2[0].x, v2[1].x);
          for (int p = lane + 64; p < n; p += 32) m = fmaxf(m, __ldcg(ml2 + (c_first + p + sgi) * G + r).x);
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
          float wl = 0.f;
          for (int p = lane, k = 0; p < n; p += 32, ++k) {
            const float2 v = k < 2 ? v2[k] : __ldcg(ml2 + (c_first + p + sgi) * G + r);
            const float w = (m == -INFINITY || v.x == -INFINITY || v.y <= 0.f) ? 0.f : v.y * exp2f(v.x - m);
            wts[r * n + p] = w;
            wl += w;
          }
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) wl += __shfl_xor_sync(0xffffffffu, wl, o);
          if (lane == 0) wsum[r] = wl;
        }
        __syncthreads();
        // Outputs as float4 column quads, every piece's load of a quad in
        // flight together (one L2 round trip per quad).
        const int64_t step4 = static_cast<int64_t>(G) * D / 4;
        const float4* po4 = reinterpret_cast<const float4*>(part_o);
        for (int e = threadIdx.x; e < G * D / 4; e += blockDim.x) {
          const int r = (4 * e) / D, d = (4 * e) % D;
          const float4* po = po4 + (((c_first + sgi) * G + r) * D + d) / 4;
          float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
          for (int p0 = 0; p0 < n; p0 += 32) {
            float4 v[32];
#pragma unroll
            for (int k = 0; k < 32; ++k)
              v[k] = p0 + k < n ? __ldcg(po + (p0 + k) * step4) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
            for (int k = 0; k < 32; ++k) {
              const float w = p0 + k < n ? wts[r * n + p0 + k] : 0.f;
              acc.x += w * v[k].x;
              acc.y += w * v[k].y;
              acc.z += w * v[k].z;
              acc.w += w * v[k].w;
            }
          }
          const float ws = wsum[r];
          const float inv = ws > 0.f ? 1.f / ws : 0.f;
          __nv_bfloat16* o16 =
              out + (static_cast<int64_t>(b) * Hq + static_cast<int64_t>(h) * G + r) * D + d;
          reinterpret_cast<uint2*>(o16)[0] =
              make_uint2(pack_bf16(acc.x * inv, acc.y * inv), pack_bf16(acc.z * inv, acc.w * inv));
        }
      }
    }
    t0 = pe;
  }
}

// Merge a segment's pieces, one CTA per segment (batch, kv head) covering
// its G query heads: out = sum_p w_p O_p / sum_p w_p, w_p = l_p 2^(m_p - M).
// Segments finished by a single piece were written by the main kernel.
constexpr int kCombineThreads = 256;

__global__ void __launch_bounds__(kCombineThreads) k_decode_combine(
    const float* __restrict__ part_o, const float* __restrict__ part_ml,
    const int64_t* __restrict__ seg_start, int64_t n_seg, int Hq, int Hkv, int D, int grid,
    __nv_bfloat16* __restrict__ out) {
  extern __shared__ float cw[];  // [rows][n] weights, then [rows] weight sums
  // Launched as a programmatic dependent of the attention kernel: everything
  // up to griddepcontrol.wait (segment bounds, piece range) overlaps its
  // tail; partials are read only after the dependency resolves.  Three
  // dependent memory round trips in all (bounds, (m, l) pairs, O pieces):
  // at small batch the combine is pure latency.
  const int64_t s = blockIdx.x;
  const int rpc = (Hq / Hkv + gridDim.y - 1) / gridDim.y;  // query rows of this CTA
  const int r_base = blockIdx.y * rpc;
  const int b = static_cast<int>(s / Hkv), h = static_cast<int>(s % Hkv);
  const int G = Hq / Hkv;
  const int64_t T = seg_start[n_seg];
  const int64_t x0 = seg_start[s], x1 = seg_start[s + 1] - 1;
  if (x1 < x0) return;
  auto cta_of = [&](int64_t x) {  // CTA whose tile range holds tile x
    int64_t c = x * grid / T;
    while (c + 1 < grid && cta_tile_start(c + 1, T, grid) <= x) ++c;
    while (c > 0 && cta_tile_start(c, T, grid) > x) --c;
    return c;
  };
  const int64_t c0 = cta_of(x0);
  const int n = static_cast<int>(cta_of(x1) - c0 + 1);
  if (n == 1) return;
  const int rows = min(rpc, G - r_base);
  if (rows <= 0) return;
  asm volatile("griddepcontrol.wait;" ::: "memory");
  float* wsum = cw + rows * n;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int rr = wid; rr < rows; rr += blockDim.x / 32) {
    const int r = r_base + rr;
    // (m, l) of up to 64 pieces per lane pass, one 8-byte load each.
    float wl = 0.f;
    float m = -INFINITY;
    float2 ml[2];
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const int p = lane + 32 * k;
      ml[k] = p < n ? __ldcg(reinterpret_cast<const float2*>(part_ml) + (c0 + p + s) * G + r)
                    : make_float2(-INFINITY, 0.f);
      m = fmaxf(m, ml[k].x);
    }
    for (int p = lane + 64; p < n; p += 32)
      m = fmaxf(m, __ldcg(reinterpret_cast<const float2*>(part_ml) + (c0 + p + s) * G + r).x);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    for (int p = lane, k = 0; p < n; p += 32, ++k) {
      const float2 v = k < 2 ? ml[k] : __ldcg(reinterpret_cast<const float2*>(part_ml) + (c0 + p + s) * G + r);
      const float w = (m == -INFINITY || v.x == -INFINITY || v.y <= 0.f) ? 0.f : v.y * exp2f(v.x - m);
      cw[rr * n + p] = w;
      wl += w;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) wl += __shfl_xor_sync(0xffffffffu, wl, o);
    if (lane == 0) wsum[rr] = wl;
  }
  __syncthreads();
  for (int e = threadIdx.x; e < rows * D; e += blockDim.x) {
    const int rr = e / D, d = e % D, r = r_base + rr;
    // All pieces' loads in flight together (one round trip for n <= 32).
    const float* po = part_o + ((c0 + s) * G + r) * D + d;
    const int64_t step = static_cast<int64_t>(G) * D;  // between consecutive pieces
    float acc0 = 0.f, acc1 = 0.f;
    int p = 0;
    if (n > 32 && n <= 64) {  // up to 64 pieces: every load in flight at once
      float v[64];
#pragma unroll
      for (int k = 0; k < 64; ++k) v[k] = k < n ? __ldcg(po + k * step) : 0.f;
#pragma unroll
      for (int k = 0; k < 64; k += 2) {
        if (k < n) acc0 += cw[rr * n + k] * v[k];
        if (k + 1 < n) acc1 += cw[rr * n + k + 1] * v[k + 1];
      }
      p = n;
    }
    for (; p + 32 <= n; p += 32) {
      float v[32];
#pragma unroll
      for (int k = 0; k < 32; ++k) v[k] = __ldcg(po + (p + k) * step);
#pragma unroll
      for (int k = 0; k < 32; k += 2) {
        acc0 += cw[rr * n + p + k] * v[k];
        acc1 += cw[rr * n + p + k + 1] * v[k + 1];
      }
    }
    auto tail = [&](auto width) {  // the last n - p < 32 pieces, predicated
      constexpr int kW = decltype(width)::value;
      float v[kW];
#pragma unroll
      for (int k = 0; k < kW; ++k) v[k] = p + k < n ? __ldcg(po + (p + k) * step) : 0.f;
#pragma unroll
      for (int k = 0; k < kW; ++k)
        if (p + k < n) acc0 += cw[rr * n + p + k] * v[k];
    };
    if (n - p > 8) tail(std::integral_constant<int, 32>{});
    else if (n > p) tail(std::integral_constant<int, 8>{});
    const float acc = acc0 + acc1;
    const float ws = wsum[rr];
    out[(static_cast<int64_t>(b) * Hq + static_cast<int64_t>(h) * G + r) * D + d] =
        __float2bfloat16_rn(ws > 0.f ? acc / ws : 0.f);
  }
}

}  // namespace

size_t decode_attn_smem(int head_dim) {
  const size_t tiles = static_cast<size_t>(kWarps) * 2 * kStages * kTile * head_dim * 2;
  const size_t red = static_cast<size_t>(kWarps) * 16 * head_dim * 4 + kWarps * 16 * 2 * 4;
  return (tiles > red ? tiles : red) + static_cast<size_t>(kTile) * head_dim * 2;
}

int decode_attn_resident_ctas(int head_dim, int num_sms) {
  const size_t smem = decode_attn_smem(head_dim);
  int per_sm = 1;
  if (head_dim == 128) {
    cudaFuncSetAttribute(k_decode_attn<128>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(smem));
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_decode_attn<128>, kWarps * 32, smem);
  } else {
    cudaFuncSetAttribute(k_decode_attn<64>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(smem));
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_decode_attn<64>, kWarps * 32, smem);
  }
  return (per_sm < 1 ? 1 : per_sm) * num_sms;
}

bool launch_decode_attn(const void* pool_l, int64_t row_elems, const int32_t* slots,
                        const int64_t* ctx_off, const int32_t* ctx_len, const int64_t* seg_start,
                        int64_t n_seg, int64_t total_tiles, const void* q, int batch, int Hq,
                        int Hkv, int D, float scale, float* part_o, float* part_ml, void* out,
                        int grid, uint32_t* seg_count, const int32_t* cta_seg,
                        cudaStream_t s) {
  const float scale_log2 = scale * 1.4426950408889634f;
  const int g = static_cast<int>(total_tiles < grid ? (total_tiles < 1 ? 1 : total_tiles) : grid);
  const size_t smem = decode_attn_smem(D);
  auto q16 = static_cast<const __nv_bfloat16*>(q);
  auto pool16 = static_cast<const __nv_bfloat16*>(pool_l);
  auto out16 = static_cast<__nv_bfloat16*>(out);
  {
    void (*kern)(const __nv_bfloat16*, int64_t, const int32_t*, const int64_t*, const int32_t*,
                 const int64_t*, int64_t, const __nv_bfloat16*, int, int, float, float*, float*,
                 __nv_bfloat16*, uint32_t*, const int32_t*) = nullptr;
    if (D == 128) kern = k_decode_attn<128>;
    else if (D == 64) kern = k_decode_attn<64>;
    else return false;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(static_cast<unsigned>(g));
    cfg.blockDim = dim3(kWarps * 32);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
#ifndef DA_NO_PDL
    attr[0].val.programmaticStreamSerializationAllowed = 1;
#else
    attr[0].val.programmaticStreamSerializationAllowed = 0;
#endif
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, kern, pool16, row_elems, slots, ctx_off, ctx_len, seg_start, n_seg, q16,
                       Hq, Hkv, scale_log2, part_o, part_ml, out16, seg_count, cta_seg);
  }
  if (seg_count != nullptr) return true;  // pieces merged by the attention kernel
  // Few segments -> one query row per CTA (more parallel merge work); many
  // segments -> all G rows per CTA (fewer, fuller CTAs).
  const int G = Hq / Hkv;
  const int row_groups = n_seg * G <= 4096 ? G : 1;
  const int rpc = (G + row_groups - 1) / row_groups;
  const size_t csmem = sizeof(float) * (static_cast<size_t>(rpc) * (g + 1) + rpc);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(static_cast<unsigned>(n_seg), row_groups);
  cfg.blockDim = dim3(rpc == 1 ? 128 : kCombineThreads);
  cfg.dynamicSmemBytes = csmem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, k_decode_combine, part_o, part_ml, seg_start, n_seg, Hq, Hkv, D, g,
                     out16);
  return true;
}


void preload_decode_attn_kernels() {
  cudaFuncAttributes a;
  cudaFuncGetAttributes(&a, k_decode_attn<128>);
  cudaFuncGetAttributes(&a, k_decode_attn<64>);
  cudaFuncGetAttributes(&a, k_decode_combine);
}

}  // namespace mkv
