// decode_attn.cu — paged GQA decode attention over the KV pool (sm_100a).
//
// No reference analogue (the reference's "attention" is the integer fold,
// kv_cache.cc:319-351); numerics are checked against a CPU fp32
// restatement (tests/test_decode_attention_gpu.py, tolerance stated there).
//
// Each (token, layer) entry of the pool is one row of dim u64 words holding
// K[Hkv][D] then V[Hkv][D] in bf16, addressed through the decode plan's
// per-position slot map (the device page table).  Split-KV (flash-decoding):
// CTA (split, kv_head, batch) folds its token chunk for the G = Hq/Hkv query
// heads of that KV head, 4 warps x 16-token tiles, then a combine kernel
// merges the splits.
//
// Why tensor cores: per 4 KiB token row the group does 2*G*D*Hkv = 16 K
// FMAs at the 70B shape (G = 8), i.e. 26 T FMA/s at the 6.5 TB/s HBM
// roofline — 72% of the FP32 CUDA-core peak before any softmax or
// conversion work — so QK^T and PV run as bf16 mma.sync m16n8k16 with
// fp32 accumulation (M = query heads of the group, padded to 16).  The
// kernel is HBM-bound; the MMA pipe is far from saturated.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

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

template <int D>
__global__ void __launch_bounds__(kWarps * 32) k_decode_attn(
    const __nv_bfloat16* __restrict__ pool_l, int64_t row_elems, const int32_t* __restrict__ slots,
    const int64_t* __restrict__ ctx_off, const int32_t* __restrict__ ctx_len,
    const __nv_bfloat16* __restrict__ q, int Hq, int Hkv, float scale_log2, int splits,
    int n_batch, float* __restrict__ part_o, float* __restrict__ part_ml) {
  static_assert(D % 16 == 0 && D <= 256, "head_dim");
  constexpr int kChunks = D / 8;             // 16-byte chunks per row
  constexpr int kTileBytes = kTile * D * 2;  // one K or V tile
  extern __shared__ __align__(128) uint8_t smem[];
  const int G = Hq / Hkv;
  const int64_t n_items = static_cast<int64_t>(splits) * Hkv * n_batch;
  // Persistent CTAs walk (split, kv_head, batch) items round-robin.
  for (int64_t item = blockIdx.x; item < n_items; item += gridDim.x) {
  const int split = static_cast<int>(item % splits);
  const int h = static_cast<int>((item / splits) % Hkv);
  const int b = static_cast<int>(item / (static_cast<int64_t>(splits) * Hkv));
  __syncthreads();  // the previous item's reduction used the tile buffers
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int len = ctx_len[b];
  int chunk = (len + splits - 1) / splits;
  chunk = (chunk + kTile - 1) / kTile * kTile;
  const int t_begin = split * chunk;
  const int t_end = min(len, t_begin + chunk);
  const int32_t* sl = slots + ctx_off[b];

  // Q fragments (A operand, rows = query heads of this group, zero-padded).
  uint32_t qa[D / 16][4];
  {
    const int r0 = lane >> 2, r1 = r0 + 8, c = 2 * (lane & 3);
    const __nv_bfloat16* qb = q + (static_cast<int64_t>(b) * Hq + static_cast<int64_t>(h) * G) * D;
#pragma unroll
    for (int kk = 0; kk < D / 16; ++kk) {
      auto ld2 = [&](int r, int col) -> uint32_t {
        if (r >= G) return 0u;
        return *reinterpret_cast<const uint32_t*>(qb + static_cast<int64_t>(r) * D + col);
      };
      qa[kk][0] = ld2(r0, kk * 16 + c);
      qa[kk][1] = ld2(r1, kk * 16 + c);
      qa[kk][2] = ld2(r0, kk * 16 + c + 8);
      qa[kk][3] = ld2(r1, kk * 16 + c + 8);
    }
  }

  float o[D / 8][4];
#pragma unroll
  for (int j = 0; j < D / 8; ++j) o[j][0] = o[j][1] = o[j][2] = o[j][3] = 0.f;
  float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;

  uint8_t* wsm = smem + warp * (4 * kTileBytes);  // [stage][K|V][16][D]
  const int n_tiles = t_end > t_begin ? (t_end - t_begin + kTile - 1) / kTile : 0;
  const int64_t k_off = static_cast<int64_t>(h) * D, v_off = static_cast<int64_t>(Hkv + h) * D;

  auto load_tile = [&](int tile, int stage) {
    const int t0 = t_begin + tile * kTile;
    const uint32_t kbase = smem_u32(wsm + stage * 2 * kTileBytes);
    const uint32_t vbase = kbase + kTileBytes;
#pragma unroll
    for (int i = lane; i < kTile * kChunks; i += 32) {
      const int r = i / kChunks, c = i % kChunks;
      const int t = t0 + r;
      const bool valid = t < t_end;
      const int64_t slot = valid ? static_cast<int64_t>(__ldg(sl + t)) : 0;
      const __nv_bfloat16* row = pool_l + slot * row_elems;
      cp_async16(kbase + tile_off<D>(r, c), row + k_off + c * 8, valid);
      cp_async16(vbase + tile_off<D>(r, c), row + v_off + c * 8, valid);
    }
  };

  int my = 0;  // tiles handled by this warp: warp, warp + 4, ...
  if (warp < n_tiles) load_tile(warp, 0);
  cp_async_commit();
  for (int tile = warp; tile < n_tiles; tile += kWarps, ++my) {
    const int stage = my & 1;
    if (tile + kWarps < n_tiles) load_tile(tile + kWarps, stage ^ 1);
    cp_async_commit();
    cp_async_wait<1>();
    __syncwarp();
    const uint32_t kbase = smem_u32(wsm + stage * 2 * kTileBytes);
    const uint32_t vbase = kbase + kTileBytes;

    // S = Q K^T over 16 tokens (two n8 tiles).
    float s[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
#pragma unroll
    for (int kk = 0; kk < D / 16; ++kk) {
      const int mi = lane >> 3, r = (lane & 7) + ((mi >> 1) << 3);
      const int c = 2 * kk + (mi & 1);
      uint32_t b0, b1, b2, b3;
      ldmatrix_x4(kbase + tile_off<D>(r, c), b0, b1, b2, b3);
      mma_bf16(s[0], qa[kk], b0, b1);
      mma_bf16(s[1], qa[kk], b2, b3);
    }
    // Mask tokens past the context, scale, online softmax per query row.
    const int t0 = t_begin + tile * kTile;
#pragma unroll
    for (int j = 0; j < 2; ++j) {
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int t = t0 + 8 * j + 2 * (lane & 3) + (e & 1);
        s[j][e] = t < t_end ? s[j][e] * scale_log2 : -INFINITY;
      }
    }
    float mx0 = fmaxf(fmaxf(s[0][0], s[0][1]), fmaxf(s[1][0], s[1][1]));
    float mx1 = fmaxf(fmaxf(s[0][2], s[0][3]), fmaxf(s[1][2], s[1][3]));
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
      p[j][0] = exp2f(s[j][0] - m0);
      p[j][1] = exp2f(s[j][1] - m0);
      p[j][2] = exp2f(s[j][2] - m1);
      p[j][3] = exp2f(s[j][3] - m1);
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
      red[(warp * 16 + r0) * D + c] = o[j][0];
      red[(warp * 16 + r0) * D + c + 1] = o[j][1];
      red[(warp * 16 + r1) * D + c] = o[j][2];
      red[(warp * 16 + r1) * D + c + 1] = o[j][3];
    }
    if ((lane & 3) == 0) {
      red_ml[(warp * 16 + r0) * 2] = m0;
      red_ml[(warp * 16 + r0) * 2 + 1] = l0;
      red_ml[(warp * 16 + r1) * 2] = m1;
      red_ml[(warp * 16 + r1) * 2 + 1] = l1;
    }
  }
  __syncthreads();
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
        const float sc = exp2f(mw - M);
        acc += sc * red[(w * 16 + r) * D + c];
        lsum += sc * red_ml[(w * 16 + r) * 2 + 1];
      }
    }
    const int64_t qh = static_cast<int64_t>(b) * Hq + static_cast<int64_t>(h) * G + r;
    part_o[(qh * splits + split) * D + c] = lsum > 0.f ? acc / lsum : 0.f;
    if (c == 0) {
      part_ml[(qh * splits + split) * 2] = M;
      part_ml[(qh * splits + split) * 2 + 1] = lsum;
    }
  }
  }  // items
}

// Merge split partials: out = sum_s w_s O_s / sum_s w_s, w_s = l_s 2^(m_s - M).
__global__ void k_decode_combine(const float* __restrict__ part_o, const float* __restrict__ part_ml,
                                 int splits, int D, __nv_bfloat16* __restrict__ out) {
  const int64_t qh = blockIdx.x;
  float M = -INFINITY;
  for (int s = 0; s < splits; ++s) M = fmaxf(M, part_ml[(qh * splits + s) * 2]);
  for (int c = threadIdx.x; c < D; c += blockDim.x) {
    float acc = 0.f, wsum = 0.f;
    if (M != -INFINITY) {
      for (int s = 0; s < splits; ++s) {
        const float ms = part_ml[(qh * splits + s) * 2];
        const float ls = part_ml[(qh * splits + s) * 2 + 1];
        if (ms == -INFINITY || ls <= 0.f) continue;
        const float w = ls * exp2f(ms - M);
        acc += w * part_o[(qh * splits + s) * D + c];
        wsum += w;
      }
    }
    out[qh * D + c] = __float2bfloat16_rn(wsum > 0.f ? acc / wsum : 0.f);
  }
}

}  // namespace

size_t decode_attn_smem(int head_dim) {
  const size_t tiles = static_cast<size_t>(kWarps) * 4 * kTile * head_dim * 2;
  const size_t red = static_cast<size_t>(kWarps) * 16 * head_dim * 4 + kWarps * 16 * 2 * 4;
  return tiles > red ? tiles : red;
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
                        const int64_t* ctx_off, const int32_t* ctx_len, const void* q, int batch,
                        int Hq, int Hkv, int D, float scale, int splits, float* part_o,
                        float* part_ml, void* out, int grid, cudaStream_t s) {
  const float scale_log2 = scale * 1.4426950408889634f;
  const int64_t items = static_cast<int64_t>(splits) * Hkv * batch;
  const int g = static_cast<int>(items < grid ? items : grid);
  const size_t smem = decode_attn_smem(D);
  auto q16 = static_cast<const __nv_bfloat16*>(q);
  auto pool16 = static_cast<const __nv_bfloat16*>(pool_l);
  if (D == 128) {
    k_decode_attn<128><<<g, kWarps * 32, smem, s>>>(pool16, row_elems, slots, ctx_off, ctx_len,
                                                    q16, Hq, Hkv, scale_log2, splits, batch,
                                                    part_o, part_ml);
  } else if (D == 64) {
    k_decode_attn<64><<<g, kWarps * 32, smem, s>>>(pool16, row_elems, slots, ctx_off, ctx_len,
                                                   q16, Hq, Hkv, scale_log2, splits, batch,
                                                   part_o, part_ml);
  } else {
    return false;
  }
  k_decode_combine<<<batch * Hq, 128, 0, s>>>(part_o, part_ml, splits, D,
                                              static_cast<__nv_bfloat16*>(out));
  return true;
}

}  // namespace mkv
