// prefill_attn.cu — paged causal GQA prefill attention on tcgen05 (sm_100a).
//
// The decode engine's tail prefill in balanced PD (SURVEY
// §8(f) #2): queries at positions [q_begin, q_end) of a sequence attend to
// keys [0, pos] read from the KV pool through the sequence's HBM page table.
// Unlike decode, this is a dense contraction (e.g. 1,639 queries x 8,192
// keys x 64 heads at the 70B shape), so QK^T and PV run on the 5th-gen
// tensor cores:
//
//   CTA = (16 query tokens x the 8 query heads of one KV head) = M 128 rows.
//   per 128-key tile:  S[128x128] = Q K^T      tcgen05.mma kind::f16, D in TMEM
//                      softmax rows (thread = TMEM lane = row), P -> smem bf16
//                      O[128x128] += P V       tcgen05.mma, V as MN-major B
//   O stays in TMEM (columns 128..255) across tiles; rescaled in place when a
//   row max grows; written once at the end.
//
// Shared memory operands use the UMMA SWIZZLE_128B canonical layout: 8-row
// x 128-byte atoms whose 16-byte chunks are XORed with the row (bits 4-6 ^
// bits 7-9 of the address), atoms 1024-byte aligned; a 128-element row spans
// two atom columns.  K and V tiles are the same bytes ([key][d], d
// contiguous): K is read as a K-major B operand, V as an MN-major one.
// Tiles are gathered row by row (paged, 256 B per (key, kv head)) with
// cp.async, double-buffered.
//
// Numerics: bf16 inputs, fp32 accumulation in TMEM, P rounded to bf16 for
// the PV product; checked against fp32 PyTorch in
// tests/test_prefill_attention_gpu.py.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

namespace mkv {

namespace {

constexpr int kRows = 128;     // M: 16 tokens x 8 heads
constexpr int kTokens = 16;    // query tokens per CTA
constexpr int kKeys = 128;     // N of S / K of PV per tile
constexpr int kD = 128;        // head dim (K of S, N of PV)
constexpr int kThreads = 128;  // 4 warps, thread = TMEM lane = row
constexpr int kAtom = kRows * 128;  // one 64-element atom column of a 128-row tile (16 KiB)
constexpr int kTile = 2 * kAtom;    // a [128][128] bf16 tile (32 KiB)

// Shared memory map (bytes, 1024-aligned regions).
constexpr int kOffQ = 0;
constexpr int kOffK = kOffQ + kTile;       // 2 stages
constexpr int kOffV = kOffK + 2 * kTile;   // 2 stages
constexpr int kOffP = kOffV + 2 * kTile;
constexpr int kOffBar = kOffP + kTile;     // mbarriers + tmem base
constexpr int kSmem = kOffBar + 64;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// Byte offset of 16-byte chunk c (0..15) of row r in a SW128 [rows][128 bf16] tile.
__device__ __forceinline__ uint32_t sw128(int r, int c) {
  return static_cast<uint32_t>((c >> 3) * kAtom + r * 128 + (((c & 7) ^ (r & 7)) << 4));
}

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, bool valid) {
  const int n = valid ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(n)
               : "memory");
}

// UMMA shared-memory descriptor, SWIZZLE_128B (layout type 2), version 1.
__device__ __forceinline__ uint64_t umma_desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  return static_cast<uint64_t>((addr >> 4) & 0x3FFFu) |
         (static_cast<uint64_t>((lbo >> 4) & 0x3FFFu) << 16) |
         (static_cast<uint64_t>((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46) | (2ull << 61);
}

// Instruction descriptor: D f32, A/B bf16, M=128, N=128, A K-major, B K- or MN-major.
__host__ __device__ constexpr uint32_t idesc_bf16(bool b_mn_major) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((b_mn_major ? 1u : 0u) << 16) |
         ((kKeys >> 3) << 17) | ((kRows >> 4) << 24);
}

__device__ __forceinline__ void mma_bf16(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void mma_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar)
               : "memory");
}

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}

// Bounded wait: a tensor-core completion that never arrives traps (the
// launch fails with an error) instead of hanging the GPU.
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
    if (clock64() - t0 > (4ll << 30)) __trap();  // ~2 s at 2 GHz
  }
}

__device__ __forceinline__ void fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// 16 consecutive fp32 columns of this thread's TMEM lane.
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
      "%11, %12, %13, %14, %15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

__device__ __forceinline__ void tmem_st16(uint32_t taddr, const float (&v)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
      "%11, %12, %13, %14, %15, %16};" ::"r"(taddr),
      "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])),
      "r"(__float_as_uint(v[3])), "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])),
      "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7])), "r"(__float_as_uint(v[8])),
      "r"(__float_as_uint(v[9])), "r"(__float_as_uint(v[10])), "r"(__float_as_uint(v[11])),
      "r"(__float_as_uint(v[12])), "r"(__float_as_uint(v[13])), "r"(__float_as_uint(v[14])),
      "r"(__float_as_uint(v[15]))
      : "memory");
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}

__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}

__global__ void __launch_bounds__(kThreads, 1) k_prefill_attn_tc(
    const __nv_bfloat16* __restrict__ pool_l, int64_t row_elems, const int32_t* __restrict__ slots,
    const __nv_bfloat16* __restrict__ q, int q_pos0, int n_q, int Hq, int Hkv,
    float scale_log2, __nv_bfloat16* __restrict__ out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // Operand atoms need 1024-byte alignment of the dynamic smem base.
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  const int tid = threadIdx.x, warp = tid >> 5;
  const int qb = blockIdx.x, h = blockIdx.y;
  const int G = Hq / Hkv;  // 8 (checked by the launcher)
  const uint32_t sQ = smem_u32(smem + kOffQ), sK = smem_u32(smem + kOffK);
  const uint32_t sV = smem_u32(smem + kOffV), sP = smem_u32(smem + kOffP);
  const uint32_t bar_s = smem_u32(smem + kOffBar), bar_o = bar_s + 8;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + kOffBar + 16);

  // Row r of the tile = (token r / 8, head r % 8) of this query block.
  const int r = tid;
  const int tok = r / G, g = r % G;
  const int qt = qb * kTokens + tok;          // query index within [0, n_q)
  const bool row_valid = qt < n_q;
  const int q_pos = q_pos0 + qt;              // absolute position (causal bound)
  const int last_pos = q_pos0 + min(n_q, (qb + 1) * kTokens) - 1;
  const int n_keys = last_pos + 1;            // keys [0, n_keys) needed by this block
  const int n_tiles = (n_keys + kKeys - 1) / kKeys;

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(
                     smem_u32(tmem_slot))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (tid == 0) {
    mbar_init(bar_s, 1);
    mbar_init(bar_o, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  // Q tile (zero rows past n_q).
  {
    const __nv_bfloat16* qrow =
        q + (static_cast<int64_t>(qt) * Hq + static_cast<int64_t>(h) * G + g) * kD;
#pragma unroll
    for (int c = 0; c < 16; ++c) cp_async16(sQ + sw128(r, c), qrow + c * 8, row_valid);
  }
  auto load_kv = [&](int tile, int stage) {
    const uint32_t kb = sK + stage * kTile, vb = sV + stage * kTile;
    const int64_t k_off = static_cast<int64_t>(h) * kD, v_off = static_cast<int64_t>(Hkv + h) * kD;
    // 128 keys x 16 chunks per operand over 128 threads.
#pragma unroll 4
    for (int i = tid; i < kKeys * 16; i += kThreads) {
      const int kk = i >> 4, c = i & 15;
      const int pos = tile * kKeys + kk;
      const bool valid = pos < n_keys;
      const int64_t slot = valid ? static_cast<int64_t>(__ldg(slots + pos)) : 0;
      const __nv_bfloat16* row = pool_l + slot * row_elems;
      cp_async16(kb + sw128(kk, c), row + k_off + c * 8, valid);
      cp_async16(vb + sw128(kk, c), row + v_off + c * 8, valid);
    }
  };
  load_kv(0, 0);
  asm volatile("cp.async.commit_group;" ::: "memory");
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t tS = tmem, tO = tmem + 128;
  const uint32_t lane_off = static_cast<uint32_t>(warp * 32) << 16;  // this warp's TMEM lanes

  float m = -INFINITY, l = 0.f;
  uint32_t ph_s = 0, ph_o = 0;
  constexpr uint32_t kIdescS = idesc_bf16(false), kIdescO = idesc_bf16(true);
  for (int j = 0; j < n_tiles; ++j) {
    const int stage = j & 1;
    // PV(j-1) read stage (j+1)&1's V and the P buffer: wait before reusing them.
    if (j > 0) {
      mbar_wait(bar_o, ph_o);
      ph_o ^= 1;
    }
    if (j + 1 < n_tiles) load_kv(j + 1, stage ^ 1);
    asm volatile("cp.async.commit_group;" ::: "memory");
    asm volatile("cp.async.wait_group 1;" ::: "memory");
    fence_proxy_async();  // cp.async bytes -> visible to the tensor core (async proxy)
    fence_before();
    __syncthreads();
    fence_after();
    if (tid == 0) {
      const uint32_t kb = sK + stage * kTile;
#pragma unroll
      for (int k = 0; k < kD / 16; ++k) {
        const uint32_t off = (k >> 2) * kAtom + (k & 3) * 32;
        mma_bf16(tS, umma_desc(sQ + off, 16, 1024), umma_desc(kb + off, 16, 1024), kIdescS,
                 k > 0 ? 1u : 0u);
      }
      mma_commit(bar_s);
    }
    mbar_wait(bar_s, ph_s);
    ph_s ^= 1;
    fence_after();
    // Row softmax over this tile's 128 keys (two passes over TMEM columns).
    const int key0 = j * kKeys;
    float tmax = -INFINITY;
#pragma unroll
    for (int c0 = 0; c0 < kKeys; c0 += 16) {
      float v[16];
      tmem_ld16(tS + lane_off + c0, v);
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const bool ok = row_valid && key0 + c0 + i <= q_pos;
        tmax = fmaxf(tmax, ok ? v[i] * scale_log2 : -INFINITY);
      }
    }
    const float m_new = fmaxf(m, tmax);
    const float alpha = m_new == -INFINITY ? 1.f : exp2f(m - m_new);
    float psum = 0.f;
#pragma unroll
    for (int c0 = 0; c0 < kKeys; c0 += 16) {
      float v[16];
      tmem_ld16(tS + lane_off + c0, v);
      uint32_t pk[8];
#pragma unroll
      for (int i = 0; i < 16; i += 2) {
        const bool ok0 = row_valid && key0 + c0 + i <= q_pos;
        const bool ok1 = row_valid && key0 + c0 + i + 1 <= q_pos;
        const float p0 = ok0 ? exp2f(v[i] * scale_log2 - m_new) : 0.f;
        const float p1 = ok1 ? exp2f(v[i + 1] * scale_log2 - m_new) : 0.f;
        psum += p0 + p1;
        pk[i / 2] = pack_bf16(p0, p1);
      }
      // P row r, keys c0..c0+15 = chunks c0/8 and c0/8+1 of the SW128 tile.
      const int c = c0 >> 3;
      asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(sP + sw128(r, c)), "r"(pk[0]),
                   "r"(pk[1]), "r"(pk[2]), "r"(pk[3])
                   : "memory");
      asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(sP + sw128(r, c + 1)),
                   "r"(pk[4]), "r"(pk[5]), "r"(pk[6]), "r"(pk[7])
                   : "memory");
    }
    l = l * alpha + psum;
    m = m_new;
    // Rescale the running O rows in TMEM when this tile raised a max.  The
    // TMEM load/store are warp-collective, so the decision is per warp.
    if (j > 0 && __any_sync(0xffffffffu, alpha != 1.f)) {
#pragma unroll
      for (int c0 = 0; c0 < kD; c0 += 16) {
        float v[16];
        tmem_ld16(tO + lane_off + c0, v);
#pragma unroll
        for (int i = 0; i < 16; ++i) v[i] *= alpha;
        tmem_st16(tO + lane_off + c0, v);
      }
    }
    fence_proxy_async();  // P stores -> async proxy
    fence_before();
    __syncthreads();
    fence_after();
    if (tid == 0) {
      const uint32_t vb = sV + stage * kTile;
#pragma unroll
      for (int k = 0; k < kKeys / 16; ++k) {
        // A = P [128 rows x 128 keys] K-major; B = V [128 keys x 128 d] MN-major:
        // 16 keys per step = two 8-key atoms (SBO 1024 B apart); the two
        // 64-d halves are LBO = one atom column (16 KiB) apart.
        const uint32_t a_off = (k >> 2) * kAtom + (k & 3) * 32;
        mma_bf16(tO, umma_desc(sP + a_off, 16, 1024), umma_desc(vb + k * 2048, kAtom, 1024),
                 kIdescO, (j > 0 || k > 0) ? 1u : 0u);
      }
      mma_commit(bar_o);
    }
  }
  mbar_wait(bar_o, ph_o);
  fence_after();
  // O row / l -> bf16 -> out[token][head][d].
  {
    const float inv = l > 0.f ? 1.f / l : 0.f;
    __nv_bfloat16* orow = out + (static_cast<int64_t>(qt) * Hq + static_cast<int64_t>(h) * G + g) * kD;
#pragma unroll
    for (int c0 = 0; c0 < kD; c0 += 16) {
      float v[16];
      tmem_ld16(tO + lane_off + c0, v);  // warp-collective: every lane loads
      if (!row_valid) continue;
      uint4 w0, w1;
      w0.x = pack_bf16(v[0] * inv, v[1] * inv);
      w0.y = pack_bf16(v[2] * inv, v[3] * inv);
      w0.z = pack_bf16(v[4] * inv, v[5] * inv);
      w0.w = pack_bf16(v[6] * inv, v[7] * inv);
      w1.x = pack_bf16(v[8] * inv, v[9] * inv);
      w1.y = pack_bf16(v[10] * inv, v[11] * inv);
      w1.z = pack_bf16(v[12] * inv, v[13] * inv);
      w1.w = pack_bf16(v[14] * inv, v[15] * inv);
      *reinterpret_cast<uint4*>(orow + c0) = w0;
      *reinterpret_cast<uint4*>(orow + c0 + 8) = w1;
    }
  }
  fence_before();
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem) : "memory");
  }
}

}  // namespace

bool launch_prefill_attn(const void* pool_l, int64_t row_elems, const int32_t* slots,
                         const void* q, int q_pos0, int n_q, int Hq, int Hkv, int D, float scale,
                         void* out, cudaStream_t s) {
  if (D != kD || Hkv <= 0 || Hq != Hkv * 8 || n_q <= 0) return false;
  const int smem = kSmem + 1024;  // + alignment slack
  cudaFuncSetAttribute(k_prefill_attn_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const dim3 grid((n_q + kTokens - 1) / kTokens, Hkv);
  k_prefill_attn_tc<<<grid, kThreads, smem, s>>>(
      static_cast<const __nv_bfloat16*>(pool_l), row_elems, slots,
      static_cast<const __nv_bfloat16*>(q), q_pos0, n_q, Hq, Hkv, scale * 1.4426950408889634f,
      static_cast<__nv_bfloat16*>(out));
  return true;
}

}  // namespace mkv
