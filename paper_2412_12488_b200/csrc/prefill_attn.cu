// prefill_attn.cu — paged causal GQA prefill attention on tcgen05 (sm_100a).
//
// The decode engine's tail prefill in balanced PD (SURVEY
// §8(f) #2): queries at positions [q_begin, q_end) of a sequence attend to
// keys [0, pos] read from the KV pool through the sequence's HBM page table.
// Unlike decode, this is a dense contraction (e.g. 1,638 queries x 8,192
// keys x 64 heads at the 70B shape), so QK^T and PV run on the 5th-gen
// tensor cores.
//
// CTA = one KV head x two M=128 query tiles of 128 / G tokens x the G query
// heads sharing the KV head (G = 8 at Llama 70B: 16 tokens per tile; G = 4
// at Llama 8B: 32), warp-specialised:
//
//   warps 8, 10 producers of K and V: per 128-key tile, one TMA box per
//               (page chunk, 64-dim half) straight from the paged pool (a
//               page's rows of one head are a 2-D box of the pool's tensor
//               map; slots that are not consecutive fall back to one-row
//               boxes), into SWIZZLE_128B shared tiles; a 2-stage ring each.
//   warp 9      MMA issuer (one elected lane): S_i = Q_i K^T into TMEM at
//               N = 128, O_i += P_i V with P_i read from TMEM (A operand in
//               tensor memory).  S_i(j+1) goes right behind PV_i(j) into the
//               columns P_i(j) held, so the S-full barrier of tile j+1 also
//               proves PV_i(j) retired; the two query tiles ping-pong on the
//               tensor core.
//   warps 0-3   softmax of query tile 0, thread = TMEM lane = row;
//   warps 4-7   softmax of query tile 1.  Each reads its S row from TMEM,
//               masks (causal), keeps a running max (O rescaled in TMEM only
//               when the max grows by more than 2^8 — exact, since l and O
//               share the stale max), writes P = exp2(.) as packed bf16 over
//               the S columns in two 64-key halves (PV starts on the first
//               half while the second is exponentiated; scale/shift and row
//               sums as f32x2 pairs), and signals the MMA warp.
//
// TMEM (512 columns): query tile i owns S_i at [128 i, 128 i + 128) (P_i(j)
// overwrites its first 64 columns) and O_i at [256 + 128 i, 384 + 128 i).
//
// Measured alternatives, removed from the library after they lost on B200
// (profiles/r01/prefill_variant_ab.txt): 64-key tiles with two
// S slots per query tile (0.65 of peak on the tail vs 0.66-0.72), a 2-SM
// cta_group::2 pair (0.45-0.52), persistent CTAs (within +-4%), two softmax
// threads per row (equal), a key split over several CTAs + merge kernel
// (slower on every tail it was meant for); round 2: a CTA pair with
// 256-key N = 256 S tiles and separate P columns (0.61 vs 0.72 on full 8K
// causal, softmax-bound; profiles/r02/prefill_pair.txt).  This layout runs
// at the N = 128 tcgen05 dispatch rate (profiles/r02/mma_rate.txt).

// Shared-memory operands use the UMMA SWIZZLE_128B canonical layout (8-row x
// 128-byte atoms, 16-byte chunks XOR row, 1024-byte aligned); a 128-element
// row spans two atom columns.  K and V tiles are the same bytes ([key][d]): K
// is read as a K-major B operand, V as an MN-major one.  Keys past the end
// of the sequence in the last tile are zeroed in V (P is 0 there, but pool
// words of other pages may hold any bit pattern, NaN included).
//
// Numerics: bf16 inputs, fp32 accumulation in TMEM, P rounded to bf16 for
// the PV product; checked against fp32 PyTorch in
// tests/test_prefill_attention_gpu.py.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <type_traits>

#include "kernels.cuh"

namespace mkv {

namespace {

constexpr int kRows = 128;     // M of one query tile: (128 / G) tokens x G heads
constexpr int kQTiles = 2;     // query tiles per CTA
constexpr int kD = 128;        // head dim (K of S, N of PV)
constexpr int kAtom = kRows * 128;   // one 64-element atom column of a 128-row tile (16 KiB)
constexpr int kTile = 2 * kAtom;     // a [128][128] bf16 query tile (32 KiB)
constexpr int kBoxRows = 64;         // rows of the page-chunk TMA box (at most one page)
constexpr int kSoftmaxThreads = 256;
constexpr int kThreads = kSoftmaxThreads + 96;  // + K producer, MMA, V producer warps

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

// Instruction descriptor: D f32, A/B bf16, M=128, N=n, A K-major, B K- or MN-major.
__host__ __device__ constexpr uint32_t idesc_bf16(bool b_mn_major, int n = 128) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((b_mn_major ? 1u : 0u) << 16) |
         ((static_cast<uint32_t>(n) >> 3) << 17) | ((kRows >> 4) << 24);
}

// Warp-converged issue: one elected lane issues; descriptors are passed as
// (lo, hi) halves so a uniform base plus compile-time offsets stays in
// uniform registers (no per-instruction R2UR broadcast loop).
__device__ __forceinline__ void mma_ss_elect(uint32_t tmem_d, uint32_t a_lo, uint32_t b_lo,
                                             uint32_t hi, uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t.reg .b64 da, db;\n\t"
      "mov.b64 da, {%1, %3};\n\tmov.b64 db, {%2, %3};\n\t"
      "setp.ne.b32 p, %5, 0;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], da, db, %4, p;\n\t}\n" ::"r"(tmem_d),
      "r"(a_lo), "r"(b_lo), "r"(hi), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void mma_ts_elect(uint32_t tmem_d, uint32_t tmem_a, uint32_t b_lo,
                                             uint32_t b_hi, uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t.reg .b64 db;\n\t"
      "mov.b64 db, {%2, %3};\n\t"
      "setp.ne.b32 p, %5, 0;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], db, %4, p;\n\t}\n" ::"r"(tmem_d),
      "r"(tmem_a), "r"(b_lo), "r"(b_hi), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void commit_elect(uint32_t bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}\n" ::"r"(
          bar)
      : "memory");
}

// Low / high 32 bits of a SWIZZLE_128B descriptor (see umma_desc).
__host__ __device__ constexpr uint32_t desc_lo(uint32_t addr, uint32_t lbo) {
  return ((addr >> 4) & 0x3FFFu) | (((lbo >> 4) & 0x3FFFu) << 16);
}
__host__ __device__ constexpr uint32_t desc_hi(uint32_t sbo) {
  return ((sbo >> 4) & 0x3FFFu) | (1u << 14) | (2u << 29);
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

// Bounded wait: a completion that never arrives traps (the launch fails with
// an error) instead of hanging the GPU.
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

// TMA: a {64 elements, rows, 1} box of the pool's 3-D tensor map.
__device__ __forceinline__ void tma_load_3d(uint32_t dst, const CUtensorMap* map, int c0, int c1,
                                            int c2, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
      "%3, %4}], [%5];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(bar)
      : "memory");
}

// 16 columns, no wait (the caller issues tmem_wait_ld once for a batch).
__device__ __forceinline__ void tmem_ld16_nowait(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
      "%11, %12, %13, %14, %15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() {
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

__device__ __forceinline__ void tmem_st16_nowait(uint32_t taddr, const uint32_t* r) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
      "%11, %12, %13, %14, %15, %16};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
      "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]),
      "r"(r[15])
      : "memory");
}
__device__ __forceinline__ void tmem_wait_st() {
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}

// 2^x on the MUFU unit (ftz: no denormal fix-up instructions).
__device__ __forceinline__ float ex2_mufu(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// Packed f32x2 arithmetic (FFMA2 / FADD2 on sm_100): two lanes per instruction.
__device__ __forceinline__ uint64_t f2pack(float a, float b) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ void f2unpack(uint64_t v, float& a, float& b) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v));
}
__device__ __forceinline__ uint64_t ffma2(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t d;
  asm("fma.rn.ftz.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ uint64_t fadd2(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("add.rn.ftz.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ uint64_t fsub2(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("sub.rn.ftz.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}

// ex2_poly for a pair, the polynomial in packed f32x2 arithmetic.
__device__ __forceinline__ void ex2_poly2(float x0, float x1, float& y0, float& y1) {
  const uint64_t x = f2pack(fmaxf(x0, -125.f), fmaxf(x1, -125.f));
  const uint64_t K = f2pack(12582912.f, 12582912.f);
  const uint64_t t = fadd2(x, K);
  const uint64_t f = fsub2(x, fsub2(t, K));
  uint64_t p = ffma2(f, f2pack(0.0555041087f, 0.0555041087f), f2pack(0.240226507f, 0.240226507f));
  p = ffma2(p, f, f2pack(0.693147181f, 0.693147181f));
  p = ffma2(p, f, f2pack(1.f, 1.f));
  float p0, p1, t0, t1;
  f2unpack(p, p0, p1);
  f2unpack(t, t0, t1);
  y0 = __int_as_float(__float_as_int(p0) + (__float_as_int(t0) << 23));
  y1 = __int_as_float(__float_as_int(p1) + (__float_as_int(t1) << 23));
}

__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}

struct PrefillArgs {
  const int32_t* slots;       // sequence page table: slot of each position
  const __nv_bfloat16* q;     // [n_q][Hq][128]
  __nv_bfloat16* out;         // [n_q][Hq][128]
  int layer, page_size, q_pos0, n_q, Hq, Hkv, n_blocks;
  int tile_tokens;            // query tokens per M = 128 tile: 128 / (Hq / Hkv)
  float scale_log2;
  int pool_rows;              // rows of the pool tensor maps (an OOB row loads zeros)
#if defined(PF_TRACE) || defined(PF_PROF)
  unsigned long long* trace;  // debug timeline of CTA (0, 0) / per-warp phase sums
#endif
};

// Debug timeline (build with -DPF_TRACE): plain stores of clock64() into a
// slot fixed by the event code (type, tile, j < 256), CTA (0, 0) only.
#ifdef PF_TRACE
#define PF_EV(code)                                                              \
  do {                                                                           \
    if (blockIdx.x == 0 && blockIdx.y == 0) a.trace[(code) & 0xffff] = clock64(); \
  } while (0)
#else
#define PF_EV(code) do {} while (0)
#endif

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return static_cast<EncodeTiledFn>(nullptr);
    return reinterpret_cast<EncodeTiledFn>(p);
  }();
  return fn;
}


// ===========================================================================
// Layout constants: 128-key KV tiles and ONE S slot per query tile (TMEM: S_i
// at 128 i, O_i at 256 + 128 i).  The S MMAs run at N = 128, which halves
// the shared-memory reads of Q per key against 64-key tiles (A is re-read
// per MMA).  S_i(j+1) is issued right behind PV_i(j) into the columns P_i(j)
// occupied (MMAs of one thread run in order), so the S-full barrier of tile
// j+1 also proves PV_i(j) retired and the O rescale needs no separate wait;
// the two query tiles ping-pong: one tile's softmax runs while the tensor
// core works on the other's PV and S.
namespace p3 {
constexpr int kKeys = 128;
constexpr int kPer = kKeys / 32;          // tile positions per producer lane
constexpr int kKvAtom = kKeys * 128;      // atom column of a [128][128] K or V tile (16 KiB)
constexpr int kKvTile = 2 * kKvAtom;      // 32 KiB
#ifndef PF3_K_STAGES
#define PF3_K_STAGES 2
#endif
#ifndef PF3_V_STAGES
#define PF3_V_STAGES 2
#endif
#ifndef PF3_POLY_EVERY
#define PF3_POLY_EVERY 4  // every 4th exponential pair on the FMA pipe (polynomial)
#endif
constexpr int kStagesK = PF3_K_STAGES, kStagesV = PF3_V_STAGES;
constexpr int kOffQ = 0;
constexpr int kOffK = kOffQ + kQTiles * kTile;
constexpr int kOffV = kOffK + kStagesK * kKvTile;
constexpr int kOffBar = kOffV + kStagesV * kKvTile;
constexpr int kSmem = kOffBar + 512;
enum : int {
  kBarQ = 0,
  kBarKFull = 1,
  kBarVFull = kBarKFull + kStagesK,
  kBarKEmpty = kBarVFull + kStagesV,
  kBarVEmpty = kBarKEmpty + kStagesK,
  kBarSFull = kBarVEmpty + kStagesV,  // +tile
  kBarPFull = kBarSFull + 2,          // +tile (count 128)
  kBarODone = kBarPFull + 2,          // +tile
  kBarPHalf = kBarODone + 2,          // +tile: first half of P_i(j)
  kBarCount = kBarPHalf + 2,
};
static_assert(kBarCount * 8 + 8 <= 512, "barrier area");
static_assert(kSmem + 1024 <= 227 * 1024, "shared memory");
}  // namespace p3

__global__ void __launch_bounds__(kThreads, 1)
    k_prefill_attn_k128(const __grid_constant__ CUtensorMap pool_map,
                        const __grid_constant__ CUtensorMap row_map, const PrefillArgs a) {
  using namespace p3;
  constexpr int kKeys = p3::kKeys, kKvAtom = p3::kKvAtom, kKvTile = p3::kKvTile;
  constexpr int kOffQ = p3::kOffQ, kOffK = p3::kOffK, kOffV = p3::kOffV, kOffBar = p3::kOffBar;
  constexpr int kBarQ = p3::kBarQ, kBarKFull = p3::kBarKFull, kBarVFull = p3::kBarVFull;
  constexpr int kBarKEmpty = p3::kBarKEmpty, kBarVEmpty = p3::kBarVEmpty;
  constexpr int kBarSFull = p3::kBarSFull, kBarPFull = p3::kBarPFull, kBarODone = p3::kBarODone;
  constexpr int kBarPHalf = p3::kBarPHalf;
  constexpr int kBarCount = p3::kBarCount;
  constexpr int kStagesV = p3::kStagesV;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // Heaviest (latest) query blocks first.
  const int qb = a.n_blocks - 1 - static_cast<int>(blockIdx.x);
  const int h = blockIdx.y;
  const uint32_t sQ = smem_u32(smem + kOffQ), sK = smem_u32(smem + kOffK);
  const uint32_t sV = smem_u32(smem + kOffV), bars = smem_u32(smem + kOffBar);
  auto bar = [&](int i) { return bars + 8u * static_cast<uint32_t>(i); };
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + kOffBar + 8 * kBarCount);

  const int tok_first = qb * kQTiles * a.tile_tokens;
  const int tok_last = min(a.n_q, tok_first + kQTiles * a.tile_tokens) - 1;
  const int n_keys = a.q_pos0 + tok_last + 1;
  const int n_tiles = (n_keys + kKeys - 1) / kKeys;
  // This CTA's key tiles [t_begin, t_begin + n_local): all of them.
  const int t_begin = 0;
  const int n_local = n_tiles;

  if (warp == 9) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                     smem_u32(tmem_slot))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (tid == kSoftmaxThreads) {
    mbar_init(bar(kBarQ), kSoftmaxThreads);
    for (int s = 0; s < kStagesK; ++s) {
      mbar_init(bar(kBarKFull + s), 1);
      mbar_init(bar(kBarKEmpty + s), 1);
    }
    for (int s = 0; s < kStagesV; ++s) {
      mbar_init(bar(kBarVFull + s), 1);
      mbar_init(bar(kBarVEmpty + s), 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(bar(kBarSFull + i), 1);
      mbar_init(bar(kBarPFull + i), kRows);
      mbar_init(bar(kBarPHalf + i), kRows);
      mbar_init(bar(kBarODone + i), 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&pool_map))
                 : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&row_map))
                 : "memory");
  }
  fence_before();
  __syncthreads();
  fence_after();
  constexpr uint32_t tmem = 0;
  if (tid == 0 && *tmem_slot != 0u) __trap();

  if (warp == 8 || warp == 10) {
    // ---------------- producers: K (warp 8) / V (warp 10), lane l owns
    // positions kPer*l .. kPer*l + kPer - 1 of the tile ----------------
    const int C = min(a.page_size, kBoxRows), lanes_per_chunk = C / kPer;
    const uint32_t chunk_mask = lanes_per_chunk >= 32 ? 0xffffffffu : ((1u << lanes_per_chunk) - 1u);
    const int my_chunk_lane0 = lane - lane % lanes_per_chunk;
    const int op = warp == 8 ? 0 : 1;
    const int nst = op == 0 ? kStagesK : kStagesV;
    const int col = op == 0 ? h * kD : (a.Hkv + h) * kD;
    for (int jj = 0; jj < n_local; ++jj) {
      const int j = t_begin + jj;
      const int s = jj % nst;
      const int p0 = j * kKeys + lane * kPer;
      int sl[kPer];
#pragma unroll
      for (int t = 0; t < kPer; ++t) sl[t] = p0 + t < n_keys ? __ldg(a.slots + p0 + t) : -1;
      const int prev_last = __shfl_up_sync(0xffffffffu, sl[kPer - 1], 1);
      bool ok = true;
#pragma unroll
      for (int t = 0; t < kPer; ++t) {
        const bool chunk_start = ((lane * kPer + t) % C) == 0;
        const int prev = t > 0 ? sl[t - 1] : prev_last;
        if (!chunk_start && sl[t] >= 0) ok = ok && sl[t] == prev + 1;
      }
      const uint32_t ballot = __ballot_sync(0xffffffffu, ok);
      const bool contiguous = ((ballot >> my_chunk_lane0) & chunk_mask) == chunk_mask;
      const int chunk_row = __shfl_sync(0xffffffffu, sl[0], my_chunk_lane0);
      const uint32_t base = (op == 0 ? sK : sV) + s * kKvTile;
      const uint32_t full = bar((op == 0 ? kBarKFull : kBarVFull) + s);
      if (lane == 0) {
        if (jj >= nst) mbar_wait(bar((op == 0 ? kBarKEmpty : kBarVEmpty) + s), ((jj / nst) + 1) & 1);
        PF_EV((op == 0 ? 0xA00 : 0xC00) | (j & 0xff));
        mbar_expect_tx(full, kKvTile);
      }
      __syncwarp();
      if (contiguous) {
        if (lane == my_chunk_lane0) {
          const uint32_t dst = base + (lane * kPer) * 128;
          const int row = chunk_row >= 0 ? chunk_row : 0;
          tma_load_3d(dst, &pool_map, col, row, a.layer, full);
          tma_load_3d(dst + kKvAtom, &pool_map, col + 64, row, a.layer, full);
        }
      } else {
#pragma unroll
        for (int t = 0; t < kPer; ++t) {
          const uint32_t dst = base + (lane * kPer + t) * 128;
          const int row = sl[t] >= 0 ? sl[t] : 0;
          tma_load_3d(dst, &row_map, col, row, a.layer, full);
          tma_load_3d(dst + kKvAtom, &row_map, col + 64, row, a.layer, full);
        }
      }
    }
  } else if (warp == 9) {
    // ---------------- MMA issuer ----------------
    //   prologue  S0(0) S1(0)
    //   tile j    [P0(j)] PV0(j) S0(j+1) [P1(j)] PV1(j) S1(j+1)
    constexpr uint32_t kIdescS = idesc_bf16(false, kKeys), kIdescO = idesc_bf16(true, kD);
    constexpr uint32_t kHi = desc_hi(1024);
    auto tS = [&](int i) { return tmem + i * 128; };
    auto tO = [&](int i) { return tmem + 256 + i * 128; };
    const uint32_t q_lo = desc_lo(sQ, 16), k_lo = desc_lo(sK, 16), v_lo = desc_lo(sV, kKvAtom);
    auto issue_s = [&](int i, int j) {
      const uint32_t a0 = q_lo + ((i * kTile) >> 4), b0 = k_lo + (((j % kStagesK) * kKvTile) >> 4);
#pragma unroll
      for (int k = 0; k < kD / 16; ++k) {
        const uint32_t ao = ((k >> 2) * kAtom + (k & 3) * 32) >> 4;
        const uint32_t bo = ((k >> 2) * kKvAtom + (k & 3) * 32) >> 4;
        mma_ss_elect(tS(i), a0 + ao, b0 + bo, kHi, kIdescS, k > 0 ? 1u : 0u);
      }
      commit_elect(bar(kBarSFull + i));
    };
    auto issue_pv = [&](int i, int j) {
      const uint32_t b0 = v_lo + (((j % kStagesV) * kKvTile) >> 4);
      mbar_wait(bar(kBarPHalf + i), j & 1);  // P_i(j) keys [0, 64) and O_i rescaled
      fence_after();
      if (lane == 0) PF_EV(0xE00 | (i << 8) | (j & 0xff));
#pragma unroll
      for (int k = 0; k < kKeys / 32; ++k)
        mma_ts_elect(tO(i), tS(i) + k * 8, b0 + ((k * 2048) >> 4), kHi, kIdescO,
                     (j > 0 || k > 0) ? 1u : 0u);
      mbar_wait(bar(kBarPFull + i), j & 1);  // keys [64, 128)
      fence_after();
#pragma unroll
      for (int k = kKeys / 32; k < kKeys / 16; ++k)
        mma_ts_elect(tO(i), tS(i) + k * 8, b0 + ((k * 2048) >> 4), kHi, kIdescO, 1u);
    };
    auto zero_tail = [&](int j, int jj) {
      const int valid = n_keys - j * kKeys;
      if (valid >= kKeys) return;
      uint8_t* vb = smem + kOffV + (jj % kStagesV) * kKvTile;
      for (int e = lane; e < (kKeys - valid) * 16; e += 32) {
        const int r = valid + (e >> 4), c = e & 15;
        *reinterpret_cast<uint4*>(vb + (c >> 3) * kKvAtom + r * 128 + (c & 7) * 16) =
            make_uint4(0, 0, 0, 0);
      }
      fence_proxy_async();
      __syncwarp();
    };
    mbar_wait(bar(kBarQ), 0);
    mbar_wait(bar(kBarKFull), 0);
    fence_after();
    issue_s(0, 0);
    issue_s(1, 0);
    commit_elect(bar(kBarKEmpty));
    for (int j = 0; j < n_local; ++j) {  // local tile index (stages, parities)
      const int sv = j % kStagesV;
      mbar_wait(bar(kBarVFull + sv), (j / kStagesV) & 1);
      if (t_begin + j == n_tiles - 1) zero_tail(t_begin + j, j);
      const bool next = j + 1 < n_local;
      const int sk = (j + 1) % kStagesK;
      if (next) mbar_wait(bar(kBarKFull + sk), ((j + 1) / kStagesK) & 1);
      fence_after();
      if (lane == 0) PF_EV(0x100 | (j & 0xff));
      for (int i = 0; i < kQTiles; ++i) {
        issue_pv(i, j);
        if (lane == 0) PF_EV(0x200 | (i << 8) | (j & 0xff));
        if (!next) commit_elect(bar(kBarODone + i));
        if (next) issue_s(i, j + 1);
      }
      commit_elect(bar(kBarVEmpty + sv));
      if (next) commit_elect(bar(kBarKEmpty + sk));
    }
  } else {
    // ---------------- softmax warpgroups ----------------
    const int i = warp >> 2;
    const int r = tid & (kRows - 1);
    const int G = a.Hq / a.Hkv;
    const int tok = tok_first + i * a.tile_tokens + r / G, g = r % G;
    const bool row_valid = tok < a.n_q;
    const int q_pos = a.q_pos0 + tok;
    const int tile_min_pos = a.q_pos0 + tok_first + i * a.tile_tokens;
    const uint32_t lane_off = static_cast<uint32_t>((warp & 3) * 32) << 16;
    const uint32_t tS = tmem + i * 128 + lane_off, tO = tmem + 256 + i * 128 + lane_off;
    {
      const __nv_bfloat16* qrow =
          a.q + (static_cast<int64_t>(tok) * a.Hq + static_cast<int64_t>(h) * G + g) * kD;
      const uint32_t qa = sQ + i * kTile;
#pragma unroll
      for (int c = 0; c < 16; ++c) cp_async16(qa + sw128(r, c), qrow + c * 8, row_valid);
      asm volatile("cp.async.commit_group;" ::: "memory");
      asm volatile("cp.async.wait_group 0;" ::: "memory");
      fence_proxy_async();
      mbar_arrive(bar(kBarQ));
    }
    const float sl2 = a.scale_log2;
    float m = -INFINITY, l = 0.f;
#ifdef PF_PROF
    long long prof[6] = {0, 0, 0, 0, 0, 0};  // wait S, load S, max, P half 1, P half 2 + stores, total
    long long tp0 = clock64(), tp1;
#define PF_LAP(k) do { tp1 = clock64(); prof[k] += tp1 - tp0; tp0 = tp1; } while (0)
#else
#define PF_LAP(k) do {} while (0)
#endif
    for (int j = 0; j < n_local; ++j) {  // local tile index (parities, rescale)
      if ((warp & 3) == 0 && lane == 0) PF_EV(0x400 | (i << 8) | (j & 0xff));
      mbar_wait(bar(kBarSFull + i), j & 1);
      fence_after();
      PF_LAP(0);
      if ((warp & 3) == 0 && lane == 0) PF_EV(0x600 | (i << 8) | (j & 0xff));
      uint32_t sr[kKeys];
#pragma unroll
      for (int c0 = 0; c0 < kKeys; c0 += 16) tmem_ld16_nowait(tS + c0, sr + c0);
      tmem_wait_ld();
      PF_LAP(1);
      const int key0 = (t_begin + j) * kKeys;
      const bool need_mask =
          __any_sync(0xffffffffu, key0 + kKeys - 1 > tile_min_pos || !row_valid);
      if (need_mask) {
        const int lim = row_valid ? q_pos - key0 : -1;
#pragma unroll
        for (int c = 0; c < kKeys; ++c) sr[c] = c > lim ? __float_as_uint(-INFINITY) : sr[c];
      }
      float mx[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
      for (int c = 0; c < kKeys; c += 8) {
#pragma unroll
        for (int k = 0; k < 4; ++k)
          mx[k] = fmaxf(mx[k], fmaxf(__uint_as_float(sr[c + 2 * k]), __uint_as_float(sr[c + 2 * k + 1])));
      }
      const float rmax = fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3]));
      PF_LAP(2);
      const float tmax = rmax * sl2;
      const bool bump = tmax > m + 8.f;
      const float m_new = bump ? tmax : m;
      const float alpha = (bump && m != -INFINITY) ? ex2_mufu(m - m_new) : 1.f;
      const float neg_m = m_new == -INFINITY ? 0.f : -m_new;
      const uint64_t sc2 = f2pack(sl2, sl2), nm2 = f2pack(neg_m, neg_m);
      uint64_t acc[2] = {0ull, 0ull};
      // P in two halves of 64 keys: the MMA warp starts PV on keys [0, 64)
      // while the second half's exponentials run (shorter softmax -> PV
      // chain per tile).
      auto make_p = [&](auto poly, auto lo) {
#pragma unroll
        for (int c = decltype(lo)::value; c < decltype(lo)::value + kKeys / 2; c += 2) {
          float x0, x1, p0, p1;
          f2unpack(ffma2(f2pack(__uint_as_float(sr[c]), __uint_as_float(sr[c + 1])), sc2, nm2),
                   x0, x1);
          if (decltype(poly)::value && PF3_POLY_EVERY > 0 &&
              ((c >> 1) % (PF3_POLY_EVERY > 0 ? PF3_POLY_EVERY : 1)) == PF3_POLY_EVERY - 1) {
            ex2_poly2(x0, x1, p0, p1);
          } else {
            p0 = ex2_mufu(x0);
            p1 = ex2_mufu(x1);
          }
          acc[(c >> 1) & 1] = fadd2(acc[(c >> 1) & 1], f2pack(p0, p1));
          sr[c / 2] = pack_bf16(p0, p1);
        }
      };
      using Lo = std::integral_constant<int, 0>;
      using Hi = std::integral_constant<int, kKeys / 2>;
      if (need_mask) make_p(std::false_type{}, Lo{});
      else make_p(std::true_type{}, Lo{});
      // S_i(j) landed behind PV_i(j-1) (same issuing thread, in order), so
      // O_i is stable here: rescale without a further wait, before PV_i(j).
      if (j > 0 && __any_sync(0xffffffffu, alpha != 1.f)) {
#pragma unroll
        for (int c0 = 0; c0 < kD; c0 += 32) {
          uint32_t o[32];
          tmem_ld16_nowait(tO + c0, o);
          tmem_ld16_nowait(tO + c0 + 16, o + 16);
          tmem_wait_ld();
#pragma unroll
          for (int k = 0; k < 32; ++k) o[k] = __float_as_uint(__uint_as_float(o[k]) * alpha);
          tmem_st16_nowait(tO + c0, o);
          tmem_st16_nowait(tO + c0 + 16, o + 16);
        }
      }
#pragma unroll
      for (int c0 = 0; c0 < kKeys / 4; c0 += 16) tmem_st16_nowait(tS + c0, sr + c0);
      tmem_wait_st();
      fence_before();
      mbar_arrive(bar(kBarPHalf + i));
      PF_LAP(3);
      if (need_mask) make_p(std::false_type{}, Hi{});
      else make_p(std::true_type{}, Hi{});
      float ps[4];
      f2unpack(acc[0], ps[0], ps[1]);
      f2unpack(acc[1], ps[2], ps[3]);
      const float psum = (ps[0] + ps[1]) + (ps[2] + ps[3]);
#pragma unroll
      for (int c0 = kKeys / 4; c0 < kKeys / 2; c0 += 16) tmem_st16_nowait(tS + c0, sr + c0);
      tmem_wait_st();
      fence_before();
      mbar_arrive(bar(kBarPFull + i));
      PF_LAP(4);
      if ((warp & 3) == 0 && lane == 0) PF_EV(0x800 | (i << 8) | (j & 0xff));
      if (lane == 0) PF_EV(0x4000 | (warp << 8) | (j & 0xff));
      l = l * alpha + psum;
      m = m_new;
    }
#ifdef PF_PROF
    if (lane == 0 && blockIdx.x == 0) {  // per warp of the heaviest CTA of each head
      unsigned long long* o = a.trace + (blockIdx.y * 8 + warp) * 8;
      for (int k = 0; k < 5; ++k) o[k] = static_cast<unsigned long long>(prof[k]);
      o[5] = static_cast<unsigned long long>(n_tiles);
    }
#endif
#undef PF_LAP
    mbar_wait(bar(kBarODone + i), 0);
    fence_after();
    const float inv = l > 0.f ? 1.f / l : 0.f;
    __nv_bfloat16* orow =
        a.out + (static_cast<int64_t>(tok) * a.Hq + static_cast<int64_t>(h) * G + g) * kD;
#pragma unroll
    for (int c0 = 0; c0 < kD; c0 += 32) {
      uint32_t o[32];
      tmem_ld16_nowait(tO + c0, o);
      tmem_ld16_nowait(tO + c0 + 16, o + 16);
      tmem_wait_ld();
      if (row_valid) {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          auto pk = [&](int e) {
            return pack_bf16(__uint_as_float(o[8 * k + e]) * inv,
                             __uint_as_float(o[8 * k + e + 1]) * inv);
          };
          reinterpret_cast<uint4*>(orow + c0)[k] = make_uint4(pk(0), pk(2), pk(4), pk(6));
        }
      }
    }
  }
  fence_before();
  __syncthreads();
  if (warp == 9) {
    fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
  }
}

}  // namespace

bool make_pool_tensor_map(void* pool, int64_t layers, int64_t rows, int64_t row_u64,
                          int box_rows, PoolTensorMap* out) {
  static_assert(sizeof(CUtensorMap) <= sizeof(out->bytes), "tensor map size");
  EncodeTiledFn fn = encode_fn();
  if (fn == nullptr) return false;
  CUtensorMap map;
  const cuuint64_t dims[3] = {static_cast<cuuint64_t>(row_u64 * 4), static_cast<cuuint64_t>(rows),
                              static_cast<cuuint64_t>(layers)};
  const cuuint64_t strides[2] = {static_cast<cuuint64_t>(row_u64 * 8),
                                 static_cast<cuuint64_t>(rows * row_u64 * 8)};
  const cuuint32_t box[3] = {64, static_cast<cuuint32_t>(box_rows), 1};
  const cuuint32_t estr[3] = {1, 1, 1};
  const CUresult r = fn(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, pool, dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return false;
  std::memcpy(out->bytes, &map, sizeof(map));
  return true;
}

bool prefill_attn_supported(int page_size, int Hq, int Hkv, int D) {
  const bool pow2 = page_size > 0 && (page_size & (page_size - 1)) == 0;
  // Any GQA group that divides a 128-row tile (Llama 70B: 8, Llama 8B: 4, MHA: 1).
  const bool group_ok = Hkv >= 1 && Hq % Hkv == 0 && Hq / Hkv <= kRows && kRows % (Hq / Hkv) == 0;
  return D == kD && group_ok && pow2 && page_size >= 8 && page_size <= 1024;
}

int prefill_attn_box_rows(int page_size) { return page_size < kBoxRows ? page_size : kBoxRows; }

int launch_prefill_attn(const PoolTensorMap& page_map, const PoolTensorMap& row_map, int layer,
                         int page_size, int64_t pool_rows, const int32_t* slots, const void* q,
                         int q_pos0, int n_q, int Hq, int Hkv, int D, float scale, void* out,
                         cudaStream_t s) {
  if (!prefill_attn_supported(page_size, Hq, Hkv, D) || n_q <= 0) return 0;
  // Shared-memory attributes are set per device by preload_prefill_attn_kernels().
  PrefillArgs a;
  a.slots = slots;
  a.q = static_cast<const __nv_bfloat16*>(q);
  a.out = static_cast<__nv_bfloat16*>(out);
  a.layer = layer;
  a.page_size = page_size;
  a.q_pos0 = q_pos0;
  a.n_q = n_q;
  a.Hq = Hq;
  a.Hkv = Hkv;
  a.tile_tokens = kRows / (Hq / Hkv);  // 16 tokens at G = 8, 32 at G = 4
  a.n_blocks = (n_q + kQTiles * a.tile_tokens - 1) / (kQTiles * a.tile_tokens);
  a.scale_log2 = scale * 1.4426950408889634f;
  a.pool_rows = static_cast<int>(pool_rows);
  const int launches = 1;
  CUtensorMap m, mr;
  std::memcpy(&m, page_map.bytes, sizeof(m));
  std::memcpy(&mr, row_map.bytes, sizeof(mr));
#if defined(PF_TRACE) || defined(PF_PROF)
  unsigned long long* tr = nullptr;
  cudaMalloc(&tr, 65536 * sizeof(unsigned long long));
  cudaMemset(tr, 0, 65536 * sizeof(unsigned long long));
  a.trace = tr;
#endif
  const dim3 grid(a.n_blocks, Hkv);
  k_prefill_attn_k128<<<grid, kThreads, p3::kSmem + 1024, s>>>(m, mr, a);
#ifdef PF_PROF
  cudaDeviceSynchronize();
  {
    static unsigned long long hp[8 * 8 * 8];
    cudaMemcpy(hp, tr, sizeof(hp), cudaMemcpyDeviceToHost);
    cudaFree(tr);
    if (FILE* f = std::fopen("gpurun_out/pf_prof.txt", "w")) {
      for (int w = 0; w < 64; ++w)
        if (hp[w * 8 + 5])
          std::fprintf(f, "head %d warp %d tiles %llu wait %llu load %llu max %llu p1 %llu p2 %llu\n",
                       w / 8, w % 8, hp[w * 8 + 5], hp[w * 8], hp[w * 8 + 1], hp[w * 8 + 2],
                       hp[w * 8 + 3], hp[w * 8 + 4]);
      std::fclose(f);
    }
  }
#endif
#ifdef PF_TRACE
  cudaDeviceSynchronize();
  static unsigned long long h[65536];
  cudaMemcpy(h, tr, sizeof(h), cudaMemcpyDeviceToHost);
  cudaFree(tr);
  if (FILE* f = std::fopen("gpurun_out/pf_trace.txt", "w")) {
    for (int i = 0; i < 65536; ++i)
      if (h[i]) std::fprintf(f, "%llu %x\n", h[i], i);
    std::fclose(f);
  }
#endif
  return launches;
}


void preload_prefill_attn_kernels() {
  // Per device (called once per device at cache creation): the kernel's
  // dynamic shared memory above 48 KiB.
  cudaFuncSetAttribute(k_prefill_attn_k128, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       p3::kSmem + 1024);
  cudaFuncAttributes a;
  cudaFuncGetAttributes(&a, k_prefill_attn_k128);
}

}  // namespace mkv
