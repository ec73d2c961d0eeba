// prefill_attn.cu — paged causal GQA prefill attention on tcgen05 (sm_100a).
//
// The decode engine's tail prefill in balanced PD (SURVEY
// §8(f) #2): queries at positions [q_begin, q_end) of a sequence attend to
// keys [0, pos] read from the KV pool through the sequence's HBM page table.
// Unlike decode, this is a dense contraction (e.g. 1,638 queries x 8,192
// keys x 64 heads at the 70B shape), so QK^T and PV run on the 5th-gen
// tensor cores.
//
// CTA = one KV head x 32 query tokens, as two M=128 query tiles (16 tokens x
// the 8 query heads sharing the KV head), warp-specialised:
//
//   warp 8      producer: per 64-key tile, one TMA box per (page, 64-dim
//               half) of K and of V straight from the paged pool (a page's P
//               rows of one head are a 2-D box of the pool's tensor map), into
//               SWIZZLE_128B shared tiles; a 4-stage ring each for K and V.
//   warp 9      MMA issuer (one elected lane): S_i = Q_i K^T into TMEM,
//               O_i += P_i V with P_i read from TMEM (A operand in tensor
//               memory).  Per KV tile j and query tile i: PV_i(j) as soon as
//               P_i(j) is ready, then S_i(j+2) into the S slot P_i(j) frees,
//               so S_i(j+1) is always computed while softmax_i(j) runs and
//               the two query tiles never wait on each other.
//   warps 0-3   softmax of query tile 0, thread = TMEM lane = row;
//   warps 4-7   softmax of query tile 1.  Each reads its S row from TMEM,
//               masks (causal), keeps a running max (O rescaled in TMEM only
//               when the max grows by more than 2^8 — exact, since l and O
//               share the stale max; warps with nothing to rescale do not
//               wait for the previous PV), writes P = exp2(.) as packed bf16
//               over the S columns (scale/shift and row sums as f32x2 pairs),
//               and signals the MMA warp.  S-full and P-full barriers are per
//               (query tile, S slot), so a warp running one tile ahead of its
//               warpgroup cannot land in the wrong phase.
//
// TMEM (512 columns): query tile i owns [128 i, 128 i + 128) as two 64-column
// S slots (KV tile j uses slot j & 1; P_i(j) overwrites the slot's first 32
// columns), O_i at [256 + 128 i, 384 + 128 i).
//
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

constexpr int kRows = 128;     // M of one query tile: 16 tokens x 8 heads
constexpr int kTokens = 16;    // query tokens per query tile
constexpr int kQTiles = 2;     // query tiles per CTA
constexpr int kKeys = 64;      // keys per KV tile (N of S, K of PV)
constexpr int kD = 128;        // head dim (K of S, N of PV)
constexpr int kAtom = kRows * 128;   // one 64-element atom column of a 128-row tile (16 KiB)
constexpr int kTile = 2 * kAtom;     // a [128][128] bf16 query tile (32 KiB)
constexpr int kKvAtom = kKeys * 128; // atom column of a [64][128] K or V tile (8 KiB)
constexpr int kKvTile = 2 * kKvAtom; // 16 KiB
constexpr int kStages = 4;           // K ring depth
#ifndef PF_V_STAGES
#define PF_V_STAGES 4  // 4, 5, 6 measured equal
#endif
constexpr int kStagesV = PF_V_STAGES; // V ring depth (V is released last: PV retires it)
constexpr int kSoftmaxThreads = 256;
constexpr int kThreads = kSoftmaxThreads + 96;  // + K producer, MMA, V producer warps

// Shared memory map (bytes; tiles 1024-aligned).
constexpr int kOffQ = 0;                             // 2 query tiles
constexpr int kOffK = kOffQ + kQTiles * kTile;       // kStages K tiles
constexpr int kOffV = kOffK + kStages * kKvTile;     // kStagesV V tiles
constexpr int kOffBar = kOffV + kStagesV * kKvTile;  // mbarriers + tmem base
constexpr int kSmem = kOffBar + 512;

// mbarrier slots (8 bytes each) from kOffBar.
enum : int {
  kBarQ = 0,                         // softmax threads loaded Q (count 256)
  kBarKFull = 1,                     // +stage: TMA bytes landed
  kBarVFull = kBarKFull + kStages,
  kBarKEmpty = kBarVFull + kStagesV, // +stage: MMAs reading it retired
  kBarVEmpty = kBarKEmpty + kStages,
  kBarSFull = kBarVEmpty + kStagesV,  // +2*tile+slot: S_i(j) ready in TMEM slot j&1
                                     // (per slot, so S_i(j+1) landing early cannot
                                     // push a barrier two phases past its waiter)
  kBarPFull = kBarSFull + 4,         // +2*tile+slot: P_i(j) written, O_i rescaled (count
                                     // 128).  Per slot: a warp that skips the O wait may
                                     // run one tile ahead of its warpgroup, and its
                                     // P_i(j+1) arrival must not land in phase j.
  kBarPVDone = kBarPFull + 4,        // +tile: PV_i(j) retired (O_i stable)
  kBarODone = kBarPVDone + 2,        // +tile: the last PV_i retired (single phase)
  kBarCount = kBarODone + 2,
};
static_assert(kBarCount * 8 + 8 <= 512, "barrier area");
static_assert(kSmem + 1024 <= 227 * 1024, "shared memory");

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

// Instruction descriptor: D f32, A/B bf16, M=128, N=n, A K-major, B K- or MN-major.
__host__ __device__ constexpr uint32_t idesc_bf16(bool b_mn_major, int n = 128) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((b_mn_major ? 1u : 0u) << 16) |
         ((static_cast<uint32_t>(n) >> 3) << 17) | ((kRows >> 4) << 24);
}

// D[tmem] (+)= A[smem] * B[smem]
__device__ __forceinline__ void mma_bf16(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(accumulate));
}

// D[tmem] (+)= A[tmem] * B[smem]
__device__ __forceinline__ void mma_bf16_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t b,
                                            uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "r"(tmem_a), "l"(b), "r"(idesc), "r"(accumulate));
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

__device__ __forceinline__ void mma_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar)
               : "memory");
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

// 16 consecutive fp32 columns of this thread's TMEM lane (waits).
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

__device__ __forceinline__ void tmem_st16(uint32_t taddr, const float (&v)[16]) {
  uint32_t r[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) r[i] = __float_as_uint(v[i]);
  tmem_st16_nowait(taddr, r);
  tmem_wait_st();
}

// 2^x on the MUFU unit (ftz: no denormal fix-up instructions).
__device__ __forceinline__ float ex2_mufu(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// 2^x on the FMA pipe: round-to-nearest split x = j + f, f in [-0.5, 0.5],
// 2^f by its degree-3 Taylor polynomial (relative error < 7e-4, below
// bf16's 2^-9 rounding of P), 2^j added to the exponent.  x is clamped at
// -125 (2^-125 ~ 0 next to the row maximum's 1); callers use it only for
// unmasked scores (x <= 8).
__device__ __forceinline__ float ex2_poly(float x) {
  x = fmaxf(x, -125.f);
  const float t = x + 12582912.f;  // 1.5 * 2^23: low mantissa bits = round(x)
  const float f = x - (t - 12582912.f);
  float p = fmaf(f, 0.0555041087f, 0.240226507f);
  p = fmaf(p, f, 0.693147181f);
  p = fmaf(p, f, 1.f);
  return __int_as_float(__float_as_int(p) + (__float_as_int(t) << 23));
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
  float scale_log2;
  int pool_rows;              // rows of the pool tensor maps (an OOB row loads zeros)
  // Key split (k_prefill_attn_k128 only): n_split CTAs per work item, each
  // over an equal share of its key tiles, writing normalised fp32 partials
  // [split][n_q][Hq][128] and (max, sum) pairs that k_prefill_combine merges.
  int n_split;
  float* part_o;
  float2* part_ml;
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

__global__ void __launch_bounds__(kThreads, 1)
    k_prefill_attn_tc(const __grid_constant__ CUtensorMap pool_map,
                      const __grid_constant__ CUtensorMap row_map, const PrefillArgs a) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // Heaviest (latest) query blocks first: causal work grows with position.
  const int qb = a.n_blocks - 1 - static_cast<int>(blockIdx.x);
  const int h = blockIdx.y;
  const uint32_t sQ = smem_u32(smem + kOffQ), sK = smem_u32(smem + kOffK);
  const uint32_t sV = smem_u32(smem + kOffV), bars = smem_u32(smem + kOffBar);
  auto bar = [&](int i) { return bars + 8u * static_cast<uint32_t>(i); };
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + kOffBar + 8 * kBarCount);

  const int tok_first = qb * kQTiles * kTokens;
  const int tok_last = min(a.n_q, tok_first + kQTiles * kTokens) - 1;
  const int n_keys = a.q_pos0 + tok_last + 1;  // keys [0, n_keys) needed by this CTA
  const int n_tiles = (n_keys + kKeys - 1) / kKeys;

  if (warp == 9) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                     smem_u32(tmem_slot))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (tid == kSoftmaxThreads) {
    mbar_init(bar(kBarQ), kSoftmaxThreads);
    for (int s = 0; s < kStages; ++s) {
      mbar_init(bar(kBarKFull + s), 1);
      mbar_init(bar(kBarKEmpty + s), 1);
    }
    for (int s = 0; s < kStagesV; ++s) {
      mbar_init(bar(kBarVFull + s), 1);
      mbar_init(bar(kBarVEmpty + s), 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(bar(kBarSFull + 2 * i), 1);
      mbar_init(bar(kBarSFull + 2 * i + 1), 1);
      mbar_init(bar(kBarPFull + 2 * i), kRows);
      mbar_init(bar(kBarPFull + 2 * i + 1), kRows);
      mbar_init(bar(kBarPVDone + i), 1);
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
  // The CTA owns all 512 columns, so the allocation starts at lane 0,
  // column 0: a compile-time constant keeps TMEM addresses uniform.
  constexpr uint32_t tmem = 0;
  if (tid == 0 && *tmem_slot != 0u) __trap();

  if (warp == 8 || warp == 10) {
    // ---------------- producers: paged K (warp 8) / V (warp 10) tiles by TMA ----
    // Separate warps so K runs ahead of V: with one producer, K(j+2) queued
    // behind V(j+1), which waits for PV(j-3) to free its stage, and the MMA
    // warp waited ~900 cycles per tile for K (profiled timeline).
    // Lane l owns tile positions 2l, 2l+1.  A chunk of C = min(P, 64)
    // positions whose slots are consecutive rows (a page, when the sequence
    // is page-aligned) is one C-row box; otherwise (a fork at a
    // non-page-aligned length) its rows are loaded one by one.  Positions
    // >= n_keys are don't-care (masked; V zeroed by the MMA warp).
    const int C = min(a.page_size, kKeys), lanes_per_chunk = C / 2;
    const uint32_t chunk_mask = lanes_per_chunk >= 32 ? 0xffffffffu : ((1u << lanes_per_chunk) - 1u);
    const int my_chunk_lane0 = lane - lane % lanes_per_chunk;
    const int ck = h * kD, cv = (a.Hkv + h) * kD;  // element column of K / V of this head
    for (int j = 0; j < n_tiles; ++j) {
      const int nst = warp == 8 ? kStages : kStagesV;
      const int s = j % nst;
      const int p0 = j * kKeys + lane * 2;
      int sl[2];
#pragma unroll
      for (int t = 0; t < 2; ++t) sl[t] = p0 + t < n_keys ? __ldg(a.slots + p0 + t) : -1;
      const int prev_last = __shfl_up_sync(0xffffffffu, sl[1], 1);
      bool ok = true;
#pragma unroll
      for (int t = 0; t < 2; ++t) {
        const bool chunk_start = ((lane * 2 + t) % C) == 0;
        const int prev = t > 0 ? sl[t - 1] : prev_last;
        if (!chunk_start && sl[t] >= 0) ok = ok && sl[t] == prev + 1;
      }
      const uint32_t ballot = __ballot_sync(0xffffffffu, ok);
      const bool contiguous = ((ballot >> my_chunk_lane0) & chunk_mask) == chunk_mask;
      const int chunk_row = __shfl_sync(0xffffffffu, sl[0], my_chunk_lane0);
      {
        const int op = warp == 8 ? 0 : 1;
        const uint32_t base = (op == 0 ? sK : sV) + s * kKvTile;
        const uint32_t full = bar((op == 0 ? kBarKFull : kBarVFull) + s);
        const int col = op == 0 ? ck : cv;
        if (lane == 0) {
          if (j >= nst)
            mbar_wait(bar((op == 0 ? kBarKEmpty : kBarVEmpty) + s), ((j / nst) + 1) & 1);
          PF_EV((op == 0 ? 0xA00 : 0xC00) | (j & 0xff));  // producer: stage free, issuing
          mbar_expect_tx(full, kKvTile);
        }
        __syncwarp();
        if (contiguous) {
          if (lane == my_chunk_lane0) {
            const uint32_t dst = base + (lane * 2) * 128;
            const int row = chunk_row >= 0 ? chunk_row : 0;
            tma_load_3d(dst, &pool_map, col, row, a.layer, full);
            tma_load_3d(dst + kKvAtom, &pool_map, col + 64, row, a.layer, full);
          }
        } else {
#pragma unroll
          for (int t = 0; t < 2; ++t) {
            const uint32_t dst = base + (lane * 2 + t) * 128;
            const int row = sl[t] >= 0 ? sl[t] : 0;
            tma_load_3d(dst, &row_map, col, row, a.layer, full);
            tma_load_3d(dst + kKvAtom, &row_map, col + 64, row, a.layer, full);
          }
        }
      }
    }
  } else if (warp == 9) {
    // ---------------- MMA issuer ----------------
    // TMEM: query tile i owns columns [128 i, 128 i + 128) as two 64-column S
    // slots (tile j uses slot j & 1; P_i(j) overwrites the first 32 columns
    // of its slot), O_i at 256 + 128 i.  Issue order per KV tile j:
    //   S0(j) S1(j) | PV0(j-1) PV1(j-1)
    // so S(j) runs on the tensor core while the softmax warpgroups work on
    // tile j-1.  S_i(j) reuses the slot of P_i(j-2), consumed by PV_i(j-2),
    // issued one iteration earlier (tcgen05 MMAs of one thread run in order).
    constexpr uint32_t kIdescS = idesc_bf16(false, kKeys), kIdescO = idesc_bf16(true, kD);
    constexpr uint32_t kHi = desc_hi(1024);  // SBO 1024 B (8-row groups), version 1, SW128
    auto tS = [&](int i, int j) { return tmem + i * 128 + (j & 1) * 64; };
    auto tO = [&](int i) { return tmem + 256 + i * 128; };
    // Low descriptor words of the tile bases; K-step offsets are added in
    // 16-byte units (start address field, no carry: smem < 256 KiB).
    const uint32_t q_lo = desc_lo(sQ, 16), k_lo = desc_lo(sK, 16), v_lo = desc_lo(sV, kKvAtom);
    auto issue_s = [&](int i, int j) {
      const uint32_t a0 = q_lo + ((i * kTile) >> 4), b0 = k_lo + (((j % kStages) * kKvTile) >> 4);
#pragma unroll
      for (int k = 0; k < kD / 16; ++k) {
        const uint32_t ao = ((k >> 2) * kAtom + (k & 3) * 32) >> 4;
        const uint32_t bo = ((k >> 2) * kKvAtom + (k & 3) * 32) >> 4;
        mma_ss_elect(tS(i, j), a0 + ao, b0 + bo, kHi, kIdescS, k > 0 ? 1u : 0u);
      }
      commit_elect(bar(kBarSFull + 2 * i + (j & 1)));
    };
    auto issue_pv = [&](int i, int j) {
      mbar_wait(bar(kBarPFull + 2 * i + (j & 1)), (j >> 1) & 1);
      fence_after();
      const uint32_t b0 = v_lo + (((j % kStagesV) * kKvTile) >> 4);
#pragma unroll
      for (int k = 0; k < kKeys / 16; ++k) {
        // A = P_i in TMEM (bf16 pairs: 8 columns per 16 keys); B = V MN-major:
        // 16 keys = two 8-key atoms (SBO 1024 B), d halves LBO = 8 KiB apart.
        mma_ts_elect(tO(i), tS(i, j) + k * 8, b0 + ((k * 2048) >> 4), kHi, kIdescO,
                     (j > 0 || k > 0) ? 1u : 0u);
      }
      commit_elect(bar(kBarPVDone + i));
    };
    // Keys past n_keys in the last tile: zero their V rows (both halves).
    auto zero_tail = [&](int j) {
      const int valid = n_keys - j * kKeys;
      if (valid >= kKeys) return;
      uint8_t* vb = smem + kOffV + (j % kStagesV) * kKvTile;
      for (int e = lane; e < (kKeys - valid) * 16; e += 32) {
        const int r = valid + (e >> 4), c = e & 15;
        *reinterpret_cast<uint4*>(vb + (c >> 3) * kKvAtom + r * 128 + (c & 7) * 16) =
            make_uint4(0, 0, 0, 0);
      }
      fence_proxy_async();
      __syncwarp();
    };
    mbar_wait(bar(kBarQ), 0);
    // Prologue: S of KV tiles 0 and 1 for both query tiles.
    for (int j = 0; j < 2 && j < n_tiles; ++j) {
      const int s = j % kStages;
      mbar_wait(bar(kBarKFull + s), (j / kStages) & 1);
      fence_after();
      issue_s(0, j);
      issue_s(1, j);
      commit_elect(bar(kBarKEmpty + s));
    }
    // Steady state, per query tile: PV_i(j) as soon as P_i(j) is ready, then
    // S_i(j+2) into the slot P_i(j) frees (tcgen05 MMAs of one thread run in
    // order), so one tile's softmax never waits on the other's.
    for (int j = 0; j < n_tiles; ++j) {
      const int sv = j % kStagesV;
      mbar_wait(bar(kBarVFull + sv), (j / kStagesV) & 1);
      if (lane == 0) PF_EV(0xE00 | (j & 0xff));  // MMA: V(j) landed
      if (j == n_tiles - 1) zero_tail(j);
      const bool next = j + 2 < n_tiles;
      const int sk = (j + 2) % kStages;
      if (next) mbar_wait(bar(kBarKFull + sk), ((j + 2) / kStages) & 1);
      fence_after();
      if (lane == 0) PF_EV(0x100 | (j & 0xff));  // MMA: V(j) and K(j+2) ready
      for (int i = 0; i < kQTiles; ++i) {
        issue_pv(i, j);
        if (lane == 0) PF_EV(0x200 | (i << 8) | (j & 0xff));  // MMA: PV_i(j) issued
        if (j == n_tiles - 1) commit_elect(bar(kBarODone + i));
        if (next) issue_s(i, j + 2);
      }
      commit_elect(bar(kBarVEmpty + sv));
      if (next) commit_elect(bar(kBarKEmpty + sk));
    }
  } else {
    // ---------------- softmax warpgroups ----------------
    const int i = warp >> 2;              // query tile
    const int r = tid & (kRows - 1);      // row = TMEM lane
    const int G = a.Hq / a.Hkv;           // 8
    const int tok = tok_first + i * kTokens + r / G, g = r % G;
    const bool row_valid = tok < a.n_q;
    const int q_pos = a.q_pos0 + tok;
    const int tile_min_pos = a.q_pos0 + tok_first + i * kTokens;  // smallest position of tile i
    const uint32_t lane_off = static_cast<uint32_t>((warp & 3) * 32) << 16;
    const uint32_t tSi = tmem + i * 128 + lane_off, tO = tmem + 256 + i * 128 + lane_off;
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
    float m = -INFINITY, l = 0.f;  // running max (scaled log2 domain) and sum
    for (int j = 0; j < n_tiles; ++j) {
      const uint32_t tS = tSi + (j & 1) * 64;
      if ((warp & 3) == 0 && lane == 0) PF_EV(0x400 | (i << 8) | (j & 0xff));  // softmax: wait S
      mbar_wait(bar(kBarSFull + 2 * i + (j & 1)), (j >> 1) & 1);
      fence_after();
      if ((warp & 3) == 0 && lane == 0) PF_EV(0x600 | (i << 8) | (j & 0xff));  // softmax: S ready
      uint32_t sr[kKeys];
#pragma unroll
      for (int c0 = 0; c0 < kKeys; c0 += 16) tmem_ld16_nowait(tS + c0, sr + c0);
      tmem_wait_ld();
      const int key0 = j * kKeys;
      // Causal mask only where this tile crosses the diagonal of query tile i.
      // Warp-uniform: the two P paths below hold warp-collective TMEM stores.
      const bool need_mask =
          __any_sync(0xffffffffu, key0 + kKeys - 1 > tile_min_pos || !row_valid);
      if (need_mask) {
        const int lim = row_valid ? q_pos - key0 : -1;  // last visible column
#pragma unroll
        for (int c = 0; c < kKeys; ++c)
          sr[c] = c > lim ? __float_as_uint(-INFINITY) : sr[c];
      }
      // Row max over 64 columns: four independent 3-input chains.
      float mx[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
      for (int c = 0; c < kKeys; c += 8) {
#pragma unroll
        for (int k = 0; k < 4; ++k)
          mx[k] = fmaxf(mx[k], fmaxf(__uint_as_float(sr[c + 2 * k]), __uint_as_float(sr[c + 2 * k + 1])));
      }
      const float rmax = fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3]));  // raw (unscaled)
      const float tmax = rmax * sl2;
      // Keep the stale max unless this tile exceeds it by > 8 (p <= 2^8 then).
      const bool bump = tmax > m + 8.f;
      const float m_new = bump ? tmax : m;
      const float alpha = (bump && m != -INFINITY) ? ex2_mufu(m - m_new) : 1.f;
      const float neg_m = m_new == -INFINITY ? 0.f : -m_new;
      // P = 2^(s*scale - m) packed in place (pair c/2 overwrites S[c/2],
      // already consumed).  Scale/shift and the row sum run as f32x2 pairs;
      // in unmasked tiles every PF_POLY_EVERY-th pair of exponentials runs on
      // the FMA pipe (polynomial) to relieve the MUFU unit.
#ifndef PF_POLY_EVERY
#define PF_POLY_EVERY 0  // measured best: the softmax is issue-bound, not MUFU-bound
#endif
      const uint64_t sc2 = f2pack(sl2, sl2), nm2 = f2pack(neg_m, neg_m);
      uint64_t acc[2] = {0ull, 0ull};
      auto make_p = [&](auto poly) {
#pragma unroll
        for (int c = 0; c < kKeys; c += 2) {
          float x0, x1, p0, p1;
          f2unpack(ffma2(f2pack(__uint_as_float(sr[c]), __uint_as_float(sr[c + 1])), sc2, nm2),
                   x0, x1);
          if (decltype(poly)::value && PF_POLY_EVERY > 0 &&
              ((c >> 1) % (PF_POLY_EVERY > 0 ? PF_POLY_EVERY : 1)) == PF_POLY_EVERY - 1) {
            ex2_poly2(x0, x1, p0, p1);
          } else {
            p0 = ex2_mufu(x0);
            p1 = ex2_mufu(x1);
          }
          acc[(c >> 1) & 1] = fadd2(acc[(c >> 1) & 1], f2pack(p0, p1));
          sr[c / 2] = pack_bf16(p0, p1);
        }
      };
      if (need_mask) make_p(std::false_type{});
      else make_p(std::true_type{});
      float ps[4];
      f2unpack(acc[0], ps[0], ps[1]);
      f2unpack(acc[1], ps[2], ps[3]);
      const float psum = (ps[0] + ps[1]) + (ps[2] + ps[3]);
#pragma unroll
      for (int c0 = 0; c0 < kKeys / 2; c0 += 16) tmem_st16_nowait(tS + c0, sr + c0);
      // O_i must be stable (PV_i(j-1) retired) before it is rescaled for
      // tile j; warps with nothing to rescale skip the wait (parity waits
      // stay exact: PV_i(j) needs this warpgroup's P_i(j), so the barrier is
      // at most one phase ahead of any later wait).
      if (j > 0 && __any_sync(0xffffffffu, alpha != 1.f)) {
        mbar_wait(bar(kBarPVDone + i), (j - 1) & 1);
        fence_after();
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
      tmem_wait_st();
      fence_before();
      mbar_arrive(bar(kBarPFull + 2 * i + (j & 1)));
      if ((warp & 3) == 0 && lane == 0) PF_EV(0x800 | (i << 8) | (j & 0xff));  // softmax: P arrived
      l = l * alpha + psum;
      m = m_new;
    }
    // The last PV of this tile (PVDone could be one phase behind or ahead
    // here, which a parity wait cannot tell apart).
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


// ===========================================================================
// 2-SM variant (tcgen05 cta_group::2): a cluster of two CTAs on one TPC
// computes S = Q K^T and O += P V for 256 query rows (2 x [16 tokens x 8
// heads]) as M = 256 MMAs issued by the leader CTA.  Each CTA keeps its own
// Q rows, S slots and O in its TMEM, but holds only half of each B operand
// (K: its 64 of the tile's 128 keys; V: its 64 of the 128 head dims), so the
// shared-memory traffic per SM per KV tile — the wall both single-CTA
// layouts hit — drops from ~160 KiB to ~96 KiB.
//   warps 0-3 softmax (own 128 rows), warp 4 K producer, warp 5 MMA (leader
//   issues; both allocate TMEM), warp 6 V producer.
// Cross-CTA signalling: TMA of both CTAs completes on the leader's full
// barriers (peer bit cleared), the follower's softmax and Q loads arrive on
// the leader's barriers through shared::cluster addresses, and the leader's
// commits multicast to both CTAs' S-full / PV-done / stage-empty barriers.
#ifndef PF2_POLY_EVERY
#define PF2_POLY_EVERY 3
#endif
namespace p2 {
constexpr int kKeys = 128;                // keys per KV tile
constexpr int kHalfKeys = kKeys / 2;      // K rows held per CTA
constexpr int kSlots = 3;                 // S slots (128 columns each) after O
constexpr int kStages = 4;                // K and V rings
constexpr int kKTile = kHalfKeys * 256;   // [64 keys][128 d] bf16, two atom columns: 16 KiB
constexpr int kKAtom = kHalfKeys * 128;   // 8 KiB
constexpr int kVTile = kKeys * 128;       // [128 keys][64 d] bf16, one atom column: 16 KiB
constexpr int kThreads = 128 + 96;
constexpr int kOffQ = 0;                  // [128][128] bf16, 32 KiB
constexpr int kOffK = kOffQ + kTile;
constexpr int kOffV = kOffK + kStages * kKTile;
constexpr int kOffBar = kOffV + kStages * kVTile;
constexpr int kSmem = kOffBar + 512;
enum : int {
  kBarQ = 0,                          // leader: both CTAs' Q rows staged (8 warps)
  kBarKFull = 1,                      // leader: +stage, 2 arrivals + both CTAs' bytes
  kBarVFull = kBarKFull + kStages,
  kBarKEmpty = kBarVFull + kStages,   // both: +stage (multicast commit)
  kBarVEmpty = kBarKEmpty + kStages,
  kBarSFull = kBarVEmpty + kStages,   // both: +slot
  kBarPFull = kBarSFull + kSlots,     // leader: +slot, one arrival per softmax warp (8)
  kBarPVDone = kBarPFull + kSlots,    // both: +slot
  kBarODone = kBarPVDone + kSlots,    // both
  kBarCount = kBarODone + 1,
};
static_assert(kBarCount * 8 + 8 <= 512, "barrier area");
static_assert(kSmem + 1024 <= 227 * 1024, "shared memory");

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::
                   : "memory");
}
// shared::cluster address of the same shared variable in CTA `rank`.
__device__ __forceinline__ uint32_t mapa(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
__device__ __forceinline__ void arrive_cluster(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr)
               : "memory");
}
__device__ __forceinline__ void expect_tx_cluster(uint32_t cluster_addr, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.release.cluster.shared::cluster.b64 _, [%0], %1;" ::"r"(
                   cluster_addr),
               "r"(bytes)
               : "memory");
}
// Bounded cluster-scope wait (a lost arrival traps instead of hanging).
__device__ __forceinline__ void wait_cluster(uint32_t bar, uint32_t phase) {
  uint32_t done = 0;
  const long long t0 = clock64();
  for (;;) {
    asm volatile(
        "{\n\t.reg .pred P;\n\t"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, P;\n\t}\n"
        : "=r"(done)
        : "r"(bar), "r"(phase)
        : "memory");
    if (done) return;
    if (clock64() - t0 > (4ll << 30)) __trap();
  }
}
// 2-SM TMA: lands in this CTA's shared memory, completes bytes on the
// leader's barrier (peer bit cleared).
__device__ __forceinline__ void tma2_load_3d(uint32_t dst, const CUtensorMap* map, int c0, int c1,
                                             int c2, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes "
      "[%0], [%1, {%2, %3, %4}], [%5];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(bar & 0xFEFFFFFFu)
      : "memory");
}
__device__ __forceinline__ void mma2_ss(uint32_t tmem_d, uint32_t a_lo, uint32_t b_lo, uint32_t hi,
                                        uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t.reg .b64 da, db;\n\t"
      "mov.b64 da, {%1, %3};\n\tmov.b64 db, {%2, %3};\n\t"
      "setp.ne.b32 p, %5, 0;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], da, db, %4, p;\n\t}\n" ::"r"(tmem_d),
      "r"(a_lo), "r"(b_lo), "r"(hi), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void mma2_ts(uint32_t tmem_d, uint32_t tmem_a, uint32_t b_lo,
                                        uint32_t b_hi, uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t.reg .b64 db;\n\t"
      "mov.b64 db, {%2, %3};\n\t"
      "setp.ne.b32 p, %5, 0;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], db, %4, p;\n\t}\n" ::"r"(tmem_d),
      "r"(tmem_a), "r"(b_lo), "r"(b_hi), "r"(idesc), "r"(accumulate));
}
// Commit to the barrier at `bar` in both CTAs of the pair.
__device__ __forceinline__ void commit2(uint32_t bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 "
      "[%0], %1;\n\t}\n" ::"r"(bar),
      "h"(static_cast<unsigned short>(3))
      : "memory");
}
// D f32, A/B bf16, M = 256 (2 SMs), N = n, A K-major, B K- or MN-major.
__host__ __device__ constexpr uint32_t idesc2(bool b_mn_major, int n) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((b_mn_major ? 1u : 0u) << 16) |
         ((static_cast<uint32_t>(n) >> 3) << 17) | ((256u >> 4) << 24);
}
}  // namespace p2

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(p2::kThreads, 1)
    k_prefill_attn_2sm(const __grid_constant__ CUtensorMap pool_map,
                       const __grid_constant__ CUtensorMap row_map, const PrefillArgs a) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t rank = p2::cluster_rank();
  const bool leader = rank == 0;
  // Heaviest (latest) pair first; CTA `rank` takes the pair's token half.
  const int pair = a.n_blocks - 1 - static_cast<int>(blockIdx.x >> 1);
  const int h = blockIdx.y;
  const uint32_t sQ = smem_u32(smem + p2::kOffQ), sK = smem_u32(smem + p2::kOffK);
  const uint32_t sV = smem_u32(smem + p2::kOffV), bars = smem_u32(smem + p2::kOffBar);
  auto bar = [&](int i) { return bars + 8u * static_cast<uint32_t>(i); };
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + p2::kOffBar + 8 * p2::kBarCount);
  const int tok_pair = pair * 2 * kTokens;
  const int tok_first = tok_pair + static_cast<int>(rank) * kTokens;
  const int tok_last = min(a.n_q, tok_pair + 2 * kTokens) - 1;  // of the pair
  const int n_keys = a.q_pos0 + tok_last + 1;
  const int n_tiles = (n_keys + p2::kKeys - 1) / p2::kKeys;

  if (warp == 5) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                     smem_u32(tmem_slot))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  if (tid == 128) {
    mbar_init(bar(p2::kBarQ), 8);  // one arrival per softmax warp of either CTA
    for (int s = 0; s < p2::kStages; ++s) {
      mbar_init(bar(p2::kBarKFull + s), 2);
      mbar_init(bar(p2::kBarVFull + s), 2);
      mbar_init(bar(p2::kBarKEmpty + s), 1);
      mbar_init(bar(p2::kBarVEmpty + s), 1);
    }
    for (int k = 0; k < p2::kSlots; ++k) {
      mbar_init(bar(p2::kBarSFull + k), 1);
      mbar_init(bar(p2::kBarPFull + k), 8);
      mbar_init(bar(p2::kBarPVDone + k), 1);
    }
    mbar_init(bar(p2::kBarODone), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&pool_map))
                 : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&row_map))
                 : "memory");
  }
  fence_before();
  p2::cluster_sync();  // barriers of both CTAs initialised, TMEM allocated
  fence_after();
  constexpr uint32_t tmem = 0;
  if (tid == 0 && *tmem_slot != 0u) __trap();

  if (warp == 4 || warp == 6) {
    // ---------------- producers ----------------
    // K (warp 4): keys [j*128 + 64*rank, +64) of tile j, all 128 dims; lane
    // l owns positions 2l, 2l+1.  V (warp 6): all 128 keys of tile j, dims
    // [64*rank, +64); lane l owns 4l .. 4l+3.  Chunks of C = min(P, 64)
    // consecutive rows are one box; otherwise rows one by one, and V rows
    // past n_keys load an out-of-range row, which TMA fills with zeros.
    const bool isK = warp == 4;
    const int per_lane = isK ? 2 : 4;
    const int C = min(a.page_size, 64), lanes_per_chunk = C / per_lane;
    const uint32_t chunk_mask =
        lanes_per_chunk >= 32 ? 0xffffffffu : ((1u << lanes_per_chunk) - 1u);
    const int my_chunk_lane0 = lane - lane % lanes_per_chunk;
    const int col = isK ? h * kD : (a.Hkv + h) * kD + 64 * static_cast<int>(rank);
    const uint32_t lead_full = p2::mapa(bar(isK ? p2::kBarKFull : p2::kBarVFull), 0);
    for (int j = 0; j < n_tiles; ++j) {
      const int s = j % p2::kStages;
      const int p0 = j * p2::kKeys + (isK ? 64 * static_cast<int>(rank) : 0) + lane * per_lane;
      int sl[4];
#pragma unroll
      for (int t = 0; t < 4; ++t)
        sl[t] = (t < per_lane && p0 + t < n_keys) ? __ldg(a.slots + p0 + t) : -1;
      const int prev_last = __shfl_up_sync(0xffffffffu, sl[per_lane - 1], 1);
      bool ok = true;
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        if (t >= per_lane) break;
        const bool chunk_start = ((lane * per_lane + t) % C) == 0;
        const int prev = t > 0 ? sl[t - 1] : prev_last;
        if (sl[t] < 0) ok = isK ? ok : false;  // V: invalid rows must load zeros
        else if (!chunk_start) ok = ok && sl[t] == prev + 1;
      }
      const uint32_t ballot = __ballot_sync(0xffffffffu, ok);
      const bool contiguous = ((ballot >> my_chunk_lane0) & chunk_mask) == chunk_mask;
      const int chunk_row = __shfl_sync(0xffffffffu, sl[0], my_chunk_lane0);
      const uint32_t base = isK ? sK + s * p2::kKTile : sV + s * p2::kVTile;
      const uint32_t bytes = isK ? p2::kKTile : p2::kVTile;
      if (lane == 0) {
        if (j >= p2::kStages)
          mbar_wait(bar((isK ? p2::kBarKEmpty : p2::kBarVEmpty) + s), ((j / p2::kStages) + 1) & 1);
        p2::expect_tx_cluster(lead_full + 8u * static_cast<uint32_t>(s), bytes);
      }
      __syncwarp();
      const uint32_t full = bar((isK ? p2::kBarKFull : p2::kBarVFull) + s);
      if (contiguous) {
        if (lane == my_chunk_lane0) {
          const uint32_t dst = base + (lane * per_lane) * 128;
          const int row = chunk_row >= 0 ? chunk_row : 0;
          p2::tma2_load_3d(dst, &pool_map, col, row, a.layer, full);
          if (isK) p2::tma2_load_3d(dst + p2::kKAtom, &pool_map, col + 64, row, a.layer, full);
        }
      } else {
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          if (t >= per_lane) break;
          const uint32_t dst = base + (lane * per_lane + t) * 128;
          const int row = sl[t] >= 0 ? sl[t] : (isK ? 0 : a.pool_rows);
          p2::tma2_load_3d(dst, &row_map, col, row, a.layer, full);
          if (isK) p2::tma2_load_3d(dst + p2::kKAtom, &row_map, col + 64, row, a.layer, full);
        }
      }
    }
  } else if (warp == 5) {
    if (leader) {
      // ---------------- MMA issuer (leader CTA) ----------------
      constexpr uint32_t kIdescS = p2::idesc2(false, p2::kKeys), kIdescO = p2::idesc2(true, kD);
      constexpr uint32_t kHi = desc_hi(1024);
      auto tS = [&](int j) { return tmem + 128 + (j % p2::kSlots) * 128; };
      const uint32_t q_lo = desc_lo(sQ, 16), k_lo = desc_lo(sK, 16), v_lo = desc_lo(sV, 16);
      auto issue_s = [&](int j) {
        const uint32_t b0 = k_lo + (((j % p2::kStages) * p2::kKTile) >> 4);
#pragma unroll
        for (int k = 0; k < kD / 16; ++k) {
          const uint32_t ao = ((k >> 2) * kAtom + (k & 3) * 32) >> 4;
          const uint32_t bo = ((k >> 2) * p2::kKAtom + (k & 3) * 32) >> 4;
          p2::mma2_ss(tS(j), q_lo + ao, b0 + bo, kHi, kIdescS, k > 0 ? 1u : 0u);
        }
        p2::commit2(bar(p2::kBarSFull + j % p2::kSlots));
      };
      p2::wait_cluster(bar(p2::kBarQ), 0);
      for (int j = 0; j < p2::kSlots && j < n_tiles; ++j) {
        const int sk = j % p2::kStages;
        p2::wait_cluster(bar(p2::kBarKFull + sk), (j / p2::kStages) & 1);
        fence_after();
        issue_s(j);
        p2::commit2(bar(p2::kBarKEmpty + sk));
      }
      for (int j = 0; j < n_tiles; ++j) {
        const int sv = j % p2::kStages;
        p2::wait_cluster(bar(p2::kBarVFull + sv), (j / p2::kStages) & 1);
        p2::wait_cluster(bar(p2::kBarPFull + j % p2::kSlots), (j / p2::kSlots) & 1);
        fence_after();
        const uint32_t b0 = v_lo + ((sv * p2::kVTile) >> 4);
#pragma unroll
        for (int k = 0; k < p2::kKeys / 16; ++k) {
          // A = P in TMEM (8 columns per 16 keys); B = V MN-major, this CTA's
          // 64 dims (one atom column), 16 keys = two 8-key groups (SBO 1 KiB).
          p2::mma2_ts(tmem, tS(j) + k * 8, b0 + ((k * 2048) >> 4), kHi, kIdescO,
                      (j > 0 || k > 0) ? 1u : 0u);
        }
        p2::commit2(bar(p2::kBarPVDone + j % p2::kSlots));
        p2::commit2(bar(p2::kBarVEmpty + sv));
        if (j == n_tiles - 1) p2::commit2(bar(p2::kBarODone));
        const int jn = j + p2::kSlots;
        if (jn < n_tiles) {
          const int sk = jn % p2::kStages;
          p2::wait_cluster(bar(p2::kBarKFull + sk), (jn / p2::kStages) & 1);
          fence_after();
          issue_s(jn);
          p2::commit2(bar(p2::kBarKEmpty + sk));
        }
      }
    }
  } else {
    // ---------------- softmax (warps 0-3, own 128 rows) ----------------
    const int r = tid;
    const int G = a.Hq / a.Hkv;
    const int tok = tok_first + r / G, g = r % G;
    const bool row_valid = tok < a.n_q;
    const int q_pos = a.q_pos0 + tok;
    const int tile_min_pos = a.q_pos0 + tok_first;
    const uint32_t lane_off = static_cast<uint32_t>(warp * 32) << 16;
    const uint32_t tO = tmem + lane_off;
    const uint32_t lead_q = p2::mapa(bar(p2::kBarQ), 0);
    const uint32_t lead_p = p2::mapa(bar(p2::kBarPFull), 0);
    {
      const __nv_bfloat16* qrow =
          a.q + (static_cast<int64_t>(row_valid ? tok : 0) * a.Hq + static_cast<int64_t>(h) * G + g) * kD;
#pragma unroll
      for (int c = 0; c < 16; ++c) cp_async16(sQ + sw128(r, c), qrow + c * 8, row_valid);
      asm volatile("cp.async.commit_group;" ::: "memory");
      asm volatile("cp.async.wait_group 0;" ::: "memory");
      fence_proxy_async();
      __syncwarp();
      if (lane == 0) p2::arrive_cluster(lead_q);
    }
    const float sl2 = a.scale_log2;
    float m = -INFINITY, l = 0.f;
    for (int j = 0; j < n_tiles; ++j) {
      const int slot = j % p2::kSlots;
      const uint32_t tS = tmem + 128 + slot * 128 + lane_off;
      mbar_wait(bar(p2::kBarSFull + slot), (j / p2::kSlots) & 1);
      fence_after();
      uint32_t sr[p2::kKeys];
#pragma unroll
      for (int c0 = 0; c0 < p2::kKeys; c0 += 16) tmem_ld16_nowait(tS + c0, sr + c0);
      tmem_wait_ld();
      const int key0 = j * p2::kKeys;
      const bool need_mask =
          __any_sync(0xffffffffu, key0 + p2::kKeys - 1 > tile_min_pos || !row_valid);
      if (need_mask) {
        const int lim = row_valid ? q_pos - key0 : -1;
#pragma unroll
        for (int c = 0; c < p2::kKeys; ++c)
          sr[c] = c > lim ? __float_as_uint(-INFINITY) : sr[c];
      }
      float mx[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
      for (int c = 0; c < p2::kKeys; c += 8) {
#pragma unroll
        for (int k = 0; k < 4; ++k)
          mx[k] = fmaxf(mx[k], fmaxf(__uint_as_float(sr[c + 2 * k]), __uint_as_float(sr[c + 2 * k + 1])));
      }
      const float tmax = fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3])) * sl2;
      const bool bump = tmax > m + 8.f;
      const float m_new = bump ? tmax : m;
      const float alpha = (bump && m != -INFINITY) ? ex2_mufu(m - m_new) : 1.f;
      const float neg_m = m_new == -INFINITY ? 0.f : -m_new;
      const uint64_t sc2 = f2pack(sl2, sl2), nm2 = f2pack(neg_m, neg_m);
      uint64_t acc[2] = {0ull, 0ull};
      // One softmax warp per SM sub-partition: in unmasked tiles every
      // PF2_POLY_EVERY-th pair of exponentials runs on the FMA pipe.
      auto make_p = [&](auto poly) {
#pragma unroll
        for (int c = 0; c < p2::kKeys; c += 2) {
          float x0, x1, p0, p1;
          f2unpack(ffma2(f2pack(__uint_as_float(sr[c]), __uint_as_float(sr[c + 1])), sc2, nm2),
                   x0, x1);
          if (decltype(poly)::value && PF2_POLY_EVERY > 0 &&
              ((c >> 1) % (PF2_POLY_EVERY > 0 ? PF2_POLY_EVERY : 1)) == PF2_POLY_EVERY - 1) {
            ex2_poly2(x0, x1, p0, p1);
          } else {
            p0 = ex2_mufu(x0);
            p1 = ex2_mufu(x1);
          }
          acc[(c >> 1) & 1] = fadd2(acc[(c >> 1) & 1], f2pack(p0, p1));
          sr[c / 2] = pack_bf16(p0, p1);
        }
      };
      if (need_mask) make_p(std::false_type{});
      else make_p(std::true_type{});
      float ps[4];
      f2unpack(acc[0], ps[0], ps[1]);
      f2unpack(acc[1], ps[2], ps[3]);
      const float psum = (ps[0] + ps[1]) + (ps[2] + ps[3]);
#pragma unroll
      for (int c0 = 0; c0 < p2::kKeys / 2; c0 += 16) tmem_st16_nowait(tS + c0, sr + c0);
      if (j > 0 && __any_sync(0xffffffffu, alpha != 1.f)) {
        mbar_wait(bar(p2::kBarPVDone + (j - 1) % p2::kSlots), ((j - 1) / p2::kSlots) & 1);
        fence_after();
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
      tmem_wait_st();
      fence_before();
      __syncwarp();
      if (lane == 0) p2::arrive_cluster(lead_p + 8u * static_cast<uint32_t>(slot));
      l = l * alpha + psum;
      m = m_new;
    }
    mbar_wait(bar(p2::kBarODone), 0);
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
  p2::cluster_sync();  // both CTAs done with TMEM and the peer's barriers
  if (warp == 5) {
    fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
  }
}

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
// 128-key variant (MICROKV_PREFILL_VARIANT=3 while it is evaluated): the
// same CTA (one KV head x two M=128 query tiles) with 128-key KV tiles and
// ONE S slot per query tile (TMEM: S_i at 128 i, O_i at 256 + 128 i).  The
// S MMAs run at N = 128 instead of 64, which halves the shared-memory reads
// of Q per key (A is re-read per MMA): per 128 keys and both tiles ~128 B/clk
// of operand traffic instead of ~160.  S_i(j+1) is issued right behind
// PV_i(j) into the columns P_i(j) occupied (MMAs of one thread run in
// order), so the S-full barrier of tile j+1 also proves PV_i(j) retired and
// the O rescale needs no separate wait; the two query tiles ping-pong: one
// tile's softmax runs while the tensor core works on the other's PV and S.
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
#define PF3_POLY_EVERY 4
#endif
constexpr int kStagesK = PF3_K_STAGES, kStagesV = PF3_V_STAGES;
constexpr int kOffQ = 0;
constexpr int kOffK = kOffQ + kQTiles * kTile;
constexpr int kOffV = kOffK + kStagesK * kKvTile;
constexpr int kOffBar = kOffV + kStagesV * kKvTile;
constexpr int kSmem = kOffBar + 512;
// Split-row softmax variant (k_prefill_attn_k128s): 16 softmax warps.
constexpr int kSoftmaxThreadsS = 512;
constexpr int kThreadsS = kSoftmaxThreadsS + 96;
constexpr int kOffRed = kOffBar + 512;          // row max / sum exchange, 6 x [2][128] floats
constexpr int kSmemS = kOffRed + 6 * 2 * 128 * 4;
enum : int {
  kBarQ = 0,
  kBarKFull = 1,
  kBarVFull = kBarKFull + kStagesK,
  kBarKEmpty = kBarVFull + kStagesV,
  kBarVEmpty = kBarKEmpty + kStagesK,
  kBarSFull = kBarVEmpty + kStagesV,  // +tile
  kBarPFull = kBarSFull + 2,          // +tile (count 128)
  kBarODone = kBarPFull + 2,          // +tile
  kBarPHalf = kBarODone + 2,          // +tile: first half of P_i(j) (k128 only)
  kBarOFree = kBarPHalf + 2,          // +tile: epilogue read O_i (persistent k128p only)
  kBarCount = kBarOFree + 2,
};
static_assert(kBarCount * 8 + 8 <= 512, "barrier area");
static_assert(kSmem + 1024 <= 227 * 1024, "shared memory");
static_assert(kSmemS + 1024 <= 227 * 1024, "shared memory");
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
  // Heaviest (latest) query blocks first; a.n_split CTAs per block split
  // its key tiles evenly (short balanced-PD tails fill the SMs).
  const int qb = a.n_blocks - 1 - static_cast<int>(blockIdx.x) / a.n_split;
  const int sp = static_cast<int>(blockIdx.x) % a.n_split;
  const int h = blockIdx.y;
  const uint32_t sQ = smem_u32(smem + kOffQ), sK = smem_u32(smem + kOffK);
  const uint32_t sV = smem_u32(smem + kOffV), bars = smem_u32(smem + kOffBar);
  auto bar = [&](int i) { return bars + 8u * static_cast<uint32_t>(i); };
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + kOffBar + 8 * kBarCount);

  const int tok_first = qb * kQTiles * kTokens;
  const int tok_last = min(a.n_q, tok_first + kQTiles * kTokens) - 1;
  const int n_keys = a.q_pos0 + tok_last + 1;
  const int n_tiles = (n_keys + kKeys - 1) / kKeys;
  // This CTA's key tiles [t_begin, t_begin + n_local); the host keeps
  // n_split <= the lightest block's tile count, so n_local >= 1.
  const int t_begin = sp * n_tiles / a.n_split;
  const int n_local = (sp + 1) * n_tiles / a.n_split - t_begin;

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
    const int C = min(a.page_size, 64), lanes_per_chunk = C / kPer;
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
    const int tok = tok_first + i * kTokens + r / G, g = r % G;
    const bool row_valid = tok < a.n_q;
    const int q_pos = a.q_pos0 + tok;
    const int tile_min_pos = a.q_pos0 + tok_first + i * kTokens;
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
    if (a.n_split > 1) {  // normalised fp32 partial + (max, sum) for k_prefill_combine
      const int64_t prow = (static_cast<int64_t>(sp) * a.n_q + tok) * a.Hq +
                           static_cast<int64_t>(h) * G + g;
#pragma unroll
      for (int c0 = 0; c0 < kD; c0 += 32) {
        uint32_t o[32];
        tmem_ld16_nowait(tO + c0, o);
        tmem_ld16_nowait(tO + c0 + 16, o + 16);
        tmem_wait_ld();
        if (row_valid) {
          float4* dst = reinterpret_cast<float4*>(a.part_o + prow * kD + c0);
#pragma unroll
          for (int k = 0; k < 8; ++k)
            dst[k] = make_float4(__uint_as_float(o[4 * k]) * inv, __uint_as_float(o[4 * k + 1]) * inv,
                                 __uint_as_float(o[4 * k + 2]) * inv, __uint_as_float(o[4 * k + 3]) * inv);
        }
      }
      if (row_valid) a.part_ml[prow] = make_float2(m, l);
    } else {
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
  }
  fence_before();
  __syncthreads();
  if (warp == 9) {
    fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
  }
}

// Merge of key-split partials: one 128-thread CTA per (token, query head)
// row, thread = head dim.  out = sum_s w_s O_s / sum_s w_s with
// w_s = l_s 2^(m_s - max_s m_s) (O_s normalised by its own l_s).
__global__ void __launch_bounds__(128) k_prefill_combine(const float* __restrict__ part_o,
                                                          const float2* __restrict__ part_ml,
                                                          int n_split, int64_t rows,
                                                          __nv_bfloat16* __restrict__ out) {
  const int64_t row = blockIdx.x;
  const int d = threadIdx.x;
  float M = -INFINITY;
  for (int s = 0; s < n_split; ++s) M = fmaxf(M, __ldg(&part_ml[s * rows + row]).x);
  float acc = 0.f, wsum = 0.f;
  for (int s = 0; s < n_split; ++s) {
    const float2 ml = __ldg(&part_ml[s * rows + row]);
    const float w = (ml.x == -INFINITY || ml.y <= 0.f) ? 0.f : ml.y * exp2f(ml.x - M);
    acc += w * __ldg(&part_o[(s * rows + row) * kD + d]);
    wsum += w;
  }
  out[row * kD + d] = __float2bfloat16_rn(wsum > 0.f ? acc / wsum : 0.f);
}

__global__ void __launch_bounds__(kThreads, 1)
    k_prefill_attn_k128p(const __grid_constant__ CUtensorMap pool_map,
                        const __grid_constant__ CUtensorMap row_map, const PrefillArgs a) {
  using namespace p3;
  constexpr int kKeys = p3::kKeys, kKvAtom = p3::kKvAtom, kKvTile = p3::kKvTile;
  constexpr int kOffQ = p3::kOffQ, kOffK = p3::kOffK, kOffV = p3::kOffV, kOffBar = p3::kOffBar;
  constexpr int kBarQ = p3::kBarQ, kBarKFull = p3::kBarKFull, kBarVFull = p3::kBarVFull;
  constexpr int kBarKEmpty = p3::kBarKEmpty, kBarVEmpty = p3::kBarVEmpty;
  constexpr int kBarSFull = p3::kBarSFull, kBarPFull = p3::kBarPFull, kBarODone = p3::kBarODone;
  constexpr int kBarPHalf = p3::kBarPHalf, kBarOFree = p3::kBarOFree;
  constexpr int kBarCount = p3::kBarCount;
  constexpr int kStagesV = p3::kStagesV;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // Persistent: CTA c serves work items c, c + gridDim.x, ... of the
  // (query block, KV head) list in heaviest-first order; ring stages and
  // barrier parities run on a per-CTA tile counter across items.
  const int n_items = a.n_blocks * a.Hkv;
  const uint32_t sQ = smem_u32(smem + kOffQ), sK = smem_u32(smem + kOffK);
  const uint32_t sV = smem_u32(smem + kOffV), bars = smem_u32(smem + kOffBar);
  auto bar = [&](int i) { return bars + 8u * static_cast<uint32_t>(i); };
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + kOffBar + 8 * kBarCount);

  struct Item {
    int h, tok_first, n_keys, n_tiles;
  };
  auto item_of = [&](int it) {
    Item x;
    // Head-major (the CTAs of a wave share one head's K/V in L2: at 32K
    // keys the 8 heads' K/V together exceed L2), heaviest block first.
    const int qb = a.n_blocks - 1 - it % a.n_blocks;
    x.h = it / a.n_blocks;
    x.tok_first = qb * kQTiles * kTokens;
    const int tok_last = min(a.n_q, x.tok_first + kQTiles * kTokens) - 1;
    x.n_keys = a.q_pos0 + tok_last + 1;
    x.n_tiles = (x.n_keys + kKeys - 1) / kKeys;
    return x;
  };

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
      mbar_init(bar(kBarOFree + i), kRows);
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
    const int C = min(a.page_size, 64), lanes_per_chunk = C / kPer;
    const uint32_t chunk_mask = lanes_per_chunk >= 32 ? 0xffffffffu : ((1u << lanes_per_chunk) - 1u);
    const int my_chunk_lane0 = lane - lane % lanes_per_chunk;
    const int op = warp == 8 ? 0 : 1;
    const int nst = op == 0 ? kStagesK : kStagesV;
    int g = 0;  // tile counter across items
    for (int it = blockIdx.x; it < n_items; it += gridDim.x) {
    const Item x = item_of(it);
    const int n_keys = x.n_keys, n_tiles = x.n_tiles;
    const int col = op == 0 ? x.h * kD : (a.Hkv + x.h) * kD;
    for (int j = 0; j < n_tiles; ++j, ++g) {
      const int s = g % nst;
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
        if (g >= nst) mbar_wait(bar((op == 0 ? kBarKEmpty : kBarVEmpty) + s), ((g / nst) + 1) & 1);
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
    auto issue_s = [&](int i, int g) {
      const uint32_t a0 = q_lo + ((i * kTile) >> 4), b0 = k_lo + (((g % kStagesK) * kKvTile) >> 4);
#pragma unroll
      for (int k = 0; k < kD / 16; ++k) {
        const uint32_t ao = ((k >> 2) * kAtom + (k & 3) * 32) >> 4;
        const uint32_t bo = ((k >> 2) * kKvAtom + (k & 3) * 32) >> 4;
        mma_ss_elect(tS(i), a0 + ao, b0 + bo, kHi, kIdescS, k > 0 ? 1u : 0u);
      }
      commit_elect(bar(kBarSFull + i));
    };
    auto issue_pv = [&](int i, int g, int j) {
      const uint32_t b0 = v_lo + (((g % kStagesV) * kKvTile) >> 4);
      mbar_wait(bar(kBarPHalf + i), g & 1);  // P_i keys [0, 64) and O_i rescaled
      fence_after();
#pragma unroll
      for (int k = 0; k < kKeys / 32; ++k)
        mma_ts_elect(tO(i), tS(i) + k * 8, b0 + ((k * 2048) >> 4), kHi, kIdescO,
                     (j > 0 || k > 0) ? 1u : 0u);
      mbar_wait(bar(kBarPFull + i), g & 1);  // keys [64, 128)
      fence_after();
#pragma unroll
      for (int k = kKeys / 32; k < kKeys / 16; ++k)
        mma_ts_elect(tO(i), tS(i) + k * 8, b0 + ((k * 2048) >> 4), kHi, kIdescO, 1u);
    };
    int g0 = 0, k_item = 0;
    for (int it = blockIdx.x; it < n_items; it += gridDim.x, ++k_item) {
      const Item x = item_of(it);
      const int n_keys = x.n_keys, n_tiles = x.n_tiles;
      auto zero_tail = [&](int j, int g) {
        const int valid = n_keys - j * kKeys;
        if (valid >= kKeys) return;
        uint8_t* vb = smem + kOffV + (g % kStagesV) * kKvTile;
        for (int e = lane; e < (kKeys - valid) * 16; e += 32) {
          const int r = valid + (e >> 4), c = e & 15;
          *reinterpret_cast<uint4*>(vb + (c >> 3) * kKvAtom + r * 128 + (c & 7) * 16) =
              make_uint4(0, 0, 0, 0);
        }
        fence_proxy_async();
        __syncwarp();
      };
      mbar_wait(bar(kBarQ), k_item & 1);
      mbar_wait(bar(kBarKFull + g0 % kStagesK), (g0 / kStagesK) & 1);
      fence_after();
      issue_s(0, g0);
      issue_s(1, g0);
      commit_elect(bar(kBarKEmpty + g0 % kStagesK));
      for (int j = 0; j < n_tiles; ++j) {
        const int g = g0 + j;
        const int sv = g % kStagesV;
        mbar_wait(bar(kBarVFull + sv), (g / kStagesV) & 1);
        if (j == n_tiles - 1) zero_tail(j, g);
        const bool next = j + 1 < n_tiles;
        const int sk = (g + 1) % kStagesK;
        if (next) mbar_wait(bar(kBarKFull + sk), ((g + 1) / kStagesK) & 1);
        fence_after();
        for (int i = 0; i < kQTiles; ++i) {
          // The previous item's epilogue must have read O_i before the first
          // PV of this item overwrites it.
          if (j == 0 && k_item > 0) {
            mbar_wait(bar(kBarOFree + i), (k_item - 1) & 1);
            fence_after();
          }
          issue_pv(i, g, j);
          if (!next) commit_elect(bar(kBarODone + i));
          if (next) issue_s(i, g + 1);
        }
        commit_elect(bar(kBarVEmpty + sv));
        if (next) commit_elect(bar(kBarKEmpty + sk));
      }
      g0 += n_tiles;
    }
  } else {
    // ---------------- softmax warpgroups (persistent) ----------------
    const int i = warp >> 2;
    const int r = tid & (kRows - 1);
    const int G = a.Hq / a.Hkv;
    const uint32_t lane_off = static_cast<uint32_t>((warp & 3) * 32) << 16;
    const uint32_t tS = tmem + i * 128 + lane_off, tO = tmem + 256 + i * 128 + lane_off;
    const uint32_t qa = sQ + i * kTile;
    // Q rows of item `it` into this tile's shared-memory slot (cp.async).
    auto load_q = [&](int it) {
      const Item x = item_of(it);
      const int tok = x.tok_first + i * kTokens + r / G, g = r % G;
      const __nv_bfloat16* qrow =
          a.q + (static_cast<int64_t>(tok) * a.Hq + static_cast<int64_t>(x.h) * G + g) * kD;
#pragma unroll
      for (int c = 0; c < 16; ++c) cp_async16(qa + sw128(r, c), qrow + c * 8, tok < a.n_q);
      asm volatile("cp.async.commit_group;" ::: "memory");
    };
    auto publish_q = [&]() {
      asm volatile("cp.async.wait_group 0;" ::: "memory");
      fence_proxy_async();
      mbar_arrive(bar(kBarQ));
    };
    if (static_cast<int>(blockIdx.x) < n_items) {
      load_q(blockIdx.x);
      publish_q();
    }
    const float sl2 = a.scale_log2;
    int g0 = 0, k_item = 0;
    for (int it = blockIdx.x; it < n_items; it += gridDim.x, ++k_item) {
    const Item x = item_of(it);
    const int h = x.h, tok_first = x.tok_first, n_tiles = x.n_tiles;
    const int tok = tok_first + i * kTokens + r / G, g = r % G;
    const bool row_valid = tok < a.n_q;
    const int q_pos = a.q_pos0 + tok;
    const int tile_min_pos = a.q_pos0 + tok_first + i * kTokens;
    float m = -INFINITY, l = 0.f;
    for (int j = 0; j < n_tiles; ++j) {
      const int gt = g0 + j;
      mbar_wait(bar(kBarSFull + i), gt & 1);
      fence_after();
      uint32_t sr[kKeys];
#pragma unroll
      for (int c0 = 0; c0 < kKeys; c0 += 16) tmem_ld16_nowait(tS + c0, sr + c0);
      tmem_wait_ld();
      const int key0 = j * kKeys;
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
      l = l * alpha + psum;
      m = m_new;
    }
    // The last PV of this item retired (S_i reads of Q_i too): the next
    // item's Q can be loaded under this item's epilogue.
    mbar_wait(bar(kBarODone + i), k_item & 1);
    fence_after();
    const int it_next = it + static_cast<int>(gridDim.x);
    if (it_next < n_items) load_q(it_next);
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
    fence_before();
    mbar_arrive(bar(kBarOFree + i));
    if (it_next < n_items) publish_q();
    g0 += n_tiles;
    }
  }
  fence_before();
  __syncthreads();
  if (warp == 9) {
    fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
  }
}


__global__ void __launch_bounds__(p3::kThreadsS, 1)
    k_prefill_attn_k128s(const __grid_constant__ CUtensorMap pool_map,
                        const __grid_constant__ CUtensorMap row_map, const PrefillArgs a) {
  using namespace p3;
  constexpr int kKeys = p3::kKeys, kKvAtom = p3::kKvAtom, kKvTile = p3::kKvTile;
  constexpr int kOffQ = p3::kOffQ, kOffK = p3::kOffK, kOffV = p3::kOffV, kOffBar = p3::kOffBar;
  constexpr int kBarQ = p3::kBarQ, kBarKFull = p3::kBarKFull, kBarVFull = p3::kBarVFull;
  constexpr int kBarKEmpty = p3::kBarKEmpty, kBarVEmpty = p3::kBarVEmpty;
  constexpr int kBarSFull = p3::kBarSFull, kBarPFull = p3::kBarPFull, kBarODone = p3::kBarODone;
  constexpr int kBarCount = p3::kBarCount;
  constexpr int kStagesV = p3::kStagesV;
  constexpr int kSoftmaxThreads = p3::kSoftmaxThreadsS;  // two threads per query row
  constexpr int kWarpK = 16, kWarpMma = 17, kWarpV = 18;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int qb = a.n_blocks - 1 - static_cast<int>(blockIdx.x);
  const int h = blockIdx.y;
  const uint32_t sQ = smem_u32(smem + kOffQ), sK = smem_u32(smem + kOffK);
  const uint32_t sV = smem_u32(smem + kOffV), bars = smem_u32(smem + kOffBar);
  auto bar = [&](int i) { return bars + 8u * static_cast<uint32_t>(i); };
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + kOffBar + 8 * kBarCount);

  const int tok_first = qb * kQTiles * kTokens;
  const int tok_last = min(a.n_q, tok_first + kQTiles * kTokens) - 1;
  const int n_keys = a.q_pos0 + tok_last + 1;
  const int n_tiles = (n_keys + kKeys - 1) / kKeys;

  if (warp == kWarpMma) {
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
      mbar_init(bar(kBarPFull + i), 2 * kRows);
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

  if (warp == kWarpK || warp == kWarpV) {
    // ---------------- producers: K (warp 8) / V (warp 10), lane l owns
    // positions kPer*l .. kPer*l + kPer - 1 of the tile ----------------
    const int C = min(a.page_size, 64), lanes_per_chunk = C / kPer;
    const uint32_t chunk_mask = lanes_per_chunk >= 32 ? 0xffffffffu : ((1u << lanes_per_chunk) - 1u);
    const int my_chunk_lane0 = lane - lane % lanes_per_chunk;
    const int op = warp == kWarpK ? 0 : 1;
    const int nst = op == 0 ? kStagesK : kStagesV;
    const int col = op == 0 ? h * kD : (a.Hkv + h) * kD;
    for (int j = 0; j < n_tiles; ++j) {
      const int s = j % nst;
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
        if (j >= nst) mbar_wait(bar((op == 0 ? kBarKEmpty : kBarVEmpty) + s), ((j / nst) + 1) & 1);
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
  } else if (warp == kWarpMma) {
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
      mbar_wait(bar(kBarPFull + i), j & 1);
      fence_after();
      if (lane == 0) PF_EV(0xE00 | (i << 8) | (j & 0xff));
      const uint32_t b0 = v_lo + (((j % kStagesV) * kKvTile) >> 4);
#pragma unroll
      for (int k = 0; k < kKeys / 16; ++k)
        mma_ts_elect(tO(i), tS(i) + k * 8, b0 + ((k * 2048) >> 4), kHi, kIdescO,
                     (j > 0 || k > 0) ? 1u : 0u);
    };
    auto zero_tail = [&](int j) {
      const int valid = n_keys - j * kKeys;
      if (valid >= kKeys) return;
      uint8_t* vb = smem + kOffV + (j % kStagesV) * kKvTile;
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
    for (int j = 0; j < n_tiles; ++j) {
      const int sv = j % kStagesV;
      mbar_wait(bar(kBarVFull + sv), (j / kStagesV) & 1);
      if (j == n_tiles - 1) zero_tail(j);
      const bool next = j + 1 < n_tiles;
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
    // ---------------- softmax: four warpgroups, two threads per row -------
    // Warps 8 i + 4 hf + q: query tile i, key/column half hf, TMEM lane
    // quarter q (= warp % 4, the quarter a warp may access).  The two halves
    // of a row exchange their maxima through shared memory (a 64-thread
    // named barrier per (tile, quarter)), so both use the same reference
    // max; row sums stay per half until the epilogue.
    const int i = warp >> 3, hf = (warp >> 2) & 1, q = warp & 3;
    const int r = q * 32 + lane;
    const int G = a.Hq / a.Hkv;
    const int tok = tok_first + i * kTokens + r / G, g = r % G;
    const bool row_valid = tok < a.n_q;
    const int q_pos = a.q_pos0 + tok;
    const int tile_min_pos = a.q_pos0 + tok_first + i * kTokens;
    const uint32_t lane_off = static_cast<uint32_t>(q * 32) << 16;
    const uint32_t tS = tmem + i * 128 + lane_off, tO = tmem + 256 + i * 128 + lane_off;
    float* red = reinterpret_cast<float*>(smem + p3::kOffRed);  // [2 buf][2 tile][2 half][128]
    const uint32_t pair_bar = 1 + i * 4 + q;
    auto pair_sync = [&]() {
      asm volatile("bar.sync %0, 64;" ::"r"(pair_bar) : "memory");
    };
    {
      const __nv_bfloat16* qrow =
          a.q + (static_cast<int64_t>(tok) * a.Hq + static_cast<int64_t>(h) * G + g) * kD;
      const uint32_t qa = sQ + i * kTile;
#pragma unroll
      for (int c = 8 * hf; c < 8 * hf + 8; ++c) cp_async16(qa + sw128(r, c), qrow + c * 8, row_valid);
      asm volatile("cp.async.commit_group;" ::: "memory");
      asm volatile("cp.async.wait_group 0;" ::: "memory");
      fence_proxy_async();
      mbar_arrive(bar(kBarQ));
    }
    constexpr int kHalf = kKeys / 2;  // S columns per thread
    const int col0 = hf * kHalf;
    const float sl2 = a.scale_log2;
    float m = -INFINITY, l = 0.f;
    for (int j = 0; j < n_tiles; ++j) {
      mbar_wait(bar(kBarSFull + i), j & 1);
      fence_after();
      uint32_t sr[kHalf];
#pragma unroll
      for (int c0 = 0; c0 < kHalf; c0 += 16) tmem_ld16_nowait(tS + col0 + c0, sr + c0);
      tmem_wait_ld();
      const int key0 = j * kKeys + col0;
      const bool need_mask =
          __any_sync(0xffffffffu, key0 + kHalf - 1 > tile_min_pos || !row_valid);
      if (need_mask) {
        const int lim = row_valid ? q_pos - key0 : -1;
#pragma unroll
        for (int c = 0; c < kHalf; ++c) sr[c] = c > lim ? __float_as_uint(-INFINITY) : sr[c];
      }
      float mx[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
      for (int c = 0; c < kHalf; c += 8) {
#pragma unroll
        for (int k = 0; k < 4; ++k)
          mx[k] = fmaxf(mx[k], fmaxf(__uint_as_float(sr[c + 2 * k]), __uint_as_float(sr[c + 2 * k + 1])));
      }
      float rmax = fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3]));
      {  // exchange with the other half of the row (double-buffered by tile parity)
        float* rb = red + (((j & 1) * 2 + i) * 2) * 128;
        rb[hf * 128 + r] = rmax;
        pair_sync();  // also orders the other half's S loads before our P stores
        rmax = fmaxf(rmax, rb[(hf ^ 1) * 128 + r]);
      }
      const float tmax = rmax * sl2;
      const bool bump = tmax > m + 8.f;
      const float m_new = bump ? tmax : m;
      const float alpha = (bump && m != -INFINITY) ? ex2_mufu(m - m_new) : 1.f;
      const float neg_m = m_new == -INFINITY ? 0.f : -m_new;
      const uint64_t sc2 = f2pack(sl2, sl2), nm2 = f2pack(neg_m, neg_m);
      uint64_t acc[2] = {0ull, 0ull};
      auto make_p = [&](auto poly) {
#pragma unroll
        for (int c = 0; c < kHalf; c += 2) {
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
      if (need_mask) make_p(std::false_type{});
      else make_p(std::true_type{});
      float ps[4];
      f2unpack(acc[0], ps[0], ps[1]);
      f2unpack(acc[1], ps[2], ps[3]);
      const float psum = (ps[0] + ps[1]) + (ps[2] + ps[3]);
      // P columns of this half: keys [col0, col0 + 64) -> packed [col0 / 2, col0 / 2 + 32).
#pragma unroll
      for (int c0 = 0; c0 < kHalf / 2; c0 += 16) tmem_st16_nowait(tS + col0 / 2 + c0, sr + c0);
      if (j > 0 && __any_sync(0xffffffffu, alpha != 1.f)) {
#pragma unroll
        for (int c0 = 0; c0 < kD / 2; c0 += 32) {
          uint32_t o[32];
          tmem_ld16_nowait(tO + hf * (kD / 2) + c0, o);
          tmem_ld16_nowait(tO + hf * (kD / 2) + c0 + 16, o + 16);
          tmem_wait_ld();
#pragma unroll
          for (int k = 0; k < 32; ++k) o[k] = __float_as_uint(__uint_as_float(o[k]) * alpha);
          tmem_st16_nowait(tO + hf * (kD / 2) + c0, o);
          tmem_st16_nowait(tO + hf * (kD / 2) + c0 + 16, o + 16);
        }
      }
      tmem_wait_st();
      fence_before();
      mbar_arrive(bar(kBarPFull + i));
      l = l * alpha + psum;
      m = m_new;
    }
    {  // row sum of both halves (buffer 0 of tile i is free: last use was >= 2 tiles ago
       // or, for n_tiles == 1, read before the pair barrier below... use the epilogue slot)
      float* rb = red + (4 * 2 + i * 2) * 128;
      rb[hf * 128 + r] = l;
      pair_sync();
      l += rb[(hf ^ 1) * 128 + r];
    }
    mbar_wait(bar(kBarODone + i), 0);
    fence_after();
    const float inv = l > 0.f ? 1.f / l : 0.f;
    __nv_bfloat16* orow =
        a.out + (static_cast<int64_t>(tok) * a.Hq + static_cast<int64_t>(h) * G + g) * kD;
#pragma unroll
    for (int c0 = hf * (kD / 2); c0 < hf * (kD / 2) + kD / 2; c0 += 32) {
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
  if (warp == kWarpMma) {
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
  return D == kD && Hkv >= 1 && Hq == 8 * Hkv && pow2 && page_size >= 8 && page_size <= 1024;
}

int prefill_attn_box_rows(int page_size) { return page_size < kKeys ? page_size : kKeys; }

int launch_prefill_attn(const PoolTensorMap& page_map, const PoolTensorMap& row_map, int layer,
                         int page_size, int64_t pool_rows, const int32_t* slots, const void* q,
                         int q_pos0, int n_q, int Hq, int Hkv, int D, float scale, void* out,
                         cudaStream_t s) {
  if (!prefill_attn_supported(page_size, Hq, Hkv, D) || n_q <= 0) return 0;
  // Kernel selection (A/B of the layouts): MICROKV_PREFILL_VARIANT
  // = "128" (default: 128-key tiles, one S slot per query tile, one CTA per
  // work item), "128p" (the same as persistent CTAs over the work items),
  // "128s" (two softmax threads per row), "64" (64-key tiles, two S slots),
  // "2sm" (CTA pair, cta_group::2).  Read per launch.
  const char* ev = std::getenv("MICROKV_PREFILL_VARIANT");
  const std::string variant = ev != nullptr ? ev : "128";
  const bool use_2sm = variant == "2sm";
  const bool use_k64 = variant == "64";
  const bool use_k128s = variant == "128s";
  const bool use_k128p = variant == "128p";
  const bool use_k128 = !use_2sm && !use_k64 && !use_k128s && !use_k128p;
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
  a.n_blocks = (n_q + kQTiles * kTokens - 1) / (kQTiles * kTokens);  // 32 tokens per CTA / pair
  a.scale_log2 = scale * 1.4426950408889634f;
  a.pool_rows = static_cast<int>(pool_rows);
  a.n_split = 1;
  a.part_o = nullptr;
  a.part_ml = nullptr;
  int launches = 1;
  CUtensorMap m, mr;
  std::memcpy(&m, page_map.bytes, sizeof(m));
  std::memcpy(&mr, row_map.bytes, sizeof(mr));
#if defined(PF_TRACE) || defined(PF_PROF)
  unsigned long long* tr = nullptr;
  cudaMalloc(&tr, 65536 * sizeof(unsigned long long));
  cudaMemset(tr, 0, 65536 * sizeof(unsigned long long));
  a.trace = tr;
#endif
  if (use_k128p) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int items = a.n_blocks * Hkv;
    k_prefill_attn_k128p<<<items < sms ? items : sms, kThreads, p3::kSmem + 1024, s>>>(m, mr, a);
  } else if (use_k128s) {
    const dim3 grid(a.n_blocks, Hkv);
    k_prefill_attn_k128s<<<grid, p3::kThreadsS, p3::kSmemS + 1024, s>>>(m, mr, a);
  } else if (use_k128) {
    // MICROKV_PREFILL_SPLIT=n: split each work item's keys over n CTAs and
    // merge by k_prefill_combine.  Off by default: for the short
    // balanced-PD tails it was meant for (fewer than two waves of items)
    // the fp32 partials' extra traffic and the second launch cost more than
    // the filled SMs gain (2K tail 47 -> 76-91 us, 4K tail 145 -> 166-209 us).
    const int lightest_keys = q_pos0 + (n_q < kQTiles * kTokens ? n_q : kQTiles * kTokens);
    const int tiles_min = (lightest_keys + p3::kKeys - 1) / p3::kKeys;
    int split = 1;
    if (const char* e = std::getenv("MICROKV_PREFILL_SPLIT")) split = std::atoi(e);
    split = split < 1 ? 1 : (split > 8 ? 8 : split);
    if (split > tiles_min) split = tiles_min;  // every split gets >= 1 key tile
    a.n_split = split;
    void* ws = nullptr;
    const int64_t rows = static_cast<int64_t>(n_q) * Hq;
    if (split > 1) {
      const size_t bytes_o = sizeof(float) * split * rows * kD;
      if (cudaMallocAsync(&ws, bytes_o + sizeof(float2) * split * rows, s) != cudaSuccess) return 0;
      a.part_o = static_cast<float*>(ws);
      a.part_ml = reinterpret_cast<float2*>(static_cast<char*>(ws) + bytes_o);
    }
    const dim3 grid(a.n_blocks * split, Hkv);
    k_prefill_attn_k128<<<grid, kThreads, p3::kSmem + 1024, s>>>(m, mr, a);
    if (split > 1) {
      k_prefill_combine<<<static_cast<unsigned>(rows), kD, 0, s>>>(a.part_o, a.part_ml, split, rows,
                                                                    a.out);
      cudaFreeAsync(ws, s);
      launches = 2;
    }
  } else if (use_2sm) {
    const dim3 grid(2 * a.n_blocks, Hkv);
    k_prefill_attn_2sm<<<grid, p2::kThreads, p2::kSmem + 1024, s>>>(m, mr, a);
  } else if (use_k64) {
    const dim3 grid(a.n_blocks, Hkv);
    k_prefill_attn_tc<<<grid, kThreads, kSmem + 1024, s>>>(m, mr, a);
  }
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
  // Per device (called once per device at cache creation): the kernels'
  // dynamic shared memory above 48 KiB.
  cudaFuncSetAttribute(k_prefill_attn_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem + 1024);
  cudaFuncSetAttribute(k_prefill_attn_2sm, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       p2::kSmem + 1024);
  cudaFuncSetAttribute(k_prefill_attn_k128, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       p3::kSmem + 1024);
  cudaFuncSetAttribute(k_prefill_attn_k128s, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       p3::kSmemS + 1024);
  cudaFuncSetAttribute(k_prefill_attn_k128p, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       p3::kSmem + 1024);
  cudaFuncAttributes a;
  cudaFuncGetAttributes(&a, k_prefill_attn_tc);
  cudaFuncGetAttributes(&a, k_prefill_attn_2sm);
  cudaFuncGetAttributes(&a, k_prefill_attn_k128);
  cudaFuncGetAttributes(&a, k_prefill_attn_k128s);
  cudaFuncGetAttributes(&a, k_prefill_attn_k128p);
  cudaFuncGetAttributes(&a, k_prefill_combine);
}

}  // namespace mkv
