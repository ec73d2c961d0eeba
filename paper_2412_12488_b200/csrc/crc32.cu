// crc32.cu — CRC-32 (IEEE 802.3, reflected, polynomial 0xEDB88320) of a
// device buffer, the checksum of the reference's KV write frames
// (Crc32, transport.cc:14-28; frame layout transport.h:6-12).
//
// The reference computes it byte by byte on the host (Sarwate's table
// loop).  Here the payload never leaves HBM before it is checksummed:
//
//  * CRC is linear over GF(2): with raw(M) the register after M from a zero
//    start, raw(A || B) = raw(A) * x^(8|B|) mod P  xor  raw(B), and the
//    standard CRC is raw(M) xor (0xFFFFFFFF * x^(8|M|)) xor 0xFFFFFFFF.
//    Leading zero bytes do not change raw(M).
//  * The 32-byte-aligned body is cut into equal items (one per warp of a
//    single wave), zero-padded at the FRONT so every item is full.  Inside
//    an item each lane owns one contiguous segment (32-byte vector loads;
//    segments of neighbouring lanes are sector-complete, so DRAM traffic is
//    exactly the body) and runs the slice-by-4 table loop over it: per
//    4-byte word four independent lookups, so a lane's dependency chain
//    waits on shared memory once per word.  The four 256-entry tables are
//    replicated 32x in shared memory (entry e, copy `lane` at word
//    32e + lane, 128 KiB per CTA): every lookup of a warp is bank-conflict
//    free.  ~3.75 instructions and one LDS per byte per lane.
//  * The grid is persistent (one 32-warp CTA per SM at most); CTA b owns
//    32 consecutive items, so the number of bytes after lane l of warp w of
//    CTA b is seg*(31-l) + item*(31-w) + chunk*(G-1-b) + tail.  The host
//    precomputes x^(8 * that) as a [32 x 32] (lane, warp) table and a
//    per-CTA factor; each lane multiplies its register by both (two
//    branch-free 32-step GF(2) products), the lanes' terms are XORed and
//    one atomicXor per warp adds them into the result.  No serial tail:
//    the unaligned head, the tail (< 32 bytes each) and the init/xorout
//    term are folded in by one thread.
//
// Bound: HBM read of the buffer (one pass), or the per-SM shared-memory
// lookup rate (1 lookup/byte, 32 per clock) — both ~7-9 TB/s on B200.
#include <cuda_runtime.h>

#include <cstdint>
#include <mutex>

#include "kernels.cuh"

namespace mkv {

namespace {

constexpr uint32_t kPoly = 0xEDB88320u;
constexpr uint32_t kOne = 1u << 31;  // x^0 in the reflected representation
constexpr int kCrcThreads = 1024;
constexpr int kCrcWarps = kCrcThreads / 32;
constexpr size_t kTabWords = 4 * 256 * 32;
constexpr size_t kCrcSmem = kTabWords * sizeof(uint32_t);  // 128 KiB

struct CrcTables {
  uint32_t v[4][256];  // slice-by-4: v[k][b] = raw CRC of byte b followed by k zero bytes
};

constexpr CrcTables MakeTables() {
  CrcTables t{};
  for (uint32_t i = 0; i < 256; ++i) {
    uint32_t c = i;
    for (int k = 0; k < 8; ++k) c = (c & 1u) ? kPoly ^ (c >> 1) : c >> 1;
    t.v[0][i] = c;
  }
  for (int k = 1; k < 4; ++k)
    for (uint32_t i = 0; i < 256; ++i)
      t.v[k][i] = (t.v[k - 1][i] >> 8) ^ t.v[0][t.v[k - 1][i] & 0xffu];
  return t;
}

__device__ const CrcTables kDevTables = MakeTables();

// a(x) * b(x) mod P(x), reflected bit order (bit 31 = x^0): host version
// (loop over the set bits of a).
inline uint32_t multmodp(uint32_t a, uint32_t b) {
  uint32_t m = 1u << 31, p = 0;
  for (;;) {
    if (a & m) {
      p ^= b;
      if ((a & (m - 1)) == 0) break;
    }
    m >>= 1;
    b = (b & 1u) ? (b >> 1) ^ kPoly : b >> 1;
  }
  return p;
}

// Device version: 32 branch-free steps (a may differ across lanes).
__device__ __forceinline__ uint32_t mulmod_dev(uint32_t a, uint32_t b) {
  uint32_t p = 0;
#pragma unroll
  for (int i = 0; i < 32; ++i) {
    p ^= b & static_cast<uint32_t>(static_cast<int32_t>(a << i) >> 31);
    b = (b >> 1) ^ (kPoly & static_cast<uint32_t>(static_cast<int32_t>(b << 31) >> 31));
  }
  return p;
}

// x^(8 n) mod P: the multiplier that appends n zero bytes.
uint32_t x8n(uint64_t n) {
  static const auto pow2 = [] {
    struct T {
      uint32_t v[64];
    } t{};
    uint32_t p = 1u << 30;  // x^1
    t.v[0] = p;
    for (int k = 1; k < 64; ++k) t.v[k] = p = multmodp(p, p);  // x^(2^k)
    return t;
  }();
  uint32_t p = kOne;
  int k = 3;  // 8 n = n * 2^3
  while (n) {
    if (n & 1) p = multmodp(pow2.v[k], p);
    n >>= 1;
    ++k;
  }
  return p;
}

struct alignas(32) V32 {
  uint32_t w[8];
};

__device__ __forceinline__ V32 ld_v32(const void* p) {
  V32 v;
  asm volatile("ld.global.nc.L1::no_allocate.v8.u32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
               : "=r"(v.w[0]), "=r"(v.w[1]), "=r"(v.w[2]), "=r"(v.w[3]), "=r"(v.w[4]),
                 "=r"(v.w[5]), "=r"(v.w[6]), "=r"(v.w[7])
               : "l"(p));
  return v;
}

constexpr int kMaxGrid = 160;  // >= SM count (148)

struct CrcParams {
  const uint8_t* head;   // unaligned prefix, head_len < 32 bytes
  const uint8_t* body;   // 32-byte aligned, n_body % 32 == 0
  const uint8_t* tail;   // tail_len < 32 bytes
  int32_t head_len, tail_len;
  int64_t pad;           // zero bytes in front of the body (grid * 32 * item_bytes - n_body)
  int32_t m;             // 32-byte vectors per lane segment
  uint32_t* out;         // zeroed before the launch; warps atomicXor into it
  uint32_t x_after_head; // x^(8 * (n - head_len))
  uint32_t init_term;    // 0xFFFFFFFF * x^(8 n) xor 0xFFFFFFFF
  uint32_t cta_k[kMaxGrid];   // x^(8 * (chunk * (G - 1 - b) + tail_len))
  uint32_t lw_k[32][32];      // [warp][lane]: x^(8 * (seg * (31 - lane) + item * (31 - warp)))
};

__global__ void __launch_bounds__(kCrcThreads, 1) k_crc32(const __grid_constant__ CrcParams p) {
  extern __shared__ uint32_t tab[];  // [4][256][32]
  {
    const uint32_t* src = &kDevTables.v[0][0];
#pragma unroll 8
    for (int i = threadIdx.x; i < static_cast<int>(kTabWords); i += kCrcThreads)
      tab[i] = src[i >> 5];
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // Byte address of lane's copy of entry 0 in table k: k * 32 KiB + lane * 4.
  const uint32_t tb = static_cast<uint32_t>(__cvta_generic_to_shared(tab)) + lane * 4;
  auto lk = [&](uint32_t byte_addr) {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(byte_addr));
    return v;
  };
  // c = raw CRC register; one 4-byte word: c ^= w, then four table reads.
  auto word = [&](uint32_t c, uint32_t w) {
    c ^= w;
    const uint32_t a3 = tb + 3 * 32768 + ((c << 7) & 0x7f80u);
    const uint32_t a2 = tb + 2 * 32768 + ((c >> 1) & 0x7f80u);
    const uint32_t a1 = tb + 1 * 32768 + ((c >> 9) & 0x7f80u);
    const uint32_t a0 = tb + ((c >> 17) & 0x7f80u);
    return (lk(a3) ^ lk(a2)) ^ (lk(a1) ^ lk(a0));
  };

  const int64_t seg_bytes = 32ll * p.m;
  const int64_t item = static_cast<int64_t>(blockIdx.x) * kCrcWarps + warp;
  // Byte offset of this lane's segment in the body (negative = padding, a
  // prefix of the message: the register stays 0 over it).
  const int64_t seg = (item * 32 + lane) * seg_bytes - p.pad;
  int k = 0;
  if (seg < 0) {
    const int64_t skip = -seg / 32;
    k = static_cast<int>(skip < p.m ? skip : p.m);
  }
  const uint8_t* src = p.body + seg;
  uint32_t c = 0;
  // Two vectors per step, the next step's pair loaded before this one is
  // folded, so each lane keeps 64 bytes in flight behind the table work.
  V32 va, vb;
  if (k + 1 < p.m) {
    va = ld_v32(src + 32ll * k);
    vb = ld_v32(src + 32ll * (k + 1));
  }
  for (; k + 1 < p.m; k += 2) {
    V32 na, nb;
    const bool more = k + 3 < p.m;
    if (more) {
      na = ld_v32(src + 32ll * (k + 2));
      nb = ld_v32(src + 32ll * (k + 3));
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) c = word(c, va.w[j]);
#pragma unroll
    for (int j = 0; j < 8; ++j) c = word(c, vb.w[j]);
    if (more) {
      va = na;
      vb = nb;
    }
  }
  if (k < p.m) {
    const V32 vl = ld_v32(src + 32ll * k);
#pragma unroll
    for (int j = 0; j < 8; ++j) c = word(c, vl.w[j]);
  }
  uint32_t t = mulmod_dev(mulmod_dev(p.cta_k[blockIdx.x], p.lw_k[warp][lane]), c);
#pragma unroll
  for (int s = 16; s > 0; s >>= 1) t ^= __shfl_xor_sync(0xffffffffu, t, s);
  if (lane == 0 && t != 0u) atomicXor(p.out, t);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    // Sarwate over the head and tail bytes (table 0, copy 0).
    uint32_t h = 0, tl = 0;
    const uint32_t t0 = static_cast<uint32_t>(__cvta_generic_to_shared(tab));
    for (int i = 0; i < p.head_len; ++i) h = lk(t0 + (((h ^ p.head[i]) & 0xffu) << 7)) ^ (h >> 8);
    for (int i = 0; i < p.tail_len; ++i) tl = lk(t0 + (((tl ^ p.tail[i]) & 0xffu) << 7)) ^ (tl >> 8);
    atomicXor(p.out, mulmod_dev(p.x_after_head, h) ^ tl ^ p.init_term);
  }
}

struct CrcPlan {
  int32_t grid = 1;  // CTAs, each 32 items (one per warp)
  int32_t m = 8;     // 32-byte vectors per lane segment
};

// One wave: G <= SM count CTAs of 32 warps, at least 8 vectors (256 bytes)
// per lane so the two per-lane products stay small next to the loop.
CrcPlan plan_crc(int64_t n_body, int num_sms) {
  CrcPlan pl;
  if (n_body <= 0) return pl;
  const int64_t g_max = num_sms < kMaxGrid ? num_sms : kMaxGrid;
  int64_t m = (n_body + 1024ll * kCrcWarps * g_max - 1) / (1024ll * kCrcWarps * g_max);
  if (m < 8) m = 8;
  pl.m = static_cast<int32_t>(m);
  const int64_t chunk = 1024ll * kCrcWarps * m;
  pl.grid = static_cast<int32_t>((n_body + chunk - 1) / chunk);
  return pl;
}

}  // namespace

uint32_t crc32_x8n(uint64_t n) { return x8n(n); }

size_t crc32_workspace_bytes(int64_t, int) { return 0; }

void launch_crc32(const void* data, int64_t n, uint32_t* out, void*, cudaStream_t s,
                  int num_sms) {
  // The 128 KiB table attribute is set per device by preload_crc32_kernels().
  const auto* d = static_cast<const uint8_t*>(data);
  const uintptr_t a = reinterpret_cast<uintptr_t>(d);
  int64_t head = static_cast<int64_t>((32 - (a & 31)) & 31);
  if (head > n) head = n;
  const int64_t rest = n - head;
  const int64_t n_body = rest & ~31ll;
  const int64_t tail = rest - n_body;
  const CrcPlan pl = plan_crc(n_body, num_sms);
  static CrcParams p;  // large (5 KB); filled under the launch mutex below
  static std::mutex mu;
  std::lock_guard<std::mutex> lock(mu);
  p.head = d;
  p.head_len = static_cast<int32_t>(head);
  p.body = d + head;
  p.tail = d + head + n_body;
  p.tail_len = static_cast<int32_t>(tail);
  p.m = pl.m;
  const int64_t seg = 32ll * pl.m, item = 32 * seg, chunk = kCrcWarps * item;
  p.pad = pl.grid * chunk - n_body;  // n_body = 0: the whole grid is padding
  p.out = out;
  p.x_after_head = x8n(static_cast<uint64_t>(n - head));
  p.init_term = multmodp(x8n(static_cast<uint64_t>(n)), 0xFFFFFFFFu) ^ 0xFFFFFFFFu;
  // Cached: the (lane, warp) table depends only on m.
  static int32_t cached_m = -1;
  if (cached_m != pl.m) {
    const uint32_t xs = x8n(static_cast<uint64_t>(seg)), xi = x8n(static_cast<uint64_t>(item));
    uint32_t wk = kOne;  // x^(8 * item * (31 - w)), w from 31 down
    for (int w = 31; w >= 0; --w) {
      uint32_t v = wk;   // times x^(8 * seg * (31 - l)), l from 31 down
      for (int l = 31; l >= 0; --l) {
        p.lw_k[w][l] = v;
        v = multmodp(xs, v);
      }
      wk = multmodp(xi, wk);
    }
    cached_m = pl.m;
  }
  {
    const uint32_t xc = x8n(static_cast<uint64_t>(chunk));
    uint32_t v = x8n(static_cast<uint64_t>(tail));
    for (int b = pl.grid - 1; b >= 0; --b) {
      p.cta_k[b] = v;
      v = multmodp(xc, v);
    }
  }
  cudaMemsetAsync(out, 0, sizeof(uint32_t), s);
  k_crc32<<<static_cast<unsigned>(pl.grid), kCrcThreads, kCrcSmem, s>>>(p);
}


void preload_crc32_kernels() {
  cudaFuncSetAttribute(k_crc32, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       static_cast<int>(kCrcSmem));
  cudaFuncAttributes a;
  cudaFuncGetAttributes(&a, k_crc32);
}

}  // namespace mkv
