// Micro-benchmark of slot-indexed row-copy variants for the DirectSend
// kernel (4 KiB rows, 8191 rows x 80 layers, 16-slot pages), against
// cudaMemcpyDeviceToDevice of the same bytes.  Standalone:
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o copy_variants copy_variants.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <vector>

#define CK(x)                                                                   \
  do {                                                                          \
    cudaError_t e = (x);                                                        \
    if (e != cudaSuccess) {                                                     \
      printf("CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
      return 1;                                                                 \
    }                                                                           \
  } while (0)

constexpr int W = 512;  // u64 words per row

__device__ __forceinline__ ulonglong2 ld_nc(const ulonglong2* p) {
  ulonglong2 v;
  asm volatile("ld.global.nc.L1::no_allocate.v2.u64 {%0, %1}, [%2];" : "=l"(v.x), "=l"(v.y) : "l"(p));
  return v;
}
__device__ __forceinline__ void st2(ulonglong2* p, ulonglong2 v) {
  asm volatile("st.global.v2.u64 [%0], {%1, %2};" ::"l"(p), "l"(v.x), "l"(v.y) : "memory");
}
struct u256 {
  unsigned long long a, b, c, d;
};
__device__ __forceinline__ u256 ld256(const void* p) {
  u256 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u64 {%0, %1, %2, %3}, [%4];"
               : "=l"(v.a), "=l"(v.b), "=l"(v.c), "=l"(v.d)
               : "l"(p));
  return v;
}
__device__ __forceinline__ void st256(void* p, u256 v) {
  asm volatile("st.global.v4.u64 [%0], {%1, %2, %3, %4};" ::"l"(p), "l"(v.a), "l"(v.b), "l"(v.c),
               "l"(v.d)
               : "memory");
}

struct P {
  const uint64_t* src;
  uint64_t* dst;
  const int32_t* si;
  const int32_t* di;
  uint8_t* fill;
  int64_t n_rows, layers, src_lw, dst_lw, fill_lw;
};

// v1: the library's current scheme (16-byte vectors, 8 per lane, fill check).
__global__ void __launch_bounds__(256) v1(P p) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
  for (int64_t it = warp; it < p.n_rows * p.layers; it += nw) {
    int64_t l = it / p.n_rows, r = it % p.n_rows;
    int64_t s = p.si[r], d = p.di[r];
    uint8_t* f = p.fill + l * p.fill_lw + d;
    uint8_t fv = *(volatile uint8_t*)f;
    const ulonglong2* s2 = (const ulonglong2*)(p.src + l * p.src_lw + s * W);
    ulonglong2* d2 = (ulonglong2*)(p.dst + l * p.dst_lw + d * W);
    ulonglong2 t[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) t[u] = ld_nc(s2 + lane + 32 * u);
    if (fv == 0) {
#pragma unroll
      for (int u = 0; u < 8; ++u) st2(d2 + lane + 32 * u, t[u]);
      __syncwarp();
      if (lane == 0) *f = 2;
    }
  }
}

// v2: 32-byte vectors (ld/st .v4.u64), 4 per lane.
__global__ void __launch_bounds__(256) v2(P p) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
  for (int64_t it = warp; it < p.n_rows * p.layers; it += nw) {
    int64_t l = it / p.n_rows, r = it % p.n_rows;
    int64_t s = p.si[r], d = p.di[r];
    uint8_t* f = p.fill + l * p.fill_lw + d;
    uint8_t fv = *(volatile uint8_t*)f;
    const u256* s4 = (const u256*)(p.src + l * p.src_lw + s * W);
    u256* d4 = (u256*)(p.dst + l * p.dst_lw + d * W);
    u256 t[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) t[u] = ld256(s4 + lane + 32 * u);
    if (fv == 0) {
#pragma unroll
      for (int u = 0; u < 4; ++u) st256(d4 + lane + 32 * u, t[u]);
      __syncwarp();
      if (lane == 0) *f = 2;
    }
  }
}

// v3: two rows per warp iteration (16 x 16-byte loads in flight per lane).
__global__ void __launch_bounds__(256) v3(P p) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
  const int64_t items = p.n_rows * p.layers;
  for (int64_t it = 2 * warp; it < items; it += 2 * nw) {
    ulonglong2 t[2][8];
    uint8_t fv[2];
    uint8_t* f[2];
    ulonglong2* d2[2];
    bool ok[2];
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      int64_t i = it + k;
      ok[k] = i < items;
      if (!ok[k]) continue;
      int64_t l = i / p.n_rows, r = i % p.n_rows;
      int64_t s = p.si[r], d = p.di[r];
      f[k] = p.fill + l * p.fill_lw + d;
      fv[k] = *(volatile uint8_t*)f[k];
      const ulonglong2* s2 = (const ulonglong2*)(p.src + l * p.src_lw + s * W);
      d2[k] = (ulonglong2*)(p.dst + l * p.dst_lw + d * W);
#pragma unroll
      for (int u = 0; u < 8; ++u) t[k][u] = ld_nc(s2 + lane + 32 * u);
    }
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      if (!ok[k] || fv[k] != 0) continue;
#pragma unroll
      for (int u = 0; u < 8; ++u) st2(d2[k] + lane + 32 * u, t[k][u]);
      __syncwarp();
      if (lane == 0) *f[k] = 2;
    }
  }
}

// v4: TMA bulk copies through a shared-memory ring (one elected thread per
// warp issues cp.async.bulk global->shared, then shared->global).
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
constexpr int kStages = 6;  // per warp
__global__ void __launch_bounds__(128) v4(P p) {
  extern __shared__ __align__(128) uint8_t sm[];
  __shared__ __align__(8) uint64_t bar[4][kStages];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  uint8_t* ring = sm + wid * kStages * 4096;
  const int64_t warp = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
  const int64_t items = p.n_rows * p.layers;
  if (lane == 0) {
    for (int s = 0; s < kStages; ++s)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[wid][s])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncwarp();
  if (lane != 0) return;
  // Issue loads kStages ahead; store each row as its load lands.
  int64_t issued = warp, done = warp;
  uint32_t phase[kStages] = {0};
  int64_t dst_of[kStages];
  uint8_t* fill_of[kStages];
  int slot = 0, dslot = 0;
  auto issue = [&](int64_t i, int s) {
    int64_t l = i / p.n_rows, r = i % p.n_rows;
    int64_t si = p.si[r], di = p.di[r];
    const uint64_t* src = p.src + l * p.src_lw + si * W;
    dst_of[s] = (l * p.dst_lw + di * W);
    fill_of[s] = p.fill + l * p.fill_lw + di;
    uint32_t b = smem_u32(&bar[wid][s]);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], 4096;" ::"r"(b) : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 4096, [%2];" ::"r"(
            smem_u32(ring + s * 4096)),
        "l"(src), "r"(b)
        : "memory");
  };
  int inflight = 0;
  while (issued < items && inflight < kStages) {
    issue(issued, slot);
    issued += nw;
    slot = (slot + 1) % kStages;
    ++inflight;
  }
  while (inflight > 0) {
    uint32_t b = smem_u32(&bar[wid][dslot]);
    asm volatile(
        "{ .reg .pred P; W: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1; @!P bra W; }" ::"r"(b),
        "r"(phase[dslot])
        : "memory");
    phase[dslot] ^= 1;
    uint8_t fv = *(volatile uint8_t*)fill_of[dslot];
    if (fv == 0) {
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], 4096;" ::"l"(p.dst + dst_of[dslot]),
                   "r"(smem_u32(ring + dslot * 4096))
                   : "memory");
      asm volatile("cp.async.bulk.commit_group;");
      *fill_of[dslot] = 2;
    }
    done += nw;
    --inflight;
    // Before refilling this stage, its store must have read the buffer.
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    if (issued < items) {
      issue(issued, dslot);
      issued += nw;
      ++inflight;
    }
    dslot = (dslot + 1) % kStages;
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}


// d1: plain dense memcpy kernel (grid-stride over 32-byte vectors, 4 in flight).
__global__ void __launch_bounds__(256) d1(const u256* __restrict__ s, u256* __restrict__ d, int64_t n) {
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  for (; i + 3 * stride < n; i += 4 * stride) {
    u256 t0 = ld256(s + i), t1 = ld256(s + i + stride), t2 = ld256(s + i + 2 * stride),
         t3 = ld256(s + i + 3 * stride);
    st256(d + i, t0);
    st256(d + i + stride, t1);
    st256(d + i + 2 * stride, t2);
    st256(d + i + 3 * stride, t3);
  }
  for (; i < n; i += stride) st256(d + i, ld256(s + i));
}

// d2: row structure of v2 without indirection or fill (dense rows).
__global__ void __launch_bounds__(256) d2(P p) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
  for (int64_t it = warp; it < p.n_rows * p.layers; it += nw) {
    int64_t l = it / p.n_rows, r = it % p.n_rows;
    const u256* s4 = (const u256*)(p.src + l * p.src_lw + r * W);
    u256* d4 = (u256*)(p.dst + l * p.dst_lw + r * W);
    u256 t[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) t[u] = ld256(s4 + lane + 32 * u);
#pragma unroll
    for (int u = 0; u < 4; ++u) st256(d4 + lane + 32 * u, t[u]);
  }
}

// v5: v2 with contiguous row blocks per CTA, cg fill load.
__global__ void __launch_bounds__(256) v5(P p, int rows_per_cta) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int64_t items = p.n_rows * p.layers;
  const int64_t chunks = (items + rows_per_cta - 1) / rows_per_cta;
  for (int64_t c = blockIdx.x; c < chunks; c += gridDim.x) {
    const int64_t hi = (c + 1) * rows_per_cta < items ? (c + 1) * rows_per_cta : items;
    for (int64_t it = c * rows_per_cta + wid; it < hi; it += 8) {
      int64_t l = it / p.n_rows, r = it % p.n_rows;
      int64_t s = p.si[r], d = p.di[r];
      uint8_t* f = p.fill + l * p.fill_lw + d;
      unsigned short fv;
      asm volatile("ld.global.cg.u8 %0, [%1];" : "=h"(fv) : "l"(f));
      const u256* s4 = (const u256*)(p.src + l * p.src_lw + s * W);
      u256* d4 = (u256*)(p.dst + l * p.dst_lw + d * W);
      u256 t[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) t[u] = ld256(s4 + lane + 32 * u);
      if (fv == 0) {
#pragma unroll
        for (int u = 0; u < 4; ++u) st256(d4 + lane + 32 * u, t[u]);
        __syncwarp();
        if (lane == 0) *f = 2;
      }
    }
  }
}

// v6: v2 + cg fill load + .cs (streaming) stores.
__device__ __forceinline__ void st256cs(void* p, u256 v) {
  asm volatile("st.global.cs.v4.u64 [%0], {%1, %2, %3, %4};" ::"l"(p), "l"(v.a), "l"(v.b), "l"(v.c),
               "l"(v.d)
               : "memory");
}
__global__ void __launch_bounds__(256) v6(P p) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
  for (int64_t it = warp; it < p.n_rows * p.layers; it += nw) {
    int64_t l = it / p.n_rows, r = it % p.n_rows;
    int64_t s = p.si[r], d = p.di[r];
    uint8_t* f = p.fill + l * p.fill_lw + d;
    unsigned short fv;
    asm volatile("ld.global.cg.u8 %0, [%1];" : "=h"(fv) : "l"(f));
    const u256* s4 = (const u256*)(p.src + l * p.src_lw + s * W);
    u256* d4 = (u256*)(p.dst + l * p.dst_lw + d * W);
    u256 t[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) t[u] = ld256(s4 + lane + 32 * u);
    if (fv == 0) {
#pragma unroll
      for (int u = 0; u < 4; ++u) st256cs(d4 + lane + 32 * u, t[u]);
      __syncwarp();
      if (lane == 0) *f = 2;
    }
  }
}

// v7: v2 + indices prefetched one item ahead + cg fill load (use_fill=0: no fill rule).
template <bool kFill>
__global__ void __launch_bounds__(256) v7(P p) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
  const int64_t items = p.n_rows * p.layers;
  int64_t ns = 0, nd = 0;
  if (warp < items) {
    int64_t r = warp % p.n_rows;
    ns = p.si[r];
    nd = p.di[r];
  }
  for (int64_t it = warp; it < items; it += nw) {
    int64_t l = it / p.n_rows;
    const int64_t s = ns, d = nd;
    if (it + nw < items) {
      int64_t r2 = (it + nw) % p.n_rows;
      ns = p.si[r2];
      nd = p.di[r2];
    }
    uint8_t* f = p.fill + l * p.fill_lw + d;
    unsigned short fv = 0;
    if (kFill) asm volatile("ld.global.cg.u8 %0, [%1];" : "=h"(fv) : "l"(f));
    const u256* s4 = (const u256*)(p.src + l * p.src_lw + s * W);
    u256* d4 = (u256*)(p.dst + l * p.dst_lw + d * W);
    u256 t[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) t[u] = ld256(s4 + lane + 32 * u);
    if (fv == 0) {
#pragma unroll
      for (int u = 0; u < 4; ++u) st256(d4 + lane + 32 * u, t[u]);
      if (kFill) {
        __syncwarp();
        if (lane == 0) *f = 2;
      }
    }
  }
}

// v8: items are groups of G consecutive rows of one layer.  Lanes 0..G-1
// load the group's indices and fill bytes in one coalesced access each;
// rows are copied with no dependent load; lanes store the fill marks.
template <int G>
__global__ void __launch_bounds__(256) v8(P p) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
  const int64_t groups_per_layer = (p.n_rows + G - 1) / G;
  const int64_t items = groups_per_layer * p.layers;
  for (int64_t it = warp; it < items; it += nw) {
    const int64_t l = it / groups_per_layer;
    const int64_t r0 = (it % groups_per_layer) * G;
    const int nr = (int)((p.n_rows - r0) < G ? (p.n_rows - r0) : G);
    int32_t my_s = 0, my_d = 0;
    unsigned short my_f = 1;
    if (lane < nr) {
      my_s = p.si[r0 + lane];
      my_d = p.di[r0 + lane];
      asm volatile("ld.global.cg.u8 %0, [%1];" : "=h"(my_f) : "l"(p.fill + l * p.fill_lw + my_d));
    }
    const unsigned empty = __ballot_sync(0xffffffffu, lane < nr && my_f == 0);
#pragma unroll 1
    for (int k = 0; k < nr; ++k) {
      const int64_t s = __shfl_sync(0xffffffffu, my_s, k);
      const int64_t d = __shfl_sync(0xffffffffu, my_d, k);
      if (!((empty >> k) & 1u)) continue;
      const u256* s4 = (const u256*)(p.src + l * p.src_lw + s * W);
      u256* d4 = (u256*)(p.dst + l * p.dst_lw + d * W);
      u256 t[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) t[u] = ld256(s4 + lane + 32 * u);
#pragma unroll
      for (int u = 0; u < 4; ++u) st256(d4 + lane + 32 * u, t[u]);
    }
    __syncwarp();
    if (lane < nr && ((empty >> lane) & 1u)) p.fill[l * p.fill_lw + my_d] = 2;
  }
}

int main() {
  const int64_t n_rows = 8191, layers = 80, pages = 8192 / 16 + 16;
  const int64_t lw = pages * 16 * W;
  const size_t bytes = size_t(lw) * layers * 8;
  uint64_t *src, *dst;
  uint8_t* fill;
  int32_t *si, *di;
  CK(cudaMalloc(&src, bytes));
  CK(cudaMalloc(&dst, bytes));
  CK(cudaMalloc(&fill, pages * 16 * layers));
  CK(cudaMalloc(&si, 4 * n_rows));
  CK(cudaMalloc(&di, 4 * n_rows));
  std::vector<int32_t> h(n_rows);
  for (int64_t i = 0; i < n_rows; ++i) h[i] = int32_t(i);
  CK(cudaMemcpy(si, h.data(), 4 * n_rows, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(di, h.data(), 4 * n_rows, cudaMemcpyHostToDevice));
  // LIFO reuse after a free hands the decode engine its pages in descending
  // order (kv_cache.cc:499-507): rows ascend within a page, pages descend.
  std::vector<int32_t> hdesc(n_rows);
  for (int64_t i = 0; i < n_rows; ++i) hdesc[i] = int32_t(((511 - i / 16) * 16) + i % 16);
  int32_t* di_desc;
  CK(cudaMalloc(&di_desc, 4 * n_rows));
  CK(cudaMemcpy(di_desc, hdesc.data(), 4 * n_rows, cudaMemcpyHostToDevice));
  CK(cudaMemset(src, 1, bytes));
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  P p{src, dst, si, di, fill, n_rows, layers, lw, lw, pages * 16};
  const double alg = 2.0 * n_rows * layers * 4096;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  auto timeit = [&](const char* name, auto&& launch) {
    for (int w = 0; w < 2; ++w) {
      cudaMemset(fill, 0, pages * 16 * layers);
      launch();
    }
    float best = 1e9;
    for (int rep = 0; rep < 5; ++rep) {
      cudaMemset(fill, 0, pages * 16 * layers);
      cudaEventRecord(a);
      launch();
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      best = ms < best ? ms : best;
    }
    cudaError_t e = cudaGetLastError();
    printf("%-28s %8.1f us  %7.1f GB/s (r+w)  %s\n", name, best * 1e3, alg / (best * 1e-3) / 1e9,
           e == cudaSuccess ? "" : cudaGetErrorString(e));
  };
  timeit("cudaMemcpy D2D", [&] {
    cudaMemcpyAsync(dst, src, size_t(n_rows) * 4096, cudaMemcpyDeviceToDevice);
    for (int l = 1; l < layers; ++l)
      cudaMemcpyAsync(dst + l * lw, src + l * lw, size_t(n_rows) * 4096, cudaMemcpyDeviceToDevice);
  });
  timeit("cudaMemcpy D2D one shot", [&] {
    cudaMemcpyAsync(dst, src, size_t(n_rows) * 4096 * layers, cudaMemcpyDeviceToDevice);
  });
  for (int mult : {4, 8}) {
    char nm[64];
    snprintf(nm, 64, "v1 16B x8 grid=%dx%d", sms, mult);
    timeit(nm, [&] { v1<<<sms * mult, 256>>>(p); });
    snprintf(nm, 64, "v2 32B x4 grid=%dx%d", sms, mult);
    timeit(nm, [&] { v2<<<sms * mult, 256>>>(p); });
    snprintf(nm, 64, "v3 2 rows grid=%dx%d", sms, mult);
    timeit(nm, [&] { v3<<<sms * mult, 256>>>(p); });
  }
  {
    const int64_t nvec = n_rows * 4096 / 32;  // per layer
    timeit("d1 dense memcpy kernel x80", [&] {
      for (int l = 0; l < layers; ++l)
        d1<<<sms * 4, 256>>>((const u256*)(src + l * lw), (u256*)(dst + l * lw), nvec);
    });
    timeit("d1 dense memcpy one launch", [&] {
      d1<<<sms * 4, 256>>>((const u256*)src, (u256*)dst, nvec * layers);
    });
    timeit("d2 dense rows (v2 loop)", [&] { d2<<<sms * 4, 256>>>(p); });
    for (int rpc : {64, 256, 1024}) {
      char nm[64];
      snprintf(nm, 64, "v5 cta blocks R=%d", rpc);
      timeit(nm, [&] { v5<<<sms * 4, 256>>>(p, rpc); });
    }
    timeit("v6 32B cg-fill .cs stores", [&] { v6<<<sms * 4, 256>>>(p); });
    {
      P pd = p;
      pd.di = di_desc;
      timeit("v8 G=4 x2 descending dst", [&] { v8<4><<<sms * 2, 256>>>(pd); });
      timeit("v8 G=4 x2 ascending  dst", [&] { v8<4><<<sms * 2, 256>>>(p); });
    }
    for (int mult : {2}) {
      char nm[64];
      snprintf(nm, 64, "v8 G=4 x%d", mult);
      timeit(nm, [&] { v8<4><<<sms * mult, 256>>>(p); });
      snprintf(nm, 64, "v8 G=8 x%d", mult);
      timeit(nm, [&] { v8<8><<<sms * mult, 256>>>(p); });
      snprintf(nm, 64, "v8 G=16 x%d", mult);
      timeit(nm, [&] { v8<16><<<sms * mult, 256>>>(p); });
    }
    for (int mult : {2, 4}) {
      char nm[64];
      snprintf(nm, 64, "v7 prefetch+fill x%d", mult);
      timeit(nm, [&] { v7<true><<<sms * mult, 256>>>(p); });
      snprintf(nm, 64, "v7 prefetch no-fill x%d", mult);
      timeit(nm, [&] { v7<false><<<sms * mult, 256>>>(p); });
    }
  }
  const int smem = 4 * kStages * 4096;
  cudaFuncSetAttribute(v4, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int mult : {1, 2}) {
    char nm[64];
    snprintf(nm, 64, "v4 TMA bulk grid=%dx%d", sms, mult);
    timeit(nm, [&] { v4<<<sms * mult, 128, smem>>>(p); });
  }
  // Correctness of the last variant.
  std::vector<uint64_t> hs(W * 4), hd(W * 4);
  cudaMemcpy(hs.data(), src + 79 * lw + 100 * W, 8 * W * 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(hd.data(), dst + 79 * lw + 100 * W, 8 * W * 4, cudaMemcpyDeviceToHost);
  printf("check %s\n", hs == hd ? "ok" : "MISMATCH");
  return 0;
}
