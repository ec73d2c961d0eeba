// grid_stride.cu — is the "odd CTAs per SM" effect of the long row copies
// (profiles/r02/copy_grid_ab.txt) a property of plain grid-stride copies on
// B200?  A dense copy of 5.37 GB (the headline DirectSend's bytes) in 16 KiB
// warp items (4 x 4 KiB rows, each lane 4 x 32-byte loads per row, then the
// stores), grid-stride over items, 256 threads per CTA, 2 CTAs resident per
// SM (dynamic shared memory sized to allow exactly 2), grid = 148 x k CTAs,
// k = 1 .. 12; CUDA events around 5 launches after 2 warm-ups.
// Build: nvcc -std=c++17 -gencode arch=compute_100a,code=sm_100a -O3 \
//          -o profiles/micro/grid_stride.bin profiles/micro/grid_stride.cu
#include <cstdint>
#include <cstdio>

struct u256 {
  unsigned long long a, b, c, d;
};
__device__ __forceinline__ u256 ld256(const void* p) {
  u256 v;
  asm volatile("ld.global.L1::no_allocate.L2::evict_first.v4.u64 {%0, %1, %2, %3}, [%4];"
               : "=l"(v.a), "=l"(v.b), "=l"(v.c), "=l"(v.d)
               : "l"(p));
  return v;
}
__device__ __forceinline__ void st256(void* p, const u256& v) {
  asm volatile("st.global.v4.u64 [%0], {%1, %2, %3, %4};" ::"l"(p), "l"(v.a), "l"(v.b), "l"(v.c),
               "l"(v.d)
               : "memory");
}

__global__ void __launch_bounds__(256) k_copy(const uint8_t* __restrict__ src, uint8_t* __restrict__ dst,
                                              int64_t items) {
  extern __shared__ uint8_t pad[];  // occupancy only
  const int lane = threadIdx.x & 31;
  const int64_t warp = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  for (int64_t it = warp; it < items; it += nw) {
#pragma unroll 1
    for (int r = 0; r < 4; ++r) {
      const int64_t off = (it * 4 + r) * 4096;
      const u256* s4 = reinterpret_cast<const u256*>(src + off) + lane;
      u256* d4 = reinterpret_cast<u256*>(dst + off) + lane;
      u256 t[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) t[u] = ld256(s4 + 32 * u);
#pragma unroll
      for (int u = 0; u < 4; ++u) st256(d4 + 32 * u, t[u]);
    }
  }
  if (items < 0) pad[0] = 0;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int64_t rows = 8191LL * 80, items = rows / 4;
  const size_t bytes = static_cast<size_t>(items) * 4 * 4096;
  uint8_t *src, *dst;
  if (cudaMalloc(&src, bytes) != cudaSuccess || cudaMalloc(&dst, bytes) != cudaSuccess) return 1;
  cudaMemset(src, 1, bytes);
  const int smem = 100 * 1024;  // 2 CTAs per SM
  cudaFuncSetAttribute(k_copy, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_copy, 256, smem);
  printf("resident CTAs per SM: %d; %.2f GB copied per launch\n", occ, bytes / 1e9);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int k = 1; k <= 12; ++k) {
    const int grid = sms * k;
    for (int w = 0; w < 2; ++w) k_copy<<<grid, 256, smem>>>(src, dst, items);
    cudaEventRecord(e0);
    for (int i = 0; i < 5; ++i) k_copy<<<grid, 256, smem>>>(src, dst, items);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double t = ms * 1e-3 / 5;
    printf("grid %2d x %d CTAs  %8.1f us  %7.1f GB/s (read + write)\n", k, sms, t * 1e6,
           2.0 * bytes / t / 1e9);
  }
  cudaError_t err = cudaDeviceSynchronize();
  if (err != cudaSuccess) printf("error %s\n", cudaGetErrorString(err));
  return 0;
}
