// read_floor.cu — how fast can one launch read S bytes of HBM on B200?
// One CTA per SM streams its contiguous 1/148 slice through a ring of bulk
// copies (cp.async.bulk global -> shared, mbarrier completion), STAGES x
// CHUNK bytes in flight per SM; 20 back-to-back launches cycle over enough
// buffers to exceed L2 (126 MB); CUDA events around the 20.  The floor a
// decode-attention launch of the same bytes can approach (decode at B = 1,
// ctx 8K, 70B heads reads 33.5 MB).
// Build: nvcc -std=c++17 -gencode arch=compute_100a,code=sm_100a -O2 \
//          -o profiles/micro/read_floor.bin profiles/micro/read_floor.cu
#include <cstdint>
#include <cstdio>
#include <vector>

__device__ __forceinline__ uint32_t su32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

template <int STAGES, int CHUNK>
__global__ void __launch_bounds__(32, 1) k_read(const uint8_t* src, size_t bytes, int* sink) {
  extern __shared__ __align__(128) uint8_t ring[];
  __shared__ __align__(8) uint64_t bars[STAGES];
  const int lane = threadIdx.x;
  const size_t per = (bytes / gridDim.x) & ~static_cast<size_t>(15);
  const uint8_t* base = src + per * blockIdx.x;
  const int n = static_cast<int>((per + CHUNK - 1) / CHUNK);
  if (lane == 0) {
    for (int s = 0; s < STAGES; ++s)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bars[s])) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  int acc = 0;
  auto issue = [&](int c) {
    const int s = c % STAGES;
    const size_t off = static_cast<size_t>(c) * CHUNK;
    const uint32_t len = static_cast<uint32_t>(per - off < CHUNK ? per - off : CHUNK);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bars[s])),
                 "r"(len)
                 : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            su32(ring + s * CHUNK)),
        "l"(base + off), "r"(len), "r"(su32(&bars[s]))
        : "memory");
  };
  if (lane == 0)
    for (int c = 0; c < STAGES && c < n; ++c) issue(c);
  for (int c = 0; c < n; ++c) {
    const int s = c % STAGES;
    uint32_t done = 0;
    while (!done) {
      asm volatile(
          "{\n\t.reg .pred P;\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2;\n\t"
          "selp.u32 %0, 1, 0, P;\n\t}\n"
          : "=r"(done)
          : "r"(su32(&bars[s])), "r"((c / STAGES) & 1)
          : "memory");
    }
    acc += ring[s * CHUNK + lane * 4];
    __syncwarp();
    if (lane == 0 && c + STAGES < n) issue(c + STAGES);
  }
  if (acc == 0x7fffffff) *sink = acc;
}

template <int STAGES, int CHUNK>
void run(const std::vector<uint8_t*>& bufs, size_t bytes, int sms, int* sink) {
  auto k = k_read<STAGES, CHUNK>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, STAGES * CHUNK);
  for (int i = 0; i < 3; ++i) k<<<sms, 32, STAGES * CHUNK>>>(bufs[i % bufs.size()], bytes, sink);
  cudaDeviceSynchronize();
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int i = 0; i < 20; ++i) k<<<sms, 32, STAGES * CHUNK>>>(bufs[i % bufs.size()], bytes, sink);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  const double t = ms * 1e-3 / 20;
  printf("read %8.1f MB  %d x %3d KiB in flight per SM  %7.2f us  %7.1f GB/s\n", bytes / 1e6, STAGES,
         CHUNK / 1024, t * 1e6, bytes / t / 1e9);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int* sink;
  cudaMalloc(&sink, 4);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  // empty-launch cost for reference
  for (int i = 0; i < 3; ++i) k_read<1, 1024><<<sms, 32, 1024>>>(nullptr, 0, sink);
  cudaEventRecord(e0);
  for (int i = 0; i < 20; ++i) k_read<1, 1024><<<sms, 32, 1024>>>(nullptr, 0, sink);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  printf("empty launch (148 CTAs)  %7.2f us\n", ms * 1e3 / 20);
  for (size_t bytes : {size_t(33554432), size_t(67108864), size_t(134217728), size_t(536870912)}) {
    const int nbuf = static_cast<int>(std::max<size_t>(2, (400ull << 20) / bytes + 1));
    std::vector<uint8_t*> bufs(nbuf);
    for (auto& b : bufs) {
      cudaMalloc(&b, bytes);
      cudaMemset(b, 1, bytes);
    }
    run<3, 65536>(bufs, bytes, sms, sink);
    run<6, 32768>(bufs, bytes, sms, sink);
    run<12, 16384>(bufs, bytes, sms, sink);
    run<7, 32768>(bufs, bytes, sms, sink);   // 224 KiB in flight per SM
    run<14, 16384>(bufs, bytes, sms, sink);
    for (auto b : bufs) cudaFree(b);
  }
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) printf("error %s\n", cudaGetErrorString(e));
  return 0;
}
