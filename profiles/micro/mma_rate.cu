// mma_rate.cu — cycles per tcgen05.mma dispatch (bf16, M = 128, K = 16) as
// the prefill kernel issues them, one CTA per SM on every SM:
//   mode 0  SS, N = 128   (S = Q K^T: A and B from shared memory)
//   mode 1  TS, N = 128   (O += P V: A from tensor memory, B MN-major)
//   mode 2  SS, N = 256
//   mode 3  mode 0 while 8 other warps stream tcgen05.ld from TMEM
//   mode 4  mode 1 while 8 other warps stream tcgen05.ld from TMEM
//   mode 5  alternating SS (N = 128) and TS (N = 128) GEMMs of K = 128
//   mode 6  SS, N = 128, consecutive dispatches into two accumulators
//   mode 7  TS, N = 128, consecutive dispatches into two accumulators
//   mode 8  SS, N = 64 (for scale)
//   mode 9  SS, N = 192     mode 10  SS, N = 160     mode 11  SS, N = 224
// (Issuing from two warps of one CTA, one accumulator each, ended the launch
// with an unspecified failure on B200: not measured.)
// and with a CTA pair (cta_group::2, M = 256, leader issues), k_rate2:
//   mode 0  SS, N = 128    mode 1  TS, N = 128    mode 2  SS, N = 256
// Build: nvcc -std=c++17 -gencode arch=compute_100a,code=sm_100a -O2 \
//          -o profiles/micro/mma_rate.bin profiles/micro/mma_rate.cu -lcuda
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../../paper_2412_12488_b200/csrc/prefill_attn.cu"

using namespace mkv;

__global__ void __launch_bounds__(288, 1) k_rate(int mode, int iters, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  __shared__ uint32_t slot;
  __shared__ uint64_t mbar;
  __shared__ volatile int stop;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < 96 * 1024 / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
  if (warp == 8) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                     smem_u32(&slot))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (tid == 0) {
    mbar_init(smem_u32(&mbar), 1);
    stop = 0;
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  fence_proxy_async();
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = slot;
  const uint32_t sA = smem_u32(smem), sB = smem_u32(smem + 32 * 1024);
  if (warp == 8) {
    const uint32_t hi = desc_hi(1024);
    const uint32_t a_lo = desc_lo(sA, 16), b_lo = desc_lo(sB, 16), v_lo = desc_lo(sB, 16384);
    const uint32_t idS = idesc_bf16(false, 128), idS256 = idesc_bf16(false, 256);
    const uint32_t idO = idesc_bf16(true, 128);
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      const bool ss = mode == 0 || mode == 2 || mode == 3 || (mode == 5 && (it & 1) == 0);
      if (mode == 6 || mode == 7) {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const uint32_t ao = ((k >> 2) * 16384 + (k & 3) * 32) >> 4;
#pragma unroll
          for (int d = 0; d < 2; ++d) {
            if (mode == 6)
              mma_ss_elect(tmem + d * 128, a_lo + ao, b_lo + ao, hi, idS, k > 0 ? 1u : 0u);
            else
              mma_ts_elect(tmem + 256 + d * 128, tmem + d * 128 + k * 8, v_lo + ((k * 2048) >> 4),
                           hi, idO, 1u);
          }
        }
        continue;
      }
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const uint32_t ao = ((k >> 2) * 16384 + (k & 3) * 32) >> 4;
        if (mode >= 8) {
          const int n = mode == 8 ? 64 : mode == 9 ? 192 : mode == 10 ? 160 : 224;
          mma_ss_elect(tmem + ((it & 1) ? 256 : 0), a_lo + ao, b_lo + ao, hi,
                       idesc_bf16(false, n), k > 0 ? 1u : 0u);
        } else if (ss) {
          mma_ss_elect(tmem + ((it & 1) ? 128 : 0), a_lo + ao, b_lo + ao, hi,
                       mode == 2 ? idS256 : idS, k > 0 ? 1u : 0u);
        } else {
          mma_ts_elect(tmem + 256, tmem + k * 8, v_lo + ((k * 2048) >> 4), hi, idO, 1u);
        }
      }
    }
    commit_elect(smem_u32(&mbar));
    mbar_wait(smem_u32(&mbar), 0);
    const long long t1 = clock64();
    if ((tid & 31) == 0) {
      out[blockIdx.x] = static_cast<unsigned long long>(t1 - t0);
      stop = 1;
    }
  } else if (mode == 3 || mode == 4) {
    // Softmax stand-in: warp w streams 128 columns of its lane quadrant.
    const uint32_t lane_off = static_cast<uint32_t>((warp & 3) * 32) << 16;
    const uint32_t base = tmem + 384 + lane_off;
    uint32_t acc = 0, r[16];
    while (!stop) {
#pragma unroll
      for (int c = 0; c < 128; c += 16) {
        tmem_ld16_nowait(base + c, r);
        tmem_wait_ld();
        acc ^= r[0] ^ r[15];
      }
    }
    if (acc == 0xdeadbeef) out[1000] = acc;
  }
  fence_before();
  __syncthreads();
  if (warp == 8) {
    fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
  }
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
__host__ __device__ constexpr uint32_t idesc2(bool b_mn_major, int n) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((b_mn_major ? 1u : 0u) << 16) |
         ((static_cast<uint32_t>(n) >> 3) << 17) | ((256u >> 4) << 24);
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1)
    k_rate2(int mode, int iters, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  __shared__ uint32_t slot;
  __shared__ uint64_t mbar;
  const int tid = threadIdx.x, warp = tid >> 5;
  uint32_t rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  for (int i = tid; i < 96 * 1024 / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                     smem_u32(&slot))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  if (tid == 0) {
    mbar_init(smem_u32(&mbar), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  fence_proxy_async();
  fence_before();
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::
                   : "memory");
  fence_after();
  const uint32_t tmem = slot;
  const uint32_t sA = smem_u32(smem), sB = smem_u32(smem + 32 * 1024);
  if (warp == 0 && rank == 0) {
    const uint32_t hi = desc_hi(1024);
    const uint32_t a_lo = desc_lo(sA, 16), b_lo = desc_lo(sB, 16), v_lo = desc_lo(sB, 8192);
    const uint32_t idS = idesc2(false, 128), idS256 = idesc2(false, 256), idO = idesc2(true, 128);
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const uint32_t ao = ((k >> 2) * 16384 + (k & 3) * 32) >> 4;
        if (mode == 1)
          mma2_ts(tmem + 256, tmem + k * 8, v_lo + ((k * 2048) >> 4), hi, idO, 1u);
        else
          mma2_ss(tmem + ((it & 1) ? 128 : 0), a_lo + ao, b_lo + ao, hi,
                  mode == 2 ? idS256 : idS, k > 0 ? 1u : 0u);
      }
    }
    asm volatile(
        "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 "
        "[%0], %1;\n\t}\n" ::"r"(smem_u32(&mbar)),
        "h"(static_cast<unsigned short>(3))
        : "memory");
    mbar_wait(smem_u32(&mbar), 0);
    const long long t1 = clock64();
    if ((tid & 31) == 0) out[blockIdx.x >> 1] = static_cast<unsigned long long>(t1 - t0);
  } else if (warp == 0) {
    mbar_wait(smem_u32(&mbar), 0);
  }
  fence_before();
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::
                   : "memory");
  if (warp == 0) {
    fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
  }
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int smem = 96 * 1024 + 1024;
  cudaFuncSetAttribute(k_rate, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  unsigned long long* d;
  cudaMalloc(&d, 2048 * sizeof(unsigned long long));
  const int iters = 4096;
  const char* names[] = {"SS N=128", "TS N=128", "SS N=256", "SS N=128 + 8 warps tcgen05.ld",
                         "TS N=128 + 8 warps tcgen05.ld", "SS/TS alternating N=128",
                         "SS N=128, 2 accumulators interleaved", "TS N=128, 2 accumulators interleaved",
                         "SS N=64", "SS N=192", "SS N=160", "SS N=224"};
  for (int mode = 0; mode < 12; ++mode) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      cudaEventRecord(e0);
      k_rate<<<sms, 288, smem>>>(mode, iters, d);
      cudaEventRecord(e1);
      cudaError_t err = cudaDeviceSynchronize();
      if (err != cudaSuccess) {
        printf("error %s\n", cudaGetErrorString(err));
        return 1;
      }
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      std::vector<unsigned long long> h(sms);
      cudaMemcpy(h.data(), d, sms * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
      double avg = 0;
      for (auto v : h) avg += v;
      avg /= sms;
      const double n = static_cast<double>(iters) * 8 * ((mode == 6 || mode == 7) ? 2 : 1);
      const int nn = mode == 2 ? 256 : mode == 8 ? 64 : mode == 9 ? 192 : mode == 10 ? 160 : mode == 11 ? 224 : 128;
      const double flop = 2.0 * 128 * nn * 16 * n * sms;
      if (rep == 1)
        printf("%-32s %6.1f cycles/dispatch  %7.1f TFLOP/s (event time %.3f ms)\n", names[mode],
               avg / n, flop / (ms * 1e-3) / 1e12, ms);
    }
  }

  cudaFuncSetAttribute(k_rate2, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const char* names2[] = {"pair SS M=256 N=128", "pair TS M=256 N=128", "pair SS M=256 N=256"};
  for (int mode = 0; mode < 3; ++mode) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      cudaEventRecord(e0);
      k_rate2<<<sms, 128, smem>>>(mode, iters, d);
      cudaEventRecord(e1);
      cudaError_t err = cudaDeviceSynchronize();
      if (err != cudaSuccess) {
        printf("error %s\n", cudaGetErrorString(err));
        return 1;
      }
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      std::vector<unsigned long long> h(sms / 2);
      cudaMemcpy(h.data(), d, (sms / 2) * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
      double avg = 0;
      for (auto v : h) avg += v;
      avg /= (sms / 2);
      const double n = static_cast<double>(iters) * 8;
      const double flop = 2.0 * 256 * (mode == 2 ? 256 : 128) * 16 * n * (sms / 2);
      if (rep == 1)
        printf("%-32s %6.1f cycles/dispatch  %7.1f TFLOP/s (event time %.3f ms)\n", names2[mode],
               avg / n, flop / (ms * 1e-3) / 1e12, ms);
    }
  }
  return 0;
}
