// Micro-benchmark: per-SM throughput of ex2.approx.ftz.f32 (MUFU), of the
// packed ex2.approx.f16x2 / ex2.approx.ftz.bf16x2, and of fma.rn.f32x2
// (FFMA2) on B200, to bound the prefill softmax.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mufu_rate mufu_rate.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_ex2(float* out, int iters) {
  float v[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) v[k] = -0.001f * (threadIdx.x + k);
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(v[k]));
  }
  float s = 0.f;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += v[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// Packed half-precision exponentials: two exps per lane per instruction.
template <bool kBf16>
__global__ void k_ex2_x2(float* out, int iters) {
  unsigned v[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) v[k] = 0xBC00BC00u - threadIdx.x - k;  // ~ -1.0 in both halves
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      if constexpr (kBf16) asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(v[k]));
      else asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(v[k]));
    }
  }
  unsigned s = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s ^= v[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = static_cast<float>(s);
}

__global__ void k_ffma2(float* out, int iters) {
  unsigned long long v[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    float a = 1.f + threadIdx.x * 1e-7f + k, b = 2.f;
    asm("mov.b64 %0, {%1, %2};" : "=l"(v[k]) : "f"(a), "f"(b));
  }
  unsigned long long m, c;
  asm("mov.b64 %0, {%1, %2};" : "=l"(m) : "f"(0.999f), "f"(0.999f));
  asm("mov.b64 %0, {%1, %2};" : "=l"(c) : "f"(0.001f), "f"(0.001f));
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) asm volatile("fma.rn.ftz.f32x2 %0, %0, %1, %2;" : "+l"(v[k]) : "l"(m), "l"(c));
  }
  float s = 0.f;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    float a, b;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v[k]));
    s += a + b;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  int sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* out;
  cudaMalloc(&out, sizeof(float) * sms * 4 * 1024);
  const int iters = 1 << 14;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const char* names[] = {"ex2", "ffma2", "ex2.f16x2", "ex2.bf16x2"};
  for (int warps : {4, 8, 16, 32}) {
    for (int which = 0; which < 4; ++which) {
      dim3 grid(sms), block(32 * warps);
      auto run = [&](int it) {
        if (which == 0) k_ex2<<<grid, block>>>(out, it);
        else if (which == 1) k_ffma2<<<grid, block>>>(out, it);
        else if (which == 2) k_ex2_x2<false><<<grid, block>>>(out, it);
        else k_ex2_x2<true><<<grid, block>>>(out, it);
      };
      run(16);
      cudaEventRecord(e0);
      run(iters);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      const double ops = double(sms) * 32 * warps * 8.0 * iters * (which == 0 ? 1 : 2);
      printf("%-10s warps/SM %2d: %8.1f G lane-ops/s per SM (%s)\n", names[which], warps,
             ops / (ms * 1e-3) / sms / 1e9, which == 1 ? "fp32 FMAs" : "exps");
    }
  }
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("max SM clock %.0f MHz\n", clk / 1e3);
  return 0;
}
