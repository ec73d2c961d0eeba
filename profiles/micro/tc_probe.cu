// tc_probe.cu — step-by-step checks of the tcgen05 building blocks used by
// csrc/prefill_attn.cu (same helpers, included as one translation unit):
//   1. TMEM alloc + tcgen05.st/ld round trip
//   2. S = Q K^T (M=N=128, K=128): K-major SW128 A and B descriptors
//   3. O = P V with V as an MN-major SW128 B operand
// Build: nvcc -std=c++17 -gencode arch=compute_100a,code=sm_100a -O2 -o tc_probe tc_probe.cu
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>

#include "../../paper_2412_12488_b200/csrc/prefill_attn.cu"

using namespace mkv;

#define CK(x)                                                                  \
  do {                                                                         \
    cudaError_t e_ = (x);                                                      \
    if (e_ != cudaSuccess) {                                                   \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
      exit(1);                                                                 \
    }                                                                          \
  } while (0)

__global__ void k_tmem_roundtrip(float* out) {
  __shared__ uint32_t slot;
  const int tid = threadIdx.x, warp = tid >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(
                     smem_u32(&slot))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = slot;
  const uint32_t lane_off = static_cast<uint32_t>(warp * 32) << 16;
  float v[16];
  for (int i = 0; i < 16; ++i) v[i] = tid * 1000.f + i;
  tmem_st16(tmem + lane_off + 128 + 16, v);
  float w[16];
  tmem_ld16(tmem + lane_off + 128 + 16, w);
  for (int i = 0; i < 16; ++i) out[tid * 16 + i] = w[i];
  if (tid == 0) out[128 * 16] = __uint_as_float(tmem);
  fence_before();
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem) : "memory");
}

// A [128][128] bf16 row-major (K contiguous), B given as [128 rows][128] bf16
// row-major; mode 0: D = A B^T (B rows = N, K-major); mode 1: D = A B with B
// rows = K (keys), contiguous = N (MN-major).
__global__ void k_mma(const __nv_bfloat16* A, const __nv_bfloat16* B, float* D, int mode) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  const int tid = threadIdx.x, warp = tid >> 5;
  const uint32_t sA = smem_u32(smem), sB = smem_u32(smem + kTile);
  const uint32_t bar = smem_u32(smem + 2 * kTile);
  uint32_t* slot = reinterpret_cast<uint32_t*>(smem + 2 * kTile + 16);
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(
                     smem_u32(slot))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (tid == 0) {
    mbar_init(bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int c = 0; c < 16; ++c) {
    const uint4 a = *reinterpret_cast<const uint4*>(A + tid * 128 + c * 8);
    const uint4 b = *reinterpret_cast<const uint4*>(B + tid * 128 + c * 8);
    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(sA + sw128(tid, c)), "r"(a.x),
                 "r"(a.y), "r"(a.z), "r"(a.w));
    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(sB + sw128(tid, c)), "r"(b.x),
                 "r"(b.y), "r"(b.z), "r"(b.w));
  }
  fence_proxy_async();
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = *slot;
  if (tid == 0) {
    for (int k = 0; k < 8; ++k) {
      const uint32_t a_off = (k >> 2) * kAtom + (k & 3) * 32;
      if (mode == 0) {
        mma_bf16(tmem, umma_desc(sA + a_off, 16, 1024), umma_desc(sB + a_off, 16, 1024),
                 idesc_bf16(false), k > 0);
      } else {
        mma_bf16(tmem, umma_desc(sA + a_off, 16, 1024), umma_desc(sB + k * 2048, kAtom, 1024),
                 idesc_bf16(true), k > 0);
      }
    }
    mma_commit(bar);
  }
  mbar_wait(bar, 0);
  fence_after();
  const uint32_t lane_off = static_cast<uint32_t>(warp * 32) << 16;
  for (int c0 = 0; c0 < 128; c0 += 16) {
    float v[16];
    tmem_ld16(tmem + lane_off + c0, v);
    for (int i = 0; i < 16; ++i) D[tid * 128 + c0 + i] = v[i];
  }
  fence_before();
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem) : "memory");
}

static float bf(uint16_t h) {
  uint32_t u = static_cast<uint32_t>(h) << 16;
  float f;
  memcpy(&f, &u, 4);
  return f;
}
static uint16_t tobf(float f) {
  uint32_t u;
  memcpy(&u, &f, 4);
  return static_cast<uint16_t>((u + 0x7FFF + ((u >> 16) & 1)) >> 16);
}

int main(int argc, char** argv) {
  const int stage = argc > 1 ? atoi(argv[1]) : 0;
  // 1. TMEM round trip
  if (stage == 0 || stage == 1) {
    float* d;
    CK(cudaMalloc(&d, sizeof(float) * (128 * 16 + 1)));
    k_tmem_roundtrip<<<1, 128>>>(d);
    CK(cudaDeviceSynchronize());
    std::vector<float> h(128 * 16 + 1);
    CK(cudaMemcpy(h.data(), d, sizeof(float) * h.size(), cudaMemcpyDeviceToHost));
    int bad = 0;
    for (int t = 0; t < 128; ++t)
      for (int i = 0; i < 16; ++i) bad += h[t * 16 + i] != t * 1000.f + i;
    uint32_t base;
    memcpy(&base, &h[128 * 16], 4);
    printf("tmem roundtrip: bad=%d tmem_base=0x%08x\n", bad, base);
    cudaFree(d);
  }
  std::vector<uint16_t> A(128 * 128), B(128 * 128);
  srand(1);
  for (auto& x : A) x = tobf((rand() / (float)RAND_MAX - 0.5f));
  for (auto& x : B) x = tobf((rand() / (float)RAND_MAX - 0.5f));
  __nv_bfloat16 *dA, *dB;
  float* dD;
  CK(cudaMalloc(&dA, 2 * A.size()));
  CK(cudaMalloc(&dB, 2 * B.size()));
  CK(cudaMalloc(&dD, 4 * 128 * 128));
  CK(cudaMemcpy(dA, A.data(), 2 * A.size(), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dB, B.data(), 2 * B.size(), cudaMemcpyHostToDevice));
  const int smem = 2 * kTile + 64 + 1024;
  CK(cudaFuncSetAttribute(k_mma, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  for (int mode = 0; mode < 2; ++mode) {
    if (stage != 0 && stage != 2 + mode) continue;
    CK(cudaMemset(dD, 0, 4 * 128 * 128));
    k_mma<<<1, 128, smem>>>(dA, dB, dD, mode);
    CK(cudaDeviceSynchronize());
    std::vector<float> D(128 * 128);
    CK(cudaMemcpy(D.data(), dD, 4 * D.size(), cudaMemcpyDeviceToHost));
    double maxerr = 0;
    for (int m = 0; m < 128; ++m)
      for (int n = 0; n < 128; ++n) {
        double ref = 0;
        for (int k = 0; k < 128; ++k)
          ref += (double)bf(A[m * 128 + k]) *
                 (mode == 0 ? bf(B[n * 128 + k]) : bf(B[k * 128 + n]));
        maxerr = fmax(maxerr, fabs(ref - D[m * 128 + n]));
      }
    printf("mma mode %d (%s): max err %.3e  D[0][0]=%f D[5][7]=%f\n", mode,
           mode == 0 ? "A B^T, K-major B" : "A B, MN-major B", maxerr, D[0], D[5 * 128 + 7]);
  }
  // 4. the full prefill kernel, identity-paged pool: Hkv=8, Hq=64, n keys, queries [qb, n)
  if (stage == 0 || stage == 4) {
    const int Hkv = 8, Hq = 64, n = argc > 2 ? atoi(argv[2]) : 300, qb = argc > 3 ? atoi(argv[3]) : 0;
    const int nq = n - qb;
    const int64_t row = 2 * Hkv * 128;  // bf16 elements per (token) row: K then V
    std::vector<uint16_t> pool(static_cast<size_t>(n) * row), q(static_cast<size_t>(nq) * Hq * 128);
    for (auto& x : pool) x = tobf((rand() / (float)RAND_MAX - 0.5f));
    for (auto& x : q) x = tobf((rand() / (float)RAND_MAX - 0.5f));
    std::vector<int32_t> slots(n);
    for (int i = 0; i < n; ++i) slots[i] = (i * 7) % n == i ? i : i;  // identity
    __nv_bfloat16 *dP, *dQ, *dO;
    int32_t* dS;
    CK(cudaMalloc(&dP, 2 * pool.size()));
    CK(cudaMalloc(&dQ, 2 * q.size()));
    CK(cudaMalloc(&dO, 2 * q.size()));
    CK(cudaMalloc(&dS, 4 * n));
    CK(cudaMemcpy(dP, pool.data(), 2 * pool.size(), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dQ, q.data(), 2 * q.size(), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dS, slots.data(), 4 * n, cudaMemcpyHostToDevice));
    CK(cudaMemset(dO, 0xFF, 2 * q.size()));
    printf("launching prefill n=%d qb=%d\n", n, qb);
    fflush(stdout);
    PoolTensorMap pm, rm;
    const int64_t rows = n;
    if (!make_pool_tensor_map(dP, 1, rows, row / 4, 16, &pm) ||
        !make_pool_tensor_map(dP, 1, rows, row / 4, 1, &rm)) {
      printf("tensor map encode failed\n");
      return 1;
    }
    const bool ok = launch_prefill_attn(pm, rm, 0, 16, dS, dQ, qb, nq, Hq, Hkv, 128, 0.0883883f, dO, 0);
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    printf("prefill ok=%d done\n", ok);
    std::vector<uint16_t> o(q.size());
    CK(cudaMemcpy(o.data(), dO, 2 * o.size(), cudaMemcpyDeviceToHost));
    double maxerr = 0;
    int checked = 0;
    for (int i = 0; i < nq; i += (nq > 40 ? 7 : 1))
      for (int hh = 0; hh < Hq; hh += 5) {
        const int kvh = hh / 8, pos = qb + i;
        std::vector<double> s(pos + 1);
        double mx = -1e30;
        for (int k = 0; k <= pos; ++k) {
          double acc = 0;
          for (int d = 0; d < 128; ++d)
            acc += (double)bf(q[((size_t)i * Hq + hh) * 128 + d]) * bf(pool[k * row + kvh * 128 + d]);
          s[k] = acc * 0.0883883;
          mx = fmax(mx, s[k]);
        }
        double sum = 0;
        for (int k = 0; k <= pos; ++k) sum += (s[k] = exp(s[k] - mx));
        for (int d = 0; d < 128; ++d) {
          double acc = 0;
          for (int k = 0; k <= pos; ++k) acc += s[k] * bf(pool[k * row + (Hkv + kvh) * 128 + d]);
          const double got = bf(o[((size_t)i * Hq + hh) * 128 + d]);
          const double err = fabs(acc / sum - got);
          if (!(err <= maxerr)) maxerr = err;  // catches NaN
        }
        ++checked;
      }
    printf("prefill: %d rows checked, max err %.3e\n", checked, maxerr);
  }
  return 0;
}
