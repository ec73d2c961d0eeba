// Times the library's own k_copy_rows (linked from kernels.cu) on the same
// synthetic DirectSend as copy_variants.cu, to separate kernel code from
// environment.  nvcc ... lib_kernel.cu ../../paper_2412_12488_b200/csrc/kernels.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <vector>
#include "../../paper_2412_12488_b200/csrc/kernels.cuh"
int main() {
  const int64_t n_rows = 8191, layers = 80, pages = 8192 / 16 + 16, W = 512;
  const int64_t lw = pages * 16 * W;
  uint64_t *src, *dst; uint8_t* fill; int32_t *si, *di, *verdict; unsigned long long* wr; uint32_t* wl; uint32_t* st;
  cudaMalloc(&src, lw * layers * 8); cudaMalloc(&dst, lw * layers * 8);
  cudaMalloc(&fill, pages * 16 * layers); cudaMalloc(&si, 4 * n_rows); cudaMalloc(&di, 4 * n_rows);
  cudaMalloc(&verdict, 8); cudaMalloc(&wr, 8 * 16); cudaMalloc(&wl, 4 * 16 * layers); cudaMalloc(&st, 4);
  std::vector<int32_t> h(n_rows); for (int64_t i = 0; i < n_rows; ++i) h[i] = int32_t(i);
  cudaMemcpy(si, h.data(), 4 * n_rows, cudaMemcpyHostToDevice); cudaMemcpy(di, h.data(), 4 * n_rows, cudaMemcpyHostToDevice);
  int32_t v[2] = {0, 0}; cudaMemcpy(verdict, v, 8, cudaMemcpyHostToDevice);
  cudaMemset(src, 1, lw * layers * 8);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int variant = 0; variant < 3; ++variant) {
    mkv::CopyParams p{};
    p.src = src; p.src_layer_words = lw; p.src_idx = si; p.dst = dst; p.dst_layer_words = lw; p.dst_idx = di;
    p.dst_fill = fill; p.dst_fill_layer = pages * 16; p.fill_value = 2; p.n_rows = n_rows; p.layer0 = 0;
    p.n_layers = layers; p.W = W;
    if (variant >= 1) { p.win_received = wr; p.win_layer_rows = wl; p.win_layers = layers; }
    if (variant >= 2) { p.verdict = verdict; p.status = st; }
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    float best = 1e9;
    for (int rep = 0; rep < 7; ++rep) {
      cudaMemset(fill, 0, pages * 16 * layers);
      cudaEventRecord(a); mkv::launch_copy_rows(p, 0, sms); cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b); if (rep >= 2 && ms < best) best = ms;
    }
    printf("library k_copy_rows variant %d (%s): %.1f us  %.1f GB/s r+w  %s\n", variant,
           variant == 0 ? "fill only" : variant == 1 ? "+window accounting" : "+verdict",
           best * 1e3, 2.0 * n_rows * layers * 4096 / (best * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
  }
}
