// Does a predicated-off DMMA cost DMMA-pipe time? Register-only m8n8k4 chains
// where chain q issues only if bit q of a runtime mask is set (warp-uniform),
// as the masked fragments of the K7 Gram. Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gpurun_out/dmma_pred_probe scripts/dmma_pred_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kIters = 4096;
constexpr int kChains = 16;

__global__ void p884_mask(double* out, unsigned mask) {
  double c[kChains][2] = {};
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  bool act[kChains];
#pragma unroll
  for (int q = 0; q < kChains; ++q) act[q] = (mask >> q) & 1u;
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int q = 0; q < kChains; ++q)
      if (act[q])
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(c[q][0]), "+d"(c[q][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int q = 0; q < kChains; ++q) s += c[q][0] + c[q][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  const int blocks = sms * 2, threads = 128;
  cudaMalloc(&out, sizeof(double) * blocks * threads);
  for (unsigned mask : {0xFFFFu, 0x00FFu, 0x000Fu, 0x0001u}) {
    p884_mask<<<blocks, threads>>>(out, mask);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    for (int r = 0; r < 5; ++r) p884_mask<<<blocks, threads>>>(out, mask);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const int active = __builtin_popcount(mask);
    const double flops = 5.0 * blocks * (threads / 32) * (double)kIters * active * 512.0;
    printf("{\"mask\": \"0x%04x\", \"active_chains\": %d, \"ms\": %.3f, \"useful_tflops\": %.2f, "
           "\"issued_equiv_tflops\": %.2f}\n", mask, active, ms / 5, flops / ms / 1e9,
           flops / ms / 1e9 * kChains / active);
  }
  return 0;
}
