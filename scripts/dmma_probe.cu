// Register-only throughput probe of the sm_100a fp64 mma.sync shapes
// (m8n8k4 vs m16n8k4 / m16n8k8 / m16n8k16). Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gpurun_out/dmma_probe scripts/dmma_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kIters = 4096;
constexpr int kChains = 8;  // independent accumulators per warp

__global__ void p884(double* out) {
  double c[kChains][2] = {};
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int q = 0; q < kChains; ++q)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[q][0]), "+d"(c[q][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int q = 0; q < kChains; ++q) s += c[q][0] + c[q][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void p1684(double* out) {
  double c[kChains][4] = {};
  double a0 = threadIdx.x * 1e-3, a1 = a0 + 1, b = 1.0 + threadIdx.x * 1e-4;
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int q = 0; q < kChains; ++q)
      asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
                   : "+d"(c[q][0]), "+d"(c[q][1]), "+d"(c[q][2]), "+d"(c[q][3]) : "d"(a0), "d"(a1), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int q = 0; q < kChains; ++q) s += c[q][0] + c[q][1] + c[q][2] + c[q][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void p1688(double* out) {
  double c[kChains][4] = {};
  double a0 = threadIdx.x * 1e-3, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, b0 = 1.0 + threadIdx.x * 1e-4, b1 = b0 + 1;
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int q = 0; q < kChains; ++q)
      asm volatile(
          "mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
          : "+d"(c[q][0]), "+d"(c[q][1]), "+d"(c[q][2]), "+d"(c[q][3])
          : "d"(a0), "d"(a1), "d"(a2), "d"(a3), "d"(b0), "d"(b1));
  }
  double s = 0;
#pragma unroll
  for (int q = 0; q < kChains; ++q) s += c[q][0] + c[q][1] + c[q][2] + c[q][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void p16816(double* out) {
  double c[kChains][4] = {};
  double a[8], b[4];
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3 + i;
  for (int i = 0; i < 4; ++i) b[i] = 1.0 + threadIdx.x * 1e-4 + i;
  for (int it = 0; it < kIters / 4; ++it) {
#pragma unroll
    for (int q = 0; q < kChains; ++q)
      asm volatile(
          "mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, "
          "{%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
          : "+d"(c[q][0]), "+d"(c[q][1]), "+d"(c[q][2]), "+d"(c[q][3])
          : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]), "d"(b[0]),
            "d"(b[1]), "d"(b[2]), "d"(b[3]));
  }
  double s = 0;
#pragma unroll
  for (int q = 0; q < kChains; ++q) s += c[q][0] + c[q][1] + c[q][2] + c[q][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <typename K>
static void run(const char* name, K kern, double flops_per_mma_iter, int warps_per_block, int blocks) {
  double* out;
  cudaMalloc(&out, sizeof(double) * blocks * warps_per_block * 32);
  kern<<<blocks, warps_per_block * 32>>>(out);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int r = 0; r < 5; ++r) kern<<<blocks, warps_per_block * 32>>>(out);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double flops = 5.0 * blocks * warps_per_block * (double)kIters * kChains * flops_per_mma_iter;
  printf("%-10s warps/blk %2d blocks %5d : %.2f TFLOP/s (%s)\n", name, warps_per_block, blocks, flops / ms / 1e9,
         cudaGetErrorString(cudaGetLastError()));
  cudaFree(out);
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int w : {4, 8, 16}) {
    run("m8n8k4", p884, 2.0 * 8 * 8 * 4, w, sms * 2);
    run("m16n8k4", p1684, 2.0 * 16 * 8 * 4, w, sms * 2);
    run("m16n8k8", p1688, 2.0 * 16 * 8 * 8, w, sms * 2);
    run("m16n8k16", p16816, 2.0 * 16 * 8 * 16 / 4, w, sms * 2);  // kIters/4 iterations of k16
  }
  // One CTA per SM with 1, 2, 3, 4 warps: does a single warp reach the SM's
  // DMMA rate, or a quarter of it (one pipe per sub-partition)?
  for (int w : {1, 2, 3, 4, 8}) run("m8n8k4/SM", p884, 2.0 * 8 * 8 * 4, w, sms);
  return 0;
}
