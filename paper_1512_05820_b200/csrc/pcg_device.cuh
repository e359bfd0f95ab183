// Device pieces shared by the multi-kernel PCG iteration (pcg.cu) and the
// persistent single-cluster solver (pcg_cluster.cu).
#pragma once

#include "common.cuh"

namespace rk {

constexpr int kFuseMax = 64;  // widths whose mu solve runs inside a block (update tail / cluster solver)

// mu = F^{-1} c for w <= kFuseMax with one 256-thread block: warp q-rows
// (rows warp + 8q), lanes over the row's entries, butterfly sums. Each batch of
// 32 entries issues all its rows' loads before any fma, so a triangular
// mat-vec costs ceil(w / 32) L2 round trips rather than one per row.
__device__ inline void solve_factor_warps(const rk_pcg_plan& P, const double* c, double* y, double* mu) {
  constexpr int R = kFuseMax / 8;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int w = (int)P.wchol, m = (int)P.m;
  const int64_t ldl = P.ldl;
  const double* __restrict__ L = P.L;
  double a[R], lv[R];
#pragma unroll
  for (int q = 0; q < R; ++q) a[q] = 0.0;
  if (P.linv_full) {  // mu_i = sum_j Finv[j, i] c_j (column i: coalesced), one pass
    for (int t = 0; 32 * t < w; ++t) {
      const int j = lane + 32 * t;
#pragma unroll
      for (int q = 0; q < R; ++q) {
        const int i = warp + 8 * q;
        lv[q] = (i < w && j < w) ? __ldg(L + j + (int64_t)i * ldl) : 0.0;
      }
      const double cj = j < w ? c[j] : 0.0;
#pragma unroll
      for (int q = 0; q < R; ++q) a[q] = fma(lv[q], cj, a[q]);
    }
    warp_sum_n(a);
#pragma unroll
    for (int q = 0; q < R; ++q) {
      const int i = warp + 8 * q;
      if (lane == 0 && i < w) mu[i] = a[q];
    }
    for (int i = threadIdx.x; i < m; i += blockDim.x) {
      if (i >= w) {
        const double d = P.sqd[i - w];
        mu[i] = c[i] / (d * d);
      }
    }
    return;
  }
  for (int t = 0; 32 * t < w; ++t) {  // y_i = sum_{j <= i} Linv[i, j] c_j
    const int j = lane + 32 * t;
#pragma unroll
    for (int q = 0; q < R; ++q) {
      const int i = warp + 8 * q;
      lv[q] = (i < w && j <= i) ? __ldg(L + i + (int64_t)j * ldl) : 0.0;
    }
    const double cj = j < w ? c[j] : 0.0;
#pragma unroll
    for (int q = 0; q < R; ++q) a[q] = fma(lv[q], cj, a[q]);
  }
  warp_sum_n(a);
#pragma unroll
  for (int q = 0; q < R; ++q) {
    const int i = warp + 8 * q;
    if (lane == 0 && i < w) y[i] = a[q];
    a[q] = 0.0;
  }
  __syncthreads();
  for (int t = 0; 32 * t < w; ++t) {  // mu_i = sum_{j >= i} Linv[j, i] y_j (column i: coalesced)
#pragma unroll
    for (int q = 0; q < R; ++q) {
      const int i = warp + 8 * q;
      const int j = lane + 32 * t;
      lv[q] = (i < w && j >= i && j < w) ? __ldg(L + j + (int64_t)i * ldl) : 0.0;
    }
    const int j = lane + 32 * t;
    const double yj = j < w ? y[j] : 0.0;
#pragma unroll
    for (int q = 0; q < R; ++q) a[q] = fma(lv[q], yj, a[q]);
  }
  warp_sum_n(a);
#pragma unroll
  for (int q = 0; q < R; ++q) {
    const int i = warp + 8 * q;
    if (lane == 0 && i < w) mu[i] = a[q];
  }
  for (int i = threadIdx.x; i < m; i += blockDim.x) {
    if (i >= w) {
      const double d = P.sqd[i - w];
      mu[i] = c[i] / (d * d);
    }
  }
}

}  // namespace rk
