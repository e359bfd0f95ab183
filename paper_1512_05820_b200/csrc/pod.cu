// Small m x m kernels of the POD truncation that keep the reduced problem on
// the device between the DMMA Gram and the basis reconstruction:
//   weighted Gram  G^ = 1/2 (W + W'),  W_ab = (gamma_a G_ab) gamma_b      (pod.py:127-129)
//   snapshot coefficients  coef_ij = (V_ij / sigma_j) gamma_i           (pod.py:91)
// Elementwise products are explicitly rounded (no fma contraction) so they
// reproduce the reference's numpy expressions bit for bit.
#include <algorithm>

#include "common.cuh"

namespace rk {

// mode 0: G is a full (not necessarily symmetric) matrix -> 1/2 (W + W').
// mode 1: only the upper triangle of G is defined (rk_gram_upper); column b of
//         that triangle is scaled by col_scale[b] (may be null), then mirrored,
//         so W is symmetric and 1/2 (W + W') = W exactly.
__global__ void k_pod_weighted_gram(int64_t m, const double* __restrict__ G, int64_t ldg, int mode,
                                    const double* __restrict__ col_scale, const double* __restrict__ gamma,
                                    double* __restrict__ out, int64_t ldo) {
  const int64_t total = m * m;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t a = e % m, b = e / m;
    double v;
    if (mode == 1) {
      const int64_t lo = min(a, b), hi = max(a, b);
      double g = G[lo + hi * ldg];
      if (col_scale) g = __dmul_rn(g, col_scale[hi]);
      v = __dmul_rn(__dmul_rn(gamma[a], g), gamma[b]);
    } else {
      const double wab = __dmul_rn(__dmul_rn(gamma[a], G[a + b * ldg]), gamma[b]);
      const double wba = __dmul_rn(__dmul_rn(gamma[b], G[b + a * ldg]), gamma[a]);
      v = __dmul_rn(0.5, __dadd_rn(wab, wba));
    }
    out[a + b * ldo] = v;
  }
}

// coef[:, j] = V[:, m-1-j] / sigma[j] * gamma  (V: eigenvectors in ascending order)
__global__ void k_pod_coef(int64_t m, int64_t y, const double* __restrict__ V, int64_t ldv,
                           const double* __restrict__ sigma, const double* __restrict__ gamma,
                           double* __restrict__ coef, int64_t ldc) {
  const int64_t total = m * y;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e % m, j = e / m;
    coef[i + j * ldc] = __dmul_rn(V[i + (m - 1 - j) * ldv] / sigma[j], gamma[i]);
  }
}

}  // namespace rk

extern "C" {

int rk_pod_weighted_gram(int64_t m, const double* G, int64_t ldg, int32_t mode, const double* col_scale,
                         const double* gamma, double* out, int64_t ldo, void* stream) {
  RK_REQUIRE(m >= 0 && ldg >= m && ldo >= m && (mode == 0 || mode == 1), RK_ERR_DIMENSION,
             "rk_pod_weighted_gram: bad shape/mode");
  if (m == 0) return RK_OK;
  RK_REQUIRE(G && gamma && out, RK_ERR_ARG, "rk_pod_weighted_gram: null pointer");
  const int64_t total = m * m;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((total + 255) / 256, 4096));
  rk::k_pod_weighted_gram<<<grid, 256, 0, rkh::as_stream(stream)>>>(m, G, ldg, mode, col_scale, gamma, out, ldo);
  rkh::note_launch();
  return rkh::cuda_check("rk_pod_weighted_gram");
}

int rk_pod_coef(int64_t m, int64_t y, const double* V, int64_t ldv, const double* sigma, const double* gamma,
                double* coef, int64_t ldc, void* stream) {
  RK_REQUIRE(m >= 0 && y >= 0 && y <= m && ldv >= m && ldc >= m, RK_ERR_DIMENSION, "rk_pod_coef: bad shape");
  if (m == 0 || y == 0) return RK_OK;
  RK_REQUIRE(V && sigma && gamma && coef, RK_ERR_ARG, "rk_pod_coef: null pointer");
  const int64_t total = m * y;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((total + 255) / 256, 4096));
  rk::k_pod_coef<<<grid, 256, 0, rkh::as_stream(stream)>>>(m, y, V, ldv, sigma, gamma, coef, ldc);
  rkh::note_launch();
  return rkh::cuda_check("rk_pod_coef");
}

}  // extern "C"
