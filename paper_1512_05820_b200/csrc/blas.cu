// Tall-skinny dense kernels on column-major N x m blocks (K4 GEMV-T, K5 GEMV-N),
// plus the small vector helpers the host layer needs.
//
// Replaces the OpenBLAS dgemv / ddot / elementwise numpy calls at
// krylov.py:80-81 (`Y @ p`, `Y.T @ full`), krylov.py:156 (`cross.T @ z`),
// krylov.py:291,326 (`Y @ mu`), krylov.py:335-337 (FOM re-orthogonalisation,
// restructured as block classical Gram-Schmidt, see pcg.cu) and
// threestage.py:482-483 (`V / sqrt_t`).
//
// Reductions are two-level and deterministic: each block owns a row chunk and
// writes one partial per column; a second kernel sums the partials of a column
// in a fixed order with one warp per column.
#include <algorithm>

#include "common.cuh"

namespace rk {

constexpr int kGemvChunk = 1024;   // rows per block of the GEMV-T partial pass
constexpr int kGemvCols = 32;      // columns per block of the GEMV-T partial pass
constexpr int kGemvThreads = 256;

// partials[col * nchunks + chunk] = sum_{rows in chunk} B[row, col] * x[row]
// Columns [0, m) with m = (m_dev ? *m_dev : m_host); skipped entirely if *done.
__global__ void __launch_bounds__(kGemvThreads) k_gemv_t_partial(
    int64_t n, int64_t m_host, const int64_t* m_dev, const int64_t* done, const double* __restrict__ B,
    int64_t ldb, const double* __restrict__ x, int64_t x_col_from_m, int64_t ldx, double* __restrict__ partials,
    int64_t nchunks) {
  pdl_wait();
  pdl_trigger();
  if (done && *done) return;
  const int64_t m = m_dev ? *m_dev : m_host;
  const int64_t c0 = (int64_t)blockIdx.y * kGemvCols;
  if (c0 >= m) return;
  __shared__ double xs[kGemvChunk];
  const int64_t chunk = blockIdx.x;
  const int64_t r0 = chunk * kGemvChunk;
  const int rows = (int)min((int64_t)kGemvChunk, n - r0);
  // x may be column m of a block (the freshly written direction, FOM sweeps)
  const double* xv = x + (x_col_from_m ? m * ldx : 0);
  for (int i = threadIdx.x; i < rows; i += blockDim.x) xs[i] = xv[r0 + i];
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int cend = (int)min((int64_t)kGemvCols, m - c0);
  for (int c = warp; c < cend; c += nw) {
    const double* __restrict__ col = B + (c0 + c) * ldb + r0;
    double acc = 0.0;
#pragma unroll 8
    for (int i = lane; i < rows; i += 32) acc = fma(__ldcs(col + i), xs[i], acc);
    acc = warp_sum(acc);
    if (lane == 0) partials[(c0 + c) * nchunks + chunk] = acc;
  }
}

// out[c] = (sum_chunk partials[c*nchunks + chunk]) [/ div[c]] for c < m.
__global__ void __launch_bounds__(256) k_gemv_t_reduce(int64_t m_host, const int64_t* m_dev,
                                                       const int64_t* done,
                                                       const double* __restrict__ partials,
                                                       int64_t nchunks, const double* __restrict__ div,
                                                       double* __restrict__ out) {
  pdl_wait();
  pdl_trigger();
  if (done && *done) return;
  const int64_t m = m_dev ? *m_dev : m_host;
  const int lane = threadIdx.x & 31;
  const int64_t c = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (c >= m) return;
  double acc = 0.0;
  for (int64_t b = lane; b < nchunks; b += 32) acc += partials[c * nchunks + b];
  acc = warp_sum(acc);
  if (lane == 0) out[c] = div ? acc / div[c] : acc;
}

// y = B c (op 0), y0 + B c (op 1), y0 - B c (op 2). Thread per row; the m
// coefficients sit in shared memory and the column loads coalesce across the
// warp. The dot is accumulated left to right (as a reference dgemv row).
template <int OP>
__global__ void __launch_bounds__(256) k_gemv_n(int64_t n, int64_t m_host, const int64_t* m_dev,
                                                const int64_t* done, const double* __restrict__ B,
                                                int64_t ldb, const double* __restrict__ c,
                                                const double* y0, double* y, int64_t y_col_from_m,
                                                int64_t ldy) {
  pdl_wait();
  pdl_trigger();
  if (done && *done) return;
  const int64_t m = m_dev ? *m_dev : m_host;
  extern __shared__ double cs[];
  for (int64_t j = threadIdx.x; j < m; j += blockDim.x) cs[j] = c[j];
  __syncthreads();
  const int64_t off = y_col_from_m ? m * ldy : 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    const double* __restrict__ row = B + i;
    int64_t j = 0;
    for (; j + 4 <= m; j += 4) {
      const double b0 = __ldcs(row + (j + 0) * ldb), b1 = __ldcs(row + (j + 1) * ldb);
      const double b2 = __ldcs(row + (j + 2) * ldb), b3 = __ldcs(row + (j + 3) * ldb);
      s = fma(b0, cs[j + 0], s);
      s = fma(b1, cs[j + 1], s);
      s = fma(b2, cs[j + 2], s);
      s = fma(b3, cs[j + 3], s);
    }
    for (; j < m; ++j) s = fma(__ldcs(row + j * ldb), cs[j], s);
    if (OP == 0) y[off + i] = s;
    else if (OP == 1) y[off + i] = __dadd_rn(y0[off + i], s);
    else y[off + i] = __dsub_rn(y0[off + i], s);
  }
}

__global__ void __launch_bounds__(256) k_dot(int64_t n, const double* __restrict__ x,
                                             const double* __restrict__ y, double* partials,
                                             uint32_t* ticket, double* out) {
  __shared__ double scratch[32];
  double acc[1] = {0.0};
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    acc[0] = fma(x[i], y[i], acc[0]);
  block_sum<1>(acc, scratch);
  if (publish_and_check_last(acc, 1, partials, ticket)) {
    __shared__ double tot[1];
    combine_partials(partials, gridDim.x, 1, tot);
    if (threadIdx.x == 0) out[0] = tot[0];
  }
}

__global__ void k_scale_columns(int64_t n, int64_t m, const double* __restrict__ V, int64_t ldv,
                                const double* __restrict__ s, double* __restrict__ out, int64_t ldo) {
  const int64_t j = blockIdx.y;
  const double d = s[j];
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i + j * ldo] = V[i + j * ldv] / d;  // threestage.py:483 `V / sqrt_t`
}

__global__ void k_axpby(int64_t n, double a, const double* __restrict__ x, double b, double* y) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    y[i] = __dadd_rn(__dmul_rn(a, x[i]), __dmul_rn(b, y[i]));
}

__global__ void k_sub_from(int64_t n, const double* __restrict__ x0, double* y) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    y[i] = __dsub_rn(x0[i], y[i]);
}

}  // namespace rk

namespace rkh {

int64_t gemv_nchunks(int64_t n) { return std::max<int64_t>(1, (n + rk::kGemvChunk - 1) / rk::kGemvChunk); }

int elementwise_grid(int64_t n) {
  const int64_t need = (n + 255) / 256;
  return (int)std::max<int64_t>(1, std::min<int64_t>(need, (int64_t)sm_count() * 16));
}

// GEMV-T in two launches; columns read from *m_dev when given (device count).
void launch_gemv_t(int64_t n, int64_t m_max, const int64_t* m_dev, const int64_t* done, const double* B,
                   int64_t ldb, const double* x, int64_t x_col_from_m, int64_t ldx, double* partials,
                   const double* div, double* out, cudaStream_t s) {
  if (m_max <= 0 || n <= 0) return;
  const int64_t nch = gemv_nchunks(n);
  dim3 g1((unsigned)nch, (unsigned)((m_max + rk::kGemvCols - 1) / rk::kGemvCols));
  launch_pdl(rk::k_gemv_t_partial, g1, dim3(rk::kGemvThreads), 0, s, n, m_max, m_dev, done, B, ldb, x,
             x_col_from_m, ldx, partials, nch);
  const int64_t g2 = (m_max + 7) / 8;
  launch_pdl(rk::k_gemv_t_reduce, dim3((unsigned)g2), dim3(256), 0, s, m_max, m_dev, done, partials, nch, div, out);
}

void launch_gemv_n(int64_t n, int64_t m_max, const int64_t* m_dev, const int64_t* done, const double* B,
                   int64_t ldb, const double* c, const double* y0, double* y, int32_t op,
                   int64_t y_col_from_m, int64_t ldy, cudaStream_t s) {
  if (n <= 0) return;
  const size_t smem = (size_t)std::max<int64_t>(m_max, 1) * sizeof(double);
  const int grid = elementwise_grid(n);
  if (op == 0) {
    launch_pdl(rk::k_gemv_n<0>, dim3(grid), dim3(256), smem, s, n, m_max, m_dev, done, B, ldb, c, y0, y,
               y_col_from_m, ldy);
  } else if (op == 1) {
    launch_pdl(rk::k_gemv_n<1>, dim3(grid), dim3(256), smem, s, n, m_max, m_dev, done, B, ldb, c, y0, y,
               y_col_from_m, ldy);
  } else {
    launch_pdl(rk::k_gemv_n<2>, dim3(grid), dim3(256), smem, s, n, m_max, m_dev, done, B, ldb, c, y0, y,
               y_col_from_m, ldy);
  }
}

int gemv_n_smem_ok(int64_t m) {
  static bool configured = false;
  const int64_t bytes = std::max<int64_t>(m, 1) * (int64_t)sizeof(double);
  if (bytes > 200 * 1024) return 0;
  if (!configured) {
    cudaFuncSetAttribute(rk::k_gemv_n<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(rk::k_gemv_n<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(rk::k_gemv_n<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    configured = true;
  }
  return 1;
}

void launch_dot(int64_t n, const double* x, const double* y, double* out, double* ws, uint32_t* ticket,
                cudaStream_t s) {
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, (int64_t)sm_count() * 4));
  rk::k_dot<<<grid, 256, 0, s>>>(n, x, y, ws, ticket, out); rkh::note_launch();
}

int dot_grid_max() { return sm_count() * 4; }

void launch_scale_columns(int64_t n, int64_t m, const double* V, int64_t ldv, const double* sc, double* out,
                          int64_t ldo, cudaStream_t s) {
  if (n <= 0 || m <= 0) return;
  const int gx = (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, std::max<int64_t>(1, (int64_t)sm_count() * 16 / std::min<int64_t>(m, 16))));
  dim3 g((unsigned)gx, (unsigned)m);
  rk::k_scale_columns<<<g, 256, 0, s>>>(n, m, V, ldv, sc, out, ldo); rkh::note_launch();
}

void launch_axpby(int64_t n, double a, const double* x, double b, double* y, cudaStream_t s) {
  if (n > 0) {
    rk::k_axpby<<<elementwise_grid(n), 256, 0, s>>>(n, a, x, b, y); rkh::note_launch();
  }
}

void launch_sub_from(int64_t n, const double* x0, double* y, cudaStream_t s) {
  if (n > 0) {
    rk::k_sub_from<<<elementwise_grid(n), 256, 0, s>>>(n, x0, y); rkh::note_launch();
  }
}

}  // namespace rkh
