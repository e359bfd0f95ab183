// Device-resident augmented PCG iteration (krylov.py:181-345).
//
// One iteration k is three kernels (plus four for the fom re-orthogonalisation):
//   k_spmv_pcg  (spmv.cu)  Ap_k = A p_k, gamma, p'p, breakdown test, alpha
//   k_pcg_update           x += alpha p_k, r -= alpha Ap_k, z = D^{-1} r, ||r||^2, r'z,
//                          c = cross' z; the last block to finish combines the
//                          block partials in a fixed order, records ||r||, decides
//                          convergence, and solves mu = F^{-1} c
//   k_pcg_direction        p_{k+1} = z + beta p_k - B mu (cg) | z - B mu (fom),
//                          written straight into V[:, k+1]; last block advances k
//   fom: 2 x (GEMV-T over [A p_0..A p_k], divide by gamma, GEMV-N over [p_0..p_k])
// All scalars stay on the device (rk_pcg_state); once a run converges or breaks
// down every later kernel returns immediately, so the host can launch
// iterations in batches and check the state once per batch.
//
// Elementwise updates use explicitly rounded operations (__dmul_rn/__dadd_rn)
// so they reproduce numpy's `x + alpha * p` bit for bit; only the summation
// order of the reductions differs from the reference.
#include <algorithm>

#include "common.cuh"

namespace rkh {
void launch_spmv_pcg(const rk_pcg_plan& P, cudaStream_t s);
void launch_curvature(const rk_pcg_plan& P, cudaStream_t s);
void launch_gemv_t(int64_t n, int64_t m_max, const int64_t* m_dev, const int64_t* done, const double* B,
                   int64_t ldb, const double* x, int64_t x_col_from_m, int64_t ldx, double* partials,
                   const double* div, double* out, cudaStream_t s);
void launch_gemv_n(int64_t n, int64_t m_max, const int64_t* m_dev, const int64_t* done, const double* B,
                   int64_t ldb, const double* c, const double* y0, double* y, int32_t op,
                   int64_t y_col_from_m, int64_t ldy, cudaStream_t s);
int gemv_n_smem_ok(int64_t m);
int64_t gemv_nchunks(int64_t n);
int spmv_grid(int64_t n, int lanes);
int auto_lanes(const rk_csr& A);
int curvature_grid(int64_t n);
int elementwise_grid(int64_t n);
}  // namespace rkh

namespace rk {

constexpr int kUpdThreads = 256;
constexpr int kRows = 4;                          // rows per thread per chunk
constexpr int kUpdChunk = kUpdThreads * kRows;    // rows per chunk
constexpr int kColGroup = 8;                      // cross columns reduced together
constexpr int kMaxProj = 4096;    // projection width supported by the fused path
constexpr int kMaxStagedChol = 96;  // dense factor staged in smem up to this width

// mu = F^{-1} c with F = blockdiag(L L', diag(sqd)^2): forward and back
// substitution on the dense block (one warp), division on the diagonal block
// (krylov.py:119-132 BlockDiagFactor.solve_spd).
__device__ void solve_factor(const rk_pcg_plan& P, const double* c, double* ysm, double* Ls, double* mu) {
  const int lane = threadIdx.x & 31;
  const int64_t w = P.wchol, m = P.m;
  // Stage the dense factor in shared memory first: the substitutions are a
  // chain of w dependent steps, and each step must not wait on L2.
  const bool staged = w <= kMaxStagedChol;
  const double* L = staged ? Ls : P.L;
  const int64_t ldl = staged ? w : P.ldl;
  if (staged) {
    for (int64_t e = threadIdx.x; e < w * w; e += blockDim.x) {
      const int64_t i = e % w, j = e / w;
      Ls[e] = (i >= j) ? P.L[i + j * P.ldl] : 0.0;
    }
    __syncthreads();
  }
  if (threadIdx.x < 32) {
    for (int64_t i = 0; i < w; ++i) {
      double s = 0.0;
      for (int64_t j = lane; j < i; j += 32) s = fma(L[i + j * ldl], ysm[j], s);
      s = warp_sum(s);
      if (lane == 0) ysm[i] = (c[i] - s) / L[i + i * ldl];
      __syncwarp();
    }
    for (int64_t i = w - 1; i >= 0; --i) {
      double s = 0.0;
      for (int64_t j = i + 1 + lane; j < w; j += 32) s = fma(L[j + i * ldl], ysm[j + w], s);
      s = warp_sum(s);
      if (lane == 0) ysm[i + w] = (ysm[i] - s) / L[i + i * ldl];
      __syncwarp();
    }
  }
  __syncthreads();
  for (int64_t i = threadIdx.x; i < m; i += blockDim.x) {
    if (i < w) mu[i] = ysm[i + w];
    else {
      const double d = P.sqd[i - w];
      mu[i] = c[i] / (d * d);
    }
  }
}

__global__ void __launch_bounds__(kUpdThreads) k_pcg_update(const rk_pcg_plan P, int entry) {
  rk_pcg_state* st = P.st;
  if (st->done) return;
  extern __shared__ double dyn[];
  double* red = dyn;                                  // 2 + m running block sums, then 2*wchol scratch
  __shared__ double scratch[64];
  __shared__ double wsum[(kUpdThreads / 32) * kColGroup];
  const int64_t k = st->k;
  const double alpha = entry ? 0.0 : st->alpha;
  const int64_t n = P.n, m = P.m;
  const double* __restrict__ p = P.V + k * P.ldv;
  const double* __restrict__ Ap = P.AV + (P.ldav ? k * P.ldav : 0);
  double* __restrict__ x = P.x;
  double* __restrict__ r = P.r;
  double* __restrict__ z = P.z;
  const double* __restrict__ dinv = P.dinv;
  const double* __restrict__ cross = P.cross;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int64_t j = threadIdx.x; j < 2 + m; j += blockDim.x) red[j] = 0.0;
  double acc[2] = {0.0, 0.0};
  const int64_t nchunks = (n + kUpdChunk - 1) / kUpdChunk;
  // Fast path: whole 1024-row chunks with 16-byte vector accesses, every load
  // of a stage issued before its first use (vectors and the columns of cross
  // are 256-byte aligned by the host layer). Each thread owns rows
  // base + 2*(u*256 + tid) + {0, 1}, u = 0, 1.
  const bool vec_ok = ((P.ldc & 1) == 0) && (((uintptr_t)p | (uintptr_t)Ap | (uintptr_t)x | (uintptr_t)r |
                                              (uintptr_t)z | (uintptr_t)dinv | (uintptr_t)cross) & 15) == 0;
  const int64_t nfull = vec_ok ? n / kUpdChunk : 0;
  for (int64_t chunk = blockIdx.x; chunk < nfull; chunk += gridDim.x) {
    const int64_t base = chunk * kUpdChunk;
    double2 rv[2], dv[2], xv[2], pv[2], av[2];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int64_t q = (base >> 1) + u * kUpdThreads + threadIdx.x;  // double2 index
      rv[u] = reinterpret_cast<const double2*>(r)[q];
      dv[u] = dinv ? __ldg(reinterpret_cast<const double2*>(dinv) + q) : make_double2(1.0, 1.0);
      if (!entry) {
        xv[u] = reinterpret_cast<const double2*>(x)[q];
        pv[u] = reinterpret_cast<const double2*>(p)[q];
        av[u] = reinterpret_cast<const double2*>(Ap)[q];
      }
    }
    double zr[4];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int64_t q = (base >> 1) + u * kUpdThreads + threadIdx.x;
      double r0 = rv[u].x, r1 = rv[u].y;
      if (!entry) {
        // krylov.py:306-307  x = x + alpha * p ; r = r - alpha * Ap
        reinterpret_cast<double2*>(x)[q] =
            make_double2(__dadd_rn(xv[u].x, __dmul_rn(alpha, pv[u].x)), __dadd_rn(xv[u].y, __dmul_rn(alpha, pv[u].y)));
        r0 = __dsub_rn(r0, __dmul_rn(alpha, av[u].x));
        r1 = __dsub_rn(r1, __dmul_rn(alpha, av[u].y));
        reinterpret_cast<double2*>(r)[q] = make_double2(r0, r1);
      }
      // preconditioners.py:61  r * inv_diag  (identity: r.copy())
      const double z0 = dinv ? __dmul_rn(r0, dv[u].x) : r0;
      const double z1 = dinv ? __dmul_rn(r1, dv[u].y) : r1;
      reinterpret_cast<double2*>(z)[q] = make_double2(z0, z1);
      zr[2 * u] = z0;
      zr[2 * u + 1] = z1;
      acc[0] = fma(r0, r0, acc[0]);
      acc[0] = fma(r1, r1, acc[0]);
      acc[1] = fma(r0, z0, acc[1]);
      acc[1] = fma(r1, z1, acc[1]);
    }
    // K4 on the chunk: 8 columns of cross at a time, 16 independent 16-byte
    // loads per thread in flight, then a fixed-order block reduction.
    for (int64_t j0 = 0; j0 < m; j0 += kColGroup) {
      double a[kColGroup];
      if (j0 + kColGroup <= m) {
        double2 cv[kColGroup][2];
#pragma unroll
        for (int c = 0; c < kColGroup; ++c)
#pragma unroll
          for (int u = 0; u < 2; ++u)
            cv[c][u] = __ldcs(reinterpret_cast<const double2*>(cross + (j0 + c) * P.ldc + base) + u * kUpdThreads +
                              threadIdx.x);
#pragma unroll
        for (int c = 0; c < kColGroup; ++c) {
          double t = 0.0;
#pragma unroll
          for (int u = 0; u < 2; ++u) {
            t = fma(cv[c][u].x, zr[2 * u], t);
            t = fma(cv[c][u].y, zr[2 * u + 1], t);
          }
          a[c] = t;
        }
      } else {
#pragma unroll
        for (int c = 0; c < kColGroup; ++c) {
          double t = 0.0;
          if (j0 + c < m) {
#pragma unroll
            for (int u = 0; u < 2; ++u) {
              const double2 v = __ldcs(reinterpret_cast<const double2*>(cross + (j0 + c) * P.ldc + base) +
                                       u * kUpdThreads + threadIdx.x);
              t = fma(v.x, zr[2 * u], t);
              t = fma(v.y, zr[2 * u + 1], t);
            }
          }
          a[c] = t;
        }
      }
#pragma unroll
      for (int c = 0; c < kColGroup; ++c) a[c] = warp_sum(a[c]);
      if (lane == 0) {
#pragma unroll
        for (int c = 0; c < kColGroup; ++c) wsum[warp * kColGroup + c] = a[c];
      }
      __syncthreads();
      if (threadIdx.x < kColGroup && j0 + threadIdx.x < m) {
        double t = 0.0;
#pragma unroll
        for (int w = 0; w < kUpdThreads / 32; ++w) t += wsum[w * kColGroup + threadIdx.x];
        red[2 + j0 + threadIdx.x] += t;
      }
      __syncthreads();
    }
  }
  // Generic path: the tail chunk (and unaligned operands), scalar and predicated.
  for (int64_t chunk = nfull + blockIdx.x; chunk < nchunks; chunk += gridDim.x) {
    const int64_t i0 = chunk * kUpdChunk + threadIdx.x;
    // K3: R rows per thread, all loads issued before use (stride = block size,
    // so each of the R passes is a fully coalesced warp access)
    double xv[kRows], pv[kRows], rv[kRows], av[kRows], dv[kRows], zr[kRows];
#pragma unroll
    for (int u = 0; u < kRows; ++u) {
      const int64_t i = i0 + (int64_t)u * kUpdThreads;
      const bool ok = i < n;
      rv[u] = ok ? r[i] : 0.0;
      dv[u] = (ok && dinv) ? __ldg(dinv + i) : 1.0;
      if (!entry) {
        xv[u] = ok ? x[i] : 0.0;
        pv[u] = ok ? p[i] : 0.0;
        av[u] = ok ? Ap[i] : 0.0;
      }
    }
#pragma unroll
    for (int u = 0; u < kRows; ++u) {
      const int64_t i = i0 + (int64_t)u * kUpdThreads;
      zr[u] = 0.0;
      if (i >= n) continue;
      double ri = rv[u];
      if (!entry) {
        // krylov.py:306-307  x = x + alpha * p ; r = r - alpha * Ap
        x[i] = __dadd_rn(xv[u], __dmul_rn(alpha, pv[u]));
        ri = __dsub_rn(ri, __dmul_rn(alpha, av[u]));
        r[i] = ri;
      }
      // preconditioners.py:61  r * inv_diag  (identity: r.copy())
      const double zi = dinv ? __dmul_rn(ri, dv[u]) : ri;
      z[i] = zi;
      zr[u] = zi;
      acc[0] = fma(ri, ri, acc[0]);
      acc[1] = fma(ri, zi, acc[1]);
    }
    // K4: this chunk's share of c = cross' z, kColGroup columns at a time; each
    // thread multiplies its own rows by its own z (no barrier needed), then the
    // group is reduced across the block in a fixed order.
    for (int64_t j0 = 0; j0 < m; j0 += kColGroup) {
      double a[kColGroup];
#pragma unroll
      for (int c = 0; c < kColGroup; ++c) a[c] = 0.0;
#pragma unroll
      for (int u = 0; u < kRows; ++u) {
        const int64_t i = i0 + (int64_t)u * kUpdThreads;
        if (i < n) {
#pragma unroll
          for (int c = 0; c < kColGroup; ++c)
            if (j0 + c < m) a[c] = fma(__ldcs(cross + (j0 + c) * P.ldc + i), zr[u], a[c]);
        }
      }
#pragma unroll
      for (int c = 0; c < kColGroup; ++c) a[c] = warp_sum(a[c]);
      if (lane == 0) {
#pragma unroll
        for (int c = 0; c < kColGroup; ++c) wsum[warp * kColGroup + c] = a[c];
      }
      __syncthreads();
      if (threadIdx.x < kColGroup && j0 + threadIdx.x < m) {
        double t = 0.0;
#pragma unroll
        for (int w = 0; w < kUpdThreads / 32; ++w) t += wsum[w * kColGroup + threadIdx.x];
        red[2 + j0 + threadIdx.x] += t;
      }
      __syncthreads();
    }
  }
  block_sum<2>(acc, scratch);
  if (threadIdx.x == 0) { red[0] = acc[0]; red[1] = acc[1]; }
  __syncthreads();
  const int nv = (int)(2 + m);
  if (!publish_and_check_last(red, nv, P.partials, P.tickets + 1)) return;

  // ---- last block: combine, record, decide, solve --------------------------
  combine_partials(P.partials, gridDim.x, nv, red);
  __shared__ int s_stop;
  if (threadIdx.x == 0) {
    const double rr = red[0], rz_next = red[1];
    const double rnorm = sqrt(rr);
    st->rr = rr;
    s_stop = 0;
    if (entry) {
      // krylov.py:268 history[0] = ||r0|| ; :292 rz = r @ z
      P.res_h[0] = rnorm;
      st->rz = rz_next;
    } else {
      P.res_h[k + 1] = rnorm;                  // krylov.py:314
      if (rnorm <= st->threshold) {            // krylov.py:317
        st->status = 1;
        st->done = 1;
        st->k = k + 1;
        s_stop = 1;
      } else {
        st->rz_next = rz_next;                 // krylov.py:321
        st->beta = rz_next / st->rz;           // krylov.py:324 (rz_next / rz)
        st->rz = rz_next;                      // krylov.py:340
      }
    }
  }
  __syncthreads();
  if (s_stop || m == 0) return;
  double* ysm = red + nv;  // 2*wchol scratch
  solve_factor(P, red + 2, ysm, ysm + 2 * P.wchol, P.mu);
}

// K5: new direction into V[:, k+1] (entry: V[:, 0]).
__global__ void __launch_bounds__(256) k_pcg_direction(const rk_pcg_plan P, int entry) {
  rk_pcg_state* st = P.st;
  if (st->done) return;
  extern __shared__ double sm[];
  const int64_t k = st->k;
  const int64_t m = P.m;
  double* mus = sm;              // m
  double* cps = sm + m;          // paper-beta coefficients, k+1
  const int paper = (P.mode == 2) && !entry;
  for (int64_t j = threadIdx.x; j < m; j += blockDim.x) mus[j] = P.mu[j];
  if (paper) {
    const double rzn = st->rz_next;
    for (int64_t i = threadIdx.x; i <= k; i += blockDim.x) cps[i] = rzn / P.rz_h[i];
  }
  __syncthreads();
  const int cg = (P.mode == 0) && !entry;
  const double beta = cg ? st->beta : 0.0;
  const double* __restrict__ pk = P.V + k * P.ldv;
  double* __restrict__ out = P.V + (entry ? k : k + 1) * P.ldv;
  const double* __restrict__ z = P.z;
  const double* __restrict__ B = P.B;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < P.n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double t = z[i];
    if (cg) t = __dadd_rn(t, __dmul_rn(beta, pk[i]));     // krylov.py:324
    if (m > 0) {                                          // krylov.py:326/328  - Y @ mu
      double s = 0.0;
      const double* row = B + i;
      int64_t j = 0;
      for (; j + 4 <= m; j += 4) {
        const double b0 = __ldcs(row + (j + 0) * P.ldb), b1 = __ldcs(row + (j + 1) * P.ldb);
        const double b2 = __ldcs(row + (j + 2) * P.ldb), b3 = __ldcs(row + (j + 3) * P.ldb);
        s = fma(b0, mus[j], s);
        s = fma(b1, mus[j + 1], s);
        s = fma(b2, mus[j + 2], s);
        s = fma(b3, mus[j + 3], s);
      }
      for (; j < m; ++j) s = fma(__ldcs(row + j * P.ldb), mus[j], s);
      t = __dsub_rn(t, s);
    }
    if (paper) {                                          // krylov.py:329-331, same order
      for (int64_t q = 0; q <= k; ++q) t = __dadd_rn(t, __dmul_rn(cps[q], P.V[i + q * P.ldv]));
    }
    out[i] = t;
  }
  if (!entry && ticket_last(P.tickets + 2)) {
    if (threadIdx.x == 0) st->k = k + 1;
  }
}

}  // namespace rk

namespace rkh {

void prof_mark(int slot, cudaStream_t s);

struct UpdGeom {
  int grid;
  size_t smem;
};

static UpdGeom update_geometry(int64_t n, int64_t m, int64_t wchol) {
  UpdGeom g;
  const int64_t nchunks = (n + rk::kUpdChunk - 1) / rk::kUpdChunk;
  g.smem = (size_t)(2 + m + 2 * wchol + (wchol <= rk::kMaxStagedChol ? wchol * wchol : 0)) * sizeof(double);
  // one resident wave; chunks are grid-strided so every block does equal work
  static int occ = [] {
    int o = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, rk::k_pcg_update, rk::kUpdThreads, 1024) != cudaSuccess ||
        o < 1)
      o = 1;
    return o;
  }();
  g.grid = (int)std::max<int64_t>(1, std::min<int64_t>(nchunks, (int64_t)occ * sm_count()));
  return g;
}

int64_t pcg_workspace_doubles(int64_t n, int64_t m, int64_t vcap) {
  int64_t need = 0;
  // spmv / curvature partials: grid x 2
  need = std::max<int64_t>(need, (int64_t)sm_count() * 8 * 2);
  // update partials: grid x (2 + m)
  need = std::max<int64_t>(need, (int64_t)update_geometry(n, m, 0).grid * (2 + m));
  // fom gemv-t partials: chunks x vcap
  need = std::max<int64_t>(need, gemv_nchunks(n) * std::max<int64_t>(vcap, 1));
  return need;
}

static int configure_once() {
  static int done = 0;
  if (!done) {
    cudaFuncSetAttribute(rk::k_pcg_update, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(rk::k_pcg_direction, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    done = 1;
  }
  return 0;
}

// need_proj: the kernels that reduce cross'z and solve with the factor (entry,
// update) need cross/L/sqd; the direction kernel only reads B and mu.
static int check_plan(const rk_pcg_plan& P, bool need_proj) {
  RK_REQUIRE(P.st && P.x && P.r && P.z && P.V && P.AV, RK_ERR_ARG, "pcg plan: null vector pointer");
  RK_REQUIRE(P.m >= 0 && P.m <= rk::kMaxProj, RK_ERR_DIMENSION, "pcg plan: projection width %lld unsupported",
             (long long)P.m);
  RK_REQUIRE(P.m == 0 || (P.B && P.mu), RK_ERR_ARG, "pcg plan: projection pointers missing");
  if (need_proj) {
    RK_REQUIRE(P.m == 0 || P.cross, RK_ERR_ARG, "pcg plan: cross pointer missing");
    RK_REQUIRE(P.wchol >= 0 && P.wchol <= P.m, RK_ERR_DIMENSION, "pcg plan: bad factor width");
    RK_REQUIRE(P.wchol == 0 || P.L, RK_ERR_ARG, "pcg plan: factor pointer missing");
    RK_REQUIRE(P.wchol == P.m || P.sqd, RK_ERR_ARG, "pcg plan: sqrt-diagonal pointer missing");
  }
  RK_REQUIRE(P.partials && P.tickets, RK_ERR_ARG, "pcg plan: workspace missing");
  const int64_t need = pcg_workspace_doubles(P.n, need_proj ? P.m : 0, P.vcap);
  RK_REQUIRE(P.partials_len >= need, RK_ERR_ARG, "pcg plan: workspace too small (%lld < %lld)",
             (long long)P.partials_len, (long long)need);
  return 0;
}

static void launch_update(const rk_pcg_plan& P, int entry, cudaStream_t s) {
  const UpdGeom g = update_geometry(P.n, P.m, P.wchol);
  rk::k_pcg_update<<<g.grid, rk::kUpdThreads, g.smem, s>>>(P, entry); rkh::note_launch();
}

static void launch_direction(const rk_pcg_plan& P, int entry, int64_t kmax, cudaStream_t s) {
  const size_t smem = (size_t)(P.m + (P.mode == 2 ? kmax + 1 : 0) + 1) * sizeof(double);
  rk::k_pcg_direction<<<elementwise_grid(P.n), 256, smem, s>>>(P, entry); rkh::note_launch();
  if (P.mode == 1 && !entry) {
    // two classical Gram-Schmidt sweeps against every previous direction
    // (krylov.py:333-337, block form): coef_i = (A p_i)'p / gamma_i ; p -= V coef
    const int64_t* kk = &P.st->k;
    const int64_t* done = &P.st->done;
    for (int sweep = 0; sweep < 2; ++sweep) {
      launch_gemv_t(P.n, kmax, kk, done, P.AV, P.ldav, P.V, 1, P.ldv, P.partials, P.gamma_h, P.coef, s);
      launch_gemv_n(P.n, kmax, kk, done, P.V, P.ldv, P.coef, P.V, P.V, 2, 1, P.ldv, s);
    }
  }
}

int pcg_entry(const rk_pcg_plan& P, cudaStream_t s) {
  configure_once();
  if (int e = check_plan(P, true)) return e;
  launch_update(P, 1, s);
  launch_direction(P, 1, 0, s);
  return cuda_check("rk_pcg_entry");
}

int pcg_steps(const rk_pcg_plan& P, int nsteps, int64_t kmax_hint, cudaStream_t s) {
  configure_once();
  if (int e = check_plan(P, true)) return e;
  RK_REQUIRE(P.A.rowptr && P.A.col && P.A.val, RK_ERR_ARG, "rk_pcg_steps: CSR operator required");
  RK_REQUIRE(P.mode != 1 || P.ldav > 0, RK_ERR_ARG, "rk_pcg_steps: fom mode keeps A p_k columns (ldav > 0)");
  RK_REQUIRE(kmax_hint + 2 <= P.vcap, RK_ERR_DIMENSION, "rk_pcg_steps: kmax_hint %lld beyond capacity %lld",
             (long long)kmax_hint, (long long)P.vcap);
  if (P.mode == 1) gemv_n_smem_ok(kmax_hint + 1);
  for (int i = 0; i < nsteps; ++i) {
    prof_mark(0, s);
    launch_spmv_pcg(P, s);
    prof_mark(1, s);
    launch_update(P, 0, s);
    prof_mark(2, s);
    launch_direction(P, 0, kmax_hint + 1, s);
    prof_mark(3, s);
  }
  return cuda_check("rk_pcg_steps");
}

int pcg_curvature(const rk_pcg_plan& P, cudaStream_t s) {
  configure_once();
  if (int e = check_plan(P, true)) return e;
  launch_curvature(P, s);
  return cuda_check("rk_pcg_curvature");
}

int pcg_update(const rk_pcg_plan& P, cudaStream_t s) {
  configure_once();
  if (int e = check_plan(P, true)) return e;
  launch_update(P, 0, s);
  return cuda_check("rk_pcg_update");
}

int pcg_direction(const rk_pcg_plan& P, int64_t kmax_hint, cudaStream_t s) {
  configure_once();
  if (int e = check_plan(P, false)) return e;
  if (P.mode == 1) gemv_n_smem_ok(kmax_hint + 1);
  launch_direction(P, 0, kmax_hint + 1, s);
  return cuda_check("rk_pcg_direction");
}

}  // namespace rkh
