// Persistent single-cluster augmented PCG for small systems (krylov.py:300-340).
//
// For the latency-bound configurations (C1: N = 4096, 20 k nonzeros; the
// reference's fixtures) the multi-kernel iteration of pcg.cu costs ~40 us per
// iteration in launch and grid-combine latency while moving a few hundred KB.
// Here ONE thread-block cluster (<= 16 CTAs, one per SM, 256 threads each)
// runs the whole loop on the device until convergence, breakdown or `kend`:
//
//   * rows are split into contiguous per-CTA ranges of 256 * RPT rows; every
//     thread owns RPT fixed rows and keeps x, r, p, 1/diag in registers;
//   * the live direction's rows sit in shared memory (p_s) and the SpMV reads
//     a neighbour CTA's entries through distributed shared memory;
//   * A, the augmenting basis B, cross = A B and the factor are read-only for
//     the run (ld.global.nc, L1-resident from the second iteration);
//   * each reduction (p'Ap and p'p; ||r||^2, r'z and cross'z) is pushed by
//     every CTA into a slot of every CTA's shared memory, one cluster barrier
//     (release/acquire), then summed in rank order: all CTAs hold bitwise the
//     same scalars and solve mu redundantly (no further exchange);
//   * three cluster barriers per cg iteration (p published, two reductions),
//     two more per block-CGS sweep in fom mode (the sweep coefficients go
//     through the plan's workspace, double-buffered by sweep).
//
// Arithmetic is that of the multi-kernel path statement by statement: the
// SpMV rows are scipy's csr_matvec (separately rounded multiply and add in CSR
// order), the vector updates are explicitly rounded; only the order of the
// dot-product partial sums differs (as it does there from numpy's).
#include <cooperative_groups.h>

#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "pcg_device.cuh"

namespace cgx = cooperative_groups;

namespace rk {

constexpr int kClThreads = 256;
constexpr int kClMaxCtas = 16;
constexpr int kClMaxRpt = 8;
constexpr int kClNv = 2 + kFuseMax;

struct ClShared {
  double red1[kClMaxCtas][2];      // p'Ap, p'p of every CTA
  double red2[kClMaxCtas][kClNv];  // ||r||^2, r'z, cross'z of every CTA
  double loc[kClNv];               // this CTA's partials before the push
  double tot[kClNv];               // combined sums (bitwise equal in every CTA)
  double mu[kFuseMax];
  double ysm[kFuseMax];
  double scratch[64];
  int64_t k0, done0;
  double rz0, thr;
};

template <int RPT>
__global__ void __launch_bounds__(kClThreads, 1) k_pcg_cluster(const rk_pcg_plan P, int64_t kend, int64_t hstride) {
  constexpr int64_t Rc = (int64_t)kClThreads * RPT;  // rows per CTA
  cgx::cluster_group cl = cgx::this_cluster();
  const int C = (int)cl.num_blocks();
  const int rank = (int)cl.block_rank();
  __shared__ ClShared S;
  extern __shared__ double dyn[];
  double* p_s = dyn;           // Rc: this CTA's rows of the live direction
  double* w_s = dyn + Rc;      // Rc: z (cross'z) / the direction being orthogonalised (fom)
  double* cf = dyn + 2 * Rc;   // kend + 1: sweep / paper-beta coefficients
  double* rzh = cf + hstride;  // kend + 1: rz history (paper beta)
  double* gah = rzh + hstride; // kend + 1: gamma history (fom)
  rk_pcg_state* st = P.st;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t n = P.n, m = P.m, base = (int64_t)rank * Rc;
  const int64_t rows = std::max<int64_t>(0, std::min<int64_t>(Rc, n - base));
  const int mode = P.mode;
  if (tid == 0) {
    S.k0 = st->k;
    S.done0 = st->done;
    S.rz0 = st->rz;
    S.thr = st->threshold;
  }
  __syncthreads();
  int64_t k = S.k0;
  double rz = S.rz0;
  const double thr = S.thr;
  const bool lead = rank == 0 && tid == 0;
  if (mode != 0)  // histories of earlier launches (this run resumes at k)
    for (int64_t q = tid; q < k; q += kClThreads) {
      rzh[q] = P.rz_h[q];
      gah[q] = P.gamma_h[q];
    }
  cl.sync();  // every CTA has read the state before rank 0 may write it
  if (S.done0 || k >= kend) return;

  const int32_t* __restrict__ rowptr = P.A.rowptr;
  const int32_t* __restrict__ colidx = P.A.col;
  const double* __restrict__ aval = P.A.val;
  double xv[RPT], rv[RPT], pv[RPT], dv[RPT];
  {
    const double* rin = (k & 1) ? P.r2 : P.r;
#pragma unroll
    for (int u = 0; u < RPT; ++u) {
      const int64_t i = (int64_t)u * kClThreads + tid, row = base + i;
      const bool ok = i < rows;
      xv[u] = ok ? P.x[row] : 0.0;
      rv[u] = ok ? rin[row] : 0.0;
      pv[u] = ok ? P.V[k * P.ldv + row] : 0.0;
      dv[u] = (ok && P.dinv) ? __ldg(P.dinv + row) : 1.0;
      p_s[i] = pv[u];
    }
  }
  int status = 0;
  double gamma = 0.0, pp = 0.0, rr = 0.0;
  cl.sync();  // p_k published
  for (;;) {
    // ---- K1: Ap = A p_k, gamma = p'Ap, p'p (krylov.py:301-305) ----
    double apv[RPT];
    double acc[2] = {0.0, 0.0};
#pragma unroll
    for (int u = 0; u < RPT; ++u) {
      const int64_t i = (int64_t)u * kClThreads + tid, row = base + i;
      apv[u] = 0.0;
      if (i < rows) {
        double s = 0.0;
        const int32_t e1 = __ldg(rowptr + row + 1);
        for (int32_t jj = __ldg(rowptr + row); jj < e1; ++jj) {
          const int32_t c = __ldg(colidx + jj);
          const int owner = (int)(c / Rc);
          const int64_t off = c - (int64_t)owner * Rc;
          const double pj = owner == rank ? p_s[off] : *cl.map_shared_rank(p_s + off, (unsigned)owner);
          s = row_madd(__ldg(aval + jj), pj, s);
        }
        apv[u] = s;
        acc[0] = fma(pv[u], s, acc[0]);
        acc[1] = fma(pv[u], pv[u], acc[1]);
        if (P.ldav) P.AV[k * P.ldav + row] = s;
      }
    }
    block_sum<2>(acc, S.scratch);
    if (tid < 2 * C) *cl.map_shared_rank(&S.red1[rank][tid & 1], (unsigned)(tid >> 1)) = acc[tid & 1];
    cl.sync();
    gamma = 0.0;
    pp = 0.0;
    for (int q = 0; q < C; ++q) {
      gamma += S.red1[q][0];
      pp += S.red1[q][1];
    }
    // krylov.py:303  `not isfinite(gamma) or gamma <= 1e-14 * (p @ p)`
    if (!isfinite(gamma) || gamma <= 1e-14 * pp) {
      status = 2;
      break;
    }
    const double alpha = rz / gamma;
    if (lead) {
      P.alpha_h[k] = alpha;
      P.gamma_h[k] = gamma;
      P.rz_h[k] = rz;
    }
    if (mode != 0 && tid == 0) {
      rzh[k] = rz;
      gah[k] = gamma;
    }

    // ---- K3/K4: x, r, z, ||r||^2, r'z, cross'z (krylov.py:306-322) ----
    double zv[RPT];
    double acc2[2] = {0.0, 0.0};
#pragma unroll
    for (int u = 0; u < RPT; ++u) {
      const int64_t i = (int64_t)u * kClThreads + tid;
      zv[u] = 0.0;
      if (i < rows) {
        xv[u] = __dadd_rn(xv[u], __dmul_rn(alpha, pv[u]));  // krylov.py:306
        rv[u] = __dsub_rn(rv[u], __dmul_rn(alpha, apv[u])); // krylov.py:307
        zv[u] = P.dinv ? __dmul_rn(rv[u], dv[u]) : rv[u];   // preconditioners.py:61
        acc2[0] = fma(rv[u], rv[u], acc2[0]);
        acc2[1] = fma(rv[u], zv[u], acc2[1]);
      }
      w_s[i] = zv[u];
    }
    block_sum<2>(acc2, S.scratch);  // its barriers also publish w_s
    if (tid == 0) {
      S.loc[0] = acc2[0];
      S.loc[1] = acc2[1];
    }
    for (int64_t j = warp; j < m; j += kClThreads / 32) {
      const double* __restrict__ col = P.cross + j * P.ldc + base;
      double a = 0.0;
      for (int64_t i = lane; i < rows; i += 32) a = fma(__ldg(col + i), w_s[i], a);
      a = warp_sum(a);
      if (lane == 0) S.loc[2 + j] = a;
    }
    __syncthreads();
    const int nv = 2 + (int)m;
    for (int t = tid; t < C * nv; t += kClThreads) {
      const int dst = t / nv, j = t - dst * nv;
      *cl.map_shared_rank(&S.red2[rank][j], (unsigned)dst) = S.loc[j];
    }
    cl.sync();
    for (int t = tid; t < nv; t += kClThreads) {
      double s = 0.0;
      for (int q = 0; q < C; ++q) s += S.red2[q][t];
      S.tot[t] = s;
    }
    __syncthreads();
    rr = S.tot[0];
    const double rzn = S.tot[1], rnorm = sqrt(rr);
    if (lead) P.res_h[k + 1] = rnorm;  // krylov.py:314
    if (rnorm <= thr) {                // krylov.py:317
      status = 1;
      ++k;
      break;
    }
    if (m > 0) {
      solve_factor_warps(P, S.tot + 2, S.ysm, S.mu);  // mu = F^{-1} cross'z (krylov.py:155-156)
      __syncthreads();
    }
    if (mode == 2)
      for (int64_t q = tid; q <= k; q += kClThreads) cf[q] = rzn / rzh[q];

    // ---- K5: the new direction (krylov.py:323-337) ----
    const double beta = rzn / rz;  // krylov.py:324
    double pn[RPT];
#pragma unroll
    for (int u = 0; u < RPT; ++u) {
      const int64_t i = (int64_t)u * kClThreads + tid, row = base + i;
      pn[u] = 0.0;
      if (i < rows) {
        double t = zv[u];
        if (mode == 0) t = __dadd_rn(t, __dmul_rn(beta, pv[u]));
        if (m > 0) {
          const double* __restrict__ brow = P.B + row;
          double s = 0.0;
          int64_t j = 0;
          for (; j + 4 <= m; j += 4) {
            const double b0 = __ldg(brow + (j + 0) * P.ldb), b1 = __ldg(brow + (j + 1) * P.ldb);
            const double b2 = __ldg(brow + (j + 2) * P.ldb), b3 = __ldg(brow + (j + 3) * P.ldb);
            s = fma(b0, S.mu[j + 0], s);
            s = fma(b1, S.mu[j + 1], s);
            s = fma(b2, S.mu[j + 2], s);
            s = fma(b3, S.mu[j + 3], s);
          }
          for (; j < m; ++j) s = fma(__ldg(brow + j * P.ldb), S.mu[j], s);
          t = __dsub_rn(t, s);
        }
        pn[u] = t;
      }
    }
    if (mode == 2) {  // krylov.py:329-331, same order
      __syncthreads();
#pragma unroll
      for (int u = 0; u < RPT; ++u) {
        const int64_t i = (int64_t)u * kClThreads + tid, row = base + i;
        if (i < rows)
          for (int64_t q = 0; q <= k; ++q) pn[u] = __dadd_rn(pn[u], __dmul_rn(cf[q], P.V[q * P.ldv + row]));
      }
    } else if (mode == 1) {
      // two classical Gram-Schmidt sweeps against every previous direction
      // (krylov.py:333-337, block form as in pcg.cu): coef_q = (A p_q)'p / gamma_q
      for (int sweep = 0; sweep < 2; ++sweep) {
        double* gws = P.partials + (int64_t)sweep * C * hstride;
#pragma unroll
        for (int u = 0; u < RPT; ++u) w_s[(int64_t)u * kClThreads + tid] = pn[u];
        __syncthreads();
        for (int64_t q = warp; q <= k; q += kClThreads / 32) {
          const double* col = P.AV + q * P.ldav + base;
          double a = 0.0;
          for (int64_t i = lane; i < rows; i += 32) a = fma(col[i], w_s[i], a);
          a = warp_sum(a);
          if (lane == 0) gws[rank * hstride + q] = a;
        }
        cl.sync();
        for (int64_t q = tid; q <= k; q += kClThreads) {
          double s = 0.0;
          for (int c = 0; c < C; ++c) s += __ldcg(gws + c * hstride + q);
          cf[q] = s / gah[q];
        }
        __syncthreads();
#pragma unroll
        for (int u = 0; u < RPT; ++u) {
          const int64_t i = (int64_t)u * kClThreads + tid, row = base + i;
          if (i < rows) {
            double s = 0.0;
            for (int64_t q = 0; q <= k; ++q) s = fma(P.V[q * P.ldv + row], cf[q], s);
            pn[u] = __dsub_rn(pn[u], s);
          }
        }
        __syncthreads();  // w_s and cf are rewritten by the next sweep
      }
    }
#pragma unroll
    for (int u = 0; u < RPT; ++u) {
      const int64_t i = (int64_t)u * kClThreads + tid, row = base + i;
      pv[u] = pn[u];
      p_s[i] = pn[u];  // every CTA finished reading p_k before the cross'z barrier
      if (i < rows) P.V[(k + 1) * P.ldv + row] = pn[u];
    }
    rz = rzn;  // krylov.py:340
    ++k;
    if (k >= kend) break;
    cl.sync();  // p_{k} published to the cluster
  }

  // ---- write back (x, the residual buffer iteration k reads) and the state ----
  double* rdst = (k & 1) ? P.r2 : P.r;
#pragma unroll
  for (int u = 0; u < RPT; ++u) {
    const int64_t i = (int64_t)u * kClThreads + tid, row = base + i;
    if (i < rows) {
      P.x[row] = xv[u];
      rdst[row] = rv[u];
    }
  }
  if (lead) {
    st->gamma = gamma;
    st->pp = pp;
    st->rr = rr;
    st->k = k;  // breakdown: the iteration whose direction failed (as curvature_epilogue)
    st->rz = rz;
    if (status == 2) {
      st->status = 2;
      st->bd_iter = k;
      st->done = 1;
    } else if (status == 1) {
      st->status = 1;
      st->done = 1;
    }
  }
  cl.sync();  // no CTA leaves while its shared memory may still be read
}

}  // namespace rk

namespace rkh {

void prof_mark(int slot, cudaStream_t s);

struct ClusterShape {
  int ctas = 0, rpt = 0;
};

// Largest cluster the device schedules for this kernel (16 needs the
// non-portable size; fall back to the portable 8 when it cannot be placed).
static int max_cluster_ctas() {
  static int cached = 0;
  if (cached) return cached;
  cudaFuncSetAttribute(rk::k_pcg_cluster<1>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(rk::kClMaxCtas);
  cfg.blockDim = dim3(rk::kClThreads);
  cfg.dynamicSmemBytes = 48 * 1024;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = rk::kClMaxCtas;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int nclusters = 0;
  if (cudaOccupancyMaxActiveClusters(&nclusters, rk::k_pcg_cluster<1>, &cfg) != cudaSuccess) {
    cudaGetLastError();
    nclusters = 0;
  }
  cached = nclusters > 0 ? rk::kClMaxCtas : 8;
  return cached;
}

static ClusterShape cluster_shape(int64_t n) {
  ClusterShape c;
  if (n <= 0) return c;
  int cmax = max_cluster_ctas();
  if (const char* e = std::getenv("RK_CLUSTER_CTAS")) cmax = std::max(1, std::min(rk::kClMaxCtas, atoi(e)));
  c.ctas = (int)std::min<int64_t>(cmax, (n + rk::kClThreads - 1) / rk::kClThreads);
  const int64_t per = (n + c.ctas - 1) / c.ctas;
  int rpt = 1;
  while ((int64_t)rpt * rk::kClThreads < per) rpt *= 2;
  c.rpt = rpt;
  if (rpt > rk::kClMaxRpt) c.ctas = 0;
  return c;
}

static size_t cluster_smem(const rk_pcg_plan& P, const ClusterShape& c, int64_t hstride) {
  return (size_t)(2 * (int64_t)rk::kClThreads * c.rpt + (P.mode != 0 ? 3 * hstride : 0)) * sizeof(double);
}

int64_t pcg_cluster_max_rows() { return (int64_t)rk::kClMaxCtas * rk::kClThreads * rk::kClMaxRpt; }

int pcg_cluster_eligible(const rk_pcg_plan& P) {
  if (const char* e = std::getenv("RK_CLUSTER")) if (e[0] == '0') return 0;
  if (!P.A.rowptr || !P.A.col || !P.A.val) return 0;
  if (P.n <= 0 || P.n > pcg_cluster_max_rows()) return 0;
  if (P.m < 0 || P.m > rk::kFuseMax) return 0;
  if (P.mode < 0 || P.mode > 2 || (P.mode == 1 && P.ldav <= 0)) return 0;
  return cluster_shape(P.n).ctas > 0 ? 1 : 0;
}

template <int RPT>
static int launch_cluster(const rk_pcg_plan& P, int ctas, int64_t kend, int64_t hstride, size_t smem,
                          cudaStream_t s) {
  auto kern = rk::k_pcg_cluster<RPT>;
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    configured = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)ctas);
  cfg.blockDim = dim3(rk::kClThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = (unsigned)ctas;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, P, kend, hstride);
  note_launch();
  if (e != cudaSuccess) {
    set_error("rk_pcg_cluster: launch of a %d-CTA cluster failed: %s", ctas, cudaGetErrorString(e));
    return RK_ERR_CUDA;
  }
  return 0;
}

int pcg_cluster_run(const rk_pcg_plan& P, int64_t kend, cudaStream_t s) {
  RK_REQUIRE(pcg_cluster_eligible(P), RK_ERR_DIMENSION,
             "rk_pcg_cluster: plan not eligible (CSR operator, n <= %lld, m <= %d, fom keeps A p_k)",
             (long long)pcg_cluster_max_rows(), rk::kFuseMax);
  RK_REQUIRE(P.st && P.x && P.r && P.r2 && P.V && P.alpha_h && P.gamma_h && P.rz_h && P.res_h, RK_ERR_ARG,
             "rk_pcg_cluster: null vector pointer");
  RK_REQUIRE(P.m == 0 || (P.B && P.cross && P.wchol >= 0 && P.wchol <= P.m && (P.wchol == 0 || P.L) &&
                          (P.wchol == P.m || P.sqd)),
             RK_ERR_ARG, "rk_pcg_cluster: projection pointers missing");
  RK_REQUIRE(kend >= 0 && kend + 1 <= P.vcap, RK_ERR_DIMENSION, "rk_pcg_cluster: kend %lld beyond capacity %lld",
             (long long)kend, (long long)P.vcap);
  const ClusterShape c = cluster_shape(P.n);
  const int64_t hstride = kend + 1;
  RK_REQUIRE(P.mode != 1 || (P.partials && P.partials_len >= 2 * (int64_t)c.ctas * hstride), RK_ERR_ARG,
             "rk_pcg_cluster: workspace too small for the fom sweeps");
  const size_t smem = cluster_smem(P, c, hstride);
  RK_REQUIRE(smem <= 200 * 1024, RK_ERR_DIMENSION, "rk_pcg_cluster: kend %lld needs %zu bytes of shared memory",
             (long long)kend, smem);
  prof_mark(8, s);
  int e;
  switch (c.rpt) {
    case 1: e = launch_cluster<1>(P, c.ctas, kend, hstride, smem, s); break;
    case 2: e = launch_cluster<2>(P, c.ctas, kend, hstride, smem, s); break;
    case 4: e = launch_cluster<4>(P, c.ctas, kend, hstride, smem, s); break;
    default: e = launch_cluster<8>(P, c.ctas, kend, hstride, smem, s); break;
  }
  prof_mark(9, s);
  return e;
}

}  // namespace rkh
