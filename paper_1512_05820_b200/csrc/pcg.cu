// Device-resident augmented PCG iteration (krylov.py:181-345).
//
// One iteration k is three kernels (plus four for the fom re-orthogonalisation):
//   k_spmv_pcg  (spmv.cu)  Ap_k = A p_k, gamma, p'p, breakdown test, alpha
//   k_pcg_update           x += alpha p_k, r -= alpha Ap_k, z = D^{-1} r, ||r||^2, r'z,
//                          c = cross' z as block partials; the last block of each
//                          group of chunks sums its group (fixed order)
//   k_pcg_direction        every block sums the group sums (fixed order, so all
//                          blocks agree bitwise), records ||r||, decides
//                          convergence and solves mu = F^{-1} c for itself (m <=
//                          64: a 60 x 60 factor is L2 resident), then
//                          p_{k+1} = z + beta p_k - B mu (cg) | z - B mu (fom),
//                          written straight into V[:, k+1]; last block advances k
//   (wider projections and the host-stepped path combine in k_pcg_finish instead)
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
#include "pcg_device.cuh"

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

// Debug-only timeline of the direction kernel's combine prologue (built with
// -DRK_TAIL_TRACE): row k % 64 holds block 0's globaltimer stamps of
// iteration k -- after the wait, after the group sums, after the mu solve,
// at the end of the row loop (see rk_debug_trace).
__device__ unsigned long long g_tail_trace[64 * 8];
#ifdef RK_TAIL_TRACE
#define RK_STAMP(slot)                                                                  \
  do {                                                                                  \
    if (blockIdx.x == 0 && threadIdx.x == 0) {                                          \
      unsigned long long t_;                                                            \
      asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t_));                            \
      g_tail_trace[(st->k % 64) * 8 + (slot)] = t_;                                     \
    }                                                                                   \
  } while (0)
#else
#define RK_STAMP(slot)
#endif

constexpr int kUpdThreads = 256;
constexpr int kProjChunk = 1024;                 // rows per update block
constexpr int kProjCols = 32;                    // cross columns per update block (4 per warp)
constexpr int64_t kMaxProj = 65535 * 32;          // projection width: the update grid's y extent (C4: ~3000)
constexpr int64_t kStageMu = 16384;              // mu / reduced sums staged in shared memory up to this width
constexpr int kStageFactor = 96;                 // Linv staged in shared memory up to this width
#ifndef RK_DIR_UNROLL
#define RK_DIR_UNROLL 12
#endif
#ifndef RK_DIR_MINB
#define RK_DIR_MINB 4
#endif
constexpr int kDirUnroll = RK_DIR_UNROLL;          // B loads in flight per row in the direction kernel
constexpr int kDirMinBlocks = RK_DIR_MINB;
constexpr int kWideSolve = 256;                  // dense factors wider than this: mu on the whole GPU
constexpr int kMaxGroups = 256;                  // chunk groups of the fused two-level combine

// mu = F^{-1} c with F = blockdiag(L L', diag(sqd)^2) (krylov.py:119-132
// BlockDiagFactor.solve_spd). P.L holds either Linv = L^{-1} (linv_full = 0;
// lower triangular, LAPACK dtrtri on the host: the two triangular solves become
// two triangular mat-vecs, y = Linv c and mu = Linv' y) or the dense block's
// F^{-1} = Linv' Linv (linv_full = 1, one symmetric mat-vec: half the
// dependent steps in the latency-bound tail); the diagonal block is a division.
__device__ void solve_factor(const rk_pcg_plan& P, const double* c, double* ysm, const double* Ls, double* mu) {
  const int64_t w = P.wchol, m = P.m;
  // Linv is either staged in shared memory (Ls, ld = w, zero above the
  // diagonal) or, for wide factors (<= 2048^2 doubles, L2 resident), read in
  // place: each thread's row loads are independent, so they are all in flight.
  const double* __restrict__ L = Ls ? Ls : P.L;
  const int64_t ldl = Ls ? w : P.ldl;
  if (P.linv_full) {  // L holds F^{-1}: one symmetric mat-vec (row i = column i)
    for (int64_t i = threadIdx.x; i < w; i += blockDim.x) {
      double s = 0.0;
      for (int64_t j = 0; j < w; ++j) s = fma(L[j + i * ldl], c[j], s);
      ysm[i + w] = s;
    }
    __syncthreads();
    for (int64_t i = threadIdx.x; i < m; i += blockDim.x) {
      if (i < w) mu[i] = ysm[i + w];
      else {
        const double d = P.sqd[i - w];
        mu[i] = c[i] / (d * d);
      }
    }
    return;
  }
  for (int64_t i = threadIdx.x; i < w; i += blockDim.x) {   // y = Linv c
    double s = 0.0;
    for (int64_t j = 0; j <= i; ++j) s = fma(L[i + j * ldl], c[j], s);
    ysm[i] = s;
  }
  __syncthreads();
  for (int64_t i = threadIdx.x; i < w; i += blockDim.x) {   // mu = Linv' y
    double s = 0.0;
    for (int64_t j = i; j < w; ++j) s = fma(L[j + i * ldl], ysm[j], s);
    ysm[i + w] = s;
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

// Fixed-order sums out[v] = sum_{c in [c0, c1)} src[v * ld + c] for v < nv
// (nv <= 2 + kFuseMax) by one 256-thread block: warp-owned values, lanes over
// c, every value's loads issued together (one L2 round trip per 32 columns).
__device__ __forceinline__ void block_row_sums(const double* src, int64_t ld, int64_t nv, int64_t c0, int64_t c1,
                                               double* out, int64_t out_stride) {
  constexpr int QV = (2 + kFuseMax + 7) / 8;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double a[QV];
#pragma unroll
  for (int q = 0; q < QV; ++q) a[q] = 0.0;
  for (int64_t c = c0 + lane; c < c1; c += 32) {
#pragma unroll
    for (int q = 0; q < QV; ++q) {
      const int64_t v = warp + 8 * q;
      if (v < nv) a[q] += __ldcg(src + v * ld + c);
    }
  }
  warp_sum_n(a);
#pragma unroll
  for (int q = 0; q < QV; ++q) {
    const int64_t v = warp + 8 * q;
    if (lane == 0 && v < nv) out[v * out_stride] = a[q];
  }
}

// Scalar bookkeeping of the combined update reductions red = [||r||^2, r'z, c]:
// history, convergence test, beta (krylov.py:268,292,314-324,340). Returns true
// when the run stopped (the caller then skips the mu solve). Block-uniform.
__device__ bool pcg_scalars(const rk_pcg_plan& P, int entry, const double* red) {
  rk_pcg_state* st = P.st;
  __shared__ int s_stop;
  if (threadIdx.x == 0) {
    const int64_t k = st->k;
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
  return s_stop != 0;
}

// Like ticket_last, for a counter that expects `expected` arrivals.
__device__ __forceinline__ bool ticket_last_of(uint32_t* ticket, uint32_t expected) {
  __shared__ bool s_last;
  __syncthreads();
  if (threadIdx.x == 0) {
    fence_acq_rel_gpu();  // release the block's writes (ordered by the barrier)
    const uint32_t t = atomicAdd(ticket, 1u);
    s_last = (t == expected - 1);
    if (s_last) {
      *ticket = 0u;
      fence_acq_rel_gpu();  // acquire: every other block's writes are visible
    }
  }
  __syncthreads();
  return s_last;
}

// Residual ping-pong: iteration k reads r_k from buffer k&1 and writes r_{k+1}
// to the other one, so every block of the 2-D update grid can recompute z for
// its rows from unmodified inputs (entry reads buffer 0 and writes nothing).
__device__ __forceinline__ const double* r_in(const rk_pcg_plan& P, int64_t k, int entry) {
  return (entry || !(k & 1)) ? P.r : P.r2;
}
__device__ __forceinline__ double* r_out(const rk_pcg_plan& P, int64_t k) { return (k & 1) ? P.r : P.r2; }

// K3 + K4 partials. Grid (row chunks, column groups of 32). Every block forms
// z = D^{-1}(r - alpha Ap) for its 1024 rows in shared memory; column group 0
// also writes x, r_{k+1}, z and the ||r||^2, r'z partials. Then each warp
// reduces 4 columns of cross' z over the chunk (lanes over rows, 16-byte
// loads, 16 in flight per lane). Partials: part[v * nchunks + chunk].
//
// ext (a preconditioner applied by its own kernels between two launches,
// SSOR): 1 = first half, column group 0 only: x, r_{k+1} and the ||r||^2
// partials, z untouched; 2 = second half: z = M^{-1} r_{k+1} is read from P.z,
// r'z and the cross'z partials follow. 0 = the fused Jacobi / identity form.
__global__ void __launch_bounds__(kUpdThreads, 4) k_pcg_update(const rk_pcg_plan P, int entry, int fused, int64_t group,
                                                               int ext) {
  rk_pcg_state* st = P.st;
  pdl_wait();
  pdl_trigger();
  if (st->done) return;
  __shared__ __align__(16) double zs[kProjChunk];
  __shared__ double scratch[64];
  const int64_t k = st->k;
  const double alpha = entry ? 0.0 : st->alpha;
  const int64_t n = P.n, m = P.m;
  const int64_t nchunks = gridDim.x;
  const int64_t chunk = blockIdx.x;
  const int64_t beg = chunk * kProjChunk;
  const int rows = (int)min((int64_t)kProjChunk, n - beg);
  const bool lead = blockIdx.y == 0;
  const double* __restrict__ p = P.V + k * P.ldv + beg;
  const double* __restrict__ Ap = P.AV + (P.ldav ? k * P.ldav : 0) + beg;
  const bool second = ext == 2;   // r_{k+1} and x are already updated; z comes from P.z
  const bool step = !entry && !second;
  // the residual this launch starts from: r_k, or (second half) the updated r_{k+1}
  const double* __restrict__ rin = ((second && !entry) ? r_out(P, k) : r_in(P, k, entry)) + beg;
  double* __restrict__ rout = r_out(P, k) + beg;
  double* __restrict__ x = P.x + beg;
  double* __restrict__ z = P.z + beg;
  const double* __restrict__ dinv = (P.dinv && ext == 0) ? P.dinv + beg : nullptr;
  double acc[2] = {0.0, 0.0};
  constexpr int R = kProjChunk / kUpdThreads;
  double rv[R], av[R], dv[R], xv[R], pv[R];
#pragma unroll
  for (int u = 0; u < R; ++u) {
    const int i = u * kUpdThreads + threadIdx.x;
    const bool ok = i < rows;
    rv[u] = ok ? rin[i] : 0.0;
    dv[u] = (ok && dinv) ? __ldg(dinv + i) : (ok && second) ? z[i] : 1.0;  // second half: dv carries z
    av[u] = (ok && step) ? Ap[i] : 0.0;
    xv[u] = (ok && step && lead) ? x[i] : 0.0;
    pv[u] = (ok && step && lead) ? p[i] : 0.0;
  }
#pragma unroll
  for (int u = 0; u < R; ++u) {
    const int i = u * kUpdThreads + threadIdx.x;
    if (i >= rows) {
      zs[i] = 0.0;
      continue;
    }
    double ri = rv[u];
    if (step) ri = __dsub_rn(ri, __dmul_rn(alpha, av[u]));       // krylov.py:307
    const double zi = second ? dv[u] : dinv ? __dmul_rn(ri, dv[u]) : ri;  // preconditioners.py:61
    zs[i] = zi;
    if (lead) {
      if (step) {
        x[i] = __dadd_rn(xv[u], __dmul_rn(alpha, pv[u]));          // krylov.py:306
        rout[i] = ri;
      }
      if (ext == 0) z[i] = zi;
      acc[0] = fma(ri, ri, acc[0]);
      acc[1] = fma(ri, zi, acc[1]);
    }
  }
  double* part = P.partials;
  if (lead) {
    block_sum<2>(acc, scratch);  // includes the barrier that publishes zs
    if (threadIdx.x == 0) {
      if (ext != 2) part[0 * nchunks + chunk] = acc[0];
      if (ext != 1) part[1 * nchunks + chunk] = acc[1];
    }
  } else {
    __syncthreads();
  }
  if (ext == 1) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const bool vec = ((P.ldc & 1) == 0) && ((((uintptr_t)P.cross) | (beg * 8)) & 15) == 0;
#pragma unroll 1
  for (int c = 0; c < kProjCols / 8; ++c) {
    const int64_t j = (int64_t)blockIdx.y * kProjCols + c * 8 + warp;
    if (j >= m) break;
    const double* __restrict__ col = P.cross + j * P.ldc + beg;
    double a = 0.0;
    if (vec && rows == kProjChunk) {
      double2 cv[kProjChunk / 64];
#pragma unroll
      for (int t = 0; t < kProjChunk / 64; ++t) cv[t] = __ldcs(reinterpret_cast<const double2*>(col) + t * 32 + lane);
#pragma unroll
      for (int t = 0; t < kProjChunk / 64; ++t) {
        const double2 zz = reinterpret_cast<const double2*>(zs)[t * 32 + lane];
        a = fma(cv[t].x, zz.x, a);
        a = fma(cv[t].y, zz.y, a);
      }
    } else {
      for (int i = lane; i < rows; i += 32) a = fma(__ldcs(col + i), zs[i], a);
    }
    a = warp_sum(a);
    if (lane == 0) part[(2 + j) * nchunks + chunk] = a;
  }
  if (!fused) return;
  // Deferred combine (m <= kFuseMax): the last block of each group of `group`
  // chunks (over all column groups) sums the group's partials into
  // gsum[v][g]; the direction kernel combines the groups. No block waits on
  // a grid-wide chain here, so the kernel ends when its slowest group does.
  const int64_t nv = 2 + m;
  const int64_t ngroups = (nchunks + group - 1) / group;
  const int64_t g = chunk / group;
  const int64_t c0 = g * group, c1 = min(nchunks, c0 + group);
  if (!ticket_last_of(P.tickets + 8 + g, (uint32_t)((c1 - c0) * gridDim.y))) return;
  block_row_sums(part, nchunks, nv, c0, c1, part + nv * nchunks + g, ngroups);
}

// Combine the update partials and, in the last block to finish, record ||r||,
// test convergence, form beta and solve mu. One block per reduced value: every
// thread sums a fixed strided subset of the chunk partials, then a fixed-order
// block reduction (deterministic, one L2 round trip instead of a serial walk).
// Linv does not change during a run, so narrow factors are staged in shared
// memory before waiting on the update kernel (overlapping its tail). P.L is
// written by the host before the run and by no kernel of the chain, so this
// read is independent of where the predecessors wait and trigger.
__global__ void __launch_bounds__(256) k_pcg_finish(const rk_pcg_plan P, int entry, int64_t nchunks, int wide) {
  rk_pcg_state* st = P.st;
  extern __shared__ double dyn[];      // Ls[w*w] (staged) | red[2 + m] (or [2]) | ysm[2 w]
  __shared__ double scratch[32];
  const int64_t m = P.m, w = P.wchol;
  const int64_t nv = 2 + m;
  const bool staged = w > 0 && w <= kStageFactor;
  // the reduced sums the last block needs in shared memory: all of them for
  // its own mu solve, only ||r||^2 and r'z when k_pcg_musolve solves (wide)
  // or when they would not fit (the solve then reads c from the global sums)
  const bool stage_red = !wide && nv <= kStageMu;
  double* Ls = dyn;
  double* red = dyn + (staged ? w * w : 0);
  if (staged) {
    for (int64_t e = threadIdx.x; e < w * w; e += blockDim.x) {
      const int64_t col = e / w, row = e - col * w;
      Ls[e] = (P.linv_full || row >= col) ? P.L[row + col * P.ldl] : 0.0;
    }
  }
  pdl_wait();
  pdl_trigger();
  if (st->done) return;
  const double* part = P.partials;
  double* sums = P.partials + nv * nchunks;
  for (int64_t v = blockIdx.x; v < nv; v += gridDim.x) {
    const double* pv = part + v * nchunks;
    double a[1] = {0.0};
#pragma unroll 4
    for (int64_t b = threadIdx.x; b < nchunks; b += blockDim.x) a[0] += __ldcg(pv + b);
    block_sum<1>(a, scratch);
    if (threadIdx.x == 0) sums[v] = a[0];
  }
  if (!ticket_last(P.tickets + 1)) return;  // fences thread 0's sums before the ticket
  __threadfence();
  const int64_t nred = stage_red ? nv : 2;
  for (int64_t j = threadIdx.x; j < nred; j += blockDim.x) red[j] = __ldcg(sums + j);
  __syncthreads();
  if (pcg_scalars(P, entry, red) || m == 0 || wide) return;  // wide: k_pcg_musolve follows
  solve_factor(P, stage_red ? red + 2 : sums + 2, red + nred, staged ? Ls : nullptr, P.mu);
}

// mu = F^{-1} c for wide dense factors (w > kWideSolve, F^{-1} held full and
// symmetric): a warp per row, lanes over the row's entries (coalesced, since
// row i of the symmetric F^{-1} is its column i), butterfly sum; trailing
// sqrt-diagonal entries are a division. Spread over the whole GPU instead of
// the finish kernel's last block (C4, w ~ 3000: 72 MB of F^{-1} per iteration
// read by one SM took 1.3 ms). c = the combined cross' z sums of k_pcg_finish.
__global__ void __launch_bounds__(256) k_pcg_musolve(const rk_pcg_plan P, int64_t nchunks) {
  rk_pcg_state* st = P.st;
  pdl_wait();
  pdl_trigger();
  if (st->done) return;
  const int64_t m = P.m, w = P.wchol;
  const double* __restrict__ c = P.partials + (2 + m) * nchunks + 2;
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t i = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); i < m; i += warps) {
    if (i < w) {
      const double* __restrict__ row = P.L + i * P.ldl;
      double s = 0.0;
      int64_t j = lane;
      for (; j + 96 < w; j += 128) {  // 4 loads in flight per lane
        const double a0 = __ldg(row + j), a1 = __ldg(row + j + 32), a2 = __ldg(row + j + 64), a3 = __ldg(row + j + 96);
        const double c0 = __ldcg(c + j), c1 = __ldcg(c + j + 32), c2 = __ldcg(c + j + 64), c3 = __ldcg(c + j + 96);
        s = fma(a0, c0, s);
        s = fma(a1, c1, s);
        s = fma(a2, c2, s);
        s = fma(a3, c3, s);
      }
      for (; j < w; j += 32) s = fma(__ldg(row + j), __ldcg(c + j), s);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      if (lane == 0) P.mu[i] = s;
    } else if (lane == 0) {
      const double d = P.sqd[i - w];
      P.mu[i] = __ldcg(c + i) / (d * d);
    }
  }
}

// K5: new direction into V[:, k+1] (entry: V[:, 0]).
//
// combine = 1 (m <= kFuseMax, after a deferred update): every block first sums
// the update's group sums, runs the scalar bookkeeping and solves mu itself.
// The sums are in a fixed order, so every block computes bitwise the same
// ||r||, r'z and mu; block 0 alone writes them to the state and histories.
// beta = r'z_{k+1} / r'z_k uses rz_h[k] (written by the SpMV kernel), never
// st->rz, which block 0 overwrites while other blocks may still start. When
// the run has converged every block returns before the k ticket (a late block
// that already sees st->done set by block 0 returns as well), so the ticket
// only ever counts complete grids.
__global__ void __launch_bounds__(256, kDirMinBlocks)
    k_pcg_direction(const rk_pcg_plan P, int entry, int combine, int64_t nchunks, int64_t group) {
  rk_pcg_state* st = P.st;
  extern __shared__ double sm[];
  const int64_t m = P.m;
  const int64_t mstage = m <= kStageMu ? m : 0;
  double* mus = sm;              // m (staged widths)
  double* cps = sm + mstage;     // paper-beta coefficients, k+1
  // (An L2 prefetch of each thread's first basis row before the wait changed
  // nothing -- 269.1 vs 271.6 us per C3 iteration: the blocks of this one-wave
  // kernel only become resident as the update kernel's blocks retire.)
  pdl_wait();
  pdl_trigger();
  if (st->done) return;
  RK_STAMP(0);
  const int64_t k = st->k;
  const int paper = (P.mode == 2) && !entry;
  const int cg = (P.mode == 0) && !entry;
  double beta = cg ? st->beta : 0.0, rz_next = st->rz_next;
  if (combine) {
    __shared__ double red[2 + kFuseMax];
    __shared__ double ysm[kFuseMax];
    const int64_t nv = 2 + m;
    const int64_t ngroups = (nchunks + group - 1) / group;
    block_row_sums(P.partials + nv * nchunks, ngroups, nv, 0, ngroups, red, 1);
    __syncthreads();
    RK_STAMP(1);
    const double rr = red[0], rnorm = sqrt(rr);
    rz_next = red[1];
    const bool lead = blockIdx.x == 0 && threadIdx.x == 0;
    if (entry) {
      if (lead) {  // krylov.py:268 history[0] = ||r0|| ; :292 rz = r @ z
        st->rr = rr;
        P.res_h[0] = rnorm;
        st->rz = rz_next;
      }
    } else {
      const bool stop = rnorm <= st->threshold;  // krylov.py:317
      if (lead) {
        st->rr = rr;
        P.res_h[k + 1] = rnorm;                  // krylov.py:314
        if (stop) {
          st->status = 1;
          st->k = k + 1;
          st->done = 1;
        } else {
          st->rz_next = rz_next;                 // krylov.py:321
          st->beta = rz_next / P.rz_h[k];        // krylov.py:324 (rz_next / rz)
          st->rz = rz_next;                      // krylov.py:340
        }
      }
      if (stop) return;  // block-uniform
      beta = cg ? rz_next / P.rz_h[k] : 0.0;
    }
    if (m > 0) {
      solve_factor_warps(P, red + 2, ysm, mus);
      __syncthreads();
      RK_STAMP(2);
      if (blockIdx.x == 0)
        for (int64_t j = threadIdx.x; j < m; j += blockDim.x) P.mu[j] = mus[j];
    }
  } else if (m <= kStageMu) {
    for (int64_t j = threadIdx.x; j < m; j += blockDim.x) mus[j] = P.mu[j];
  }
  const double* __restrict__ muv = (combine || m <= kStageMu) ? mus : P.mu;  // wider: read in place (L2)
  if (paper) {
    for (int64_t i = threadIdx.x; i <= k; i += blockDim.x) cps[i] = rz_next / P.rz_h[i];
  }
  __syncthreads();
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
      // kDirUnroll loads of B issued before their fmas (same j order)
      for (; j + kDirUnroll <= m; j += kDirUnroll) {
        double b[kDirUnroll];
#pragma unroll
        for (int u = 0; u < kDirUnroll; ++u) b[u] = __ldcs(row + (j + u) * P.ldb);
#pragma unroll
        for (int u = 0; u < kDirUnroll; ++u) s = fma(b[u], muv[j + u], s);
      }
      for (; j < m; ++j) s = fma(__ldcs(row + j * P.ldb), muv[j], s);
      t = __dsub_rn(t, s);
    }
    if (paper) {                                          // krylov.py:329-331, same order
      for (int64_t q = 0; q <= k; ++q) t = __dadd_rn(t, __dmul_rn(cps[q], P.V[i + q * P.ldv]));
    }
    out[i] = t;
  }
  RK_STAMP(3);
  if (!entry && ticket_last(P.tickets + 2)) {
    if (threadIdx.x == 0) st->k = k + 1;
  }
}

}  // namespace rk

namespace rkh {

void prof_mark(int slot, cudaStream_t s);
bool prof_sample();

static int64_t update_chunks(int64_t n) { return std::max<int64_t>(1, (n + rk::kProjChunk - 1) / rk::kProjChunk); }

static size_t finish_smem(int64_t m, int64_t wchol, bool wide) {
  const int64_t staged = (wchol > 0 && wchol <= rk::kStageFactor) ? wchol * wchol : 0;
  const int64_t red = (!wide && 2 + m <= rk::kStageMu) ? 2 + m : 2;
  return (size_t)(staged + red + (wide ? 0 : 2 * wchol)) * sizeof(double);
}

int64_t pcg_workspace_doubles(int64_t n, int64_t m, int64_t vcap) {
  int64_t need = 0;
  // spmv / curvature partials: grid x 2
  need = std::max<int64_t>(need, (int64_t)sm_count() * 8 * 2);
  // update partials (2 + m) x chunks, plus the (2 + m) sums or the
  // (2 + m) x groups group sums of the fused finish
  const int64_t nch = update_chunks(n);
  need = std::max<int64_t>(need, (2 + m) * (nch + std::max<int64_t>(1, (nch + 31) / 32)));
  // fom gemv-t partials: chunks x vcap
  need = std::max<int64_t>(need, gemv_nchunks(n) * std::max<int64_t>(vcap, 1));
  // cluster solver (pcg_cluster.cu), fom: two sweeps x 16 CTAs x (vcap + 1) partials
  need = std::max<int64_t>(need, 2 * 16 * (vcap + 1));
  return need;
}

static int configure_once() {
  static int done = 0;
  if (!done) {
    cudaFuncSetAttribute(rk::k_pcg_finish, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(rk::k_pcg_direction, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    done = 1;
  }
  return 0;
}

// need_proj: the kernels that reduce cross'z and solve with the factor (entry,
// update) need cross/L/sqd; the direction kernel only reads B and mu.
static int check_plan(const rk_pcg_plan& P, bool need_proj) {
  RK_REQUIRE(P.st && P.x && P.r && P.r2 && P.z && P.V && P.AV, RK_ERR_ARG, "pcg plan: null vector pointer");
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

static int64_t fuse_group(int64_t nch) { return std::max<int64_t>(32, (nch + rk::kMaxGroups - 1) / rk::kMaxGroups); }

// deferred: the fused path of rk_pcg_entry / rk_pcg_steps (m <= kFuseMax),
// whose direction kernel combines the update's group sums; the host-stepped
// rk_pcg_update resolves the scalars itself (k_pcg_finish), since the host
// reads the convergence state right after it.
static bool deferred_combine(const rk_pcg_plan& P) { return P.m <= rk::kFuseMax; }

static void launch_update(const rk_pcg_plan& P, int entry, bool defer, cudaStream_t s, bool mark = false,
                          int ext = 0) {
  const int64_t nch = update_chunks(P.n);
  const int64_t groups = std::max<int64_t>(1, (P.m + rk::kProjCols - 1) / rk::kProjCols);
  dim3 grid((unsigned)nch, (unsigned)(ext == 1 ? 1 : groups));
  launch_pdl(rk::k_pcg_update, grid, dim3(rk::kUpdThreads), 0, s, P, entry, defer ? 1 : 0, fuse_group(nch), ext);
  if (mark) prof_mark(2, s);
  if (defer || ext == 1) return;
  const unsigned fgrid = (unsigned)std::min<int64_t>(2 + P.m, 4096);
  const int wide = (P.linv_full && P.wchol > rk::kWideSolve) ? 1 : 0;
  launch_pdl(rk::k_pcg_finish, dim3(fgrid), dim3(256), finish_smem(P.m, wide ? 0 : P.wchol, wide), s, P, entry, nch,
             wide);
  if (wide) {
    const unsigned mgrid = (unsigned)std::min<int64_t>((P.m + 7) / 8, (int64_t)sm_count() * 8);
    launch_pdl(rk::k_pcg_musolve, dim3(mgrid), dim3(256), 0, s, P, nch);
  }
}

static void launch_direction(const rk_pcg_plan& P, int entry, bool combine, int64_t kmax, cudaStream_t s) {
  const size_t smem =
      (size_t)((P.m <= rk::kStageMu ? P.m : 0) + (P.mode == 2 ? kmax + 1 : 0) + 1) * sizeof(double);
  const int64_t nch = update_chunks(P.n);
  // With the combine prologue every block pays a few microseconds of
  // dependent L2 round trips before its rows: one resident wave of blocks
  // (kDirMinBlocks per SM) pays them once, overlapped, instead of per wave.
  const int grid = combine ? (int)std::min<int64_t>((P.n + 255) / 256, (int64_t)sm_count() * rk::kDirMinBlocks)
                           : elementwise_grid(P.n);
  launch_pdl(rk::k_pcg_direction, dim3(std::max(grid, 1)), dim3(256), smem, s, P, entry, combine ? 1 : 0, nch,
             fuse_group(nch));
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

int debug_trace(unsigned long long* out, int64_t n) {
  const int64_t cnt = std::min<int64_t>(n, 64 * 8);
  if (cnt <= 0) return 0;
  if (cudaMemcpyFromSymbol(out, rk::g_tail_trace, cnt * sizeof(unsigned long long)) != cudaSuccess)
    return cuda_check("rk_debug_trace");
  return 0;
}

int pcg_entry(const rk_pcg_plan& P, cudaStream_t s) {
  configure_once();
  if (int e = check_plan(P, true)) return e;
  const bool defer = deferred_combine(P);
  launch_update(P, 1, defer, s);
  launch_direction(P, 1, defer, 0, s);
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
  const bool defer = deferred_combine(P);
  for (int i = 0; i < nsteps; ++i) {
    const bool mark = prof_sample();  // 1 iteration in 8 is bracketed by events (bench only)
    if (mark) prof_mark(0, s);
    launch_spmv_pcg(P, s);
    if (mark) prof_mark(1, s);
    launch_update(P, 0, defer, s, mark);
    if (mark) prof_mark(3, s);
    launch_direction(P, 0, defer, kmax_hint + 1, s);
    if (mark) prof_mark(4, s);
  }
  return cuda_check("rk_pcg_steps");
}

// Device-stepped PCG with the SSOR sweeps between the two halves of the update
// (rk_pcg_entry_ssor / rk_pcg_steps_ssor). The sweeps are ordinary launches:
// they start when the first half has completed and the second half (launched
// with programmatic serialisation) starts when they have.
int launch_ssor_apply(const rk_csr& A, const double* dw, const double* d, const double* r, double* z, double* u,
                      int* flags, unsigned int* counters, int epoch, cudaStream_t s, const rk_pcg_state* st,
                      const double* r_even, const int32_t* order_fwd, const int32_t* order_bwd);

int pcg_entry_ssor(const rk_pcg_plan& P, const rk_ssor_plan& S, cudaStream_t s) {
  configure_once();
  if (int e = check_plan(P, true)) return e;
  const bool defer = deferred_combine(P);
  launch_update(P, 1, defer, s, false, 1);
  if (int e = launch_ssor_apply(P.A, S.dw, S.d, P.r, P.z, S.work, reinterpret_cast<int*>(S.flags), S.counters,
                                S.epoch + 1, s, nullptr, nullptr, S.order_fwd, S.order_bwd))
    return e;
  launch_update(P, 1, defer, s, false, 2);
  launch_direction(P, 1, defer, 0, s);
  return cuda_check("rk_pcg_entry_ssor");
}

int pcg_steps_ssor(const rk_pcg_plan& P, const rk_ssor_plan& S, int nsteps, int64_t kmax_hint, cudaStream_t s) {
  configure_once();
  if (int e = check_plan(P, true)) return e;
  RK_REQUIRE(P.mode != 1 || P.ldav > 0, RK_ERR_ARG, "rk_pcg_steps_ssor: fom mode keeps A p_k columns (ldav > 0)");
  RK_REQUIRE(kmax_hint + 2 <= P.vcap, RK_ERR_DIMENSION, "rk_pcg_steps_ssor: kmax_hint %lld beyond capacity %lld",
             (long long)kmax_hint, (long long)P.vcap);
  if (P.mode == 1) gemv_n_smem_ok(kmax_hint + 1);
  const bool defer = deferred_combine(P);
  for (int i = 0; i < nsteps; ++i) {
    launch_spmv_pcg(P, s);
    launch_update(P, 0, defer, s, false, 1);
    // r_{k+1} is in P.r for odd k, in P.r2 for even k (the kernel reads st->k)
    if (int e = launch_ssor_apply(P.A, S.dw, S.d, P.r, P.z, S.work, reinterpret_cast<int*>(S.flags), S.counters,
                                  S.epoch + 1 + i, s, P.st, P.r2, S.order_fwd, S.order_bwd))
      return e;
    launch_update(P, 0, defer, s, false, 2);
    launch_direction(P, 0, defer, kmax_hint + 1, s);
  }
  return cuda_check("rk_pcg_steps_ssor");
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
  launch_update(P, 0, false, s);
  return cuda_check("rk_pcg_update");
}

int pcg_direction(const rk_pcg_plan& P, int64_t kmax_hint, cudaStream_t s) {
  configure_once();
  if (int e = check_plan(P, false)) return e;
  if (P.mode == 1) gemv_n_smem_ok(kmax_hint + 1);
  launch_direction(P, 0, false, kmax_hint + 1, s);
  return cuda_check("rk_pcg_direction");
}

}  // namespace rkh
