// K1 CSR SpMV (plain and fused into the PCG iteration), K2 SpMM, CSR diagonal and
// symmetry validation.
//
// Replaces scipy csr_matvec / csr_matvecs behind linalg.spmv (linalg.py:138-148),
// assemble_gram's A @ B (linalg.py:173), MatrixOperator.apply (krylov.py:56-57),
// SparseSpdMatrix._validate (linalg.py:105-119) and JacobiPreconditioner's
// diagonal (preconditioners.py:54-58).
//
// Layout: CSR with int32 indices, both triangles stored (as the reference).
// A group of LANES consecutive lanes owns one row; each lane walks the row's
// entries with stride LANES (coalesced within the group) and the group sums
// with an xor butterfly. The matrix stream is loaded with ld.global.cs
// (evict-first) so the gathered vector stays resident in L2.
#include <algorithm>

#include <cstdlib>

#include "common.cuh"

namespace rk {

constexpr int kSpmvThreads = 256;


// Entries per lane per pass for each group width: LANES * U covers the
// typical row in one pass (2 x 4 = 8 for 7-point rows, 16 x 6 = 96 for the
// 81-entry Q1 elasticity rows).
template <int LANES>
struct RowUnroll {
  static constexpr int U = (LANES == 8 || LANES == 16) ? 6 : 4;
};

template <int LANES>
__device__ __forceinline__ double csr_row_dot(const int32_t* __restrict__ rp,
                                              const int32_t* __restrict__ ci,
                                              const double* __restrict__ val,
                                              const double* __restrict__ x, int64_t row,
                                              bool valid, int sub) {
  // Each pass issues U independent (value, index) loads per lane before the
  // dependent gathers, so a short row (81 entries at 32 lanes, 7 at 4 lanes)
  // is a single pass with all its loads in flight at once.
  constexpr int U = RowUnroll<LANES>::U;
  double s = 0.0;
  if (valid) {
    const int32_t beg = __ldg(rp + row), end = __ldg(rp + row + 1);
    for (int32_t j0 = beg + sub; j0 < end; j0 += LANES * U) {
      double v[U];
      int32_t c[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int32_t j = j0 + u * LANES;
        const bool ok = j < end;
        v[u] = ok ? __ldcs(val + j) : 0.0;
        c[u] = ok ? __ldcs(ci + j) : 0;
      }
      double xv[U];
#pragma unroll
      for (int u = 0; u < U; ++u) xv[u] = __ldg(x + c[u]);
#pragma unroll
      for (int u = 0; u < U; ++u) s = row_madd(v[u], xv[u], s);
    }
  }
#pragma unroll
  for (int o = LANES / 2; o > 0; o >>= 1) s += __shfl_xor_sync(kFull, s, o);
  return s;
}

template <int LANES>
__global__ void __launch_bounds__(kSpmvThreads) k_spmv(int64_t n, const int32_t* __restrict__ rp,
                                                       const int32_t* __restrict__ ci,
                                                       const double* __restrict__ val,
                                                       const double* __restrict__ x,
                                                       double* __restrict__ y) {
  constexpr int RPB = kSpmvThreads / LANES;
  const int sub = threadIdx.x % LANES;
  for (int64_t base = (int64_t)blockIdx.x * RPB; base < n; base += (int64_t)gridDim.x * RPB) {
    const int64_t row = base + threadIdx.x / LANES;
    const bool valid = row < n;
    const double s = csr_row_dot<LANES>(rp, ci, val, x, row, valid, sub);
    if (valid && sub == 0) y[row] = s;
  }
}

// K1 fused: Ap_k = A p_k with gamma = p'Ap and p'p reduced in the same pass.
template <int LANES>
__global__ void __launch_bounds__(kSpmvThreads) k_spmv_pcg(const rk_pcg_plan P) {
  pdl_wait();
  pdl_trigger();
  if (P.st->done) return;
  constexpr int RPB = kSpmvThreads / LANES;
  __shared__ double scratch[64];
  const int64_t k = P.st->k;
  const double* __restrict__ p = P.V + k * P.ldv;
  double* __restrict__ Ap = P.AV + (P.ldav ? k * P.ldav : 0);
  const int32_t* __restrict__ rp = P.A.rowptr;
  const int32_t* __restrict__ ci = P.A.col;
  const double* __restrict__ val = P.A.val;
  const int64_t n = P.n;
  const int sub = threadIdx.x % LANES;
  double acc[2] = {0.0, 0.0};
  for (int64_t base = (int64_t)blockIdx.x * RPB; base < n; base += (int64_t)gridDim.x * RPB) {
    const int64_t row = base + threadIdx.x / LANES;
    const bool valid = row < n;
    const double s = csr_row_dot<LANES>(rp, ci, val, p, row, valid, sub);
    if (valid && sub == 0) {
      Ap[row] = s;
      const double pr = p[row];
      acc[0] = fma(pr, s, acc[0]);
      acc[1] = fma(pr, pr, acc[1]);
    }
  }
  block_sum<2>(acc, scratch);
  if (publish_and_check_last(acc, 2, P.partials, P.tickets + 0)) {
    __shared__ double tot[2];
    combine_partials(P.partials, gridDim.x, 2, tot);
    if (threadIdx.x == 0) curvature_epilogue(P, tot[0], tot[1]);
  }
}

// Generic-operator variant: the caller already wrote A p_k; reduce gamma, p'p.
__global__ void __launch_bounds__(kSpmvThreads) k_curvature(const rk_pcg_plan P) {
  pdl_wait();
  pdl_trigger();
  if (P.st->done) return;
  __shared__ double scratch[64];
  const int64_t k = P.st->k;
  const double* __restrict__ p = P.V + k * P.ldv;
  const double* __restrict__ Ap = P.AV + (P.ldav ? k * P.ldav : 0);
  double acc[2] = {0.0, 0.0};
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < P.n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double pr = p[i];
    acc[0] = fma(pr, Ap[i], acc[0]);
    acc[1] = fma(pr, pr, acc[1]);
  }
  block_sum<2>(acc, scratch);
  if (publish_and_check_last(acc, 2, P.partials, P.tickets + 0)) {
    __shared__ double tot[2];
    combine_partials(P.partials, gridDim.x, 2, tot);
    if (threadIdx.x == 0) curvature_epilogue(P, tot[0], tot[1]);
  }
}

// K2 SpMM: Y[:, c0:c0+CT] = A X[:, c0:c0+CT]; the matrix row is read once per
// column tile, the CT gathered columns share each (value, index) load.
template <int LANES, int CT>
__global__ void __launch_bounds__(kSpmvThreads) k_spmm(int64_t n, const int32_t* __restrict__ rp,
                                                       const int32_t* __restrict__ ci,
                                                       const double* __restrict__ val, int64_t m,
                                                       const double* __restrict__ X, int64_t ldx,
                                                       double* __restrict__ Y, int64_t ldy) {
  constexpr int RPB = kSpmvThreads / LANES;
  const int sub = threadIdx.x % LANES;
  const int64_t c0 = (int64_t)blockIdx.y * CT;
  const int ct = (int)min((int64_t)CT, m - c0);
  for (int64_t base = (int64_t)blockIdx.x * RPB; base < n; base += (int64_t)gridDim.x * RPB) {
    const int64_t row = base + threadIdx.x / LANES;
    double acc[CT];
#pragma unroll
    for (int t = 0; t < CT; ++t) acc[t] = 0.0;
    if (row < n) {
      const int32_t beg = __ldg(rp + row), end = __ldg(rp + row + 1);
      for (int32_t j = beg + sub; j < end; j += LANES) {
        const double v = __ldg(val + j);
        const double* xc = X + (int64_t)__ldg(ci + j) + c0 * ldx;
#pragma unroll
        for (int t = 0; t < CT; ++t)
          if (t < ct) acc[t] = row_madd(v, __ldg(xc + t * ldx), acc[t]);
      }
    }
#pragma unroll
    for (int t = 0; t < CT; ++t) {
#pragma unroll
      for (int o = LANES / 2; o > 0; o >>= 1) acc[t] += __shfl_xor_sync(kFull, acc[t], o);
    }
    if (row < n && sub == 0) {
#pragma unroll
      for (int t = 0; t < CT; ++t)
        if (t < ct) Y[row + (c0 + t) * ldy] = acc[t];
    }
  }
}

__global__ void k_csr_diagonal(int64_t n, const int32_t* __restrict__ rp,
                               const int32_t* __restrict__ ci, const double* __restrict__ val,
                               double* __restrict__ diag, double* __restrict__ dinv,
                               unsigned long long* bad) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    int32_t lo = rp[i], hi = rp[i + 1] - 1;
    double d = 0.0;
    while (lo <= hi) {  // columns sorted: binary search for the diagonal
      const int32_t mid = (lo + hi) >> 1;
      const int32_t c = ci[mid];
      if (c == i) { d = val[mid]; break; }
      if (c < i) lo = mid + 1; else hi = mid - 1;
    }
    if (diag) diag[i] = d;
    if (dinv) dinv[i] = 1.0 / d;  // preconditioners.py:58 `1.0 / diag` (IEEE division)
    if (!(d > 0.0)) atomicMin(bad, (unsigned long long)i);
  }
}

// max |A_ij - A_ji| over stored entries (missing transpose entries count as 0)
// and max |A_ij|; max is order independent, so this is deterministic.
__global__ void __launch_bounds__(256) k_csr_asymmetry(int64_t n, const int32_t* __restrict__ rp,
                                                       const int32_t* __restrict__ ci,
                                                       const double* __restrict__ val,
                                                       double* partials, uint32_t* ticket,
                                                       double* out2) {
  double worst = 0.0, scale = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    for (int32_t e = rp[i]; e < rp[i + 1]; ++e) {
      const int32_t j = ci[e];
      const double v = val[e];
      scale = fmax(scale, fabs(v));
      int32_t lo = rp[j], hi = rp[j + 1] - 1;
      double vt = 0.0;
      while (lo <= hi) {
        const int32_t mid = (lo + hi) >> 1;
        const int32_t c = ci[mid];
        if (c == i) { vt = val[mid]; break; }
        if (c < i) lo = mid + 1; else hi = mid - 1;
      }
      worst = fmax(worst, fabs(v - vt));
    }
  }
  __shared__ double sw[32], ss[32];
  for (int o = 16; o > 0; o >>= 1) {
    worst = fmax(worst, __shfl_xor_sync(kFull, worst, o));
    scale = fmax(scale, __shfl_xor_sync(kFull, scale, o));
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  if (lane == 0) { sw[warp] = worst; ss[warp] = scale; }
  __syncthreads();
  double v2[2] = {0.0, 0.0};
  if (threadIdx.x == 0) {
    for (int w = 0; w < nw; ++w) { v2[0] = fmax(v2[0], sw[w]); v2[1] = fmax(v2[1], ss[w]); }
  }
  __shared__ double vs[2];
  if (threadIdx.x == 0) { vs[0] = v2[0]; vs[1] = v2[1]; }
  __syncthreads();
  if (publish_and_check_last(vs, 2, partials, ticket)) {
    if (threadIdx.x == 0) {
      double a = 0.0, b = 0.0;
      for (unsigned blk = 0; blk < gridDim.x; ++blk) {
        a = fmax(a, __ldcg(partials + 2 * blk));
        b = fmax(b, __ldcg(partials + 2 * blk + 1));
      }
      out2[0] = a;
      out2[1] = b;
    }
  }
}

// ---------------------------------------------------------------------------
// 3x3-block SpMV in sliced-ELL form (SELL-32 of 3x3 blocks) for vector-valued
// problems such as the Q1 elasticity operator. A warp owns a slice of 32 block
// rows, one block row (3 matrix rows) per lane; slot t of the slice is read by
// all 32 lanes at once, so every load of the block column and of each of the 9
// values is a fully coalesced 128- or 256-byte warp access, the 9 value planes
// of a slot row are one contiguous 2304-byte tile (one DRAM stream per warp
// step), and the 3 consecutive x entries of the block column are gathered per
// lane. 76 bytes per stored block (vs 108 for the same 9
// nonzeros in CSR); slices are padded only to their widest row.
// ---------------------------------------------------------------------------
// Software-pipelined variant (U = 0), two stages: while the fmas of slot row t
// run, the x gather of slot row t+1 (whose block column arrived an iteration
// ago) and the column + values of slot row t+2 are in flight, so in-order
// issue never waits on a load issued in the same iteration.
__device__ __forceinline__ void sell3_row_pipe(const rk_csr& A, const double* __restrict__ x, int64_t slice,
                                               int lane, double& s0, double& s1, double& s2) {
  s0 = s1 = s2 = 0.0;
  const int32_t base = __ldg(A.browptr + slice);
  const int32_t width = (__ldg(A.browptr + slice + 1) - base) >> 5;
  if (width == 0) return;
  const int32_t* __restrict__ col = A.bcol + base + lane;
  const double* __restrict__ val = A.bval + 9 * (int64_t)base + lane;
  double v0[9], v1[9], v2[9], x0[3], x1[3];
  int32_t c1 = 0, c2 = 0;
  // prologue: slot 0 gathered, slot 1 loaded
  {
    const int32_t c0 = __ldcs(col);
#pragma unroll
    for (int e = 0; e < 9; ++e) v0[e] = __ldcs(val + 32 * e);
    if (width > 1) {
      c1 = __ldcs(col + 32);
#pragma unroll
      for (int e = 0; e < 9; ++e) v1[e] = __ldcs(val + 288 + 32 * e);
    }
    const double* xp = x + 3 * (int64_t)c0;
    x0[0] = __ldg(xp); x0[1] = __ldg(xp + 1); x0[2] = __ldg(xp + 2);
  }
  for (int32_t t = 0; t < width; ++t) {
    if (t + 1 < width) {  // gather for slot t+1
      const double* xp = x + 3 * (int64_t)c1;
      x1[0] = __ldg(xp); x1[1] = __ldg(xp + 1); x1[2] = __ldg(xp + 2);
    }
    if (t + 2 < width) {  // column + values for slot t+2
      c2 = __ldcs(col + 32 * (t + 2));
#pragma unroll
      for (int e = 0; e < 9; ++e) v2[e] = __ldcs(val + 288 * (t + 2) + 32 * e);
    }
    s0 = row_madd(v0[0], x0[0], s0); s0 = row_madd(v0[1], x0[1], s0); s0 = row_madd(v0[2], x0[2], s0);
    s1 = row_madd(v0[3], x0[0], s1); s1 = row_madd(v0[4], x0[1], s1); s1 = row_madd(v0[5], x0[2], s1);
    s2 = row_madd(v0[6], x0[0], s2); s2 = row_madd(v0[7], x0[1], s2); s2 = row_madd(v0[8], x0[2], s2);
#pragma unroll
    for (int e = 0; e < 9; ++e) {
      v0[e] = v1[e];
      v1[e] = v2[e];
    }
    x0[0] = x1[0]; x0[1] = x1[1]; x0[2] = x1[2];
    c1 = c2;
  }
}

// Streaming loads the compiler may not reorder among themselves (volatile asm):
// with them, every column and value load of U slot rows is issued before the
// first dependent gather, whatever the scheduler's register heuristics.
__device__ __forceinline__ double ld_stream_f64(const double* p) {
  double v;
  asm volatile("ld.global.cs.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ int32_t ld_stream_s32(const int32_t* p) {
  int32_t v;
  asm volatile("ld.global.cs.s32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}

template <int U>
__device__ __forceinline__ void sell3_row_issue(const rk_csr& A, const double* __restrict__ x, int64_t slice,
                                                int lane, double& s0, double& s1, double& s2) {
  s0 = s1 = s2 = 0.0;
  const int32_t base = __ldg(A.browptr + slice);
  const int32_t width = (__ldg(A.browptr + slice + 1) - base) >> 5;
  const int32_t* __restrict__ col = A.bcol + base + lane;
  const double* __restrict__ val = A.bval + 9 * (int64_t)base + lane;
  int32_t t = 0;
  for (; t + U <= width; t += U) {
    int32_t c[U];
    double v[U][9];
#pragma unroll
    for (int u = 0; u < U; ++u) c[u] = ld_stream_s32(col + 32 * (t + u));
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int e = 0; e < 9; ++e) v[u][e] = ld_stream_f64(val + 288 * (t + u) + 32 * e);
    double xs[U][3];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const double* xc = x + 3 * (int64_t)c[u];
      xs[u][0] = __ldg(xc);
      xs[u][1] = __ldg(xc + 1);
      xs[u][2] = __ldg(xc + 2);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      s0 = row_madd(v[u][0], xs[u][0], s0); s0 = row_madd(v[u][1], xs[u][1], s0); s0 = row_madd(v[u][2], xs[u][2], s0);
      s1 = row_madd(v[u][3], xs[u][0], s1); s1 = row_madd(v[u][4], xs[u][1], s1); s1 = row_madd(v[u][5], xs[u][2], s1);
      s2 = row_madd(v[u][6], xs[u][0], s2); s2 = row_madd(v[u][7], xs[u][1], s2); s2 = row_madd(v[u][8], xs[u][2], s2);
    }
  }
  for (; t < width; ++t) {
    const int32_t ca = ld_stream_s32(col + 32 * t);
    double va[9];
#pragma unroll
    for (int e = 0; e < 9; ++e) va[e] = ld_stream_f64(val + 288 * t + 32 * e);
    const double* xa = x + 3 * (int64_t)ca;
    const double a0 = __ldg(xa), a1 = __ldg(xa + 1), a2 = __ldg(xa + 2);
    s0 = row_madd(va[0], a0, s0); s0 = row_madd(va[1], a1, s0); s0 = row_madd(va[2], a2, s0);
    s1 = row_madd(va[3], a0, s1); s1 = row_madd(va[4], a1, s1); s1 = row_madd(va[5], a2, s1);
    s2 = row_madd(va[6], a0, s2); s2 = row_madd(va[7], a1, s2); s2 = row_madd(va[8], a2, s2);
  }
}

template <int U>
__device__ __forceinline__ void sell3_row(const rk_csr& A, const double* __restrict__ x, int64_t slice, int lane,
                                          double& s0, double& s1, double& s2) {
  s0 = s1 = s2 = 0.0;
  const int32_t base = __ldg(A.browptr + slice);
  const int32_t width = (__ldg(A.browptr + slice + 1) - base) >> 5;
  const int32_t* __restrict__ col = A.bcol + base + lane;
  // slot row t of the slice: 9 x 32 values, contiguous (entry e at 32 e + lane)
  const double* __restrict__ val = A.bval + 9 * (int64_t)base + lane;
  int32_t t = 0;
  for (; t + U <= width; t += U) {  // U slot rows in flight per lane
    int32_t c[U];
    double v[U][9];
#pragma unroll
    for (int u = 0; u < U; ++u) c[u] = __ldcs(col + 32 * (t + u));
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int e = 0; e < 9; ++e) v[u][e] = __ldcs(val + 288 * (t + u) + 32 * e);
    double xs[U][3];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const double* xc = x + 3 * (int64_t)c[u];
      xs[u][0] = __ldg(xc);
      xs[u][1] = __ldg(xc + 1);
      xs[u][2] = __ldg(xc + 2);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {  // slots in order: the same fma chain for every U
      s0 = row_madd(v[u][0], xs[u][0], s0); s0 = row_madd(v[u][1], xs[u][1], s0); s0 = row_madd(v[u][2], xs[u][2], s0);
      s1 = row_madd(v[u][3], xs[u][0], s1); s1 = row_madd(v[u][4], xs[u][1], s1); s1 = row_madd(v[u][5], xs[u][2], s1);
      s2 = row_madd(v[u][6], xs[u][0], s2); s2 = row_madd(v[u][7], xs[u][1], s2); s2 = row_madd(v[u][8], xs[u][2], s2);
    }
  }
  for (; t < width; ++t) {
    const int32_t ca = __ldcs(col + 32 * t);
    double va[9];
#pragma unroll
    for (int e = 0; e < 9; ++e) va[e] = __ldcs(val + 288 * t + 32 * e);
    const double* xa = x + 3 * (int64_t)ca;
    const double a0 = __ldg(xa), a1 = __ldg(xa + 1), a2 = __ldg(xa + 2);
    s0 = row_madd(va[0], a0, s0); s0 = row_madd(va[1], a1, s0); s0 = row_madd(va[2], a2, s0);
    s1 = row_madd(va[3], a0, s1); s1 = row_madd(va[4], a1, s1); s1 = row_madd(va[5], a2, s1);
    s2 = row_madd(va[6], a0, s2); s2 = row_madd(va[7], a1, s2); s2 = row_madd(va[8], a2, s2);
  }
}

__global__ void __launch_bounds__(kSpmvThreads, 2) k_bsr3_spmv(const rk_csr A, const double* __restrict__ x,
                                                            double* __restrict__ y) {
  const int lane = threadIdx.x & 31;
  const int64_t nbr = A.n / 3;
  const int64_t nsl = (nbr + 31) / 32;
  const int64_t wpb = kSpmvThreads / 32;
  for (int64_t sl = (int64_t)blockIdx.x * wpb + (threadIdx.x >> 5); sl < nsl; sl += (int64_t)gridDim.x * wpb) {
    double s0, s1, s2;
    sell3_row<3>(A, x, sl, lane, s0, s1, s2);
    const int64_t br = sl * 32 + lane;
    if (br < nbr) {
      y[3 * br] = s0;
      y[3 * br + 1] = s1;
      y[3 * br + 2] = s2;
    }
  }
}

template <int U>
__global__ void __launch_bounds__(kSpmvThreads, (U == 14 || U == 4 || U == 3) ? 2 : (U == 5 ? 3 : 1)) k_bsr3_spmv_pcg(const rk_pcg_plan P) {
  pdl_wait();
  pdl_trigger();
  if (P.st->done) return;
  __shared__ double scratch[64];
  const int64_t k = P.st->k;
  const double* __restrict__ p = P.V + k * P.ldv;
  double* __restrict__ Ap = P.AV + (P.ldav ? k * P.ldav : 0);
  const int lane = threadIdx.x & 31;
  const int64_t nbr = P.n / 3;
  const int64_t nsl = (nbr + 31) / 32;
  const int64_t wpb = kSpmvThreads / 32;
  double acc[2] = {0.0, 0.0};
  for (int64_t sl = (int64_t)blockIdx.x * wpb + (threadIdx.x >> 5); sl < nsl; sl += (int64_t)gridDim.x * wpb) {
    double s0, s1, s2;
    if constexpr (U == 0) sell3_row_pipe(P.A, p, sl, lane, s0, s1, s2);
    else if constexpr (U >= 12) sell3_row_issue<U - 10>(P.A, p, sl, lane, s0, s1, s2);
    else if constexpr (U == 5) sell3_row<4>(P.A, p, sl, lane, s0, s1, s2);
    else sell3_row<U>(P.A, p, sl, lane, s0, s1, s2);
    const int64_t br = sl * 32 + lane;
    if (br < nbr) {
      const int64_t row = 3 * br;
      Ap[row] = s0;
      Ap[row + 1] = s1;
      Ap[row + 2] = s2;
      const double p0 = p[row], p1 = p[row + 1], p2 = p[row + 2];
      acc[0] = fma(p0, s0, acc[0]);
      acc[0] = fma(p1, s1, acc[0]);
      acc[0] = fma(p2, s2, acc[0]);
      acc[1] = fma(p0, p0, acc[1]);
      acc[1] = fma(p1, p1, acc[1]);
      acc[1] = fma(p2, p2, acc[1]);
    }
  }
  block_sum<2>(acc, scratch);
  if (publish_and_check_last(acc, 2, P.partials, P.tickets + 0)) {
    __shared__ double tot[2];
    combine_partials(P.partials, gridDim.x, 2, tot);
    if (threadIdx.x == 0) curvature_epilogue(P, tot[0], tot[1]);
  }
}

// K2 on the 3x3 SELL view: Y[:, c0:c0+CT] = A X[:, c0:c0+CT] (blockIdx.y = column
// tile). A warp owns a slice (32 block rows, one per lane); per slot the 9 values
// and the block column are loaded once and applied to CT columns (x gathered per
// column: 3 contiguous doubles). Per column the fma order is exactly the SpMV's
// (sell3_row), so A X[:, j] is bitwise the SpMV of X[:, j]. Each column tile
// streams the matrix (HBM-bound at ceil(m/CT) matrix reads; CT = 4 keeps 64
// registers and full occupancy, measured 1.44 ms for m = 60 at C3 against
// 5.3 ms for the CSR kernel).
template <int CT>
__global__ void __launch_bounds__(kSpmvThreads) k_bsr3_spmm(const rk_csr A, int64_t m, const double* __restrict__ X,
                                                            int64_t ldx, double* __restrict__ Y, int64_t ldy) {
  const int lane = threadIdx.x & 31;
  const int64_t nbr = A.n / 3;
  const int64_t nsl = (nbr + 31) / 32;
  const int64_t wpb = kSpmvThreads / 32;
  const int64_t c0 = (int64_t)blockIdx.y * CT;
  const int ncol = (int)(m - c0 < CT ? m - c0 : CT);
  for (int64_t sl = (int64_t)blockIdx.x * wpb + (threadIdx.x >> 5); sl < nsl; sl += (int64_t)gridDim.x * wpb) {
    double acc[3][CT];
#pragma unroll
    for (int j = 0; j < CT; ++j) acc[0][j] = acc[1][j] = acc[2][j] = 0.0;
    const int32_t base = __ldg(A.browptr + sl);
    const int32_t width = (__ldg(A.browptr + sl + 1) - base) >> 5;
    const int32_t* __restrict__ col = A.bcol + base + lane;
    const double* __restrict__ val = A.bval + 9 * (int64_t)base + lane;
    for (int32_t t = 0; t < width; ++t) {
      const int32_t c = __ldcs(col + 32 * t);
      double v[9];
#pragma unroll
      for (int e = 0; e < 9; ++e) v[e] = __ldcs(val + 288 * t + 32 * e);
      const double* xc = X + c0 * ldx + 3 * (int64_t)c;
#pragma unroll
      for (int j = 0; j < CT; ++j) {
        if (j < ncol) {
          const double x0 = __ldg(xc + j * ldx), x1 = __ldg(xc + j * ldx + 1), x2 = __ldg(xc + j * ldx + 2);
          acc[0][j] = row_madd(v[0], x0, acc[0][j]); acc[0][j] = row_madd(v[1], x1, acc[0][j]); acc[0][j] = row_madd(v[2], x2, acc[0][j]);
          acc[1][j] = row_madd(v[3], x0, acc[1][j]); acc[1][j] = row_madd(v[4], x1, acc[1][j]); acc[1][j] = row_madd(v[5], x2, acc[1][j]);
          acc[2][j] = row_madd(v[6], x0, acc[2][j]); acc[2][j] = row_madd(v[7], x1, acc[2][j]); acc[2][j] = row_madd(v[8], x2, acc[2][j]);
        }
      }
    }
    const int64_t br = sl * 32 + lane;
    if (br < nbr) {
#pragma unroll
      for (int j = 0; j < CT; ++j) {
        if (j < ncol) {
          double* yj = Y + (c0 + j) * ldy + 3 * br;
          yj[0] = acc[0][j];
          yj[1] = acc[1][j];
          yj[2] = acc[2][j];
        }
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Scalar sliced-ELL (SELL-32, bdim == 1) for short uniform rows such as the
// 7-point stencils of C2 and C5: a warp owns a slice of 32 rows, one row per
// lane, and slot row t of the slice (32 values, 32 columns) is one 256-byte
// and one 128-byte fully coalesced warp load. Each lane sums its row in CSR
// order (padding slots hold 0 and a valid column), i.e. exactly scipy's
// sequential csr_matvec order. 12 bytes per stored slot, no row pointers.
// ---------------------------------------------------------------------------
template <int U>
__device__ __forceinline__ double sell1_row(const rk_csr& A, const double* __restrict__ x, int32_t base, int32_t width,
                                            int lane) {
  const int32_t* __restrict__ col = A.bcol + base + lane;
  const double* __restrict__ val = A.bval + base + lane;
  double s = 0.0;
  for (int32_t t = 0; t < width; t += U) {  // U slot rows in flight per lane
    int32_t c[U];
    double v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const bool ok = t + u < width;
      c[u] = ok ? ld_stream_s32(col + 32 * (t + u)) : 0;
      v[u] = ok ? ld_stream_f64(val + 32 * (t + u)) : 0.0;
    }
    double xs[U];
#pragma unroll
    for (int u = 0; u < U; ++u) xs[u] = __ldg(x + c[u]);
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (t + u < width) s = row_madd(v[u], xs[u], s);
  }
  return s;
}

constexpr int kSell1U = 8;

// A warp's walk over its slices with the slice pointers one step ahead: a
// slice's work is three dependent round trips (slice pointers -> slot columns
// and values -> gathered x); fetching the next slice's pointers before the
// current slice's loads takes the first one off the chain.
struct SliceWalk {
  const int32_t* __restrict__ ptr;
  int64_t sl, stride, nsl;
  int32_t base, end;
  __device__ __forceinline__ SliceWalk(const int32_t* p, int64_t first, int64_t stride_, int64_t nsl_)
      : ptr(p), sl(first), stride(stride_), nsl(nsl_), base(0), end(0) {
    if (sl < nsl) {
      base = __ldg(ptr + sl);
      end = __ldg(ptr + sl + 1);
    }
  }
  __device__ __forceinline__ bool valid() const { return sl < nsl; }
  __device__ __forceinline__ int32_t width() const { return (end - base) >> 5; }
  __device__ __forceinline__ void advance() {
    sl += stride;
    if (sl < nsl) {
      base = __ldg(ptr + sl);
      end = __ldg(ptr + sl + 1);
    }
  }
};

__global__ void __launch_bounds__(kSpmvThreads) k_sell1_spmv(const rk_csr A, const double* __restrict__ x,
                                                            double* __restrict__ y) {
  const int lane = threadIdx.x & 31;
  const int64_t nsl = (A.n + 31) / 32;
  const int64_t wpb = kSpmvThreads / 32;
  SliceWalk w(A.browptr, (int64_t)blockIdx.x * wpb + (threadIdx.x >> 5), (int64_t)gridDim.x * wpb, nsl);
  while (w.valid()) {
    const int64_t sl = w.sl;
    const int32_t base = w.base, width = w.width();
    w.advance();  // the next slice's pointers load in the shadow of this slice's work
    const double s = sell1_row<kSell1U>(A, x, base, width, lane);
    const int64_t row = sl * 32 + lane;
    if (row < A.n) y[row] = s;
  }
}

__global__ void __launch_bounds__(kSpmvThreads) k_sell1_spmv_pcg(const rk_pcg_plan P) {
  pdl_wait();
  pdl_trigger();
  if (P.st->done) return;
  __shared__ double scratch[64];
  const int64_t k = P.st->k;
  const double* __restrict__ p = P.V + k * P.ldv;
  double* __restrict__ Ap = P.AV + (P.ldav ? k * P.ldav : 0);
  const int lane = threadIdx.x & 31;
  const int64_t nsl = (P.n + 31) / 32;
  const int64_t wpb = kSpmvThreads / 32;
  double acc[2] = {0.0, 0.0};
  SliceWalk w(P.A.browptr, (int64_t)blockIdx.x * wpb + (threadIdx.x >> 5), (int64_t)gridDim.x * wpb, nsl);
  while (w.valid()) {
    const int64_t sl = w.sl;
    const int32_t base = w.base, width = w.width();
    w.advance();
    const double s = sell1_row<kSell1U>(P.A, p, base, width, lane);
    const int64_t row = sl * 32 + lane;
    if (row < P.n) {
      Ap[row] = s;
      const double pr = p[row];
      acc[0] = fma(pr, s, acc[0]);
      acc[1] = fma(pr, pr, acc[1]);
    }
  }
  block_sum<2>(acc, scratch);
  if (publish_and_check_last(acc, 2, P.partials, P.tickets + 0)) {
    __shared__ double tot[2];
    combine_partials(P.partials, gridDim.x, 2, tot);
    if (threadIdx.x == 0) curvature_epilogue(P, tot[0], tot[1]);
  }
}

// K2 on the scalar SELL view (blockIdx.y = column tile of CT columns): each
// slot's value and column are loaded once for CT gathered columns; per column
// the fma order is the SpMV's, so A X[:, j] is bitwise the SpMV of X[:, j].
constexpr int kSpmmJ = 4;  // columns whose gathers are issued together in the scalar SELL SpMM
template <int CT>
__global__ void __launch_bounds__(kSpmvThreads) k_sell1_spmm(const rk_csr A, int64_t m, const double* __restrict__ X,
                                                            int64_t ldx, double* __restrict__ Y, int64_t ldy) {
  const int lane = threadIdx.x & 31;
  const int64_t nsl = (A.n + 31) / 32;
  const int64_t wpb = kSpmvThreads / 32;
  // blockIdx.x = column tile, blockIdx.y = slice group: the tiles of one row
  // range are adjacent in launch order and share the matrix slice and the
  // gathered neighbour rows in L2
  const int64_t c0 = (int64_t)blockIdx.x * CT;
  const int ncol = (int)(m - c0 < CT ? m - c0 : CT);
  for (int64_t sl = (int64_t)blockIdx.y * wpb + (threadIdx.x >> 5); sl < nsl; sl += (int64_t)gridDim.y * wpb) {
    double acc[CT];
#pragma unroll
    for (int j = 0; j < CT; ++j) acc[j] = 0.0;
    const int32_t base = __ldg(A.browptr + sl);
    const int32_t width = (__ldg(A.browptr + sl + 1) - base) >> 5;
    const int32_t* __restrict__ col = A.bcol + base + lane;
    const double* __restrict__ val = A.bval + base + lane;
    for (int32_t t = 0; t < width; t += kSell1U) {  // all slot loads of a pass before the gathers
      int32_t c[kSell1U];
      double v[kSell1U];
#pragma unroll
      for (int u = 0; u < kSell1U; ++u) {
        const bool ok = t + u < width;
        c[u] = ok ? ld_stream_s32(col + 32 * (t + u)) : 0;
        v[u] = ok ? ld_stream_f64(val + 32 * (t + u)) : 0.0;
      }
      if (ncol == CT) {
        // full tile: no per-column branch, so the gathers of kSpmmJ columns
        // (kSpmmJ x kSell1U loads) are all in flight before their sums
#pragma unroll
        for (int j0 = 0; j0 < CT; j0 += kSpmmJ) {
          double xs[kSpmmJ][kSell1U];
#pragma unroll
          for (int jj = 0; jj < kSpmmJ; ++jj) {
            const double* xc = X + (c0 + j0 + jj) * ldx;
#pragma unroll
            for (int u = 0; u < kSell1U; ++u) xs[jj][u] = __ldg(xc + c[u]);
          }
#pragma unroll
          for (int jj = 0; jj < kSpmmJ; ++jj)
#pragma unroll
            for (int u = 0; u < kSell1U; ++u)
              if (t + u < width) acc[j0 + jj] = row_madd(v[u], xs[jj][u], acc[j0 + jj]);
        }
      } else {
#pragma unroll
        for (int j = 0; j < CT; ++j) {
          if (j < ncol) {
            const double* xc = X + (c0 + j) * ldx;
            double xs[kSell1U];
#pragma unroll
            for (int u = 0; u < kSell1U; ++u) xs[u] = __ldg(xc + c[u]);
#pragma unroll
            for (int u = 0; u < kSell1U; ++u)
              if (t + u < width) acc[j] = row_madd(v[u], xs[u], acc[j]);
          }
        }
      }
    }
    const int64_t row = sl * 32 + lane;
    if (row < A.n) {
#pragma unroll
      for (int j = 0; j < CT; ++j)
        if (j < ncol) Y[(c0 + j) * ldy + row] = acc[j];
    }
  }
}

// Slot values from CSR values; perm < 0 marks padding (value 0).
__global__ void k_bsr3_gather(int64_t total, const int32_t* __restrict__ perm, const double* __restrict__ val,
                              double* __restrict__ bval) {
  for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < total; s += (int64_t)gridDim.x * blockDim.x) {
    const int32_t q = __ldg(perm + s);
    bval[s] = q >= 0 ? __ldg(val + q) : 0.0;
  }
}

}  // namespace rk

// ---------------------------------------------------------------------------
// Launchers
// ---------------------------------------------------------------------------
namespace rkh {

static int spmv_blocks_per_sm() {
  static const int v = [] {
    const char* e = getenv("RK_SPMV_BPS");
    const int x = e ? atoi(e) : 4;
    return x > 0 ? x : 4;
  }();
  return v;
}

static int resident_blocks(const void* kern, int threads) {
  int occ = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, threads, 0) != cudaSuccess || occ < 1) occ = 1;
  return occ * sm_count();
}

static int launch_bsr3_spmv(const rk_csr& A, const double* x, double* y, cudaStream_t s) {
  static const int cap = resident_blocks((const void*)rk::k_bsr3_spmv, rk::kSpmvThreads);
  const int64_t need = ((A.n / 3 + 31) / 32 + rk::kSpmvThreads / 32 - 1) / (rk::kSpmvThreads / 32);
  rk::k_bsr3_spmv<<<(int)std::max<int64_t>(1, std::min<int64_t>(cap, need)), rk::kSpmvThreads, 0, s>>>(A, x, y);
  rkh::note_launch();
  return cuda_check("rk_spmv (bsr3)");
}

template <int U>
static void launch_bsr3_spmv_pcg_u(const rk_pcg_plan& P, cudaStream_t s) {
  // a fixed number of blocks per SM (when resident), so the order of the
  // p'Ap / p'p partial sums does not follow register allocation
  static const int cap = std::min(resident_blocks((const void*)rk::k_bsr3_spmv_pcg<U>, rk::kSpmvThreads),
                                  sm_count() * spmv_blocks_per_sm());
  const int64_t need = ((P.n / 3 + 31) / 32 + rk::kSpmvThreads / 32 - 1) / (rk::kSpmvThreads / 32);
  launch_pdl(rk::k_bsr3_spmv_pcg<U>, dim3((unsigned)std::max<int64_t>(1, std::min<int64_t>(cap, need))),
             dim3(rk::kSpmvThreads), 0, s, P);
}

static int sell_unroll() {
  static const int v = [] {
    const char* e = getenv("RK_SELL_U");
    // 3 slot rows in flight with room for 110 registers (2 blocks/SM), so every
    // column and value load of the 3 rows is issued before the first gather:
    // measured 94.6 us vs 98.5 us for 2 rows at 48 registers (C3). Others are
    // kept for measurement: 0 = two-stage software pipeline, 12/14 = explicit
    // issue order with 2/4 rows, 5 = 4 rows at 3 blocks/SM.
    const int x = e ? atoi(e) : 3;
    return ((x >= 0 && x <= 5) || x == 12 || x == 14) ? x : 3;
  }();
  return v;
}

static void launch_bsr3_spmv_pcg(const rk_pcg_plan& P, cudaStream_t s) {
  switch (sell_unroll()) {
    case 0: launch_bsr3_spmv_pcg_u<0>(P, s); break;
    case 1: launch_bsr3_spmv_pcg_u<1>(P, s); break;
    case 4: launch_bsr3_spmv_pcg_u<4>(P, s); break;
    case 5: launch_bsr3_spmv_pcg_u<5>(P, s); break;
    case 12: launch_bsr3_spmv_pcg_u<12>(P, s); break;  // volatile-issue variants: 2 / 4 slot rows
    case 14: launch_bsr3_spmv_pcg_u<14>(P, s); break;
    case 2: launch_bsr3_spmv_pcg_u<2>(P, s); break;
    default: launch_bsr3_spmv_pcg_u<3>(P, s); break;
  }
}

static int launch_sell1_spmv(const rk_csr& A, const double* x, double* y, cudaStream_t s) {
  static const int cap = resident_blocks((const void*)rk::k_sell1_spmv, rk::kSpmvThreads);
  const int64_t need = ((A.n + 31) / 32 + rk::kSpmvThreads / 32 - 1) / (rk::kSpmvThreads / 32);
  rk::k_sell1_spmv<<<(int)std::max<int64_t>(1, std::min<int64_t>(cap, need)), rk::kSpmvThreads, 0, s>>>(A, x, y);
  rkh::note_launch();
  return cuda_check("rk_spmv (sell1)");
}

static void launch_sell1_spmv_pcg(const rk_pcg_plan& P, cudaStream_t s) {
  // fixed blocks per SM (when resident) so the p'Ap / p'p partial order is fixed
  static const int cap = std::min(resident_blocks((const void*)rk::k_sell1_spmv_pcg, rk::kSpmvThreads),
                                  sm_count() * spmv_blocks_per_sm());
  const int64_t need = ((P.n + 31) / 32 + rk::kSpmvThreads / 32 - 1) / (rk::kSpmvThreads / 32);
  launch_pdl(rk::k_sell1_spmv_pcg, dim3((unsigned)std::max<int64_t>(1, std::min<int64_t>(cap, need))),
             dim3(rk::kSpmvThreads), 0, s, P);
}

int launch_sell_gather(int64_t total, const int32_t* perm, const double* val, double* out, cudaStream_t s) {
  if (total > 0) {
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((total + 255) / 256, (int64_t)sm_count() * 16));
    rk::k_bsr3_gather<<<grid, 256, 0, s>>>(total, perm, val, out);
    rkh::note_launch();
  }
  return cuda_check("rk_sell_gather");
}

int launch_bsr3_gather(int64_t nblk, const int32_t* perm, const double* val, double* bval, cudaStream_t s) {
  const int64_t total = 9 * nblk;
  if (total > 0) {
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((total + 255) / 256, (int64_t)sm_count() * 16));
    rk::k_bsr3_gather<<<grid, 256, 0, s>>>(total, perm, val, bval);
    rkh::note_launch();
  }
  return cuda_check("rk_bsr3_gather");
}

int auto_lanes(const rk_csr& A) {
  if (A.lanes > 0) return A.lanes;
  const double avg = A.n > 0 ? (double)A.nnz / (double)A.n : 1.0;
  if (avg <= 3.0) return 1;
  if (avg <= 7.5) return 2;
  if (avg <= 14.0) return 4;
  if (avg <= 44.0) return 8;
  if (avg <= 90.0) return 16;
  return 32;
}

int spmv_grid(int64_t n, int lanes) {
  const int64_t rpb = rk::kSpmvThreads / lanes;
  const int64_t need = (n + rpb - 1) / rpb;
  const int64_t cap = (int64_t)sm_count() * 8;
  return (int)std::max<int64_t>(1, std::min(need, cap));
}

// One resident wave: grid = (resident blocks per SM) x SMs, rows grid-strided.
template <typename Kern>
static int resident_grid(Kern kern, int threads, int64_t need) {
  int occ = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, threads, 0) != cudaSuccess || occ < 1) occ = 1;
  return (int)std::max<int64_t>(1, std::min<int64_t>(need, (int64_t)occ * sm_count()));
}

template <int L>
static void launch_spmv_l(const rk_csr& A, const double* x, double* y, cudaStream_t s) {
  static const int cap = resident_grid(rk::k_spmv<L>, rk::kSpmvThreads, INT64_MAX);
  const int grid = (int)std::min<int64_t>(cap, (A.n + rk::kSpmvThreads / L - 1) / (rk::kSpmvThreads / L));
  rk::k_spmv<L><<<std::max(grid, 1), rk::kSpmvThreads, 0, s>>>(A.n, A.rowptr, A.col, A.val, x, y); rkh::note_launch();
}

int launch_spmv(const rk_csr& A, const double* x, double* y, cudaStream_t s) {
  if (A.bval) return A.bdim == 1 ? launch_sell1_spmv(A, x, y, s) : launch_bsr3_spmv(A, x, y, s);
  switch (auto_lanes(A)) {
    case 1: launch_spmv_l<1>(A, x, y, s); break;
    case 2: launch_spmv_l<2>(A, x, y, s); break;
    case 4: launch_spmv_l<4>(A, x, y, s); break;
    case 8: launch_spmv_l<8>(A, x, y, s); break;
    case 16: launch_spmv_l<16>(A, x, y, s); break;
    default: launch_spmv_l<32>(A, x, y, s); break;
  }
  return cuda_check("rk_spmv");
}

template <int L>
static void launch_spmv_pcg_l(const rk_pcg_plan& P, cudaStream_t s) {
  static const int cap = std::min(resident_grid(rk::k_spmv_pcg<L>, rk::kSpmvThreads, INT64_MAX), sm_count() * 8);
  const int grid = (int)std::min<int64_t>(cap, (P.n + rk::kSpmvThreads / L - 1) / (rk::kSpmvThreads / L));
  launch_pdl(rk::k_spmv_pcg<L>, dim3(std::max(grid, 1)), dim3(rk::kSpmvThreads), 0, s, P);
}

void launch_spmv_pcg(const rk_pcg_plan& P, cudaStream_t s) {
  if (P.A.bval) {
    if (P.A.bdim == 1)
      launch_sell1_spmv_pcg(P, s);
    else
      launch_bsr3_spmv_pcg(P, s);
    return;
  }
  switch (auto_lanes(P.A)) {
    case 1: launch_spmv_pcg_l<1>(P, s); break;
    case 2: launch_spmv_pcg_l<2>(P, s); break;
    case 4: launch_spmv_pcg_l<4>(P, s); break;
    case 8: launch_spmv_pcg_l<8>(P, s); break;
    case 16: launch_spmv_pcg_l<16>(P, s); break;
    default: launch_spmv_pcg_l<32>(P, s); break;
  }
}

int curvature_grid(int64_t n) {
  const int64_t need = (n + 255) / 256;
  return (int)std::max<int64_t>(1, std::min<int64_t>(need, (int64_t)sm_count() * 4));
}

void launch_curvature(const rk_pcg_plan& P, cudaStream_t s) {
  launch_pdl(rk::k_curvature, dim3(curvature_grid(P.n)), dim3(256), 0, s, P);
}

// Columns per pass of the CSR / scalar-SELL SpMM (RK_SPMM_CT = 8, 16 or 32):
// the matrix is streamed once per pass, so wider passes cut its share of the
// traffic (C5, 7 nonzeros per row: 84 + 16 CT bytes per row and pass).
static int spmm_ct() {
  static const int v = [] {
    const char* e = getenv("RK_SPMM_CT");
    const int c = e ? atoi(e) : 8;
    return (c == 16 || c == 32) ? c : 8;
  }();
  return v;
}

template <int L, int CT>
static void launch_spmm_lc(const rk_csr& A, int64_t m, const double* X, int64_t ldx, double* Y,
                           int64_t ldy, cudaStream_t s) {
  const int64_t tiles = (m + CT - 1) / CT;
  const int64_t rpb = rk::kSpmvThreads / L;
  int64_t gx = (A.n + rpb - 1) / rpb;
  gx = std::max<int64_t>(1, std::min<int64_t>(gx, std::max<int64_t>(1, (int64_t)sm_count() * 8 / std::max<int64_t>(1, std::min<int64_t>(tiles, 8)))));
  dim3 grid((unsigned)gx, (unsigned)tiles);
  rk::k_spmm<L, CT><<<grid, rk::kSpmvThreads, 0, s>>>(A.n, A.rowptr, A.col, A.val, m, X, ldx, Y, ldy); rkh::note_launch();
}

template <int L>
static void launch_spmm_l(const rk_csr& A, int64_t m, const double* X, int64_t ldx, double* Y,
                          int64_t ldy, cudaStream_t s) {
  switch (spmm_ct()) {
    case 16: launch_spmm_lc<L, 16>(A, m, X, ldx, Y, ldy, s); break;
    case 32: launch_spmm_lc<L, 32>(A, m, X, ldx, Y, ldy, s); break;
    default: launch_spmm_lc<L, 8>(A, m, X, ldx, Y, ldy, s); break;
  }
}

template <int CT>
static void launch_sell1_spmm(const rk_csr& A, int64_t m, const double* X, int64_t ldx, double* Y, int64_t ldy,
                              cudaStream_t s) {
  const int64_t tiles = (m + CT - 1) / CT;
  const int64_t need = ((A.n + 31) / 32 + rk::kSpmvThreads / 32 - 1) / (rk::kSpmvThreads / 32);
  const int64_t gy = std::max<int64_t>(1, std::min<int64_t>(need, 65535));
  rk::k_sell1_spmm<CT><<<dim3((unsigned)tiles, (unsigned)gy), rk::kSpmvThreads, 0, s>>>(A, m, X, ldx, Y, ldy);
  note_launch();
}

template <int CT>
static void launch_bsr3_spmm(const rk_csr& A, int64_t m, const double* X, int64_t ldx, double* Y, int64_t ldy,
                             cudaStream_t s) {
  static const int cap = resident_blocks((const void*)rk::k_bsr3_spmm<CT>, rk::kSpmvThreads);
  const int64_t tiles = (m + CT - 1) / CT;
  const int64_t nsl = (A.n / 3 + 31) / 32;
  const int64_t need = (nsl + rk::kSpmvThreads / 32 - 1) / (rk::kSpmvThreads / 32);
  const int64_t gx = std::max<int64_t>(1, std::min<int64_t>(need, std::max<int64_t>(1, cap / tiles)));
  rk::k_bsr3_spmm<CT><<<dim3((unsigned)gx, (unsigned)tiles), rk::kSpmvThreads, 0, s>>>(A, m, X, ldx, Y, ldy);
  note_launch();
}

static int spmm_bsr_ct() {
  static const int v = [] {
    const char* e = getenv("RK_SPMM_CT");
    const int x = e ? atoi(e) : 4;
    return (x == 2 || x == 4 || x == 8) ? x : 4;
  }();
  return v;
}

int launch_spmm(const rk_csr& A, int64_t m, const double* X, int64_t ldx, double* Y, int64_t ldy,
                cudaStream_t s) {
  if (m <= 0 || A.n <= 0) return 0;
  // The scalar SELL SpMM (k_sell1_spmm) measured 1.35-1.85 TB/s at C5 against
  // 3.4 TB/s for the lanes-per-row CSR kernel, so it is opt-in (RK_SELL1_SPMM=1).
  static const bool sell1_spmm = [] {
    const char* e = getenv("RK_SELL1_SPMM");
    return e && atoi(e) == 1;
  }();
  if (A.bval && A.bdim == 1 && sell1_spmm) {
    switch (spmm_ct()) {
      case 16: launch_sell1_spmm<16>(A, m, X, ldx, Y, ldy, s); break;
      case 32: launch_sell1_spmm<32>(A, m, X, ldx, Y, ldy, s); break;
      default: launch_sell1_spmm<8>(A, m, X, ldx, Y, ldy, s); break;
    }
    return cuda_check("rk_spmm (sell1)");
  }
  if (A.bval && A.bdim != 1) {
    switch (spmm_bsr_ct()) {
      case 2: launch_bsr3_spmm<2>(A, m, X, ldx, Y, ldy, s); break;
      case 8: launch_bsr3_spmm<8>(A, m, X, ldx, Y, ldy, s); break;
      default: launch_bsr3_spmm<4>(A, m, X, ldx, Y, ldy, s); break;
    }
    return cuda_check("rk_spmm (bsr3)");
  }
  switch (auto_lanes(A)) {
    case 1: launch_spmm_l<1>(A, m, X, ldx, Y, ldy, s); break;
    case 2: launch_spmm_l<2>(A, m, X, ldx, Y, ldy, s); break;
    case 4: launch_spmm_l<4>(A, m, X, ldx, Y, ldy, s); break;
    case 8: launch_spmm_l<8>(A, m, X, ldx, Y, ldy, s); break;
    case 16: launch_spmm_l<16>(A, m, X, ldx, Y, ldy, s); break;
    default: launch_spmm_l<32>(A, m, X, ldx, Y, ldy, s); break;
  }
  return cuda_check("rk_spmm");
}

int launch_csr_diagonal(const rk_csr& A, double* diag, double* dinv, int64_t* bad, cudaStream_t s) {
  if (cudaMemsetAsync(bad, 0xff, sizeof(int64_t), s) != cudaSuccess) return cuda_check("rk_csr_diagonal");
  if (A.n > 0) {
    const int grid = curvature_grid(A.n);
    rk::k_csr_diagonal<<<grid, 256, 0, s>>>(A.n, A.rowptr, A.col, A.val, diag, dinv,
                                            reinterpret_cast<unsigned long long*>(bad)); rkh::note_launch();
  }
  return cuda_check("rk_csr_diagonal");
}

int launch_csr_asymmetry(const rk_csr& A, double* out2, double* ws, int64_t ws_len, uint32_t* tickets,
                         cudaStream_t s) {
  const int grid = curvature_grid(std::max<int64_t>(A.n, 1));
  RK_REQUIRE(ws_len >= 2 * grid, RK_ERR_ARG, "rk_csr_asymmetry: workspace too small (%lld < %d)",
             (long long)ws_len, 2 * grid);
  rk::k_csr_asymmetry<<<grid, 256, 0, s>>>(A.n, A.rowptr, A.col, A.val, ws, tickets, out2); rkh::note_launch();
  return cuda_check("rk_csr_asymmetry");
}

}  // namespace rkh
