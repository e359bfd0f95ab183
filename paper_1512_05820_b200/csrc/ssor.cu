// SSOR preconditioner application (preconditioners.py:64-90):
//   M = (D/w + L) D^{-1} (D/w + L)',  z = M^{-1} r:
//   forward sweep   (D/w + L) u = r          (rows ascending, j < i of A's CSR)
//   scale           v = u * d                (fused into the backward sweep's rhs)
//   backward sweep  (D/w + L') z = v         (rows descending, j > i of A's CSR;
//                                             L' is A's strict upper part, A = A')
// Both sweeps read A's own CSR (no triangular copies). They are "sync-free"
// sparse triangular solves: one warp per row, rows handed out in solve order by
// an atomic counter, so every row a warp waits on was handed out earlier and is
// running or done (no deadlock); a row publishes its value, then its ready flag
// (= the sweep's epoch) with release semantics, and dependants spin on the flag
// with acquire loads. Lanes stride the row's entries; the row sum is a fixed
// butterfly, so results are deterministic.
//
// Hand-out order. In natural row order only ~one window of consecutive rows is
// in flight, and inside it a 7-point stencil's rows form chains (row i waits
// for i - 1): 13.5 ms per application at 64^3. With the rows sorted by
// dependency level (rk_ssor_levels once per matrix: level = 1 + max level of
// the row's dependencies, computed by the same sync-free scheme) whole levels
// are in flight together and the sweep takes (number of levels) x (one flag
// round trip). Every dependency still has a smaller hand-out index, and a
// row's arithmetic does not depend on the order, so z is bit for bit the same.
#include <algorithm>

#include "common.cuh"

namespace rk {

constexpr int kSsorThreads = 256;

__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(int* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// UPPER = false: forward sweep, out[i] = (rhs[i] - sum_{j<i} a_ij out[j]) / dw[i]
// UPPER = true : backward sweep with rhs[i] = fl(u[i] * d[i]),
//                out[i] = (rhs[i] - sum_{j>i} a_ij out[j]) / dw[i]
template <bool UPPER>
__global__ void __launch_bounds__(kSsorThreads) k_ssor_sweep(int64_t n, const int32_t* __restrict__ rowptr,
                                                             const int32_t* __restrict__ col,
                                                             const double* __restrict__ val,
                                                             const double* __restrict__ dw,
                                                             const double* __restrict__ d, const double* rhs,
                                                             double* out, int* flags, int epoch,
                                                             unsigned int* counter, const rk_pcg_state* st,
                                                             const double* rhs_even,
                                                             const int32_t* __restrict__ order) {
  // Inside a device-stepped PCG run (st != NULL): nothing to do once the run
  // has stopped, and the residual of iteration k sits in the ping-pong buffer
  // the update kernel wrote (rhs for odd k, rhs_even for even k).
  if (st) {
    if (st->done) return;
    if (rhs_even && !(st->k & 1)) rhs = rhs_even;
  }
  const int lane = threadIdx.x & 31;
  for (;;) {
    unsigned int t = 0;
    if (lane == 0) t = atomicAdd(counter, 1u);
    t = __shfl_sync(kFull, t, 0);
    if ((int64_t)t >= n) break;
    const int64_t i = order ? (int64_t)__ldg(order + t) : UPPER ? n - 1 - (int64_t)t : (int64_t)t;
    const int32_t lo = __ldg(rowptr + i), hi = __ldg(rowptr + i + 1);
    double s = 0.0;
    for (int32_t q = lo + lane; q < hi; q += 32) {
      const int32_t j = __ldg(col + q);
      if (UPPER ? (j > i) : (j < i)) {
        while (ld_acquire(flags + j) != epoch) {
        }
        s = fma(__ldg(val + q), __ldcg(out + j), s);
      }
    }
    s = warp_sum(s);
    if (lane == 0) {
      const double b = UPPER ? __dmul_rn(__ldcg(rhs + i), __ldg(d + i)) : __ldcg(rhs + i);
      out[i] = __ddiv_rn(__dsub_rn(b, s), __ldg(dw + i));
      st_release(flags + i, epoch);
    }
  }
}

// Dependency level of every row of a sweep: lvl[i] = 1 + max lvl[j] over the
// row's strictly lower (UPPER: strictly upper) entries, rows handed out in
// natural solve order (a dependency always precedes its dependants there).
template <bool UPPER>
__global__ void __launch_bounds__(kSsorThreads) k_ssor_levels(int64_t n, const int32_t* __restrict__ rowptr,
                                                              const int32_t* __restrict__ col, int32_t* lvl,
                                                              int* flags, int epoch, unsigned int* counter) {
  const int lane = threadIdx.x & 31;
  for (;;) {
    unsigned int t = 0;
    if (lane == 0) t = atomicAdd(counter, 1u);
    t = __shfl_sync(kFull, t, 0);
    if ((int64_t)t >= n) break;
    const int64_t i = UPPER ? n - 1 - (int64_t)t : (int64_t)t;
    const int32_t lo = __ldg(rowptr + i), hi = __ldg(rowptr + i + 1);
    int32_t l = 0;
    for (int32_t q = lo + lane; q < hi; q += 32) {
      const int32_t j = __ldg(col + q);
      if (UPPER ? (j > i) : (j < i)) {
        while (ld_acquire(flags + j) != epoch) {
        }
        l = max(l, __ldcg(lvl + j));
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) l = max(l, __shfl_xor_sync(kFull, l, o));
    if (lane == 0) {
      lvl[i] = l + 1;
      st_release(flags + i, epoch);
    }
  }
}

}  // namespace rk

namespace rkh {

static int ssor_grid() {
  static const int grid = [] {
    int occ = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, rk::k_ssor_sweep<false>, rk::kSsorThreads, 0) !=
            cudaSuccess || occ < 1)
      occ = 1;
    return occ * sm_count();
  }();
  return grid;
}

int launch_ssor_levels(const rk_csr& A, int upper, int32_t* lvl, int* flags, unsigned int* counter, int epoch,
                       cudaStream_t s) {
  if (A.n <= 0) return 0;
  const int g = (int)std::max<int64_t>(1, std::min<int64_t>(ssor_grid(), (A.n + 7) / 8));
  cudaMemsetAsync(counter, 0, sizeof(unsigned int), s);
  if (upper)
    rk::k_ssor_levels<true><<<g, rk::kSsorThreads, 0, s>>>(A.n, A.rowptr, A.col, lvl, flags, epoch, counter);
  else
    rk::k_ssor_levels<false><<<g, rk::kSsorThreads, 0, s>>>(A.n, A.rowptr, A.col, lvl, flags, epoch, counter);
  note_launch();
  return cuda_check("rk_ssor_levels");
}

int launch_ssor_apply(const rk_csr& A, const double* dw, const double* d, const double* r, double* z, double* u,
                      int* flags, unsigned int* counters, int epoch, cudaStream_t s, const rk_pcg_state* st,
                      const double* r_even, const int32_t* order_fwd, const int32_t* order_bwd) {
  if (A.n <= 0) return 0;
  const int g = (int)std::max<int64_t>(1, std::min<int64_t>(ssor_grid(), (A.n + 7) / 8));
  cudaMemsetAsync(counters, 0, 2 * sizeof(unsigned int), s);
  rk::k_ssor_sweep<false><<<g, rk::kSsorThreads, 0, s>>>(A.n, A.rowptr, A.col, A.val, dw, d, r, u, flags, epoch,
                                                         counters, st, r_even, order_fwd);
  note_launch();
  rk::k_ssor_sweep<true><<<g, rk::kSsorThreads, 0, s>>>(A.n, A.rowptr, A.col, A.val, dw, d, u, z, flags + A.n,
                                                        epoch, counters + 1, st, nullptr, order_bwd);
  note_launch();
  return cuda_check("rk_ssor_apply");
}

}  // namespace rkh
