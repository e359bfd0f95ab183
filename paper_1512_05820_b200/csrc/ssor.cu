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
                                                             unsigned int* counter) {
  const int lane = threadIdx.x & 31;
  for (;;) {
    unsigned int t = 0;
    if (lane == 0) t = atomicAdd(counter, 1u);
    t = __shfl_sync(kFull, t, 0);
    if ((int64_t)t >= n) break;
    const int64_t i = UPPER ? n - 1 - (int64_t)t : (int64_t)t;
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

}  // namespace rk

namespace rkh {

int launch_ssor_apply(const rk_csr& A, const double* dw, const double* d, const double* r, double* z, double* u,
                      int* flags, unsigned int* counters, int epoch, cudaStream_t s) {
  if (A.n <= 0) return 0;
  static const int grid = [] {
    int occ = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, rk::k_ssor_sweep<false>, rk::kSsorThreads, 0) !=
            cudaSuccess || occ < 1)
      occ = 1;
    return occ * sm_count();
  }();
  const int g = (int)std::max<int64_t>(1, std::min<int64_t>(grid, (A.n + 7) / 8));
  cudaMemsetAsync(counters, 0, 2 * sizeof(unsigned int), s);
  rk::k_ssor_sweep<false><<<g, rk::kSsorThreads, 0, s>>>(A.n, A.rowptr, A.col, A.val, dw, d, r, u, flags, epoch,
                                                         counters);
  note_launch();
  rk::k_ssor_sweep<true><<<g, rk::kSsorThreads, 0, s>>>(A.n, A.rowptr, A.col, A.val, dw, d, u, z, flags + A.n,
                                                        epoch, counters + 1);
  note_launch();
  return cuda_check("rk_ssor_apply");
}

}  // namespace rkh
