// Shared device helpers: deterministic warp/block/grid reductions, error plumbing.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <utility>

#include "../../include/podcg.h"

namespace rk {

constexpr int kWarp = 32;
constexpr unsigned kFull = 0xffffffffu;

// Xor butterfly: every lane ends with the bitwise-identical sum.
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
  return v;
}

// N independent butterflies interleaved level by level (ILP across the N
// values); each result is bitwise what warp_sum gives for that value.
template <int N>
__device__ __forceinline__ void warp_sum_n(double (&v)[N]) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    double t[N];
#pragma unroll
    for (int q = 0; q < N; ++q) t[q] = __shfl_xor_sync(kFull, v[q], o);
#pragma unroll
    for (int q = 0; q < N; ++q) v[q] += t[q];
  }
}

// Release/acquire fence at GPU scope (cheaper than __threadfence's fence.sc):
// orders this thread's (and, after a barrier, its block's) prior writes before
// a following ticket atomic, and the ticket before later reads.
// Row-sum step of every SpMV / SpMM kernel: a separately rounded multiply and
// add, entries in CSR order, so a SELL row sum is scipy's csr_matvec loop
// `sum += Ax[jj] * Xx[Aj[jj]]` (linalg.py:148) bit for bit. Measured at full
// C3 size against the reference: with fused multiply-adds the first system
// took 746 iterations instead of the reference's 748 (x off by 4.5e-8); with
// the scipy arithmetic 748 (x within 1.3e-9), at no cost in a memory-bound
// kernel. RK_SPMV_FMA=1 builds the fused variant.
#ifndef RK_SPMV_FMA
#define RK_SPMV_FMA 0
#endif
__device__ __forceinline__ double row_madd(double a, double b, double s) {
#if RK_SPMV_FMA
  return fma(a, b, s);
#else
  return __dadd_rn(s, __dmul_rn(a, b));
#endif
}

// Breakdown test and step length of one iteration (krylov.py:302-305); run by
// the single last block once gamma = p'Ap and p'p are known.
__device__ __forceinline__ void curvature_epilogue(const rk_pcg_plan& P, double gamma, double pp) {
  rk_pcg_state* st = P.st;
  const int64_t k = st->k;
  st->gamma = gamma;
  st->pp = pp;
  // krylov.py:303  `not isfinite(gamma) or gamma <= 1e-14 * (p @ p)`
  if (!isfinite(gamma) || gamma <= 1e-14 * pp) {
    st->status = 2;
    st->bd_iter = k;
    st->done = 1;
    return;
  }
  const double alpha = st->rz / gamma;
  st->alpha = alpha;
  P.alpha_h[k] = alpha;
  P.gamma_h[k] = gamma;
  P.rz_h[k] = st->rz;
}

__device__ __forceinline__ void fence_acq_rel_gpu() { asm volatile("fence.acq_rel.gpu;\n" ::: "memory"); }

// Block-wide sum of NV values; result valid in every thread. scratch >= 32*NV.
template <int NV>
__device__ __forceinline__ void block_sum(double (&v)[NV], double* scratch) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nw = (blockDim.x + 31) >> 5;
#pragma unroll
  for (int j = 0; j < NV; ++j) v[j] = warp_sum(v[j]);
  __syncthreads();  // scratch may still be read by a previous call
  if (lane == 0) {
#pragma unroll
    for (int j = 0; j < NV; ++j) scratch[j * 32 + warp] = v[j];
  }
  __syncthreads();
#pragma unroll
  for (int j = 0; j < NV; ++j) {
    double t = (lane < nw) ? scratch[j * 32 + lane] : 0.0;
    v[j] = warp_sum(t);
  }
}

// Publish this block's partials and find out whether it is the last block to
// finish. partials is [gridDim.x][nv]; the ticket is reset by the last block.
// Release/acquire at GPU scope by thread 0 around the ticket (the barrier
// orders the block's writes before the release).
__device__ __forceinline__ bool publish_and_check_last(const double* vals, int nv,
                                                       double* partials, uint32_t* ticket) {
  __shared__ bool s_last;
  for (int j = threadIdx.x; j < nv; j += blockDim.x)
    partials[(int64_t)blockIdx.x * nv + j] = vals[j];
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("fence.acq_rel.gpu;\n" ::: "memory");
    uint32_t t = atomicAdd(ticket, 1u);
    s_last = (t == gridDim.x - 1);
    if (s_last) {
      *ticket = 0u;
      asm volatile("fence.acq_rel.gpu;\n" ::: "memory");
    }
  }
  __syncthreads();
  return s_last;
}

// Last block: out[j] = sum over blocks (fixed order) of partials[b][j], j < nv.
// One warp per value, lanes stride over blocks, then a butterfly: deterministic.
// (A block-parallel variant measured slower inside the SpMV: kept simple.)
__device__ __forceinline__ void combine_partials(const double* partials, int nb, int nv,
                                                 double* out) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nw = blockDim.x >> 5;
  for (int j = warp; j < nv; j += nw) {
    double acc = 0.0;
    for (int b = lane; b < nb; b += 32) acc += __ldcg(partials + (int64_t)b * nv + j);
    acc = warp_sum(acc);
    if (lane == 0) out[j] = acc;
  }
  __syncthreads();
}

// Programmatic dependent launch (sm_90+): a kernel launched with programmatic
// stream serialisation may start while its predecessor drains; it must wait
// for the predecessor's completion (and memory) before touching its outputs,
// and lets its own dependents launch early. Both are no-ops without PDL.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;\n" :::); }

// Marks a ticket-synchronised completion without data (used to advance state).
__device__ __forceinline__ bool ticket_last(uint32_t* ticket) {
  __shared__ bool s_last;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    uint32_t t = atomicAdd(ticket, 1u);
    s_last = (t == gridDim.x - 1);
    if (s_last) *ticket = 0u;
  }
  __syncthreads();
  return s_last;
}

}  // namespace rk

// Host-side helpers shared by the launchers.
namespace rkh {
void set_error(const char* fmt, ...);
void note_launch();  // process-wide count of kernels launched (rk_launch_count)
int cuda_check(const char* where);
int sm_count();
inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }
bool pdl_enabled();  // RK_PDL=0 disables programmatic dependent launch

// Launch with programmatic stream serialisation (the kernel must call
// rk::pdl_wait() before reading its predecessor's results).
template <typename... KArgs, typename... Args>
inline void launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                       Args&&... args) {
  if (pdl_enabled()) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
  } else {
    kern<<<grid, block, smem, s>>>(std::forward<Args>(args)...);
  }
  note_launch();
}
}  // namespace rkh

#define RK_REQUIRE(cond, code, ...)      \
  do {                                   \
    if (!(cond)) {                       \
      rkh::set_error(__VA_ARGS__);       \
      return (code);                     \
    }                                    \
  } while (0)
