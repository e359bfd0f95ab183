// FP64 tensor-core (DMMA) contractions for the POD truncation:
//   K7  G = X' Y            snapshot Gram S'(AS), W'(AW), Y'(AW)   (linalg.py:174,
//                           krylov.py:152, threestage.py:320, pod.py:119)
//   K8  Out = S C           basis reconstruction S @ coef          (pod.py:91-93)
//
// tcgen05 has no f64 kind, so the fp64 tensor path on sm_100a is the warp-level
// DMMA (mma.sync.m8n8k4.f64, SASS DMMA.8x8x4). K7 stages its operand panels
// with TMA (cp.async.bulk.tensor.2d, SASS UTMALDG; 128-byte swizzle, so the
// dense 16-row boxes are read without bank conflicts) issued by one producer
// warp into an mbarrier full/empty ring that the DMMA warps consume without
// block barriers; it runs over work units of (tile, row range) balanced by
// issued DMMAs (see below). K8 gives each CTA a 64 x 64 output tile computed
// by 4 warps of 32 x 32 from a cp.async ring.
#include <cuda.h>  // CUtensorMap and its enums only; the encoder is fetched from the driver at run time

#include <algorithm>
#include <vector>

#include "common.cuh"

namespace rk {

constexpr int kTile = 64;
constexpr int kStep = 16;             // K rows per pipeline stage
#ifndef RK_GRAM_STAGES
#define RK_GRAM_STAGES 4
#endif
#ifndef RK_GRAM_MINB
#define RK_GRAM_MINB 2
#endif
constexpr int kStages = RK_GRAM_STAGES;
constexpr int kPadK = kStep + 4;      // 20 doubles: conflict-free 8-byte fragment loads
constexpr int kPadM = kTile + 4;      // 68 doubles: conflict-free for the S tile of K8
constexpr int kDmmaThreads = 128;

__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gsrc, int src_bytes) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(d), "l"(gsrc), "r"(src_bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// --------------------------------------------------------------------------
// K7: G = X' Y over work units.
//
// A unit is (tile a, tile b, row range [k0, k1)). Every unit carries about the
// same number of ISSUED DMMAs: a warp issues only the 8 x 8 fragments of its
// WM x WN block that hold at least one wanted entry (inside m1 x m2 and, in
// upper mode, not strictly below the diagonal of the enclosing symmetric
// matrix), and the host gives each tile a number of row splits proportional
// to its active fragments. So the narrow last tile row / column of a width
// that is not a multiple of the tile (C2: m = 386 = 6 x 64 + 2) and the
// diagonal tiles of a triangle cost what they compute instead of a full tile,
// and no SM idles behind a light tile. Units with a tile to themselves write
// G directly; split tiles write dense BM x BN partials that k_gram_reduce
// sums in a fixed order (no fp64 atomics: deterministic).
//
// Templated on the CTA tile (BM x BN) and the warp tile (WM x WN). Per K step
// of 4 a warp issues WM/8 + WN/8 fragment loads for (WM/8)(WN/8) DMMAs and the
// CTA stages (BM + BN) x 16 doubles per 2 BM BN 16 flops, so the 128 x 64 tile
// moves 3/4 of the L2 -> SM bytes per flop of the 64 x 64 one.
// --------------------------------------------------------------------------
constexpr int kMaxUnits = 2048;
constexpr int kMaxTiles = 2048;
constexpr int kChunk = 32;  // unit row ranges are multiples of 32 rows

// Unit table passed by value in kernel parameter space (no device allocation,
// capturable in graphs, re-entrant). u = a | b << 11 | direct << 22 |
// k0 / 32 << 23 | k1 / 32 << 43; slot = partial index of a split tile.
struct GramUnits {
  uint64_t u[kMaxUnits];
  uint16_t slot[kMaxUnits];
};
struct GramTiles {  // split tiles for the reduce: a | b << 11, first slot, count
  uint32_t ab[kMaxTiles];
  uint16_t first[kMaxTiles];
  uint16_t count[kMaxTiles];
};

// ---- warp shapes of K7 -------------------------------------------------------
// A warp owns FA x FB fragments of 8 x 8. Its shape code says which of them to
// issue: 0 none; 1 .. FA*FB the leading RA x CB rectangle (the edge of a width
// that is not a multiple of 8 fragments); FA*FB + 1 .. the upper staircase
// i <= j + S (a warp on the diagonal of a symmetric Gram), S in [1 - FB, FA - 2].
constexpr int kNoStair = 1 << 20;

template <int FA, int FB>
constexpr int kFullShape = FA * FB;  // RA = FA, CB = FB

__host__ __device__ __forceinline__ int warp_shape_code(int FA, int FB, int64_t r0, int64_t c0, int64_t m1,
                                                        int64_t m2, int64_t upper_off) {
  if (r0 >= m1 || c0 >= m2) return 0;
  if (upper_off >= 0) {
    // fragment (i, j) wanted iff r0 + 8i <= c0 + 8j + off + 7, i.e. i <= j + S
    const int64_t d = c0 + upper_off + 7 - r0;
    const int64_t S = d >= 0 ? d / 8 : -((-d + 7) / 8);
    if (S < 1 - FB) return 0;                // strictly below the diagonal
    if (S <= FA - 2) return FA * FB + 1 + (int)(S + FB - 1);
  }
  const int64_t ra = (m1 - r0 + 7) / 8, cb = (m2 - c0 + 7) / 8;
  const int RA = (int)(ra < FA ? ra : FA), CB = (int)(cb < FB ? cb : FB);
  return (RA - 1) * FB + CB;
}

// DMMAs a warp of this shape issues per K step of 4 (host cost model)
static inline int shape_frags(int FA, int FB, int code) {
  if (code == 0) return 0;
  if (code <= FA * FB) return ((code - 1) / FB + 1) * ((code - 1) % FB + 1);
  const int S = code - FA * FB - 1 - (FB - 1);
  int c = 0;
  for (int i = 0; i < FA; ++i)
    for (int j = 0; j < FB; ++j) c += i <= j + S;
  return c;
}

// Fixed-order sum of a split tile's partials: G[a0 + r, b0 + c] = sum_q
// ws[first + q][r + c BM]. blockIdx.x = split tile, blockIdx.y = one of
// gridDim.y interleaved shares of its entries (a C3 truncation Gram has 55
// split tiles: one CTA per tile left two thirds of the SMs idle and took
// 0.7 ms for 57 MB of partials).
template <int BM, int BN>
__global__ void __launch_bounds__(256) k_gram_reduce(int64_t m1, int64_t m2, const double* __restrict__ ws,
                                                     double* __restrict__ G, int64_t ldg,
                                                     const __grid_constant__ GramTiles T) {
  const uint32_t ab = T.ab[blockIdx.x];
  const int64_t a0 = (int64_t)(ab & 2047u) * BM, b0 = (int64_t)((ab >> 11) & 2047u) * BN;
  const double* p = ws + (int64_t)T.first[blockIdx.x] * (BM * BN);
  const int cnt = T.count[blockIdx.x];
  for (int e = blockIdx.y * blockDim.x + threadIdx.x; e < BM * BN; e += blockDim.x * gridDim.y) {
    const int r = e % BM, c = e / BM;
    if (a0 + r >= m1 || b0 + c >= m2) continue;
    double s = 0.0;
    for (int q = 0; q < cnt; ++q) s += __ldcs(p + (int64_t)q * (BM * BN) + e);
    G[(a0 + r) + (b0 + c) * ldg] = s;
  }
}

// --------------------------------------------------------------------------
// K7 with TMA staging. Per stage the producer (lane 0 of warp 0) arms
// full[stage] with the box bytes and issues two cp.async.bulk.tensor.2d loads:
// 16 rows x BM columns of X and 16 rows x BN columns of Y (or Y2). A box lands
// dense, one 128-byte line per column, XOR-swizzled in 16-byte chunks by the
// line index mod 8 (CU_TENSOR_MAP_SWIZZLE_128B), so the 8 columns x 4 rows an
// 8 x 4 fragment load touches fall in 32 distinct banks per half warp: two
// wavefronts per 256-byte fragment, the minimum. Rows past n and columns past
// the map's extent arrive as zeros (TMA out-of-bounds fill): no predicates.
// The right operand may live in two buffers (columns [0, c1) in Y, [c1, m2)
// in Y2): a tile on one side takes one box from that buffer's map; the one
// tile that straddles c1 takes a (c1 - b0)-column box of Y and a (b0 + BN -
// c1)-column box of Y2 from two maps encoded with those box widths -- the
// swizzle is a function of the shared-memory address, so a box that starts
// at any 128-byte line lands in the same pattern.
// Each warp waits on full[stage] and issues its fragments' DMMAs; it releases
// a stage (one lane arrives on empty[stage]) only after the full-wait of the
// NEXT step, and the producer then refills that stage once all warps have
// left it (STAGES - 1 steps ahead of the consumers). No block barrier in the
// K loop. The deferred release matters: ptxas gives mbarrier.arrive no
// scoreboard wait on earlier ld.shared, so an arrive placed right after a
// step's DMMAs is hoisted to just behind the step's last LDS *issue*, the
// producer's next box can land before those loads have read the stage, and a
// few lines of one fragment come back from the wrong K step (measured: one
// wrong 16-row step in ~1e5, scripts/gram_stress.py). Behind the spin loop of
// the next wait, every DMMA of the step -- hence every load feeding it -- has
// issued. (A fifth, producer-only warp
// was tried first: 15 warps per SM put 4 on one sub-partition, which caps the
// kernel at 128 registers per thread and spills the 128 x 64 tile.)
// --------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  uint32_t ok;
  do {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        "selp.u32 %0, 1, 0, p;\n"
        "}\n"
        : "=r"(ok)
        : "r"(bar), "r"(parity)
        : "memory");
  } while (!ok);
}
__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, uint32_t bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];\n" ::"r"(dst),
      "l"(map), "r"(bar), "r"(c0), "r"(c1)
      : "memory");
}

constexpr int kLine = kStep * 8;  // bytes of one staged column: 16 rows

// One K step of a warp from a swizzled stage: xs / ys are the warp's first
// line, koff[kq] this lane's byte offset within a group of 8 lines.
template <int FA, int FB, int RA, int CB, int S>
__device__ __forceinline__ void warp_step_sw(double (&acc)[FA][FB][2], const unsigned char* xs,
                                             const unsigned char* ys, const uint32_t (&koff)[kStep / 4]) {
#pragma unroll
  for (int kq = 0; kq < kStep / 4; ++kq) {
    double af[RA], bf[CB];
#pragma unroll
    for (int i = 0; i < RA; ++i) af[i] = *reinterpret_cast<const double*>(xs + i * 8 * kLine + koff[kq]);
#pragma unroll
    for (int j = 0; j < CB; ++j) bf[j] = *reinterpret_cast<const double*>(ys + j * 8 * kLine + koff[kq]);
#pragma unroll
    for (int i = 0; i < RA; ++i)
#pragma unroll
      for (int j = 0; j < CB; ++j)
        if (i <= j + S) dmma884(acc[i][j][0], acc[i][j][1], af[i], bf[j]);  // compile-time test
  }
}

template <int FA, int FB, int C>
__device__ __forceinline__ void warp_step_sw_dispatch(int code, double (&acc)[FA][FB][2], const unsigned char* xs,
                                                      const unsigned char* ys, const uint32_t (&koff)[kStep / 4]) {
  if constexpr (C <= FA * FB) {
    if (code == C) {
      warp_step_sw<FA, FB, (C - 1) / FB + 1, (C - 1) % FB + 1, kNoStair>(acc, xs, ys, koff);
      return;
    }
    warp_step_sw_dispatch<FA, FB, C + 1>(code, acc, xs, ys, koff);
  } else if constexpr (C <= FA * FB + FA + FB - 2) {
    if (code == C) {
      warp_step_sw<FA, FB, FA, FB, C - FA * FB - 1 - (FB - 1)>(acc, xs, ys, koff);
      return;
    }
    warp_step_sw_dispatch<FA, FB, C + 1>(code, acc, xs, ys, koff);
  }
}

template <int BM, int BN, int WM, int WN, int MINB, int STAGES>
__global__ void __launch_bounds__((BM / WM) * (BN / WN) * 32, MINB)
    k_gram_tma(int64_t n, int64_t m1, int64_t m2, int64_t c1, double* __restrict__ G, int64_t ldg,
               double* __restrict__ ws, int64_t upper_off, const __grid_constant__ CUtensorMap mapx,
               const __grid_constant__ CUtensorMap mapy, const __grid_constant__ CUtensorMap mapy2,
               const __grid_constant__ CUtensorMap mapya, const __grid_constant__ CUtensorMap mapyb,
               const __grid_constant__ GramUnits U) {
  constexpr int NW = (BM / WM) * (BN / WN);
  constexpr int FA = WM / 8, FB = WN / 8;
  constexpr uint32_t kXBytes = BM * kLine, kYBytes = BN * kLine, kStageBytes = kXBytes + kYBytes;
  static_assert(kXBytes % 1024 == 0 && kYBytes % 1024 == 0, "boxes keep the 1024-byte swizzle period");
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;           // swizzle period alignment
  const unsigned char* sbase = smem_raw + (base - raw);
  const uint32_t bars = base + STAGES * kStageBytes;       // full[STAGES], empty[STAGES]

  const uint64_t unit = U.u[blockIdx.x];
  const int64_t a0 = (int64_t)(unit & 2047u) * BM, b0 = (int64_t)((unit >> 11) & 2047u) * BN;
  const bool direct = (unit >> 22) & 1u;
  const int64_t kbeg = (int64_t)((unit >> 23) & 0xFFFFFu) * kChunk;
  const int64_t kend = min(n, (int64_t)((unit >> 43) & 0xFFFFFu) * kChunk);
  const int nsteps = kend > kbeg ? (int)((kend - kbeg + kStep - 1) / kStep) : 0;

  if (threadIdx.x == 0) {
#pragma unroll
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(bars + 8 * s, 1);              // the producer's arrive + the boxes' bytes
      mbar_init(bars + 8 * (STAGES + s), NW);  // one lane of every warp
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const bool producer = threadIdx.x == 0;
  // source of the Y box: 0 all in Y, 1 all in Y2, 2 straddling c1
  const int ysrc = (b0 + BN <= c1 || c1 >= m2) ? 0 : (b0 >= c1 ? 1 : 2);
  const uint32_t w1 = ysrc == 2 ? (uint32_t)(c1 - b0) : 0u;  // lines of the straddling tile that come from Y
  auto produce = [&](int step) {  // producer thread only: refill the stage of `step`
    const int stg = step % STAGES, round = step / STAGES;
    if (round > 0) mbar_wait(bars + 8 * (STAGES + stg), (round - 1) & 1);
    const uint32_t full = bars + 8 * stg;
    mbar_expect_tx(full, kStageBytes);
    const int krow = (int)(kbeg + (int64_t)step * kStep);
    tma_load_2d(base + stg * kStageBytes, &mapx, full, krow, (int)a0);
    const uint32_t ydst = base + stg * kStageBytes + kXBytes;
    if (ysrc == 0) {
      tma_load_2d(ydst, &mapy, full, krow, (int)b0);
    } else if (ysrc == 1) {
      tma_load_2d(ydst, &mapy2, full, krow, (int)(b0 - c1));
    } else {
      tma_load_2d(ydst, &mapya, full, krow, (int)b0);
      tma_load_2d(ydst + w1 * kLine, &mapyb, full, krow, 0);
    }
  };
  if (producer)
    for (int st = 0; st < STAGES - 1 && st < nsteps; ++st) produce(st);

  const int g = lane >> 2, t = lane & 3;
  const int wa = (warp % (BM / WM)) * WM, wb = (warp / (BM / WM)) * WN;
  uint32_t koff[kStep / 4];
#pragma unroll
  for (int kq = 0; kq < kStep / 4; ++kq)
    koff[kq] = (uint32_t)(g * kLine + ((((kq << 1) | (t >> 1)) ^ g) << 4) + ((t & 1) << 3));
  const int code = warp_shape_code(FA, FB, a0 + wa, b0 + wb, m1, m2, upper_off);
  double acc[FA][FB][2];
#pragma unroll
  for (int i = 0; i < FA; ++i)
#pragma unroll
    for (int j = 0; j < FB; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  const unsigned char* xw = sbase + wa * kLine;
  const unsigned char* yw = sbase + kXBytes + wb * kLine;
  // Step prologue shared by both loops: wait for the step's boxes, release
  // the previous step's stage, let the producer refill it.
  auto next_stage = [&](int step) {
    const int stg = step % STAGES;
    mbar_wait(bars + 8 * stg, (step / STAGES) & 1);
    if (step > 0) {
      __syncwarp();
      if (lane == 0) mbar_arrive(bars + 8 * (STAGES + (step - 1) % STAGES));
    }
    if (producer && step + STAGES - 1 < nsteps) produce(step + STAGES - 1);
    return stg * kStageBytes;
  };
  if (code == kFullShape<FA, FB>) {
    for (int step = 0; step < nsteps; ++step) {
      const uint32_t so = next_stage(step);
      warp_step_sw<FA, FB, FA, FB, kNoStair>(acc, xw + so, yw + so, koff);
    }
  } else {
    for (int step = 0; step < nsteps; ++step) {
      const uint32_t so = next_stage(step);
      if (code != 0) warp_step_sw_dispatch<FA, FB, 1>(code, acc, xw + so, yw + so, koff);
    }
  }

  if (direct) {
#pragma unroll
    for (int i = 0; i < FA; ++i) {
      const int64_t ga = a0 + wa + i * 8 + g;
#pragma unroll
      for (int j = 0; j < FB; ++j) {
        const int64_t gb = b0 + wb + j * 8 + 2 * t;
        if (ga < m1) {
          if (gb < m2) G[ga + gb * ldg] = acc[i][j][0];
          if (gb + 1 < m2) G[ga + (gb + 1) * ldg] = acc[i][j][1];
        }
      }
    }
  } else {
    // dense BM x BN partial (column-major, ld BM); inactive fragments are zeros
    double* o = ws + (int64_t)U.slot[blockIdx.x] * (BM * BN);
#pragma unroll
    for (int i = 0; i < FA; ++i) {
      const int la = wa + i * 8 + g;
#pragma unroll
      for (int j = 0; j < FB; ++j) {
        const int lb = wb + j * 8 + 2 * t;
        o[la + lb * BM] = acc[i][j][0];
        o[la + (lb + 1) * BM] = acc[i][j][1];
      }
    }
  }
}

// --------------------------------------------------------------------------
// K8: Out[i0:i0+64, c0:c0+64] = S[i0:i0+64, :] C[:, c0:c0+64]
// --------------------------------------------------------------------------
__global__ void __launch_bounds__(kDmmaThreads, 2)
    k_gemm_nn(int64_t n, int64_t s, int64_t y, const double* __restrict__ S, int64_t lds,
              const double* __restrict__ C, int64_t ldc, double* __restrict__ Out, int64_t ldo) {
  extern __shared__ __align__(16) double smem[];
  double* Ss = smem;                                  // [stage][k][kPadM]  (rows contiguous)
  double* Cs = smem + kStages * kStep * kPadM;        // [stage][c][kPadK]  (k contiguous)
  const int64_t i0 = (int64_t)blockIdx.x * kTile;
  const int64_t c0 = (int64_t)blockIdx.y * kTile;
  const int nsteps = (int)((s + kStep - 1) / kStep);

  // Fixed per-thread chunks (as in K7): S rows i0 + 2 sch of columns
  // kc0 + 4 i, and C columns c0 + cc0 + 16 i at rows 2 cch; only the K offset
  // changes per step.
  constexpr int LS = kStep * (kTile / 2) / kDmmaThreads, LC = kTile * (kStep / 2) / kDmmaThreads;
  const int sch = threadIdx.x % (kTile / 2), kc0 = threadIdx.x / (kTile / 2);
  const int cch = threadIdx.x % (kStep / 2), cc0 = threadIdx.x / (kStep / 2);
  const int64_t srow = i0 + 2 * sch;
  const int srb = srow < n ? (srow + 1 < n ? 16 : 8) : 0;
  const double* sbase = S + (int64_t)kc0 * lds + srow;
  const double* cbase[LC];
#pragma unroll
  for (int i = 0; i < LC; ++i) {
    const int64_t col = c0 + cc0 + i * (kDmmaThreads / (kStep / 2));
    cbase[i] = col < y ? C + col * ldc + 2 * cch : nullptr;
  }
  auto load_stage = [&](int stage, int step) {
    const int64_t k0 = (int64_t)step * kStep;
#pragma unroll
    for (int i = 0; i < LS; ++i) {
      const int kc = kc0 + i * (kDmmaThreads / (kTile / 2));
      const int rb = k0 + kc < s ? srb : 0;
      cp_async16(Ss + (stage * kStep + kc) * kPadM + 2 * sch,
                 rb ? (const void*)(sbase + (k0 + i * (kDmmaThreads / (kTile / 2))) * lds) : (const void*)S, rb);
    }
    const int64_t crow = k0 + 2 * cch;
    const int crb = crow < s ? (crow + 1 < s ? 16 : 8) : 0;
#pragma unroll
    for (int i = 0; i < LC; ++i) {
      const int cc = cc0 + i * (kDmmaThreads / (kStep / 2));
      const bool ok = cbase[i] != nullptr && crb > 0;
      cp_async16(Cs + (stage * kTile + cc) * kPadK + 2 * cch, ok ? (const void*)(cbase[i] + k0) : (const void*)C,
                 ok ? crb : 0);
    }
  };

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int wi = (warp & 1) * 32, wc = (warp >> 1) * 32;
  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

#pragma unroll
  for (int st = 0; st < kStages - 1; ++st) {
    if (st < nsteps) load_stage(st, st);
    cp_async_commit();
  }
  for (int step = 0; step < nsteps; ++step) {
    cp_async_wait<kStages - 2>();
    __syncthreads();
    const int nxt = step + kStages - 1;
    if (nxt < nsteps) load_stage(nxt % kStages, nxt);
    cp_async_commit();
    const int stg = step % kStages;
    const double* ss = Ss + (stg * kStep) * kPadM;
    const double* cs = Cs + (stg * kTile) * kPadK;
#pragma unroll
    for (int kq = 0; kq < kStep / 4; ++kq) {
      double af[4], bf[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) af[i] = ss[(kq * 4 + t) * kPadM + wi + i * 8 + g];
#pragma unroll
      for (int j = 0; j < 4; ++j) bf[j] = cs[(wc + j * 8 + g) * kPadK + kq * 4 + t];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma884(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
  }
  cp_async_wait<0>();

#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t gi = i0 + wi + i * 8 + g;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t gc = c0 + wc + j * 8 + 2 * t;
      if (gi < n) {
        if (gc < y) Out[gi + gc * ldo] = acc[i][j][0];
        if (gc + 1 < y) Out[gi + (gc + 1) * ldo] = acc[i][j][1];
      }
    }
  }
}

}  // namespace rk

namespace rkh {

static size_t gemm_smem() {
  return (size_t)(rk::kStages * rk::kStep * rk::kPadM + rk::kStages * rk::kTile * rk::kPadK) * sizeof(double);
}

// One instantiation of the templated K7 with its launch shape and measured
// residency (CTAs per SM at its register / shared-memory footprint).
typedef void (*GramTmaFn)(int64_t, int64_t, int64_t, int64_t, double*, int64_t, double*, int64_t, const CUtensorMap,
                          const CUtensorMap, const CUtensorMap, const CUtensorMap, const CUtensorMap,
                          const rk::GramUnits);
struct GramVariant {
  GramTmaFn fn;
  void (*reduce)(int64_t, int64_t, const double*, double*, int64_t, const rk::GramTiles);
  int bm, bn, wm, wn, threads;
  size_t smem;
  int64_t per_sm;
};

template <int BM, int BN, int WM, int WN, int MINB, int STAGES>
static GramVariant make_variant() {
  GramVariant v;
  v.fn = rk::k_gram_tma<BM, BN, WM, WN, MINB, STAGES>;
  v.reduce = rk::k_gram_reduce<BM, BN>;
  v.bm = BM;
  v.bn = BN;
  v.wm = WM;
  v.wn = WN;
  v.threads = (BM / WM) * (BN / WN) * 32;
  // stages, 1024 bytes of alignment slack (swizzle period), the full / empty barriers
  v.smem = (size_t)STAGES * (BM + BN) * rk::kLine + 1024 + 2 * STAGES * sizeof(uint64_t);
  cudaFuncSetAttribute(v.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)v.smem);
  int occ = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, v.fn, v.threads, v.smem) != cudaSuccess || occ < 1) occ = 1;
  v.per_sm = occ;
  return v;
}

// 0: 64 x 64 CTA tile, 4 warps of 32 x 32 (2 CTAs / SM)
// 1: 128 x 64, 4 warps of 64 x 32 (2 CTAs / SM): full Grams
// 2: 64 x 64 (3 CTAs / SM)
// 3: 64 x 80, 4 warps of 32 x 40 (3 CTAs / SM)
// 4: 64 x 48, 4 warps of 32 x 24 (3 CTAs / SM)
// 2-4 differ only in the tile width, so a width that leaves a sliver past
// the last multiple of 64 (C2's truncation Gram: 386 = 6 x 64 + 2) can take
// a width whose last tile column is mostly full (386 = 4 x 80 + 66).
constexpr int kVariants = 5;
static const GramVariant& gram_variant(int which) {
  static const GramVariant v0 = make_variant<64, 64, 32, 32, RK_GRAM_MINB, rk::kStages>();
  static const GramVariant v1 = make_variant<128, 64, 64, 32, 2, 4>();
  static const GramVariant v2 = make_variant<64, 64, 32, 32, 3, 4>();
  static const GramVariant v3 = make_variant<64, 80, 32, 40, 3, 3>();
  static const GramVariant v4 = make_variant<64, 48, 32, 24, 3, 4>();
  switch (which) {
    case 1: return v1;
    case 2: return v2;
    case 3: return v3;
    case 4: return v4;
    default: return v0;
  }
}

// DMMAs per K step of 4 that the warps of tile (a, b) issue.
static int64_t tile_cost(const GramVariant& v, int64_t a, int64_t b, int64_t m1, int64_t m2, int64_t upper_off) {
  int64_t c = 0;
  const int fa = v.wm / 8, fb = v.wn / 8;
  for (int64_t wa = 0; wa < v.bm; wa += v.wm)
    for (int64_t wb = 0; wb < v.bn; wb += v.wn)
      c += rk::shape_frags(fa, fb, rk::warp_shape_code(fa, fb, a * v.bm + wa, b * v.bn + wb, m1, m2, upper_off));
  return c;
}

// Modelled slot time of a Gram with variant v and uniform row splits: every
// tile streams all n rows, a K step costing its issued DMMAs but at least
// half of a full tile's (a step of a light tile still waits for its panels).
static double model_cost(const GramVariant& v, int64_t m1, int64_t m2, int64_t upper_off) {
  const int64_t ta = (m1 + v.bm - 1) / v.bm, tb = (m2 + v.bn - 1) / v.bn;
  const double full = (double)(v.bm / 8) * (v.bn / 8);
  double t = 0.0;
  for (int64_t b = 0; b < tb; ++b)
    for (int64_t a = 0; a < ta; ++a) {
      const int64_t c = tile_cost(v, a, b, m1, m2, upper_off);
      if (c) t += std::max((double)c, 0.5 * full);
    }
  return t;
}

// Work plan of one Gram: variant, units (launch order) and split tiles.
struct GramPlan {
  int which = 0;
  int64_t ws_doubles = 0;
  std::vector<uint64_t> code;   // units in launch order (batched kMaxUnits per launch)
  std::vector<uint16_t> slot;
  std::vector<uint32_t> split_ab;  // split tiles for the reduce (batched kMaxTiles per launch)
  std::vector<uint16_t> split_first, split_count;
};

// Variant: full Grams at least 128 rows tall take 128 x 64 (fewer L2 -> SM
// bytes per flop: measured 0.91 of the DMMA peak at C5 against 0.89 for 64 x
// 64); otherwise the 64-row tile width (48 / 64 / 80) with the least modelled
// slot time. RK_GRAM_TILE=0..4 forces one.
static int forced_variant() {
  static const int forced = [] {
    const char* e = getenv("RK_GRAM_TILE");
    const int v = e ? atoi(e) : -1;
    return (v >= 0 && v < kVariants) ? v : -1;
  }();
  return forced;
}

static int pick_variant(int64_t m1, int64_t m2, int64_t upper_off) {
  if (forced_variant() >= 0) return forced_variant();
  if (upper_off < 0 && m1 >= 128 && m1 % 128 == 0 && m2 % 64 == 0) return 1;
  int best = 2;
  double best_cost = 0.0;
  for (int w : {2, 3, 4}) {
    const double c = model_cost(gram_variant(w), m1, m2, upper_off);  // in 8 x 8 fragments of G
    if (w == 2 || c < 0.98 * best_cost) {  // ties keep the 64-wide tile
      best = w;
      best_cost = c;
    }
  }
  return best;
}

// Split-K plan: the units of all tiles fill about `waves` (4) rounds of the
// resident CTA slots, each unit at least 512 rows. By default every tile gets
// the same row splits, so the CTAs that run together stream the same row
// band of X and Y (L2 reuse; measured 0.80 against 0.74 of the DMMA peak on
// the C3 truncation Gram for splits in proportion to a tile's DMMAs,
// RK_GRAM_UNIFORM=0). Units are launched by row band, tiles within a band.
// A width that leaves at most 16 columns past the last multiple of 64 (C2's
// truncation Gram: 386 = 6 x 64 + 2) would give the 64-wide tiling a last
// tile column whose every tile streams full panels for one or two fragment
// columns. Such a Gram runs as two launches: columns [0, cut) with 64-wide
// tiles and columns [cut, m2) -- 65 to 80 of them -- as one 80-wide tile
// column. 0: no cut (RK_GRAM_TAIL=0 disables it).
static int64_t tail_cut(int64_t m2) {
  static const bool on = [] {
    const char* e = getenv("RK_GRAM_TAIL");
    return e ? atoi(e) != 0 : true;
  }();
  const int64_t r = m2 % 64;
  if (!on || forced_variant() >= 0 || m2 < 128 || r == 0 || r > 16) return 0;
  return m2 - 64 - r;
}

// An upper-triangle Gram whose tiles come out 64 x 64 runs as two launches
// when enough of it lies off the diagonal: the 128 x 64 tiles wholly above the
// diagonal (all entries wanted: full-mode shapes), then 64 x 64 tiles for the
// band they leave. A 128 x 64 tile moves 3/4 of the L2 -> SM bytes per flop of
// a 64 x 64 one -- measured on full Grams, 0.95 against 0.90 of the DMMA peak
// -- and the triangle ran at the 64 x 64 rate times its useful fraction.
// filter 1 keeps tile (A, b) of the 128-row tiling iff A*128 + 127 <= b*64 +
// off; filter 2 drops tile (a, b) of the 64-row tiling iff tile (a / 2, b) was
// kept by filter 1. RK_GRAM_BAND=0 disables the split.
struct GramPart {
  int64_t shape_off;  // upper_off the kernel's warp shapes see (-1: every fragment)
  int force, filter;
  int64_t filter_off;
};

static bool above_band(int64_t A, int64_t b, int64_t off) { return A * 128 + 127 <= b * 64 + off; }

static int gram_parts(int64_t m1, int64_t m2, int64_t upper_off, int force, GramPart (&parts)[2]) {
  static const bool band = [] {
    const char* e = getenv("RK_GRAM_BAND");
    return e ? atoi(e) != 0 : true;
  }();
  const int which = force >= 0 ? force : pick_variant(m1, m2, upper_off);
  if (band && upper_off >= 0 && which == 2 && forced_variant() < 0) {
    int64_t above = 0;
    for (int64_t b = 0; b * 64 < m2; ++b)
      for (int64_t A = 0; A * 128 < m1; ++A) above += above_band(A, b, upper_off);
    if (above >= 6) {
      parts[0] = {-1, 1, 1, upper_off};
      parts[1] = {upper_off, 2, 2, upper_off};
      return 2;
    }
  }
  parts[0] = {upper_off, force, 0, 0};
  return 1;
}

// force: the variant to use, or -1 for the modelled choice. filter: see GramPart.
static int build_plan(int64_t n, int64_t m1, int64_t m2, int64_t upper_off, int force, GramPlan& P, int filter = 0,
                      int64_t filter_off = 0) {
  P.which = force >= 0 ? force : pick_variant(m1, m2, upper_off);
  const GramVariant& v = gram_variant(P.which);
  const int64_t ta = (m1 + v.bm - 1) / v.bm, tb = (m2 + v.bn - 1) / v.bn;
  RK_REQUIRE(ta <= 2048 && tb <= 2048, RK_ERR_DIMENSION, "rk_gram: too many columns (%lld x %lld)",
             (long long)m1, (long long)m2);
  const int64_t nchunk = (n + rk::kChunk - 1) / rk::kChunk;
  RK_REQUIRE(nchunk < (1 << 20), RK_ERR_DIMENSION, "rk_gram: too many rows (%lld)", (long long)n);
  struct Tile { int64_t a, b, cost, ns; };
  static thread_local std::vector<Tile> tiles;
  tiles.clear();
  int64_t total = 0;
  // A K step of a light tile is not free: it still waits for its operand
  // panels, so a unit of a tile with few active fragments is latency-bound.
  // Splits follow max(active, half of a full tile), which keeps such units
  // as short as the DMMA-bound ones (else they form the tail of the launch).
  const int64_t floor_cost = (v.bm / 8) * (v.bn / 8) / 2;
  for (int64_t b = 0; b < tb; ++b)
    for (int64_t a = 0; a < ta; ++a) {
      if (filter == 1 && !above_band(a, b, filter_off)) continue;
      if (filter == 2 && above_band(a / 2, b, filter_off)) continue;
      const int64_t c = tile_cost(v, a, b, m1, m2, upper_off);
      if (c) {
        tiles.push_back({a, b, std::max(c, floor_cost), 1});
        total += std::max(c, floor_cost);
      }
    }
  P.code.clear();
  P.slot.clear();
  P.split_ab.clear();
  P.split_first.clear();
  P.split_count.clear();
  P.ws_doubles = 0;
  if (tiles.empty()) return 0;
  const int64_t slots = (int64_t)sm_count() * v.per_sm;
  const int64_t max_split = std::max<int64_t>(1, nchunk / 16);  // >= 512 rows per unit
  static const int64_t waves = [] {
    const char* e = getenv("RK_GRAM_WAVES");
    return e ? std::max(1, atoi(e)) : 4;
  }();
  // Wide Grams (more tiles than `waves` rounds of slots) run one unit per
  // tile, in as many launches as the unit table needs; narrower ones split
  // the rows (partial slots are uint16).
  const int64_t target = std::max<int64_t>((int64_t)tiles.size(), std::min<int64_t>(waves * slots, 60000));
  static const bool uniform = [] {
    const char* e = getenv("RK_GRAM_UNIFORM");
    return e ? atoi(e) != 0 : true;
  }();
  const int64_t ns_u = std::min(max_split, std::max<int64_t>(1, target / (int64_t)tiles.size()));
  for (Tile& t : tiles)
    t.ns = uniform ? ns_u : std::min(max_split, std::max<int64_t>(1, (target * t.cost + total / 2) / total));
  // split tiles get partial slots (tile-major, so a tile's partials are contiguous)
  int64_t slot = 0;
  struct U { int64_t k0; uint64_t code; int64_t slot; };
  static thread_local std::vector<U> units;
  units.clear();
  for (const Tile& t : tiles) {
    const bool direct = t.ns == 1;
    if (!direct) {
      RK_REQUIRE(slot + t.ns <= 65535, RK_ERR_DIMENSION, "rk_gram: too many split units");
      P.split_ab.push_back((uint32_t)(t.a | (t.b << 11)));
      P.split_first.push_back((uint16_t)slot);
      P.split_count.push_back((uint16_t)t.ns);
    }
    for (int64_t q = 0; q < t.ns; ++q) {
      const int64_t k0 = nchunk * q / t.ns, k1 = nchunk * (q + 1) / t.ns;
      const uint64_t code = (uint64_t)t.a | ((uint64_t)t.b << 11) | ((uint64_t)direct << 22) | ((uint64_t)k0 << 23) |
                            ((uint64_t)k1 << 43);
      units.push_back({k0, code, direct ? 0 : slot++});
    }
  }
  std::stable_sort(units.begin(), units.end(), [](const U& x, const U& y) { return x.k0 < y.k0; });
  P.code.resize(units.size());
  P.slot.resize(units.size());
  for (size_t i = 0; i < units.size(); ++i) {
    P.code[i] = units[i].code;
    P.slot[i] = (uint16_t)units[i].slot;
  }
  P.ws_doubles = slot * v.bm * v.bn;
  return 0;
}

int64_t gram_workspace_doubles(int64_t n, int64_t m1, int64_t m2, int64_t upper_off) {
  if (m1 <= 0 || m2 <= 0) return 0;
  static thread_local GramPlan P;
  n = std::max<int64_t>(n, 1);
  // every launch of a Gram runs after the previous one on the stream: they share the workspace
  auto piece = [&](int64_t mm2, int64_t off, int force) -> int64_t {
    GramPart parts[2];
    const int np = gram_parts(m1, mm2, off, force, parts);
    int64_t need = 0;
    for (int i = 0; i < np; ++i) {
      if (build_plan(n, m1, mm2, parts[i].shape_off, parts[i].force, P, parts[i].filter, parts[i].filter_off) != 0)
        return 0;
      need = std::max(need, P.ws_doubles);
    }
    return need;
  };
  const int64_t cut = tail_cut(m2);
  if (cut > 0) return std::max(piece(cut, upper_off, 2), piece(m2 - cut, upper_off >= 0 ? upper_off + cut : -1, 3));
  return piece(m2, upper_off, -1);
}

static bool aligned16(const void* p) { return ((uintptr_t)p & 15u) == 0; }

// cuTensorMapEncodeTiled through the runtime's driver entry point lookup (no libcuda link).
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static EncodeTiledFn encode_tiled() {
  static const EncodeTiledFn fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q = cudaDriverEntryPointSymbolNotFound;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      p = nullptr;
    return (EncodeTiledFn)p;
  }();
  return fn;
}

// Map of a column-major fp64 panel: dimension 0 = rows (contiguous), dimension
// 1 = columns (stride ld); boxes of 16 rows x box_cols columns, 128-byte
// swizzle, zero fill outside [0, rows) x [0, cols).
static int panel_map(CUtensorMap* map, const double* base, int64_t rows, int64_t cols, int64_t ld, int box_cols) {
  const EncodeTiledFn enc = encode_tiled();
  RK_REQUIRE(enc != nullptr, RK_ERR_CUDA, "rk_gram: the driver has no cuTensorMapEncodeTiled");
  const cuuint64_t gdim[2] = {(cuuint64_t)rows, (cuuint64_t)std::max<int64_t>(cols, 1)};
  const cuuint64_t gstride[1] = {(cuuint64_t)ld * sizeof(double)};
  const cuuint32_t box[2] = {(cuuint32_t)rk::kStep, (cuuint32_t)box_cols};
  const cuuint32_t estride[2] = {1, 1};
  const CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(base), gdim, gstride, box, estride,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  RK_REQUIRE(r == CUDA_SUCCESS, RK_ERR_CUDA, "rk_gram: cuTensorMapEncodeTiled failed (%d)", (int)r);
  return 0;
}

static int launch_gram_one(int64_t n, int64_t m1, const double* X, int64_t ldx, int64_t m2, const double* Y,
                           int64_t ldy, const double* Y2, int64_t ldy2, int64_t c1, double* G, int64_t ldg, double* ws,
                           int64_t ws_len, int64_t upper_off, int force, cudaStream_t s);

int launch_gram(int64_t n, int64_t m1, const double* X, int64_t ldx, int64_t m2, const double* Y, int64_t ldy,
                const double* Y2, int64_t ldy2, int64_t c1, double* G, int64_t ldg, double* ws, int64_t ws_len,
                int64_t upper_off, cudaStream_t s) {
  if (m1 <= 0 || m2 <= 0) return 0;
  if (Y2 == nullptr || c1 >= m2) {
    Y2 = Y;
    ldy2 = ldy;
    c1 = m2;
  }
  const int64_t cut = tail_cut(m2);
  if (cut <= 0) return launch_gram_one(n, m1, X, ldx, m2, Y, ldy, Y2, ldy2, c1, G, ldg, ws, ws_len, upper_off, -1, s);
  // head: columns [0, cut), 64-wide tiles
  if (int e = launch_gram_one(n, m1, X, ldx, cut, Y, ldy, Y2, ldy2, std::min(c1, cut), G, ldg, ws, ws_len, upper_off, 2, s))
    return e;
  // tail: columns [cut, m2) as one 80-wide tile column; its first buffer is
  // whatever holds column `cut`, its boundary moves with it
  const double* Yt = c1 > cut ? Y + cut * ldy : Y2 + (cut - c1) * ldy2;
  const int64_t ldyt = c1 > cut ? ldy : ldy2;
  return launch_gram_one(n, m1, X, ldx, m2 - cut, Yt, ldyt, Y2, ldy2, std::max<int64_t>(c1 - cut, 0) == 0 ? m2 - cut : c1 - cut,
                         G + cut * ldg, ldg, ws, ws_len, upper_off >= 0 ? upper_off + cut : -1, 3, s);
}

static int launch_gram_one(int64_t n, int64_t m1, const double* X, int64_t ldx, int64_t m2, const double* Y,
                           int64_t ldy, const double* Y2, int64_t ldy2, int64_t c1, double* G, int64_t ldg, double* ws,
                           int64_t ws_len, int64_t upper_off, int force, cudaStream_t s) {
  if (Y2 == nullptr || c1 >= m2) {
    Y2 = Y;
    ldy2 = ldy;
    c1 = m2;
  }
  RK_REQUIRE(aligned16(X) && aligned16(Y) && aligned16(Y2) && (ldx % 2 == 0) && (ldy % 2 == 0) && (ldy2 % 2 == 0),
             RK_ERR_ARG, "rk_gram: operands need 16-byte aligned columns with even leading dimension");
  RK_REQUIRE(ldx >= n && ldy >= n && ldy2 >= n && ldg >= m1 && c1 >= 0, RK_ERR_DIMENSION,
             "rk_gram: leading dimension too small");
  static thread_local GramPlan P;  // per calling thread (re-entrant C-ABI)
  static thread_local rk::GramUnits U;  // kernel-parameter tables, ~20 KB: never on the stack
  static thread_local rk::GramTiles T;
  GramPart parts[2];
  const int nparts = gram_parts(m1, m2, upper_off, force, parts);
  for (int part = 0; part < nparts; ++part) {
  const int64_t shape_off = parts[part].shape_off;
  const int rc = build_plan(std::max<int64_t>(n, 1), m1, m2, shape_off, parts[part].force, P, parts[part].filter,
                            parts[part].filter_off);
  if (rc != 0) return rc;
  if (P.code.empty()) continue;
  RK_REQUIRE(P.ws_doubles == 0 || (ws && ws_len >= P.ws_doubles), RK_ERR_ARG,
             "rk_gram: workspace too small (%lld < %lld)", (long long)ws_len, (long long)P.ws_doubles);
  const GramVariant& v = gram_variant(P.which);
  CUtensorMap mx, my, my2, mya, myb;
  if (int e = panel_map(&mx, X, n, m1, ldx, v.bm)) return e;
  if (int e = panel_map(&my, Y, n, c1, ldy, v.bn)) return e;
  if (int e = panel_map(&my2, Y2, n, m2 - c1, ldy2, v.bn)) return e;
  // the tile that straddles c1: w1 columns of Y, then bn - w1 columns of Y2
  const int w1 = (int)(c1 % v.bn);
  if (c1 < m2 && w1 != 0) {
    if (int e = panel_map(&mya, Y, n, c1, ldy, w1)) return e;
    if (int e = panel_map(&myb, Y2, n, m2 - c1, ldy2, v.bn - w1)) return e;
  } else {
    mya = my;
    myb = my2;
  }
  for (size_t u0 = 0; u0 < P.code.size(); u0 += rk::kMaxUnits) {
    const size_t cnt = std::min<size_t>(rk::kMaxUnits, P.code.size() - u0);
    std::copy_n(P.code.begin() + u0, cnt, U.u);
    std::copy_n(P.slot.begin() + u0, cnt, U.slot);
    v.fn<<<(unsigned)cnt, v.threads, v.smem, s>>>(n, m1, m2, c1, G, ldg, ws, shape_off, mx, my, my2, mya, myb, U);
    rkh::note_launch();
  }
  for (size_t t0 = 0; t0 < P.split_ab.size(); t0 += rk::kMaxTiles) {
    const size_t cnt = std::min<size_t>(rk::kMaxTiles, P.split_ab.size() - t0);
    std::copy_n(P.split_ab.begin() + t0, cnt, T.ab);
    std::copy_n(P.split_first.begin() + t0, cnt, T.first);
    std::copy_n(P.split_count.begin() + t0, cnt, T.count);
    v.reduce<<<dim3((unsigned)cnt, 8), 256, 0, s>>>(m1, m2, ws, G, ldg, T);
    rkh::note_launch();
  }
  }  // parts
  return cuda_check("rk_gram");
}

int launch_gemm_nn(int64_t n, int64_t sdim, int64_t y, const double* S, int64_t lds, const double* C, int64_t ldc,
                   double* Out, int64_t ldo, cudaStream_t s) {
  if (n <= 0 || y <= 0) return 0;
  RK_REQUIRE(aligned16(S) && aligned16(C) && (lds % 2 == 0) && (ldc % 2 == 0), RK_ERR_ARG,
             "rk_gemm_nn: operands need 16-byte aligned columns with even leading dimension");
  RK_REQUIRE(lds >= n && ldc >= sdim && ldo >= n, RK_ERR_DIMENSION, "rk_gemm_nn: leading dimension too small");
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(rk::k_gemm_nn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)gemm_smem());
    configured = true;
  }
  dim3 grid((unsigned)((n + rk::kTile - 1) / rk::kTile), (unsigned)((y + rk::kTile - 1) / rk::kTile));
  rk::k_gemm_nn<<<grid, rk::kDmmaThreads, gemm_smem(), s>>>(n, sdim, y, S, lds, C, ldc, Out, ldo); rkh::note_launch();
  return cuda_check("rk_gemm_nn");
}

}  // namespace rkh
