// FP64 tensor-core (DMMA) contractions for the POD truncation:
//   K7  G = X' Y            snapshot Gram S'(AS), W'(AW), Y'(AW)   (linalg.py:174,
//                           krylov.py:152, threestage.py:320, pod.py:119)
//   K8  Out = S C           basis reconstruction S @ coef          (pod.py:91-93)
//
// tcgen05 has no f64 kind, so the fp64 tensor path on sm_100a is the warp-level
// DMMA (mma.sync.m8n8k4.f64, SASS DMMA.8x8x4). Operands are staged through a
// 4-stage cp.async (LDGSTS, 16-byte, L2-only) shared-memory ring; each CTA owns
// a 64x64 output tile computed by 4 warps of 32x32 (16 DMMA accumulators).
// K7 splits the N (row) dimension across CTAs so a single 64x64 tile still
// fills the 148 SMs; the split partials are summed in a fixed order (no fp64
// atomics), so results are deterministic.
#include <algorithm>

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
// K7: out[split] (m1 x m2 tile region, col-major ldo) = X[kbeg:kend, :]' Y[kbeg:kend, :]
// --------------------------------------------------------------------------
__global__ void __launch_bounds__(kDmmaThreads, RK_GRAM_MINB)
    k_gram(int64_t n, int64_t m1, const double* __restrict__ X, int64_t ldx, int64_t m2,
           const double* __restrict__ Y, int64_t ldy, double* __restrict__ out, int64_t ldo,
           int64_t split_stride, int64_t rows_per_split, int64_t upper_off) {
  extern __shared__ __align__(16) double smem[];
  double* Xs = smem;                                  // [stage][a][kPadK]
  double* Ys = smem + kStages * kTile * kPadK;        // [stage][b][kPadK]
  const int64_t a0 = (int64_t)blockIdx.x * kTile;
  const int64_t b0 = (int64_t)blockIdx.y * kTile;
  // upper mode: G is a block of a symmetric matrix whose column b sits at global
  // column b + upper_off; tiles strictly below the diagonal are skipped (their
  // entries are left undefined and mirrored by the caller).
  if (upper_off >= 0 && a0 > b0 + upper_off + kTile - 1) return;
  const int64_t kbeg = (int64_t)blockIdx.z * rows_per_split;
  const int64_t kend = min(n, kbeg + rows_per_split);
  const int nsteps = kend > kbeg ? (int)((kend - kbeg + kStep - 1) / kStep) : 0;

  auto load_stage = [&](int stage, int step) {
    const int64_t kr = kbeg + (int64_t)step * kStep;
    for (int q = threadIdx.x; q < kTile * (kStep / 2); q += kDmmaThreads) {
      const int col = q / (kStep / 2), ch = q % (kStep / 2);
      const int64_t row = kr + 2 * ch;
      const int rb = row < kend ? (row + 1 < kend ? 16 : 8) : 0;
      {
        const int64_t ga = a0 + col;
        const bool ok = ga < m1 && rb > 0;
        cp_async16(Xs + (stage * kTile + col) * kPadK + 2 * ch, ok ? (const void*)(X + ga * ldx + row) : (const void*)X,
                   ok ? rb : 0);
      }
      {
        const int64_t gb = b0 + col;
        const bool ok = gb < m2 && rb > 0;
        cp_async16(Ys + (stage * kTile + col) * kPadK + 2 * ch, ok ? (const void*)(Y + gb * ldy + row) : (const void*)Y,
                   ok ? rb : 0);
      }
    }
  };

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int wa = (warp & 1) * 32, wb = (warp >> 1) * 32;
  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

#pragma unroll
  for (int s = 0; s < kStages - 1; ++s) {
    if (s < nsteps) load_stage(s, s);
    cp_async_commit();
  }
  for (int step = 0; step < nsteps; ++step) {
    cp_async_wait<kStages - 2>();
    __syncthreads();
    const int nxt = step + kStages - 1;
    if (nxt < nsteps) load_stage(nxt % kStages, nxt);
    cp_async_commit();
    const int stg = step % kStages;
    const double* xs = Xs + (stg * kTile) * kPadK;
    const double* ys = Ys + (stg * kTile) * kPadK;
#pragma unroll
    for (int kq = 0; kq < kStep / 4; ++kq) {
      double af[4], bf[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) af[i] = xs[(wa + i * 8 + g) * kPadK + kq * 4 + t];
#pragma unroll
      for (int j = 0; j < 4; ++j) bf[j] = ys[(wb + j * 8 + g) * kPadK + kq * 4 + t];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma884(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
  }
  cp_async_wait<0>();

  double* o = out + (int64_t)blockIdx.z * split_stride;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t ga = a0 + wa + i * 8 + g;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t gb = b0 + wb + j * 8 + 2 * t;
      if (ga < m1) {
        if (gb < m2) o[ga + gb * ldo] = acc[i][j][0];
        if (gb + 1 < m2) o[ga + (gb + 1) * ldo] = acc[i][j][1];
      }
    }
  }
}

// Fixed-order sum of the split partials: G[a + b*ldg] = sum_s ws[s][a + b*m1].
__global__ void k_gram_reduce(int64_t m1, int64_t m2, int64_t splits, const double* __restrict__ ws,
                              double* __restrict__ G, int64_t ldg) {
  const int64_t total = m1 * m2;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int64_t q = 0; q < splits; ++q) s += ws[q * total + e];
    const int64_t a = e % m1, b = e / m1;
    G[a + b * ldg] = s;
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

  auto load_stage = [&](int stage, int step) {
    const int64_t k0 = (int64_t)step * kStep;
    // S tile: kStep columns x 64 rows, 32 chunks of 2 rows per column
    for (int q = threadIdx.x; q < kStep * (kTile / 2); q += kDmmaThreads) {
      const int kc = q / (kTile / 2), ch = q % (kTile / 2);
      const int64_t col = k0 + kc, row = i0 + 2 * ch;
      const int rb = (col < s && row < n) ? (row + 1 < n ? 16 : 8) : 0;
      cp_async16(Ss + (stage * kStep + kc) * kPadM + 2 * ch, rb ? (const void*)(S + col * lds + row) : (const void*)S, rb);
    }
    // C tile: 64 columns x kStep rows, 8 chunks per column
    for (int q = threadIdx.x; q < kTile * (kStep / 2); q += kDmmaThreads) {
      const int cc = q / (kStep / 2), ch = q % (kStep / 2);
      const int64_t col = c0 + cc, row = k0 + 2 * ch;
      const int rb = (col < y && row < s) ? (row + 1 < s ? 16 : 8) : 0;
      cp_async16(Cs + (stage * kTile + cc) * kPadK + 2 * ch, rb ? (const void*)(C + col * ldc + row) : (const void*)C, rb);
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

static size_t gram_smem() { return (size_t)2 * rk::kStages * rk::kTile * rk::kPadK * sizeof(double); }
static size_t gemm_smem() {
  return (size_t)(rk::kStages * rk::kStep * rk::kPadM + rk::kStages * rk::kTile * rk::kPadK) * sizeof(double);
}

struct GramGeom {
  int64_t ta, tb, splits, rows_per_split;
};

// Tiles the kernel computes: all of them, or (upper_off >= 0) those not strictly
// below the diagonal of the enclosing symmetric matrix.
static int64_t active_tiles(int64_t ta, int64_t tb, int64_t upper_off) {
  if (upper_off < 0) return ta * tb;
  int64_t count = 0;
  for (int64_t b = 0; b < tb; ++b) {
    const int64_t last_a = (b * rk::kTile + upper_off + rk::kTile - 1) / rk::kTile;  // a0 <= b0 + off + 63
    count += std::min(ta, last_a + 1);
  }
  return count;
}

// Split N so the (tile, split) units fill whole waves of the resident CTA slots
// (2 per SM): each unit is the same amount of work, so the tail of a partial
// wave is the loss. Picks the fewest waves (<= 8) within 3% of the best fill.
static GramGeom gram_geometry(int64_t n, int64_t m1, int64_t m2, int64_t upper_off) {
  GramGeom g;
  g.ta = (m1 + rk::kTile - 1) / rk::kTile;
  g.tb = (m2 + rk::kTile - 1) / rk::kTile;
  const int64_t tiles = std::max<int64_t>(1, active_tiles(g.ta, g.tb, upper_off));
  static const int64_t per_sm = [] {
    int occ = 0;
    cudaFuncSetAttribute(rk::k_gram, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)gram_smem());
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, rk::k_gram, rk::kDmmaThreads, gram_smem()) != cudaSuccess ||
        occ < 1)
      occ = 2;
    return (int64_t)occ;
  }();
  const int64_t slots = (int64_t)sm_count() * per_sm;
  const int64_t max_splits = std::max<int64_t>(1, n / 512);
  double fill[9] = {0};
  int64_t pick[9] = {0};
  double best = 0.0;
  for (int w = 1; w <= 8; ++w) {
    const int64_t sp = std::max<int64_t>(1, std::min(max_splits, slots * w / tiles));
    const int64_t units = sp * tiles;
    fill[w] = (double)units / (double)(slots * ((units + slots - 1) / slots));
    pick[w] = sp;
    best = std::max(best, fill[w]);
  }
  int64_t splits = pick[8];
  for (int w = 1; w <= 8; ++w)
    if (fill[w] >= best - 0.03) {
      splits = pick[w];
      break;
    }
  int64_t rps = (n + splits - 1) / splits;
  rps = (rps + rk::kStep - 1) / rk::kStep * rk::kStep;
  splits = std::max<int64_t>(1, (n + rps - 1) / rps);
  g.splits = splits;
  g.rows_per_split = std::max<int64_t>(rps, rk::kStep);
  return g;
}

int64_t gram_workspace_doubles(int64_t n, int64_t m1, int64_t m2, int64_t upper_off) {
  const GramGeom g = gram_geometry(std::max<int64_t>(n, 1), m1, m2, upper_off);
  return g.splits > 1 ? g.splits * m1 * m2 : 0;
}

static bool aligned16(const void* p) { return ((uintptr_t)p & 15u) == 0; }

int launch_gram(int64_t n, int64_t m1, const double* X, int64_t ldx, int64_t m2, const double* Y, int64_t ldy,
                double* G, int64_t ldg, double* ws, int64_t ws_len, int64_t upper_off, cudaStream_t s) {
  if (m1 <= 0 || m2 <= 0) return 0;
  RK_REQUIRE(aligned16(X) && aligned16(Y) && (ldx % 2 == 0) && (ldy % 2 == 0), RK_ERR_ARG,
             "rk_gram: operands need 16-byte aligned columns with even leading dimension");
  RK_REQUIRE(ldx >= n && ldy >= n && ldg >= m1, RK_ERR_DIMENSION, "rk_gram: leading dimension too small");
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(rk::k_gram, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)gram_smem());
    configured = true;
  }
  const GramGeom g = gram_geometry(std::max<int64_t>(n, 1), m1, m2, upper_off);
  dim3 grid((unsigned)g.ta, (unsigned)g.tb, (unsigned)g.splits);
  if (g.splits == 1) {
    rk::k_gram<<<grid, rk::kDmmaThreads, gram_smem(), s>>>(n, m1, X, ldx, m2, Y, ldy, G, ldg, 0, g.rows_per_split,
                                                           upper_off); rkh::note_launch();
  } else {
    RK_REQUIRE(ws && ws_len >= g.splits * m1 * m2, RK_ERR_ARG, "rk_gram: workspace too small (%lld < %lld)",
               (long long)ws_len, (long long)(g.splits * m1 * m2));
    rk::k_gram<<<grid, rk::kDmmaThreads, gram_smem(), s>>>(n, m1, X, ldx, m2, Y, ldy, ws, m1, m1 * m2,
                                                            g.rows_per_split, upper_off); rkh::note_launch();
    const int64_t total = m1 * m2;
    const int rg = (int)std::max<int64_t>(1, std::min<int64_t>((total + 255) / 256, (int64_t)sm_count() * 8));
    rk::k_gram_reduce<<<rg, 256, 0, s>>>(m1, m2, g.splits, ws, G, ldg); rkh::note_launch();
  }
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
