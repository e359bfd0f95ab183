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
#ifndef RK_GRAM_SKIP
#define RK_GRAM_SKIP 1
#endif
constexpr bool kSkipLower = RK_GRAM_SKIP;

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
//
// Templated on the CTA tile (BM x BN) and the warp tile (WM x WN). Per K step
// of 4 a warp issues WM/8 + WN/8 fragment loads for (WM/8)(WN/8) DMMAs and the
// CTA stages (BM + BN) x 16 doubles per 2 BM BN 16 flops, so the 128 x 128
// tile halves the L2 -> SM traffic per flop of the 64 x 64 one (16 vs 8
// flop/B) at the price of coarser triangle and edge tiles.
// --------------------------------------------------------------------------
template <int BM, int BN, int WM, int WN, int MINB, int STAGES>
__global__ void __launch_bounds__((BM / WM) * (BN / WN) * 32, MINB)
    k_gram(int64_t n, int64_t m1, const double* __restrict__ X, int64_t ldx, int64_t m2,
           const double* __restrict__ Y, int64_t ldy, const double* __restrict__ Y2, int64_t ldy2, int64_t c1,
           double* __restrict__ out, int64_t ldo, int64_t split_stride, int64_t rows_per_split, int64_t upper_off) {
  constexpr int kThreads = (BM / WM) * (BN / WN) * 32;
  constexpr int FA = WM / 8, FB = WN / 8;
  extern __shared__ __align__(16) double smem[];
  double* Xs = smem;                                  // [stage][a][kPadK]
  double* Ys = smem + STAGES * BM * kPadK;           // [stage][b][kPadK]
  const int64_t a0 = (int64_t)blockIdx.x * BM;
  const int64_t b0 = (int64_t)blockIdx.y * BN;
  // upper mode: G is a block of a symmetric matrix whose column b sits at global
  // column b + upper_off; tiles strictly below the diagonal are skipped (their
  // entries are left undefined and mirrored by the caller).
  if (upper_off >= 0 && a0 > b0 + upper_off + BN - 1) return;
  const int64_t kbeg = (int64_t)blockIdx.z * rows_per_split;
  const int64_t kend = min(n, kbeg + rows_per_split);
  const int nsteps = kend > kbeg ? (int)((kend - kbeg + kStep - 1) / kStep) : 0;

  // Each thread stages fixed (column, row pair) chunks: LX of the left panel
  // and LY of the right one. Their column base pointers do not change with the
  // K step, so they are resolved once (column bound and the Y / Y2 segment
  // choice included) and every step only adds the row offset.
  constexpr int LX = BM * (kStep / 2) / kThreads, LY = BN * (kStep / 2) / kThreads;
  static_assert(LX * kThreads == BM * (kStep / 2) && LY * kThreads == BN * (kStep / 2), "loader shape");
  const int ch = threadIdx.x % (kStep / 2);
  const double* xcol[LX];
  const double* ycol[LY];
#pragma unroll
  for (int i = 0; i < LX; ++i) {
    const int64_t ga = a0 + (threadIdx.x + i * kThreads) / (kStep / 2);
    xcol[i] = ga < m1 ? X + ga * ldx + kbeg + 2 * ch : nullptr;
  }
#pragma unroll
  for (int i = 0; i < LY; ++i) {
    const int64_t gb = b0 + (threadIdx.x + i * kThreads) / (kStep / 2);
    // columns [0, c1) of the right operand live in Y, [c1, m2) in Y2
    ycol[i] = gb >= m2 ? nullptr : gb < c1 ? Y + gb * ldy + kbeg + 2 * ch : Y2 + (gb - c1) * ldy2 + kbeg + 2 * ch;
  }
  auto load_stage = [&](int stage, int step) {
    const int64_t off = (int64_t)step * kStep;
    const int64_t row = kbeg + off + 2 * ch;
    const int rb = row < kend ? (row + 1 < kend ? 16 : 8) : 0;
#pragma unroll
    for (int i = 0; i < LX; ++i) {
      const int col = (threadIdx.x + i * kThreads) / (kStep / 2);
      const bool ok = xcol[i] != nullptr && rb > 0;
      cp_async16(Xs + (stage * BM + col) * kPadK + 2 * ch, ok ? (const void*)(xcol[i] + off) : (const void*)X,
                 ok ? rb : 0);
    }
#pragma unroll
    for (int i = 0; i < LY; ++i) {
      const int col = (threadIdx.x + i * kThreads) / (kStep / 2);
      const bool ok = ycol[i] != nullptr && rb > 0;
      cp_async16(Ys + (stage * BN + col) * kPadK + 2 * ch, ok ? (const void*)(ycol[i] + off) : (const void*)Y,
                 ok ? rb : 0);
    }
  };

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int wa = (warp % (BM / WM)) * WM, wb = (warp / (BM / WM)) * WN;
  double acc[FA][FB][2];
#pragma unroll
  for (int i = 0; i < FA; ++i)
#pragma unroll
    for (int j = 0; j < FB; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < nsteps) load_stage(s, s);
    cp_async_commit();
  }
  // upper mode: a warp whose whole WM x WN block lies strictly below the
  // diagonal only helps stage operands (its entries are undefined anyway)
  const bool compute = !(kSkipLower && upper_off >= 0 && a0 + wa > b0 + wb + upper_off + WN - 1);
  for (int step = 0; step < nsteps; ++step) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    const int nxt = step + STAGES - 1;
    if (nxt < nsteps) load_stage(nxt % STAGES, nxt);
    cp_async_commit();
    const int stg = step % STAGES;
    const double* xs = Xs + (stg * BM) * kPadK;
    const double* ys = Ys + (stg * BN) * kPadK;
    if (!compute) continue;
#pragma unroll
    for (int kq = 0; kq < kStep / 4; ++kq) {
      double af[FA], bf[FB];
#pragma unroll
      for (int i = 0; i < FA; ++i) af[i] = xs[(wa + i * 8 + g) * kPadK + kq * 4 + t];
#pragma unroll
      for (int j = 0; j < FB; ++j) bf[j] = ys[(wb + j * 8 + g) * kPadK + kq * 4 + t];
#pragma unroll
      for (int i = 0; i < FA; ++i)
#pragma unroll
        for (int j = 0; j < FB; ++j) dmma884(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
  }
  cp_async_wait<0>();

  double* o = out + (int64_t)blockIdx.z * split_stride;
#pragma unroll
  for (int i = 0; i < FA; ++i) {
    const int64_t ga = a0 + wa + i * 8 + g;
#pragma unroll
    for (int j = 0; j < FB; ++j) {
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
struct GramVariant {
  void (*fn)(int64_t, int64_t, const double*, int64_t, int64_t, const double*, int64_t, const double*, int64_t, int64_t,
             double*, int64_t, int64_t, int64_t, int64_t);
  int bm, bn, threads;
  size_t smem;
  int64_t per_sm;
};

template <int BM, int BN, int WM, int WN, int MINB, int STAGES>
static GramVariant make_variant() {
  GramVariant v;
  v.fn = rk::k_gram<BM, BN, WM, WN, MINB, STAGES>;
  v.bm = BM;
  v.bn = BN;
  v.threads = (BM / WM) * (BN / WN) * 32;
  v.smem = (size_t)STAGES * (BM + BN) * rk::kPadK * sizeof(double);
  cudaFuncSetAttribute(v.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)v.smem);
  int occ = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, v.fn, v.threads, v.smem) != cudaSuccess || occ < 1) occ = 1;
  v.per_sm = occ;
  return v;
}

// 0: 64 x 64 CTA tile, 4 warps of 32 x 32 (2 CTAs / SM)
// 1: 128 x 64, 4 warps of 64 x 32, 3 stages (2 CTAs / SM)
// 2: 128 x 128, 8 warps of 64 x 32 (1 CTA / SM)
static const GramVariant& gram_variant(int which) {
  static const GramVariant v0 = make_variant<64, 64, 32, 32, RK_GRAM_MINB, rk::kStages>();
  static const GramVariant v1 = make_variant<128, 64, 64, 32, 2, 3>();
  static const GramVariant v2 = make_variant<128, 128, 64, 32, 1, 4>();
  return which == 2 ? v2 : which == 1 ? v1 : v0;
}

struct GramGeom {
  int which;
  int64_t ta, tb, splits, rows_per_split;
};

// Tiles the kernel computes: all of them, or (upper_off >= 0) those not strictly
// below the diagonal of the enclosing symmetric matrix.
static int64_t active_tiles(int64_t ta, int64_t tb, int bm, int bn, int64_t upper_off) {
  if (upper_off < 0) return ta * tb;
  int64_t count = 0;
  for (int64_t b = 0; b < tb; ++b) {
    const int64_t last_a = (b * bn + upper_off + bn - 1) / bm;  // a0 <= b0 + off + bn - 1
    count += std::min(ta, last_a + 1);
  }
  return count;
}

// Tile choice: 128x64 when it computes no more area (edge and triangle tiles
// included) than 64x64, else 64x64; RK_GRAM_TILE=0/1/2 forces one.
static int pick_variant(int64_t m1, int64_t m2, int64_t upper_off) {
  static const int forced = [] {
    const char* e = getenv("RK_GRAM_TILE");
    return e ? atoi(e) : -1;
  }();
  if (forced >= 0 && forced <= 2) return forced;
  double area[3];
  for (int w = 0; w < 3; ++w) {
    const GramVariant& v = gram_variant(w);
    const int64_t ta = (m1 + v.bm - 1) / v.bm, tb = (m2 + v.bn - 1) / v.bn;
    area[w] = (double)active_tiles(ta, tb, v.bm, v.bn, upper_off) * v.bm * v.bn;
  }
  // measured (scripts/gram_probe.py): 128x64 beats 64x64 by 2-5% on full
  // Grams, 128x128 never wins (one CTA of 8 warps per SM hides less latency)
  return area[1] <= 1.02 * area[0] ? 1 : 0;
}

// Split N so the (tile, split) units fill whole waves of the resident CTA slots:
// each unit is the same amount of work, so the tail of a partial wave is the
// loss. Picks the fewest waves (<= 8) within 3% of the best fill.
static GramGeom gram_geometry(int64_t n, int64_t m1, int64_t m2, int64_t upper_off) {
  GramGeom g;
  g.which = pick_variant(m1, m2, upper_off);
  const GramVariant& v = gram_variant(g.which);
  g.ta = (m1 + v.bm - 1) / v.bm;
  g.tb = (m2 + v.bn - 1) / v.bn;
  const int64_t tiles = std::max<int64_t>(1, active_tiles(g.ta, g.tb, v.bm, v.bn, upper_off));
  const int64_t slots = (int64_t)sm_count() * v.per_sm;
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
                const double* Y2, int64_t ldy2, int64_t c1, double* G, int64_t ldg, double* ws, int64_t ws_len,
                int64_t upper_off, cudaStream_t s) {
  if (m1 <= 0 || m2 <= 0) return 0;
  if (Y2 == nullptr || c1 >= m2) {
    Y2 = Y;
    ldy2 = ldy;
    c1 = m2;
  }
  RK_REQUIRE(aligned16(X) && aligned16(Y) && aligned16(Y2) && (ldx % 2 == 0) && (ldy % 2 == 0) && (ldy2 % 2 == 0),
             RK_ERR_ARG, "rk_gram: operands need 16-byte aligned columns with even leading dimension");
  RK_REQUIRE(ldx >= n && ldy >= n && ldy2 >= n && ldg >= m1 && c1 >= 0, RK_ERR_DIMENSION,
             "rk_gram: leading dimension too small");
  const GramGeom g = gram_geometry(std::max<int64_t>(n, 1), m1, m2, upper_off);
  const GramVariant& v = gram_variant(g.which);
  dim3 grid((unsigned)g.ta, (unsigned)g.tb, (unsigned)g.splits);
  if (g.splits == 1) {
    v.fn<<<grid, v.threads, v.smem, s>>>(n, m1, X, ldx, m2, Y, ldy, Y2, ldy2, c1, G, ldg, 0, g.rows_per_split,
                                         upper_off);
    rkh::note_launch();
  } else {
    RK_REQUIRE(ws && ws_len >= g.splits * m1 * m2, RK_ERR_ARG, "rk_gram: workspace too small (%lld < %lld)",
               (long long)ws_len, (long long)(g.splits * m1 * m2));
    v.fn<<<grid, v.threads, v.smem, s>>>(n, m1, X, ldx, m2, Y, ldy, Y2, ldy2, c1, ws, m1, m1 * m2,
                                         g.rows_per_split, upper_off);
    rkh::note_launch();
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
