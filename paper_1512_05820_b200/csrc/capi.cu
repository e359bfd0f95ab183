// extern "C" boundary (include/podcg.h): argument checks, thread-local error
// text, and dispatch to the launchers. No allocation, no synchronisation.
#include <cstdarg>
#include <cstdio>
#include <atomic>
#include <mutex>
#include <utility>
#include <vector>

#include <algorithm>

#include "common.cuh"

namespace rkh {

static thread_local char g_err[512] = "";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

int cuda_check(const char* where) {
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error("%s: %s", where, cudaGetErrorString(e));
    return RK_ERR_CUDA;
  }
  return RK_OK;
}

int sm_count() {
  static int cached = 0;
  static std::once_flag once;
  std::call_once(once, [] {
    int dev = 0, v = 0;
    if (cudaGetDevice(&dev) == cudaSuccess &&
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess && v > 0)
      cached = v;
    else
      cached = 148;
  });
  return cached;
}

// ---- optional per-kernel event timing of rk_pcg_steps (bench only) ---------
// Marks are recorded between the kernels of each iteration; slot s -> s+1
// brackets kernel s (0: K1 spmv+curvature, 1: K3/K4 update, 2: K5 direction).
// Not thread-safe: enable it from one host thread only.
struct ProfState {
  bool on = false;
  std::vector<cudaEvent_t> pool;
  std::vector<std::pair<int, cudaEvent_t>> marks;
  size_t used = 0;
};
static ProfState g_prof;
double g_cluster_ms = 0.0;  // rk_profile_end: total ms / launches of the cluster solver (slots 8 -> 9)
int64_t g_cluster_n = 0;

static std::atomic<int64_t> g_launches{0};
void note_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

bool pdl_enabled() {
  static const bool on = [] {
    const char* e = getenv("RK_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}

bool prof_sample() {
  static uint64_t counter = 0;
  return g_prof.on && ((counter++ & 7u) == 0);
}

void prof_mark(int slot, cudaStream_t s) {
  if (!g_prof.on) return;
  if (g_prof.used == g_prof.pool.size()) {
    cudaEvent_t e;
    cudaEventCreate(&e);
    g_prof.pool.push_back(e);
  }
  cudaEvent_t e = g_prof.pool[g_prof.used++];
  cudaEventRecord(e, s);
  g_prof.marks.emplace_back(slot, e);
}

// launchers defined in the kernel files
int launch_spmv(const rk_csr& A, const double* x, double* y, cudaStream_t s);
int launch_spmm(const rk_csr& A, int64_t m, const double* X, int64_t ldx, double* Y, int64_t ldy, cudaStream_t s);
int launch_csr_diagonal(const rk_csr& A, double* diag, double* dinv, int64_t* bad, cudaStream_t s);
int launch_csr_asymmetry(const rk_csr& A, double* out2, double* ws, int64_t ws_len, uint32_t* tickets, cudaStream_t s);
int launch_ssor_apply(const rk_csr& A, const double* dw, const double* d, const double* r, double* z, double* u,
                      int* flags, unsigned int* counters, int epoch, cudaStream_t s, const rk_pcg_state* st,
                      const double* r_even, const int32_t* order_fwd, const int32_t* order_bwd);
int launch_ssor_levels(const rk_csr& A, int upper, int32_t* lvl, int* flags, unsigned int* counter, int epoch,
                       cudaStream_t s);
int pcg_entry_ssor(const rk_pcg_plan& P, const rk_ssor_plan& S, cudaStream_t s);
int pcg_steps_ssor(const rk_pcg_plan& P, const rk_ssor_plan& S, int nsteps, int64_t kmax_hint, cudaStream_t s);
int pcg_entry(const rk_pcg_plan& P, cudaStream_t s);
int pcg_steps(const rk_pcg_plan& P, int nsteps, int64_t kmax_hint, cudaStream_t s);
int pcg_cluster_eligible(const rk_pcg_plan& P);
int pcg_cluster_run(const rk_pcg_plan& P, int64_t kend, cudaStream_t s);
int64_t pcg_cluster_max_rows();
int pcg_curvature(const rk_pcg_plan& P, cudaStream_t s);
int pcg_update(const rk_pcg_plan& P, cudaStream_t s);
int pcg_direction(const rk_pcg_plan& P, int64_t kmax_hint, cudaStream_t s);
int64_t pcg_workspace_doubles(int64_t n, int64_t m, int64_t vcap);
void launch_gemv_t(int64_t n, int64_t m_max, const int64_t* m_dev, const int64_t* done, const double* B,
                   int64_t ldb, const double* x, int64_t x_col_from_m, int64_t ldx, double* partials,
                   const double* div, double* out, cudaStream_t s);
void launch_gemv_n(int64_t n, int64_t m_max, const int64_t* m_dev, const int64_t* done, const double* B,
                   int64_t ldb, const double* c, const double* y0, double* y, int32_t op, int64_t y_col_from_m,
                   int64_t ldy, cudaStream_t s);
int gemv_n_smem_ok(int64_t m);
int64_t gemv_nchunks(int64_t n);
void launch_dot(int64_t n, const double* x, const double* y, double* out, double* ws, uint32_t* ticket,
                cudaStream_t s);
int dot_grid_max();
void launch_scale_columns(int64_t n, int64_t m, const double* V, int64_t ldv, const double* sc, double* out,
                          int64_t ldo, cudaStream_t s);
void launch_axpby(int64_t n, double a, const double* x, double b, double* y, cudaStream_t s);
void launch_sub_from(int64_t n, const double* x0, double* y, cudaStream_t s);
int launch_gram(int64_t n, int64_t m1, const double* X, int64_t ldx, int64_t m2, const double* Y, int64_t ldy,
                const double* Y2, int64_t ldy2, int64_t c1, double* G, int64_t ldg, double* ws, int64_t ws_len,
                int64_t upper_off, cudaStream_t s);
int64_t gram_workspace_doubles(int64_t n, int64_t m1, int64_t m2, int64_t upper_off);
int sell_plan(int64_t n, const int32_t* rp, const int32_t* col, int32_t bdim, int32_t max_len, int32_t* len_ws,
              int32_t* sptr, int64_t* nslot, int32_t* bad, cudaStream_t s);
int sell_fill(int64_t n, const int32_t* rp, const int32_t* col, int32_t bdim, const int32_t* len_ws,
              const int32_t* sptr, int64_t nslot, int32_t* scol, int32_t* perm, cudaStream_t s);
int debug_trace(unsigned long long* out, int64_t n);
int launch_gemm_nn(int64_t n, int64_t sdim, int64_t y, const double* S, int64_t lds, const double* C, int64_t ldc,
                   double* Out, int64_t ldo, cudaStream_t s);

static int check_csr(const rk_csr* A) {
  RK_REQUIRE(A != nullptr, RK_ERR_ARG, "null CSR descriptor");
  RK_REQUIRE(A->n >= 0 && A->nnz >= 0 && A->nnz < (int64_t)INT32_MAX, RK_ERR_DIMENSION, "CSR: bad n/nnz");
  RK_REQUIRE(A->n == 0 || (A->rowptr && (A->nnz == 0 || (A->col && A->val))), RK_ERR_ARG, "CSR: null array");
  RK_REQUIRE(A->lanes == 0 || A->lanes == 1 || A->lanes == 2 || A->lanes == 4 || A->lanes == 8 ||
                 A->lanes == 16 || A->lanes == 32,
             RK_ERR_ARG, "CSR: lanes must be 0 or a power of two <= 32");
  RK_REQUIRE(A->bdim == 0 || A->bdim == 1 || A->bdim == 3, RK_ERR_ARG, "CSR: bdim must be 0, 1 or 3");
  RK_REQUIRE(!A->bval || A->bdim == 1 || (A->browptr && A->bcol && A->n % 3 == 0 && A->nblk * 9 >= A->nnz),
             RK_ERR_ARG, "CSR: inconsistent 3x3 block view");
  RK_REQUIRE(!A->bval || A->bdim != 1 || (A->browptr && A->bcol && A->nblk >= A->nnz), RK_ERR_ARG,
             "CSR: inconsistent sliced-ELL view");
  return RK_OK;
}

int launch_bsr3_gather(int64_t nblk, const int32_t* perm, const double* val, double* bval, cudaStream_t s);
int launch_sell_gather(int64_t total, const int32_t* perm, const double* val, double* out, cudaStream_t s);

}  // namespace rkh

using rkh::as_stream;

extern "C" {

const char* rk_last_error(void) { return rkh::g_err; }

int rk_device_sm_count(void) { return rkh::sm_count(); }

int64_t rk_pcg_workspace_doubles(int64_t n, int64_t m, int64_t vcap) {
  return rkh::pcg_workspace_doubles(n, m, vcap);
}

int64_t rk_reduce_workspace_doubles(int64_t n, int64_t m) {
  const int64_t a = rkh::gemv_nchunks(n) * std::max<int64_t>(m, 1);
  const int64_t b = (int64_t)rkh::dot_grid_max() * 2;
  return std::max(a, b);
}

int64_t rk_gram_workspace_doubles(int64_t n, int64_t m1, int64_t m2) {
  return rkh::gram_workspace_doubles(n, m1, m2, -1);
}

int64_t rk_gram_upper_workspace_doubles(int64_t n, int64_t m1, int64_t m2, int64_t col_off) {
  if (n <= 0 || m1 <= 0 || m2 <= 0 || col_off < 0) return 0;
  return rkh::gram_workspace_doubles(n, m1, m2, col_off);
}

int rk_pcg_entry(const rk_pcg_plan* plan, void* stream) {
  RK_REQUIRE(plan, RK_ERR_ARG, "rk_pcg_entry: null plan");
  return rkh::pcg_entry(*plan, as_stream(stream));
}

int rk_pcg_steps(const rk_pcg_plan* plan, int32_t nsteps, int64_t kmax_hint, void* stream) {
  RK_REQUIRE(plan, RK_ERR_ARG, "rk_pcg_steps: null plan");
  if (int e = rkh::check_csr(&plan->A)) return e;
  return rkh::pcg_steps(*plan, nsteps, kmax_hint, as_stream(stream));
}

static int check_ssor(const rk_pcg_plan* plan, const rk_ssor_plan* S, const char* who) {
  RK_REQUIRE(plan && S, RK_ERR_ARG, "%s: null plan", who);
  if (int e = rkh::check_csr(&plan->A)) return e;
  RK_REQUIRE(plan->A.rowptr && plan->A.col && plan->A.val, RK_ERR_ARG, "%s: CSR operator required", who);
  RK_REQUIRE(S->dw && S->d && S->work && S->flags && S->counters && S->epoch >= 0, RK_ERR_ARG, "%s: bad SSOR state", who);
  return RK_OK;
}

int rk_pcg_entry_ssor(const rk_pcg_plan* plan, const rk_ssor_plan* ssor, void* stream) {
  if (int e = check_ssor(plan, ssor, "rk_pcg_entry_ssor")) return e;
  return rkh::pcg_entry_ssor(*plan, *ssor, as_stream(stream));
}

int rk_pcg_steps_ssor(const rk_pcg_plan* plan, const rk_ssor_plan* ssor, int32_t nsteps, int64_t kmax_hint,
                      void* stream) {
  if (int e = check_ssor(plan, ssor, "rk_pcg_steps_ssor")) return e;
  return rkh::pcg_steps_ssor(*plan, *ssor, nsteps, kmax_hint, as_stream(stream));
}

int rk_pcg_cluster_eligible(const rk_pcg_plan* plan) { return plan ? rkh::pcg_cluster_eligible(*plan) : 0; }

int64_t rk_pcg_cluster_max_rows(void) { return rkh::pcg_cluster_max_rows(); }

int rk_pcg_run_cluster(const rk_pcg_plan* plan, int64_t kend, void* stream) {
  RK_REQUIRE(plan, RK_ERR_ARG, "rk_pcg_run_cluster: null plan");
  if (int e = rkh::check_csr(&plan->A)) return e;
  if (int e = rkh::pcg_cluster_run(*plan, kend, as_stream(stream))) return e;
  return rkh::cuda_check("rk_pcg_run_cluster");
}

int rk_pcg_curvature(const rk_pcg_plan* plan, void* stream) {
  RK_REQUIRE(plan, RK_ERR_ARG, "rk_pcg_curvature: null plan");
  return rkh::pcg_curvature(*plan, as_stream(stream));
}

int rk_pcg_update(const rk_pcg_plan* plan, void* stream) {
  RK_REQUIRE(plan, RK_ERR_ARG, "rk_pcg_update: null plan");
  return rkh::pcg_update(*plan, as_stream(stream));
}

int rk_pcg_direction(const rk_pcg_plan* plan, int64_t kmax_hint, void* stream) {
  RK_REQUIRE(plan, RK_ERR_ARG, "rk_pcg_direction: null plan");
  RK_REQUIRE(kmax_hint + 2 <= plan->vcap, RK_ERR_DIMENSION, "rk_pcg_direction: kmax_hint beyond capacity");
  return rkh::pcg_direction(*plan, kmax_hint, as_stream(stream));
}

int rk_spmv(const rk_csr* A, const double* x, double* y, void* stream) {
  if (int e = rkh::check_csr(A)) return e;
  RK_REQUIRE(A->n == 0 || (x && y), RK_ERR_ARG, "rk_spmv: null vector");
  if (A->n == 0) return RK_OK;
  return rkh::launch_spmv(*A, x, y, as_stream(stream));
}

int rk_spmm(const rk_csr* A, int64_t m, const double* X, int64_t ldx, double* Y, int64_t ldy, void* stream) {
  if (int e = rkh::check_csr(A)) return e;
  RK_REQUIRE(m >= 0 && ldx >= A->n && ldy >= A->n, RK_ERR_DIMENSION, "rk_spmm: bad shape");
  RK_REQUIRE(m == 0 || (X && Y), RK_ERR_ARG, "rk_spmm: null block");
  RK_REQUIRE(m <= 65535 * 8, RK_ERR_DIMENSION, "rk_spmm: too many columns");
  return rkh::launch_spmm(*A, m, X, ldx, Y, ldy, as_stream(stream));
}

int rk_csr_diagonal(const rk_csr* A, double* diag, double* dinv, int64_t* bad_row, void* stream) {
  if (int e = rkh::check_csr(A)) return e;
  RK_REQUIRE(bad_row, RK_ERR_ARG, "rk_csr_diagonal: null bad_row");
  return rkh::launch_csr_diagonal(*A, diag, dinv, bad_row, as_stream(stream));
}

int rk_ssor_apply(const rk_csr* A, const double* dw, const double* d, const double* r, double* z, double* work,
                  int32_t* flags, uint32_t* counters, int32_t epoch, const int32_t* order_fwd,
                  const int32_t* order_bwd, void* stream) {
  if (int e = rkh::check_csr(A)) return e;
  RK_REQUIRE(A->n == 0 || (dw && d && r && z && work && flags && counters), RK_ERR_ARG, "rk_ssor_apply: null pointer");
  RK_REQUIRE(epoch > 0, RK_ERR_ARG, "rk_ssor_apply: epoch must be positive");
  return rkh::launch_ssor_apply(*A, dw, d, r, z, work, reinterpret_cast<int*>(flags),
                                reinterpret_cast<unsigned int*>(counters), epoch, as_stream(stream), nullptr, nullptr,
                                order_fwd, order_bwd);
}

int rk_ssor_levels(const rk_csr* A, int32_t upper, int32_t* levels, int32_t* flags, uint32_t* counter, int32_t epoch,
                   void* stream) {
  if (int e = rkh::check_csr(A)) return e;
  RK_REQUIRE(A->n == 0 || (levels && flags && counter), RK_ERR_ARG, "rk_ssor_levels: null pointer");
  RK_REQUIRE(epoch > 0, RK_ERR_ARG, "rk_ssor_levels: epoch must be positive");
  return rkh::launch_ssor_levels(*A, upper, levels, reinterpret_cast<int*>(flags),
                                 reinterpret_cast<unsigned int*>(counter), epoch, as_stream(stream));
}

int rk_bsr3_gather(int64_t nblk, const int32_t* perm, const double* val, double* bval, void* stream) {
  RK_REQUIRE(nblk >= 0, RK_ERR_DIMENSION, "rk_bsr3_gather: bad size");
  RK_REQUIRE(nblk == 0 || (perm && val && bval), RK_ERR_ARG, "rk_bsr3_gather: null pointer");
  return rkh::launch_bsr3_gather(nblk, perm, val, bval, as_stream(stream));
}

int rk_sell_gather(int64_t total, const int32_t* perm, const double* val, double* out, void* stream) {
  RK_REQUIRE(total >= 0, RK_ERR_DIMENSION, "rk_sell_gather: bad size");
  RK_REQUIRE(total == 0 || (perm && val && out), RK_ERR_ARG, "rk_sell_gather: null pointer");
  return rkh::launch_sell_gather(total, perm, val, out, as_stream(stream));
}

int rk_sell_plan(int64_t n, const int32_t* rowptr, const int32_t* col, int32_t bdim, int32_t max_len,
                 int32_t* len_ws, int32_t* sptr, int64_t* nslot, int32_t* bad, void* stream) {
  return rkh::sell_plan(n, rowptr, col, bdim, max_len, len_ws, sptr, nslot, bad, as_stream(stream));
}

int rk_sell_fill(int64_t n, const int32_t* rowptr, const int32_t* col, int32_t bdim, const int32_t* len_ws,
                 const int32_t* sptr, int64_t nslot, int32_t* scol, int32_t* perm, void* stream) {
  return rkh::sell_fill(n, rowptr, col, bdim, len_ws, sptr, nslot, scol, perm, as_stream(stream));
}

int rk_csr_asymmetry(const rk_csr* A, double* out2, double* ws, int64_t ws_len, uint32_t* tickets, void* stream) {
  if (int e = rkh::check_csr(A)) return e;
  RK_REQUIRE(out2 && ws && tickets, RK_ERR_ARG, "rk_csr_asymmetry: null pointer");
  return rkh::launch_csr_asymmetry(*A, out2, ws, ws_len, tickets, as_stream(stream));
}

int rk_gemv_t(int64_t n, int64_t m, const double* B, int64_t ldb, const double* x, double* out, double* ws,
              int64_t ws_len, void* stream) {
  RK_REQUIRE(n >= 0 && m >= 0 && ldb >= n, RK_ERR_DIMENSION, "rk_gemv_t: bad shape");
  if (m == 0) return RK_OK;
  RK_REQUIRE(B && x && out && ws, RK_ERR_ARG, "rk_gemv_t: null pointer");
  if (n == 0) {
    RK_REQUIRE(cudaMemsetAsync(out, 0, m * sizeof(double), as_stream(stream)) == cudaSuccess, RK_ERR_CUDA,
               "rk_gemv_t: memset failed");
    return RK_OK;
  }
  RK_REQUIRE(ws_len >= rkh::gemv_nchunks(n) * m, RK_ERR_ARG, "rk_gemv_t: workspace too small");
  rkh::launch_gemv_t(n, m, nullptr, nullptr, B, ldb, x, 0, 0, ws, nullptr, out, as_stream(stream));
  return rkh::cuda_check("rk_gemv_t");
}

int rk_gemv_n(int64_t n, int64_t m, const double* B, int64_t ldb, const double* c, const double* y0, double* y,
              int32_t op, void* stream) {
  RK_REQUIRE(n >= 0 && m >= 0 && ldb >= n, RK_ERR_DIMENSION, "rk_gemv_n: bad shape");
  RK_REQUIRE(op >= 0 && op <= 2, RK_ERR_ARG, "rk_gemv_n: op must be 0, 1 or 2");
  RK_REQUIRE(n == 0 || (y && (m == 0 || (B && c)) && (op == 0 || y0)), RK_ERR_ARG, "rk_gemv_n: null pointer");
  RK_REQUIRE(rkh::gemv_n_smem_ok(m), RK_ERR_DIMENSION, "rk_gemv_n: too many columns (%lld)", (long long)m);
  rkh::launch_gemv_n(n, m, nullptr, nullptr, B, ldb, c, y0, y, op, 0, 0, as_stream(stream));
  return rkh::cuda_check("rk_gemv_n");
}

int rk_dot(int64_t n, const double* x, const double* y, double* out, double* ws, int64_t ws_len, uint32_t* tickets,
           void* stream) {
  RK_REQUIRE(n >= 0 && out && ws && tickets, RK_ERR_ARG, "rk_dot: null pointer");
  RK_REQUIRE(ws_len >= rkh::dot_grid_max(), RK_ERR_ARG, "rk_dot: workspace too small");
  if (n == 0) {
    RK_REQUIRE(cudaMemsetAsync(out, 0, sizeof(double), as_stream(stream)) == cudaSuccess, RK_ERR_CUDA,
               "rk_dot: memset failed");
    return RK_OK;
  }
  rkh::launch_dot(n, x, y, out, ws, tickets, as_stream(stream));
  return rkh::cuda_check("rk_dot");
}

int rk_scale_columns(int64_t n, int64_t m, const double* V, int64_t ldv, const double* s, double* out, int64_t ldo,
                     void* stream) {
  RK_REQUIRE(n >= 0 && m >= 0 && ldv >= n && ldo >= n && m <= 65535, RK_ERR_DIMENSION, "rk_scale_columns: bad shape");
  rkh::launch_scale_columns(n, m, V, ldv, s, out, ldo, as_stream(stream));
  return rkh::cuda_check("rk_scale_columns");
}

int rk_axpby(int64_t n, double a, const double* x, double b, double* y, void* stream) {
  rkh::launch_axpby(n, a, x, b, y, as_stream(stream));
  return rkh::cuda_check("rk_axpby");
}

int rk_sub_from(int64_t n, const double* x0, double* y, void* stream) {
  rkh::launch_sub_from(n, x0, y, as_stream(stream));
  return rkh::cuda_check("rk_sub_from");
}

int rk_gram(int64_t n, int64_t m1, const double* X, int64_t ldx, int64_t m2, const double* Y, int64_t ldy, double* G,
            int64_t ldg, double* ws, int64_t ws_len, void* stream) {
  RK_REQUIRE(n >= 0 && m1 >= 0 && m2 >= 0, RK_ERR_DIMENSION, "rk_gram: bad shape");
  RK_REQUIRE(m1 < 65535 * 64 && m2 < 65535 * 64, RK_ERR_DIMENSION, "rk_gram: too many columns");
  if (n == 0 && m1 > 0 && m2 > 0) {
    for (int64_t b = 0; b < m2; ++b)
      RK_REQUIRE(cudaMemsetAsync(G + b * ldg, 0, m1 * sizeof(double), as_stream(stream)) == cudaSuccess, RK_ERR_CUDA,
                 "rk_gram: memset failed");
    return RK_OK;
  }
  return rkh::launch_gram(n, m1, X, ldx, m2, Y, ldy, nullptr, 0, m2, G, ldg, ws, ws_len, -1, as_stream(stream));
}

int rk_gram_upper(int64_t n, int64_t m1, const double* X, int64_t ldx, int64_t m2, const double* Y, int64_t ldy,
                  int64_t col_off, double* G, int64_t ldg, double* ws, int64_t ws_len, void* stream) {
  RK_REQUIRE(n >= 0 && m1 >= 0 && m2 >= 0 && col_off >= 0, RK_ERR_DIMENSION, "rk_gram_upper: bad shape");
  if (n == 0) return rk_gram(n, m1, X, ldx, m2, Y, ldy, G, ldg, ws, ws_len, stream);
  return rkh::launch_gram(n, m1, X, ldx, m2, Y, ldy, nullptr, 0, m2, G, ldg, ws, ws_len, col_off, as_stream(stream));
}

int rk_gram_upper_split(int64_t n, int64_t m, const double* X, int64_t ldx, int64_t c1, const double* Y1, int64_t ldy1,
                        const double* Y2, int64_t ldy2, double* G, int64_t ldg, double* ws, int64_t ws_len,
                        void* stream) {
  RK_REQUIRE(n >= 0 && m >= 0 && c1 >= 0 && c1 <= m, RK_ERR_DIMENSION, "rk_gram_upper_split: bad shape");
  RK_REQUIRE(c1 == m || Y2 != nullptr, RK_ERR_ARG, "rk_gram_upper_split: second segment missing");
  if (n == 0) return rk_gram(n, m, X, ldx, m, Y1, ldy1, G, ldg, ws, ws_len, stream);
  return rkh::launch_gram(n, m, X, ldx, m, c1 > 0 ? Y1 : Y2, c1 > 0 ? ldy1 : ldy2, Y2, ldy2, c1, G, ldg, ws, ws_len,
                          0, as_stream(stream));
}

int rk_gemm_nn(int64_t n, int64_t s, int64_t y, const double* S, int64_t lds, const double* C, int64_t ldc,
               double* Out, int64_t ldo, void* stream) {
  RK_REQUIRE(n >= 0 && s >= 0 && y >= 0, RK_ERR_DIMENSION, "rk_gemm_nn: bad shape");
  RK_REQUIRE((n + 63) / 64 < 2147483647 && (y + 63) / 64 < 65535, RK_ERR_DIMENSION, "rk_gemm_nn: too large");
  return rkh::launch_gemm_nn(n, s, y, S, lds, C, ldc, Out, ldo, as_stream(stream));
}

}  // extern "C"

extern "C" {

// Debug timeline of the fused update tail (zeros unless built with -DRK_TAIL_TRACE).
int rk_debug_trace(uint64_t* out, int64_t n) {
  return rkh::debug_trace(reinterpret_cast<unsigned long long*>(out), n);
}

// Kernels launched by this library since load (all threads).
int64_t rk_launch_count(void) { return rkh::g_launches.load(std::memory_order_relaxed); }

// Start collecting per-kernel event timings of rk_pcg_steps.
int rk_profile_cluster(double* ms, int64_t* launches) {
  *ms = rkh::g_cluster_ms;
  *launches = rkh::g_cluster_n;
  return RK_OK;
}

int rk_profile_begin(void) {
  rkh::g_prof.on = true;
  rkh::g_prof.used = 0;
  rkh::g_prof.marks.clear();
  return RK_OK;
}

// Stop; synchronises and writes total milliseconds and launch counts per kernel
// slot (4 slots: spmv, update, finish, direction). Iterations launched after
// the run had converged (a batch's overshoot: every kernel returns at once) are
// left out: a sampled iteration counts only when its SpMV took more than a
// quarter of the 90th-percentile sampled SpMV.
int rk_profile_end(double* ms4, int64_t* count4) {
  rkh::g_prof.on = false;
  for (int i = 0; i < 4; ++i) { ms4[i] = 0.0; count4[i] = 0; }
  auto& mk = rkh::g_prof.marks;
  if (!mk.empty() && cudaEventSynchronize(mk.back().second) != cudaSuccess) return rkh::cuda_check("rk_profile_end");
  std::vector<float> dur(mk.size(), -1.f), spmv;
  rkh::g_cluster_ms = 0.0;
  rkh::g_cluster_n = 0;
  for (size_t i = 0; i + 1 < mk.size(); ++i) {
    const int a = mk[i].first, b = mk[i + 1].first;
    if (a == 8 && b == 9) {  // one persistent cluster solve (pcg_cluster.cu)
      float ms = 0.f;
      if (cudaEventElapsedTime(&ms, mk[i].second, mk[i + 1].second) == cudaSuccess) {
        rkh::g_cluster_ms += ms;
        rkh::g_cluster_n += 1;
      }
      continue;
    }
    if (b == a + 1 && a < 4) {
      float ms = 0.f;
      if (cudaEventElapsedTime(&ms, mk[i].second, mk[i + 1].second) == cudaSuccess) {
        dur[i] = ms;
        if (a == 0) spmv.push_back(ms);
      }
    }
  }
  // reference SpMV time: the 90th percentile (robust to a cold first launch)
  float ref = 0.f;
  if (!spmv.empty()) {
    const size_t q = (spmv.size() * 9) / 10;
    std::nth_element(spmv.begin(), spmv.begin() + q, spmv.end());
    ref = spmv[std::min(q, spmv.size() - 1)];
  }
  bool live = false;
  for (size_t i = 0; i + 1 < mk.size(); ++i) {
    const int a = mk[i].first;
    if (a == 0) live = dur[i] > 0.25f * ref;
    if (dur[i] >= 0.f && live) {
      ms4[a] += dur[i];
      count4[a] += 1;
    }
  }
  mk.clear();
  rkh::g_prof.used = 0;
  return rkh::cuda_check("rk_profile_end");
}

}  // extern "C"
