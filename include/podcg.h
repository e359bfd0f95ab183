/*
 * podcg.h -- C-ABI of the B200-native POD-augmented CG hot path.
 *
 * The reference (recykl, pure Python on numpy/scipy) has no FFI of its own;
 * every entry point below replaces one numpy/scipy call site on the hot path
 * and is cited against that site (paths under the reference's pkg/src/recykl).
 * INTEGRATION.md shows the ctypes stubs a maintainer of the reference would
 * add to bind these.
 *
 * Conventions:
 *   - every pointer is DEVICE memory owned by the caller (torch tensors);
 *   - dense N x m blocks are column-major with leading dimension ld >= N;
 *     the DMMA kernels additionally want ld even and 16-byte aligned columns
 *     (the host layer pads to multiples of 32 rows);
 *   - scalars that feed later kernels stay in device memory; nothing here
 *     synchronises the stream;
 *   - no allocation visible to the caller: reductions use the caller's
 *     workspace (double partials + uint32 tickets that start at zero and are
 *     left at zero);
 *   - all reductions are deterministic (fixed-order partial combine, no fp64
 *     atomics), so two runs on the same inputs are bitwise identical;
 *   - the last argument of every launcher is the cudaStream_t (as void*);
 *   - return 0 on success, < 0 on error; rk_last_error() gives a
 *     thread-local message.  Every entry point is re-entrant.
 */
#ifndef PODCG_H
#define PODCG_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  RK_OK = 0,
  RK_ERR_DIMENSION = -1, /* maps to recykl.errors.DimensionMismatch */
  RK_ERR_NOT_SPD = -2,   /* maps to recykl.errors.NotPositiveDefinite */
  RK_ERR_CUDA = -3,      /* CUDA launch/runtime error */
  RK_ERR_ARG = -4        /* bad argument (null pointer, misalignment) */
};

/* Immutable CSR descriptor borrowing caller-owned device arrays.
 * Replaces SparseSpdMatrix's scipy csr_matrix (linalg.py:63-135); indices
 * are int32 (nnz < 2^31 for every configuration). */
typedef struct rk_csr {
  int64_t n;
  int64_t nnz;
  const int32_t* rowptr; /* n+1 */
  const int32_t* col;    /* nnz, sorted within each row */
  const double* val;     /* nnz */
  int32_t lanes;         /* lanes cooperating on one row: 1,2,4,8,16,32 (0 = auto) */
  int32_t bdim;          /* block size of the sliced-ELL view below: 0 or 3 = 3x3 blocks, 1 = scalar */
  /* Optional sliced-ELL view of the same matrix in 3x3 blocks (vector-valued
   * problems such as the Q1 elasticity operator; SELL-32: 32 block rows per
   * slice, padded to the slice's widest row). When bval != NULL the SpMV
   * kernels stream 9 values + 1 block index per stored block instead of
   * 9 x (value + index), i.e. 76 instead of 108 bytes per 9 nonzeros.
   * Slot (slice s, position t, lane l) = browptr[s] + 32 t + l. Values come
   * in one contiguous 9 x 32 tile per slot row: entry e = 3*a + c (row a,
   * column c) of the block in slot q is bval[9 * (q - q % 32) + 32 e + q % 32]
   * (0 for padding); rk_bsr3_gather fills them from val.
   * With bdim == 1 the same fields hold a scalar SELL-32 view for short
   * uniform rows (7-point stencils): browptr has ceil(n/32) + 1 slice offsets,
   * slot (s, t, l) = browptr[s] + 32 t + l holds one column in bcol and one
   * value in bval (12 bytes per slot), filled by rk_sell_gather. */
  int64_t nblk;           /* number of slots (stored blocks + padding) */
  const int32_t* browptr; /* ceil(n/96) + 1 slice offsets, in slots */
  const int32_t* bcol;    /* nblk block columns (padding: a valid column) */
  const double* bval;     /* 9 * nblk */
} rk_csr;

/* Device-resident state of one augmented-PCG run (krylov.py:267-345). */
typedef struct rk_pcg_state {
  int64_t k;          /* completed iterations; p_k = V[:, k] is the live direction */
  int64_t done;       /* 1 once converged or broken down: later kernels are no-ops */
  int64_t status;     /* 0 running, 1 converged, 2 breakdown (krylov.py:303-304) */
  int64_t bd_iter;    /* iteration of the breakdown */
  double rz;          /* r'z of the live direction */
  double gamma;       /* p'Ap of the live direction */
  double pp;          /* p'p (breakdown scale) */
  double alpha;       /* rz / gamma */
  double rr;          /* ||r||^2 after the last update */
  double beta;        /* rz_next / rz (cg mode) */
  double threshold;   /* exit threshold on ||r|| (krylov.py:267) */
  double rz_next;     /* r'z of the new residual */
} rk_pcg_state;

/* Everything one augmented-PCG iteration touches.  Replaces the loop body of
 * augmented_pcg (krylov.py:300-340) with device kernels:
 *   K1  Ap = A p_k, gamma = p'Ap, p'p, breakdown test, alpha  (krylov.py:301-305)
 *   K3  x += alpha p; r -= alpha Ap; z = M^{-1} r; ||r||, r'z  (krylov.py:306-321)
 *   K4  c = cross' z and mu = F^{-1} c                         (krylov.py:155-156,322)
 *   K5  p_{k+1} = z + beta p_k - B mu  (cg)                     (krylov.py:323-326)
 *       p_{k+1} = z - B mu, then 2 block-CGS sweeps (fom)       (krylov.py:327-337)
 *       p_{k+1} = z - B mu + sum_i rz'/rz_i p_i  (fom, paper beta) (krylov.py:329-331) */
/* Counters a PCG plan's ticket array holds (0-3 kernel tickets, 8.. chunk groups). */
#define RK_PCG_TICKETS 272

typedef struct rk_pcg_plan {
  int64_t n;
  rk_csr A;                 /* A.rowptr == NULL: generic operator, caller fills AV */
  double* x;
  double* r;                /* residual buffer 0 (holds r_0 at entry) */
  double* r2;               /* residual buffer 1: iteration k reads buffer k&1, writes the other */
  double* z;
  double* V;                /* directions, column k = p_k */
  int64_t ldv;
  int64_t vcap;             /* allocated columns of V (and AV when ldav > 0) */
  double* AV;               /* A p_k: column k (ldav > 0, kept) or one vector (ldav == 0) */
  int64_t ldav;
  const double* dinv;       /* Jacobi inverse diagonal; NULL = no preconditioner */
  int64_t m;                /* projection width (0 = no augmenting basis) */
  const double* B;          /* augmenting basis, N x m */
  int64_t ldb;
  const double* cross;      /* cached A*B, N x m (DirectReducedProjection.cross) */
  int64_t ldc;
  const double* L;          /* Linv = L^{-1}, inverse of the lower Cholesky factor of the
                               leading wchol block (host dtrtri), lower triangular */
  int64_t ldl;
  int64_t wchol;
  const double* sqd;        /* sqrt-diagonal factor blocks for rows wchol..m-1 */
  double* mu;               /* m */
  double* coef;             /* vcap: block-CGS coefficients */
  rk_pcg_state* st;
  double* alpha_h;          /* vcap */
  double* gamma_h;          /* vcap */
  double* rz_h;             /* vcap */
  double* res_h;            /* vcap + 1: residual norms, res_h[0] = ||r_0|| */
  double* partials;         /* workspace, rk_pcg_workspace_doubles() */
  int64_t partials_len;
  uint32_t* tickets;        /* RK_PCG_TICKETS zero-initialised counters */
  int32_t mode;             /* 0 cg, 1 fom (two CGS sweeps), 2 fom with paper beta */
  int32_t linv_full;        /* 1: L holds F^{-1} = L^{-T} L^{-1} of the dense block (full,
                             * symmetric); 0: L holds L^{-1} (lower triangular) */
} rk_pcg_plan;

/* SSOR preconditioner state for a device-stepped PCG run (rk_pcg_*_ssor): the
 * arguments of rk_ssor_apply. Every application inside a call uses the next
 * epoch after `epoch`; the caller advances `epoch` by the applications made
 * (1 for the entry, nsteps for a batch of steps). */
typedef struct rk_ssor_plan {
  const double* dw;    /* fl(diag / omega) */
  const double* d;     /* diag(A) */
  double* work;        /* n doubles */
  int32_t* flags;      /* 2n, zero-initialised once */
  uint32_t* counters;  /* 2 */
  const int32_t* order_fwd; /* rows of the forward / backward sweep by dependency */
  const int32_t* order_bwd; /* level (rk_ssor_levels, sorted); NULL = natural order */
  int32_t epoch;       /* last epoch used */
} rk_ssor_plan;

const char* rk_last_error(void);
int rk_device_sm_count(void);

/* Doubles of workspace a plan needs for n rows, projection width m, vcap columns. */
int64_t rk_pcg_workspace_doubles(int64_t n, int64_t m, int64_t vcap);
/* Doubles of workspace the reductions below need for n rows / m columns. */
int64_t rk_reduce_workspace_doubles(int64_t n, int64_t m);
/* Doubles of split-K workspace rk_gram needs. */
int64_t rk_gram_workspace_doubles(int64_t n, int64_t m1, int64_t m2);
/* Doubles of split-K workspace rk_gram_upper needs for the same col_off. */
int64_t rk_gram_upper_workspace_doubles(int64_t n, int64_t m1, int64_t m2, int64_t col_off);

/* ---- augmented PCG (krylov.py:181-345) ------------------------------------ */
/* Entry: z = M^{-1} r0, rz, ||r0|| into res_h[0], mu = F^{-1} cross'z, p_0 = z - B mu
 * (krylov.py:268,290-292). Sets st->rz and st->rr; leaves st->k = 0. */
int rk_pcg_entry(const rk_pcg_plan* plan, void* stream);
/* nsteps full iterations for a CSR operator (K1,K3,K4,K5 per step); steps after
 * convergence/breakdown are no-ops, so the host may overshoot. */
int rk_pcg_steps(const rk_pcg_plan* plan, int32_t nsteps, int64_t kmax_hint, void* stream);
/* The same with z = M^{-1} r applied by the SSOR sweeps over plan->A
 * (preconditioners.py:64-90) instead of the fused Jacobi scaling (plan->dinv is
 * ignored): per step SpMV, update of x and r (+ ||r||^2), forward and backward
 * sweep, r'z and cross'z, direction -- all from the device state, no host
 * synchronisation inside a batch (krylov.py:294-340 with M = SSOR). */
int rk_pcg_entry_ssor(const rk_pcg_plan* plan, const rk_ssor_plan* ssor, void* stream);
int rk_pcg_steps_ssor(const rk_pcg_plan* plan, const rk_ssor_plan* ssor, int32_t nsteps, int64_t kmax_hint,
                      void* stream);
/* Persistent single-cluster solver for small systems (pcg_cluster.cu): ONE
 * thread-block cluster of <= 16 CTAs runs the iterations of rk_pcg_steps
 * (same statements, cg / fom / paper beta) from st->k until convergence,
 * breakdown or k == kend, with the scalars exchanged through distributed
 * shared memory and no further launches (krylov.py:300-340 for latency-bound
 * sizes such as BASELINE configs[0]). Eligible: a CSR operator, n <=
 * rk_pcg_cluster_max_rows(), m <= 64, fom keeps A p_k (ldav > 0); needs
 * kend + 1 <= vcap. Like rk_pcg_steps it follows rk_pcg_entry and may be
 * called again to continue (e.g. after the caller grew V). */
int rk_pcg_cluster_eligible(const rk_pcg_plan* plan);
int64_t rk_pcg_cluster_max_rows(void);
int rk_pcg_run_cluster(const rk_pcg_plan* plan, int64_t kend, void* stream);
/* Generic-operator pieces (ReducedSpdOperator, krylov.py:60-83): the caller writes
 * A p_k into AV column k (or the AV vector), then calls these three in order. */
int rk_pcg_curvature(const rk_pcg_plan* plan, void* stream);
int rk_pcg_update(const rk_pcg_plan* plan, void* stream);
int rk_pcg_direction(const rk_pcg_plan* plan, int64_t kmax_hint, void* stream);

/* ---- sparse kernels (linalg.py:138-174, preconditioners.py:50-61) -------- */
/* y = A x (linalg.py:138-148, scipy csr_matvec). */
int rk_spmv(const rk_csr* A, const double* x, double* y, void* stream);
/* Y = A X for m columns (linalg.py:173, scipy csr_matvecs). */
int rk_spmm(const rk_csr* A, int64_t m, const double* X, int64_t ldx, double* Y,
            int64_t ldy, void* stream);
/* diag(A) and 1/diag(A); *bad_row (device int64) = first row with diag <= 0, or -1
 * (preconditioners.py:54-58, linalg.py:114-119). */
int rk_csr_diagonal(const rk_csr* A, double* diag, double* dinv, int64_t* bad_row,
                    void* stream);
/* SSOR application z = M^{-1} r, M = (D/w + L) D^{-1} (D/w + L)' with A = L + D + L'
 * (preconditioners.py:64-90): forward sweep over A's lower triangle into work
 * (n doubles), then the backward sweep over its upper triangle with rhs work * d.
 * dw = fl(d / w), d = diag(A). Sync-free triangular solves: flags (2n int32,
 * zero-initialised once) are compared against epoch, which the caller increases
 * with every application; counters: 2 uint32 (reset by the call). order_fwd /
 * order_bwd (n int32 each, or NULL for the natural order): the rows of each
 * sweep sorted by dependency level, so whole levels are in flight together;
 * the result does not depend on them. */
int rk_ssor_apply(const rk_csr* A, const double* dw, const double* d, const double* r, double* z, double* work,
                  int32_t* flags, uint32_t* counters, int32_t epoch, const int32_t* order_fwd,
                  const int32_t* order_bwd, void* stream);
/* levels[i] = 1 + max levels[j] over row i's strictly lower (upper != 0: strictly
 * upper) entries: the dependency depth of row i in the forward (backward)
 * sweep. flags: n int32 compared against epoch as in rk_ssor_apply. */
int rk_ssor_levels(const rk_csr* A, int32_t upper, int32_t* levels, int32_t* flags, uint32_t* counter,
                   int32_t epoch, void* stream);
/* bval[s] = perm[s] >= 0 ? val[perm[s]] : 0 for s < 9*nblk: refresh the
 * 3x3-block slot values of a matrix whose pattern (and perm) was built once
 * for the sequence. */
int rk_bsr3_gather(int64_t nblk, const int32_t* perm, const double* val, double* bval, void* stream);
/* out[s] = perm[s] >= 0 ? val[perm[s]] : 0 for s < total (the scalar SELL-32
 * values of a new matrix on a known pattern). */
int rk_sell_gather(int64_t total, const int32_t* perm, const double* val, double* out, void* stream);
/* Sliced-ELL view of a CSR pattern built on the device (host
 * specification: linalg.py _bsr3_from_host / _sell1_from_host, which these
 * replace; the reference has no such view -- its SpMV is scipy csr_matvec,
 * recykl/linalg.py:138-148). bdim = 3: 3x3 blocks (rows 3b..3b+2 of equal
 * length with aligned column triples), bdim = 1: scalar rows of at most
 * max_len entries. Pass 1 (plan): len_ws[n / bdim] = (block) row lengths,
 * sptr[nsl + 1] = slice offsets in slots (nsl = ceil(n / bdim / 32)),
 * *nslot (device int64) = total slots, *bad (device int32) = 1 when the
 * pattern does not qualify. Pass 2 (fill, after the caller read *nslot and
 * allocated): scol[nslot] = (block) column per slot, perm[vals * nslot]
 * (vals = 9 or 1) = CSR index gathered into each value slot or -1 -- the
 * operands of rk_bsr3_gather / rk_sell_gather. */
int rk_sell_plan(int64_t n, const int32_t* rowptr, const int32_t* col, int32_t bdim, int32_t max_len,
                 int32_t* len_ws, int32_t* sptr, int64_t* nslot, int32_t* bad, void* stream);
int rk_sell_fill(int64_t n, const int32_t* rowptr, const int32_t* col, int32_t bdim, const int32_t* len_ws,
                 const int32_t* sptr, int64_t nslot, int32_t* scol, int32_t* perm, void* stream);
/* Largest |A_ij - A_ji| over stored entries and max|A_ij| (device doubles [2]);
 * replaces the scipy transpose difference of SparseSpdMatrix._validate
 * (linalg.py:105-113). Requires sorted columns. */
int rk_csr_asymmetry(const rk_csr* A, double* out2, double* ws, int64_t ws_len,
                     uint32_t* tickets, void* stream);

/* ---- dense tall-skinny kernels (krylov.py:80-81,151-156,291,326; linalg.py:174;
 *      pod.py:91-93) ---------------------------------------------------------- */
/* out[0:m] = B' x (deterministic split reduction). */
int rk_gemv_t(int64_t n, int64_t m, const double* B, int64_t ldb, const double* x,
              double* out, double* ws, int64_t ws_len, void* stream);
/* y = B c (op 0), y = y0 + B c (op 1), y = y0 - B c (op 2); y may alias y0. */
int rk_gemv_n(int64_t n, int64_t m, const double* B, int64_t ldb, const double* c,
              const double* y0, double* y, int32_t op, void* stream);
/* out[0] = x'y (deterministic). */
int rk_dot(int64_t n, const double* x, const double* y, double* out, double* ws,
           int64_t ws_len, uint32_t* tickets, void* stream);
/* Out[:, j] = V[:, j] / s[j] (threestage.py:482-483). */
int rk_scale_columns(int64_t n, int64_t m, const double* V, int64_t ldv, const double* s,
                     double* out, int64_t ldo, void* stream);
/* y = a x + b y with numpy's rounding (no fma contraction). */
int rk_axpby(int64_t n, double a, const double* x, double b, double* y, void* stream);
/* y = x0 - y (b - A x, krylov.py:263, threestage.py:277) */
int rk_sub_from(int64_t n, const double* x0, double* y, void* stream);

/* ---- FP64 tensor-core (DMMA) contractions ---------------------------------- */
/* G (m1 x m2, col-major ldg) = X' Y, X: N x m1, Y: N x m2 (linalg.py:174
 * `B.T @ AB`, krylov.py:152, threestage.py:320). Split-K over N with a fixed-order
 * combine. ws: rk_gram_workspace_doubles(n, m1, m2). */
int rk_gram(int64_t n, int64_t m1, const double* X, int64_t ldx, int64_t m2,
            const double* Y, int64_t ldy, double* G, int64_t ldg, double* ws,
            int64_t ws_len, void* stream);
/* Upper-triangle variant for a block G = X'Y of a symmetric matrix whose column b
 * is global column b + col_off (row a is global row a): 64x64 tiles strictly below
 * the diagonal are skipped and left undefined; the caller mirrors the upper part.
 * Halves the flops of the POD snapshot Gram S'(AS) (pod.py:119, symmetrised by
 * the reference at pod.py:129 anyway). ws: rk_gram_upper_workspace_doubles(n, m1, m2, col_off). */
int rk_gram_upper(int64_t n, int64_t m1, const double* X, int64_t ldx, int64_t m2,
                  const double* Y, int64_t ldy, int64_t col_off, double* G, int64_t ldg,
                  double* ws, int64_t ws_len, void* stream);
/* The whole snapshot Gram Z'AZ (m x m, upper triangle, col_off 0) when A Z is
 * held as two column segments: columns [0, c1) of AZ in Y1 (the stage-1 product
 * A W), columns [c1, m) in Y2 (the A p_k the PCG run stored). One launch with
 * tiles aligned to the diagonal (pod.py:119 `S.T @ AS` on the grown block,
 * threestage.py:510-524). ws: rk_gram_upper_workspace_doubles(n, m, m, 0). */
int rk_gram_upper_split(int64_t n, int64_t m, const double* X, int64_t ldx, int64_t c1,
                        const double* Y1, int64_t ldy1, const double* Y2, int64_t ldy2,
                        double* G, int64_t ldg, double* ws, int64_t ws_len, void* stream);
/* Out (N x y) = S (N x s) C (s x y) (pod.py:91-93 `S @ coef`). */
int rk_gemm_nn(int64_t n, int64_t s, int64_t y, const double* S, int64_t lds,
               const double* C, int64_t ldc, double* Out, int64_t ldo, void* stream);

/* ---- POD reduced problem on the device (pod.py:86-97,123-131) -------------- */
/* out = 1/2 (W + W'), W_ab = (gamma_a G_ab) gamma_b. mode 0: full G. mode 1: only
 * the upper triangle of G is defined (rk_gram_upper output); its column b is
 * first multiplied by col_scale[b] (NULL = 1) and the triangle mirrored. */
int rk_pod_weighted_gram(int64_t m, const double* G, int64_t ldg, int32_t mode, const double* col_scale,
                         const double* gamma, double* out, int64_t ldo, void* stream);
/* coef[:, j] = V[:, m-1-j] / sigma[j] * gamma for j < y (V: eigenvectors of the
 * weighted Gram in ascending eigenvalue order, as LAPACK/cuSOLVER return them). */
int rk_pod_coef(int64_t m, int64_t y, const double* V, int64_t ldv, const double* sigma,
                const double* gamma, double* coef, int64_t ldc, void* stream);

/* ---- measurement hooks (bench.py only; not thread-safe) --------------------
 * Between begin and end, rk_pcg_steps brackets each of its three kernels
 * (0: K1 SpMV+curvature, 1: K3/K4 update+projection, 2: K5 direction) with
 * CUDA events on the launching stream; end synchronises and returns the
 * summed milliseconds and launch counts per kernel. */
int rk_profile_begin(void);
/* Number of kernels this library has launched since it was loaded. */
int64_t rk_launch_count(void);
/* Debug: copies up to n of the 64 x 8 globaltimer stamps of the fused update
 * tail (iteration k in row k % 64); zeros unless built with -DRK_TAIL_TRACE. */
int rk_debug_trace(uint64_t* out, int64_t n);
int rk_profile_end(double* ms4, int64_t* count4);  /* slots: spmv, update, finish, direction */
/* After rk_profile_end: total milliseconds and launches of the persistent
 * cluster solver (rk_pcg_run_cluster) between begin and end. */
int rk_profile_cluster(double* ms, int64_t* launches);

#ifdef __cplusplus
}
#endif

#endif /* PODCG_H */
