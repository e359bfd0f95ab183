"""CPU oracle for the POD-augmented CG hot path -- TEST INFRASTRUCTURE ONLY.

A numpy/scipy restatement of the reference algorithm (recykl, pure Python on
numpy/scipy, /root/reference/pkg/src/recykl). Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` leg may import this module, and only as the checker or the
CPU baseline; the product (``paper_1512_05820_b200``) never touches it.

Pinning: ``tests/test_oracle.py`` replays the reference's frozen fixtures
(``pkg/tests/fixtures/{identity_like,invariant_matrix,drifting_pod}.json``,
counters exact) and golden vectors produced by running the reference itself
(``oracle/make_golden.py`` -> ``tests/golden/*.npz``), so this restatement is
"parity pinned" against the reference's own outputs.

The arithmetic lives in numpy/scipy as in the reference (CSR products by
scipy's csr_matvec(s), BLAS dot/gemv/gemm, LAPACK dpotrf/dtrtrs/dsyevd).
Each function names the reference lines it restates.
"""

from __future__ import annotations

import math
import time
import warnings
from dataclasses import dataclass, field

import numpy as np
import scipy.linalg
import scipy.sparse

BREAKDOWN_RTOL = 1e-14   # krylov.py:36
RANK_RTOL = 1e-12        # pod.py:30


class OracleBreakdown(Exception):
    pass


class OracleNotConverged(Exception):
    def __init__(self, msg, partial):
        super().__init__(msg)
        self.partial = partial


@dataclass
class Tally:
    """Cost counters with the semantics of InstrumentationSink (linalg.py:29-60)."""

    matvecs: int = 0
    precond: int = 0
    grams: int = 0


def as_csr(A) -> scipy.sparse.csr_matrix:
    if scipy.sparse.issparse(A):
        return scipy.sparse.csr_matrix(A)
    if hasattr(A, "to_scipy"):
        return A.to_scipy()
    return scipy.sparse.csr_matrix((A.values, A.col_indices, A.row_offsets), shape=(A.n, A.n))


# --- kernels ----------------------------------------------------------------
def matvec(A, x, tally: Tally | None):
    """linalg.py:138-148: one scipy CSR product, one matvec charged."""
    if tally is not None:
        tally.matvecs += 1
    return A @ x


def gram_with_product(A, B, tally: Tally | None):
    """linalg.py:160-174: AB by SpMM, B'(AB); 1 gram + B.cols matvecs."""
    B = np.atleast_2d(B)
    if tally is not None:
        tally.grams += 1
        tally.matvecs += B.shape[1]
    AB = A @ B
    return B.T @ AB, AB


def cholesky_lower(G):
    """linalg.py:250-267: dpotrf, raising on a failed pivot."""
    if G.shape[0] == 0:
        return np.zeros((0, 0))
    L, info = scipy.linalg.lapack.dpotrf(G, lower=1, clean=1, overwrite_a=0)
    if info != 0:
        raise np.linalg.LinAlgError(f"dpotrf info={info}")
    return L


def spd_solve(L, rhs):
    """linalg.py:239-247: forward then transposed back substitution."""
    t = scipy.linalg.solve_triangular(L, rhs, lower=True)
    return scipy.linalg.solve_triangular(L, t, lower=True, trans="T")


def eig_descending(G):
    """linalg.py:270-280: eigh with the order reversed."""
    w, V = np.linalg.eigh(G)
    return w[::-1].copy(), V[:, ::-1].copy()


class Factor:
    """Block-diagonal factor: dense Cholesky blocks and sqrt-diagonal blocks
    (krylov.py:97-132)."""

    def __init__(self):
        self.parts: list = []

    @property
    def size(self):
        return sum(p[1].shape[0] for p in self.parts)

    def add_dense(self, L):
        self.parts.append(("L", L))

    def add_sqrt_diag(self, d):
        self.parts.append(("d", np.asarray(d, dtype=np.float64)))

    def solve(self, rhs):
        out = np.empty_like(rhs, dtype=np.float64)
        i = 0
        for kind, blk in self.parts:
            m = blk.shape[0]
            out[i : i + m] = spd_solve(blk, rhs[i : i + m]) if kind == "L" else rhs[i : i + m] / (blk * blk)
            i += m
        return out


class Projection:
    """krylov.py:135-156: mu = F^{-1} (cross' z) from the cached cross = A B."""

    def __init__(self, cross, factor):
        self.cross = np.asarray(cross, dtype=np.float64)
        self.factor = factor

    def __call__(self, z):
        return self.factor.solve(self.cross.T @ z)


def assembled_projection(apply, B):
    """krylov.py:147-153: m operator applications, Cholesky of B'AB."""
    cross = np.column_stack([apply(B[:, i]) for i in range(B.shape[1])])
    G = B.T @ cross
    f = Factor()
    f.add_dense(cholesky_lower(0.5 * (G + G.T)))
    return Projection(cross, f)


@dataclass
class PcgOut:
    k: int
    vhat: np.ndarray
    V: np.ndarray
    gamma: np.ndarray
    history: np.ndarray
    x: np.ndarray
    converged: bool = True


def aug_pcg(apply, b, yhat0=None, Y=None, proj=None, dinv=None, tol=0.0, *, mode="cg", paper_beta=False,
            relative=False, max_iter=None, r0=None, tally=None, precond_counted=None, monitor=None,
            identity_precond=False):
    """Restatement of augmented_pcg (krylov.py:181-345).

    ``apply`` charges its own matvecs; ``dinv`` is the Jacobi inverse diagonal or
    a callable preconditioner (None: no preconditioner, or the identity when
    ``identity_precond``).
    """
    b = np.asarray(b, dtype=np.float64)
    n = b.shape[0]
    has_pc = dinv is not None or identity_precond

    def precondition(r):
        if has_pc and tally is not None:
            tally.precond += 1
        if callable(dinv):
            return dinv(r)
        return r * dinv if dinv is not None else r.copy()

    if Y is not None and Y.shape[1] == 0:
        Y = None
    if Y is not None:
        x = Y @ yhat0
        if proj is None:
            proj = assembled_projection(apply, Y)
    else:
        x = np.zeros(n)
    if r0 is not None:
        r = np.array(r0, dtype=np.float64)
    elif Y is not None and np.any(x):
        r = b - apply(x)
    else:
        r = b.copy()
    thr = tol * np.linalg.norm(b) if relative else tol
    hist = [float(np.linalg.norm(r))]
    if monitor is not None:
        monitor(0, x.copy())

    alphas, dirs, gammas, adirs, rzs = [], [], [], [], []

    def pack(k, ok):
        V = np.column_stack(dirs) if dirs else np.zeros((n, 0))
        return PcgOut(k, np.asarray(alphas), V, np.asarray(gammas), np.asarray(hist), x, ok)

    if hist[0] <= thr:
        return pack(0, True)
    if max_iter is None:
        max_iter = n
    z = precondition(r)
    p = z - Y @ proj(z) if Y is not None else z.copy()
    rz = float(r @ z)
    for k in range(max_iter):
        Ap = apply(p)
        gamma = float(p @ Ap)
        if not np.isfinite(gamma) or gamma <= BREAKDOWN_RTOL * float(p @ p):
            raise OracleBreakdown(f"curvature {gamma:.3e} at iteration {k}")
        alpha = rz / gamma
        x = x + alpha * p
        r = r - alpha * Ap
        alphas.append(alpha)
        dirs.append(p)
        gammas.append(gamma)
        rzs.append(rz)
        if mode == "fom":
            adirs.append(Ap)
        hist.append(float(np.linalg.norm(r)))
        if monitor is not None:
            monitor(k + 1, x.copy())
        if hist[-1] <= thr:
            return pack(k + 1, True)
        z = precondition(r)
        rz_next = float(r @ z)
        mu = proj(z) if Y is not None else None
        if mode == "cg":
            p = z + (rz_next / rz) * p
            if Y is not None:
                p -= Y @ mu
        elif mode == "fom":
            p = z - Y @ mu if Y is not None else z.copy()
            if paper_beta:
                for i in range(len(dirs)):
                    p = p + (rz_next / rzs[i]) * dirs[i]
            else:
                for _sweep in range(2):          # modified Gram-Schmidt, twice
                    for i in range(len(dirs)):
                        p = p - (float(adirs[i] @ p) / gammas[i]) * dirs[i]
        else:
            raise ValueError(mode)
        rz = rz_next
    raise OracleNotConverged("max_iter", pack(max_iter, False))


def direct_solve(A, b, W, tally):
    """krylov.py:396-411: (what, L, AW)."""
    G, AW = gram_with_product(A, W, tally)
    L = cholesky_lower(0.5 * (G + G.T))
    return spd_solve(L, W.T @ b), L, AW


class ReducedOp:
    """krylov.py:60-83: p -> Y'(A(Yp)), products recorded."""

    def __init__(self, A, Y, tally):
        self.A, self.Y, self.tally = A, Y, tally
        self.full, self.reduced = [], []

    def __call__(self, p):
        f = matvec(self.A, self.Y @ p, self.tally)
        red = self.Y.T @ f
        self.full.append(f)
        self.reduced.append(red)
        return red


# --- POD / truncation -------------------------------------------------------
def energy_dim(s2, eps):
    """pod.py:58-83."""
    s2 = np.asarray(s2, dtype=np.float64)
    total = float(np.sum(s2))
    rank = int(np.sum(s2 > RANK_RTOL * s2[0]))
    hit = np.nonzero((np.cumsum(s2) / total)[:rank] >= eps)[0]
    return rank if hit.size == 0 else int(hit[0]) + 1


def pod_from_gram(G, S, gamma, eps):
    """pod.py:86-97,123-131: (basis, sigma, y, coef)."""
    Gw = gamma[:, None] * G * gamma[None, :]
    lam, V = eig_descending(0.5 * (Gw + Gw.T))
    sigma = np.sqrt(np.maximum(lam, 0.0))
    y = energy_dim(np.maximum(sigma, 0.0) ** 2, eps)
    coef = (V[:, :y] / sigma[:y]) * gamma[:, None]
    return S @ coef, np.maximum(sigma, 0.0), y, coef


def rbf_weights(history, window):
    """weights.py:119-128 with zero padding (weights.py:76-80)."""
    width = max(e.shape[0] for e in history)
    w = max(1, min(int(window), len(history)))
    out = np.zeros(width)
    for i in range(1, w + 1):
        e = history[len(history) - i]
        pad = np.zeros(width)
        pad[: e.shape[0]] = e
        out += (1.0 / 2.0 ** (i - 1)) * pad
    return out


def prev_weights(history):
    width = max(e.shape[0] for e in history)
    out = np.zeros(width)
    out[: history[-1].shape[0]] = history[-1]
    return out


def pod_svd(S, gamma, chalf, eps):
    """pod.py:134-157: thin SVD of chalf (S gamma), zero-padded spectrum."""
    factored = np.atleast_2d(chalf) @ (S * gamma)
    _, sigma, Vt = np.linalg.svd(factored, full_matrices=False)
    V = Vt.T
    s = S.shape[1]
    if sigma.shape[0] < s:
        sigma = np.concatenate([sigma, np.zeros(s - sigma.shape[0])])
        Vf = np.zeros((s, s))
        Vf[:, : V.shape[1]] = V
        V = Vf
    y = energy_dim(sigma**2, eps)
    coef = (V[:, :y] / sigma[:y]) * gamma[:, None]
    return S @ coef, sigma, y, coef


def enforce_a_orth(Y, A, tally):
    """truncation.py:191-206: Y L^{-T} with Y'AY = L L'."""
    G, _ = gram_with_product(A, Y, tally)
    L = cholesky_lower(0.5 * (G + G.T))
    return scipy.linalg.solve_triangular(L, Y.T, lower=True).T, L


def deflation(Z, A, m, stage1_dim, tally):
    """truncation.py:152-188 (linalg.py:293-307 for the generalized EVD)."""
    m = min(int(m), Z.shape[1])
    G, AZ = gram_with_product(A, Z, tally)
    K = AZ.T @ AZ
    w, V = scipy.linalg.eigh(0.5 * (K + K.T), 0.5 * (G + G.T))
    keep = V[:, :m]  # the m smallest harmonic Ritz values (scipy's order is ascending)
    Y = Z @ keep
    gy = keep.T @ G @ keep
    L = cholesky_lower(0.5 * (gy + gy.T))
    Yo = scipy.linalg.solve_triangular(L, Y.T, lower=True).T
    return Yo, (m if stage1_dim is None else min(stage1_dim, m)), w[:m]


class Ssor:
    """preconditioners.py:64-90: M = (D/w + L) D^{-1} (D/w + L)', z = M^{-1} r by
    a forward and a backward triangular sweep."""

    def __init__(self, A, omega=1.0):
        A = as_csr(A)
        d = A.diagonal()
        self.d = d
        low = scipy.sparse.tril(A, k=-1) + scipy.sparse.diags(d / omega)
        self.low = scipy.sparse.csr_matrix(low)
        self.up = scipy.sparse.csr_matrix(low.T)

    def __call__(self, r):
        import scipy.sparse.linalg as spla

        u = spla.spsolve_triangular(self.low, r, lower=True)
        u = u * self.d
        return spla.spsolve_triangular(self.up, u, lower=False)


@dataclass
class Config:
    """SolverConfig + TruncationConfig fields the hot path reads
    (threestage.py:63-72, truncation.py:40-83)."""

    strategy: str = "pod-a-rbf"
    nu_y: float = 1.0
    nu_w: float = 0.5
    storage_cap: float = math.inf
    stage1_threshold: float = 1.0
    full_orth: bool = False
    max_dim: int | None = None
    stage1_dim: int | None = None
    mode: str = "fom"
    recycle: bool = True
    max_iter: int | None = None
    rbf_window: int | None = None
    deflate_dim: int | None = None


def _cap(v, pin, hard):
    out = v if pin is None else min(v, pin)
    return max(1, min(out, hard))


@dataclass
class State:
    n: int
    Y: np.ndarray
    idx: list = field(default_factory=list)
    seen: int = 0
    history: list = field(default_factory=list)
    last_trunc: int = 0


@dataclass
class Report:
    j: int
    stage1_dim: int = 0
    stage2_iters: int = 0
    stage3_iters: int = 0
    matvecs: int = 0
    precond_applies: int = 0
    final_residual: float = float("nan")
    converged: bool = True
    truncated: bool = False
    spectrum: np.ndarray | None = None
    wall_time: float = 0.0
    stage3_basis: np.ndarray | None = None


class InnerProjection:
    """threestage.py:143-220 (phi = 1)."""

    def __init__(self, A, Y, tally, tol, mode):
        self.A, self.Y, self.tally, self.tol, self.mode = A, Y, tally, tol, mode
        self.max_iter = 3 * Y.shape[1] + 10
        self.op = ReducedOp(A, Y, tally)
        self.factor = Factor()
        self.bases, self.crosses = [], []

    def add(self, B, cross, kind, payload):
        if B.shape[1] == 0:
            return
        self.bases.append(B)
        self.crosses.append(cross)
        (self.factor.add_dense if kind == "L" else self.factor.add_sqrt_diag)(payload)

    def __call__(self, z):
        bhat = self.Y.T @ matvec(self.A, z, self.tally)
        y = self.Y.shape[1]
        B = np.hstack(self.bases) if self.bases else np.zeros((y, 0))
        cross = np.hstack(self.crosses) if self.crosses else np.zeros((y, 0))
        tol = max(self.tol, 1e-13 * float(np.linalg.norm(bhat)))
        if B.shape[1]:
            ybase = self.factor.solve(B.T @ bhat)
            r0 = bhat - cross @ ybase
            handle = Projection(cross, self.factor)
        else:
            ybase, r0, handle = None, bhat.copy(), None
        mark = len(self.op.reduced)
        try:
            res = aug_pcg(self.op, bhat, ybase, B if B.shape[1] else None, handle, None, tol, mode=self.mode,
                          max_iter=self.max_iter, r0=r0)
        except OracleNotConverged as exc:
            res = exc.partial
        if res.k > 0:
            self.add(res.V, np.column_stack(self.op.reduced[mark : mark + res.k]), "d", np.sqrt(res.gamma))
        return res.x


def solve_one(A, b, xbar, state: State, eps, cfg: Config, dinv=None, identity_precond=False, eps_hat=None,
              eps_inner=None, chalf=None):
    """threestage.py:230-452 (solve_system) + 455-547 (update_basis)."""
    A = as_csr(A)
    tally = Tally()
    t0 = time.perf_counter()
    j = state.seen + 1
    rep = Report(j=j)
    b = np.asarray(b, dtype=np.float64)
    if xbar is not None and not np.any(xbar):
        xbar = None
    r0 = b - matvec(A, xbar, tally) if xbar is not None else b.copy()
    eps_hat = 1e-4 * eps if eps_hat is None else eps_hat
    eps_inner = 1e-2 * eps if eps_inner is None else eps_inner
    apply = lambda v: matvec(A, v, tally)  # noqa: E731
    y = state.Y.shape[1]
    Y = state.Y
    stage1_gram = None
    idx: list = []
    yhat = np.zeros(0)

    def run3(*args, **kw):
        try:
            return aug_pcg(*args, **kw), True
        except OracleNotConverged as exc:
            return exc.partial, False

    kw3 = dict(mode=cfg.mode, max_iter=cfg.max_iter, tally=tally, identity_precond=identity_precond)
    if y == 0 or not cfg.recycle:
        res3, rep.converged = run3(apply, r0, dinv=dinv, tol=eps, **kw3)
        basis3 = np.zeros((A.shape[0], 0))
    else:
        idx = list(state.idx)
        W = Y[:, idx]
        w = len(idx)
        what, L, AW = direct_solve(A, r0, W, tally)
        stage1_gram = L @ L.T if w == y else None
        if y > w:
            What = np.eye(y)[:, idx]
            cross_w = Y.T @ AW
            red = ReducedOp(A, Y, tally)
            bhat = Y.T @ r0
            f1 = Factor()
            f1.add_dense(L)
            try:
                res2 = aug_pcg(red, bhat, what, What, Projection(cross_w, f1), None, eps_hat, mode=cfg.mode,
                               max_iter=3 * y + 10, r0=bhat - cross_w @ what)
            except OracleNotConverged as exc:
                res2 = exc.partial
            yhat = res2.x
            vhat2, Phat, ghat = res2.vhat, res2.V, res2.gamma
            AVhat = np.column_stack(red.full[: res2.k]) if res2.k else np.zeros((A.shape[0], 0))
            rep.stage2_iters = res2.k
        else:
            yhat = np.zeros(y)
            yhat[idx] = what
            vhat2, Phat, ghat, AVhat = np.zeros(0), np.zeros((y, 0)), np.zeros(0), np.zeros((A.shape[0], 0))
        if not cfg.full_orth:
            basis3 = np.hstack([W, Y @ Phat if Phat.shape[1] else np.zeros((A.shape[0], 0))])
            cross3 = np.hstack([AW, AVhat])
            f3 = Factor()
            f3.add_dense(L)
            if ghat.size:
                f3.add_sqrt_diag(np.sqrt(ghat))
            start = np.concatenate([what, vhat2])
            res3, rep.converged = run3(apply, r0, start, basis3, Projection(cross3, f3), dinv, eps,
                                       r0=r0 - cross3 @ start, **kw3)
        else:
            proj = InnerProjection(A, Y, tally, eps_inner, cfg.mode)
            proj.add(np.eye(y)[:, idx], Y.T @ AW, "L", L)
            if Phat.shape[1]:
                proj.add(Phat, Y.T @ AVhat, "d", np.sqrt(ghat))
            basis3 = Y
            r03 = r0 - AW @ what - (AVhat @ vhat2 if vhat2.size else 0.0)
            res3, rep.converged = run3(apply, r0, yhat, Y, proj, dinv, eps, r0=r03, **kw3)
    x = res3.x if xbar is None else xbar + res3.x
    rep.stage1_dim = len(idx)
    rep.stage3_iters = res3.k
    rep.final_residual = float(res3.history[-1])
    rep.stage3_basis = basis3
    _fold(state, yhat, res3, cfg, A, tally, stage1_gram, rep, chalf=chalf)
    rep.matvecs, rep.precond_applies = tally.matvecs, tally.precond
    rep.wall_time = time.perf_counter() - t0
    return x, rep


def _fold(state: State, yhat, res3: PcgOut, cfg: Config, A, tally, stage1_gram, rep, chalf=None):
    """update_basis (threestage.py:455-547) with compress (truncation.py:209-257):
    pod-a-*, pod-ctc-* (then A-orthonormalised), deflate and none."""
    j = state.seen + 1
    if not cfg.recycle:
        state.seen = j
        return
    k = res3.k
    if k > 0:
        sq = np.sqrt(res3.gamma)
        y_old = state.Y.shape[1]
        if cfg.stage1_threshold >= 1.0:
            admitted = list(range(k))
        else:
            share = res3.gamma / np.sum(res3.gamma)
            admitted = [i for i in range(k) if share[i] > cfg.stage1_threshold]
        Z = np.hstack([state.Y, res3.V / sq]) if y_old else res3.V / sq
        idx = state.idx + [y_old + i for i in admitted]
        eta = np.concatenate([np.asarray(yhat, dtype=np.float64), res3.vhat * sq])
    else:
        Z = state.Y
        idx = list(state.idx)
        eta = np.asarray(yhat, dtype=np.float64).copy()
    if eta.size:
        state.history.append(eta.copy())
    if Z.shape[1] > cfg.storage_cap and cfg.strategy != "none":
        if cfg.strategy == "deflate":
            basis, wk, mu = deflation(Z, A, cfg.deflate_dim, cfg.stage1_dim, tally)
            state.history.clear()
            state.Y, state.idx, state.last_trunc = basis, list(range(wk)), j
            rep.truncated, rep.spectrum = True, mu
            state.seen = j
            return
        if cfg.strategy.endswith("prev"):
            gam = prev_weights(state.history)
        else:
            window = cfg.rbf_window if cfg.rbf_window is not None else len(state.history)
            gam = rbf_weights(state.history, window)
        if cfg.strategy.startswith("pod-ctc"):
            basis, sigma, ycrit, coef = pod_svd(Z, gam, chalf, cfg.nu_y)
        else:
            if stage1_gram is not None and cfg.mode == "fom" and k > 0:
                y_old = state.Y.shape[1]
                G = np.zeros((y_old + k, y_old + k))
                G[:y_old, :y_old] = stage1_gram
                G[y_old:, y_old:] = np.eye(k)
            else:
                G, _ = gram_with_product(A, Z, tally)
            basis, sigma, ycrit, coef = pod_from_gram(G, Z, gam, cfg.nu_y)
        yk = _cap(ycrit, cfg.max_dim, ycrit)
        wk = _cap(energy_dim(sigma ** 2, cfg.nu_w), cfg.stage1_dim, yk)
        if cfg.strategy.startswith("pod-ctc"):
            basis, _ = enforce_a_orth(basis[:, :yk], A, tally)
        state.history.clear()
        state.Y = basis[:, :yk]
        state.idx = list(range(wk))
        state.last_trunc = j
        rep.truncated = True
        rep.spectrum = sigma
    else:
        state.Y = Z
        state.idx = idx
    state.seen = j


def run_sequence(seq, cfg: Config, precond: str | None = "jacobi", *, max_systems=None, keep=False):
    """threestage.py:550-596 with a Jacobi, SSOR ("ssor" / "ssor:<omega>",
    preconditioners.py:64-104) or no / identity preconditioner per system.

    Returns (solutions, reports, bases) where bases[j] is the basis after system j
    when ``keep``."""
    state = None
    xs, reps, bases = [], [], []
    for j, spec in enumerate(seq, start=1):
        if max_systems is not None and j > max_systems:
            break
        A = as_csr(spec.A)
        if state is None:
            state = State(n=A.shape[0], Y=np.zeros((A.shape[0], 0)))
        if precond == "jacobi":
            dinv = 1.0 / A.diagonal()
        elif precond is not None and precond.startswith("ssor"):
            dinv = Ssor(A, float(precond.split(":")[1]) if ":" in precond else 1.0)
        else:
            dinv = None
        x, rep = solve_one(A, spec.b, spec.xbar, state, spec.tol, cfg, dinv=dinv,
                           identity_precond=(precond == "identity"), chalf=getattr(seq, "C", None))
        xs.append(x)
        reps.append(rep)
        if keep:
            bases.append(state.Y.copy())
        if not rep.converged:
            break
    return xs, reps, bases
