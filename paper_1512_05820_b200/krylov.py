"""Augmented preconditioned CG on the device (``recykl/krylov.py``).

Same public surface as the reference: ``LinearOperator`` (krylov.py:39-45),
``MatrixOperator`` (48-57), ``ReducedSpdOperator`` (60-83),
``BlockDiagFactor`` (97-132), ``DirectReducedProjection`` (135-156),
``AugmentedPcgResult`` (159-178), ``augmented_pcg`` (181-345), ``pcg``
(348-386), ``direct_reduced_solve`` (396-411).

Two drivers run the same kernels:

* the fused path (CSR operator, Jacobi/identity/no preconditioner, no
  monitor, direct projection): every iteration is launched from C
  (``rk_pcg_steps``) in batches; convergence, breakdown and the step scalars
  live in device memory and the host reads the 96-byte state once per batch;
* the stepped path (any ``LinearOperator``, a callable reduced solver, or a
  monitor): the same update/direction kernels, one host synchronisation per
  iteration so Python callbacks can run in between.

Directions are written straight into the column-major block V (column k is
p_k), so the result's ``V`` needs no ``column_stack`` (krylov.py:273).
Returned ``x`` and ``V`` are device tensors; ``vhat``, ``gamma`` and
``residual_history`` are small host arrays, as in the reference.
"""

from __future__ import annotations

import os
from dataclasses import dataclass

import numpy as np
import torch

from . import _native as nat
from .errors import Breakdown, DimensionMismatch, NotConverged, NotPositiveDefinite
from .linalg import (
    F64,
    DenseLowerTriangular,
    InstrumentationSink,
    SparseSpdMatrix,
    as_block,
    as_matrix,
    as_vector,
    block_ld,
    dense_cholesky,
    dot,
    empty_block,
    gemv_n,
    gemv_t,
    gram,
    norm,
    spmm,
    spmv,
    spmv_into,
    to_numpy,
)
from .preconditioners import IdentityPreconditioner, JacobiPreconditioner, SsorPreconditioner

_BREAKDOWN_RTOL = 1e-14  # krylov.py:36 (applied on the device, spmv.cu)


class LinearOperator:
    """SPD operator on R^dim acting on device vectors."""

    dim: int
    device: torch.device

    def apply(self, x) -> torch.Tensor:
        raise NotImplementedError


class MatrixOperator(LinearOperator):
    """A device CSR matrix as an operator, charging a shared sink."""

    def __init__(self, A, sink: InstrumentationSink | None = None):
        self.A = as_matrix(A)
        self.sink = sink
        self.dim = self.A.n
        self.device = self.A.device

    def apply(self, x):
        return spmv(self.A, x, self.sink)


class ReducedSpdOperator(LinearOperator):
    """p -> Y'(A(Yp)) without forming Y'AY (krylov.py:60-83): GEMV-N, SpMV,
    GEMV-T on the device. With ``record_products`` the full-space products
    A(Yp) are kept (as columns of one device block) for later stages."""

    def __init__(self, A, Y, sink=None, record_products: bool = False):
        self.A = as_matrix(A)
        self.device = self.A.device
        self.Y = as_block(Y, self.device)
        self.sink = sink
        self.dim = int(self.Y.shape[1])
        self._record = record_products
        self._full = None
        self._count = 0
        self.reduced_products: list | None = [] if record_products else None

    def apply(self, p):
        pd = as_vector(p, self.device)
        full = spmv(self.A, gemv_n(self.Y, pd), self.sink)
        reduced = gemv_t(self.Y, full)
        if self._record:
            if self._full is None or self._count >= self._full.shape[1]:
                cap = max(16, 2 * self._count)
                grown = empty_block(self.A.n, cap, self.device)
                if self._count:
                    grown[:, : self._count].copy_(self._full[:, : self._count])
                self._full = grown
            self._full[:, self._count].copy_(full)
            self._count += 1
            self.reduced_products.append(reduced)
        return reduced

    @property
    def full_products(self):
        if not self._record:
            return None
        return [self._full[:, i] for i in range(self._count)]

    def full_products_block(self, count: int | None = None) -> torch.Tensor:
        """Column-stacked A(Y p_i) for the first ``count`` applications."""
        c = self._count if count is None else int(count)
        if c == 0 or self._full is None:
            return empty_block(self.A.n, 0, self.device)
        return self._full[:, :c]


def _as_operator(op, sink):
    if isinstance(op, LinearOperator):
        return op
    if isinstance(op, SparseSpdMatrix):
        return MatrixOperator(op, sink)
    if hasattr(op, "row_offsets") or hasattr(op, "tocsr"):
        return MatrixOperator(SparseSpdMatrix.from_host(op), sink)
    arr = to_numpy(op) if isinstance(op, torch.Tensor) else np.asarray(op, dtype=np.float64)
    if arr.ndim == 2 and arr.shape[0] == arr.shape[1]:
        return MatrixOperator(SparseSpdMatrix.from_dense(arr), sink)
    raise DimensionMismatch("unsupported operator type")


class DenseReducedOperator(LinearOperator):
    """p -> G p with the reduced matrix G = Y'AY already formed (y x y, host).

    Stands in for ReducedSpdOperator (krylov.py:60-83) in the nested reduced
    solves (stage 2, the phi = 1 inner projection) once Y'AY is known -- the
    stage-1 Gram when W = Y, otherwise one SpMM + DMMA Gram per system. Every
    application is charged one matvec to the sink, exactly as the reference's
    implicit operator, and the reduced products are recorded. Equal to
    Y'(A(Y p)) up to rounding; an application costs y^2 host flops instead of
    two N x y GEMVs, an SpMV and a host round trip on the device."""

    def __init__(self, G, sink=None, record_products: bool = False):
        self.G = np.ascontiguousarray(np.asarray(to_numpy(G), dtype=np.float64))
        self.dim = int(self.G.shape[0])
        self.device = None
        self.sink = sink
        self.reduced_products: list | None = [] if record_products else None

    def apply(self, p):
        if self.sink is not None:
            self.sink.add_matvec()
        out = self.G @ np.asarray(to_numpy(p), dtype=np.float64)
        if self.reduced_products is not None:
            self.reduced_products.append(out)
        return out


def _host_augmented_pcg(op: DenseReducedOperator, b, yhat0, B, reduced_solver, tol, mode, paper_fom_beta,
                        relative, max_iter, r0, monitor):
    """augmented_pcg (krylov.py:181-345) for a small dense reduced operator, in
    host numpy: the same statements in the same order (so the same rounding as
    the reference's reduced-space arithmetic), no preconditioner. Returns host
    arrays (V is y x k)."""
    n = op.dim
    b = np.asarray(to_numpy(b), dtype=np.float64)
    if b.shape[0] != n:
        raise DimensionMismatch("augmented_pcg: rhs length mismatch")
    Y = None
    if B is not None:
        Y = np.asarray(to_numpy(B), dtype=np.float64)
        if Y.ndim != 2 or Y.shape[0] != n:
            raise DimensionMismatch("augmented_pcg: basis shape mismatch")
        if Y.shape[1] == 0:
            Y = None
    if Y is not None:
        if yhat0 is None:
            raise DimensionMismatch("augmented_pcg: yhat0 required with a nonempty basis")
        yhat0 = np.asarray(to_numpy(yhat0), dtype=np.float64)
        if yhat0.shape[0] != Y.shape[1]:
            raise DimensionMismatch("augmented_pcg: yhat0 length mismatch")
        x = Y @ yhat0
        if reduced_solver is None:
            cross = np.column_stack([op.apply(Y[:, i]) for i in range(Y.shape[1])])
            g = Y.T @ cross
            L = dense_cholesky(0.5 * (g + g.T))
            reduced_solver = lambda z: L.solve_spd(cross.T @ z)  # noqa: E731
    else:
        x = np.zeros(n)
    if r0 is not None:
        r = np.array(to_numpy(r0), dtype=np.float64)
    elif Y is not None and np.any(x):
        r = b - op.apply(x)
    else:
        r = b.copy()
    threshold = tol * np.linalg.norm(b) if relative else tol
    history = [float(np.linalg.norm(r))]
    if monitor is not None:
        monitor(0, x.copy())

    def result(k, alphas, dirs, gammas, converged):
        return AugmentedPcgResult(k=k, vhat=np.asarray(alphas, dtype=np.float64),
                                  V=np.column_stack(dirs) if dirs else np.zeros((n, 0)),
                                  gamma=np.asarray(gammas, dtype=np.float64),
                                  residual_history=np.asarray(history), x=x, converged=converged)

    if history[0] <= threshold:
        return result(0, [], [], [], True)
    if max_iter is None:
        max_iter = n
    z = r.copy()
    p = z - Y @ reduced_solver(z) if Y is not None else z.copy()
    rz = float(r @ z)
    alphas, dirs, gammas, a_dirs, rz_hist = [], [], [], [], []
    for k in range(max_iter):
        Ap = op.apply(p)
        gamma = float(p @ Ap)
        if not np.isfinite(gamma) or gamma <= _BREAKDOWN_RTOL * float(p @ p):
            raise Breakdown(f"direction curvature {gamma:.3e} at iteration {k}")
        alpha = rz / gamma
        x = x + alpha * p
        r = r - alpha * Ap
        alphas.append(alpha)
        dirs.append(p)
        gammas.append(gamma)
        rz_hist.append(rz)
        if mode == "fom":
            a_dirs.append(Ap)
        history.append(float(np.linalg.norm(r)))
        if monitor is not None:
            monitor(k + 1, x.copy())
        if history[-1] <= threshold:
            return result(k + 1, alphas, dirs, gammas, True)
        z = r.copy()
        rz_next = float(r @ z)
        mu = reduced_solver(z) if Y is not None else None
        if mode == "cg":
            p = z + (rz_next / rz) * p
            if Y is not None:
                p -= Y @ mu
        elif mode == "fom":
            p = z - Y @ mu if Y is not None else z.copy()
            if paper_fom_beta:
                for i in range(len(dirs)):
                    p = p + (rz_next / rz_hist[i]) * dirs[i]
            else:
                for _ in range(2):
                    for i in range(len(dirs)):
                        p = p - (float(a_dirs[i] @ p) / gammas[i]) * dirs[i]
        else:
            raise ValueError(f"unknown mode {mode!r}")
        rz = rz_next
    raise NotConverged(f"no convergence to {threshold:.3e} within {max_iter} iterations",
                       partial=result(max_iter, alphas, dirs, gammas, False))


class BlockDiagFactor:
    """Cholesky factor of a block-diagonal Gram matrix (krylov.py:97-132):
    dense lower-triangular blocks or square roots of diagonal blocks."""

    def __init__(self):
        self._blocks: list = []
        self.size = 0
        self._dev = {}

    def append_cholesky(self, factor: DenseLowerTriangular):
        self._blocks.append(("chol", factor))
        self.size += factor.m
        self._dev.clear()

    def append_sqrt_diag(self, sqrt_diag):
        sd = np.asarray(to_numpy(sqrt_diag), dtype=np.float64)
        self._blocks.append(("sqrtdiag", sd))
        self.size += sd.shape[0]
        self._dev.clear()

    def solve_spd(self, rhs):
        rhs = np.asarray(to_numpy(rhs), dtype=np.float64)
        if rhs.shape[0] != self.size:
            raise DimensionMismatch("block factor: rhs length mismatch")
        out = np.empty_like(rhs)
        at = 0
        for kind, block in self._blocks:
            if kind == "chol":
                m = block.m
                out[at : at + m] = block.solve_spd(rhs[at : at + m])
            else:
                m = block.shape[0]
                out[at : at + m] = rhs[at : at + m] / (block * block)
            at += m
        return out

    def device_form(self, device):
        """(F^{-1} of the dense block, wchol, sqd, full=True) for the fused
        kernels: one leading dense block and a trailing sqrt-diagonal; other
        block patterns are densified."""
        key = (device.type, device.index)
        hit = self._dev.get(key)
        if hit is not None:
            return hit
        kinds = [k for k, _ in self._blocks]
        if all(k == "sqrtdiag" for k in kinds[1:]) and (not kinds or kinds[0] in ("chol", "sqrtdiag")):
            if kinds and kinds[0] == "chol":
                L = self._blocks[0][1]
                w = L.m
                Ld = L.device_spd_inverse(device)
                rest = [b for _, b in self._blocks[1:]]
            else:
                w, Ld = 0, None
                rest = [b for _, b in self._blocks]
            sqd = np.concatenate(rest) if rest else np.zeros(0)
            sqd_d = torch.from_numpy(np.ascontiguousarray(sqd)).to(device) if sqd.size else None
            out = (Ld, w, sqd_d, True)
        else:
            Lfull = np.zeros((self.size, self.size))
            at = 0
            for kind, block in self._blocks:
                if kind == "chol":
                    Lfull[at : at + block.m, at : at + block.m] = block.full()
                    at += block.m
                else:
                    m = block.shape[0]
                    Lfull[np.arange(at, at + m), np.arange(at, at + m)] = block
                    at += m
            Finv = DenseLowerTriangular.from_full(Lfull).device_spd_inverse(device)
            out = (Finv, self.size, None, True)
        self._dev[key] = out
        return out


class DirectReducedProjection:
    """mu = (B'AB)^{-1} B'Az from the cached product cross = A B
    (krylov.py:135-156). Inside the fused PCG kernels the GEMV-T and the
    factor solve run on the device; called directly it returns mu (host)."""

    def __init__(self, cross, factor):
        self.cross = as_block(cross)
        self.factor = factor

    @classmethod
    def assemble(cls, op, B) -> "DirectReducedProjection":
        """A*B with m operator applications (charged m matvecs, no gram) and a
        Cholesky of B'AB (krylov.py:147-153)."""
        Bd = as_block(B, getattr(op, "device", None))
        m = int(Bd.shape[1])
        if isinstance(op, MatrixOperator):
            cross = spmm(op.A, Bd)
            if op.sink is not None:
                op.sink.add_matvec(m)
        else:
            cross = empty_block(Bd.shape[0], m, Bd.device)
            for i in range(m):
                cross[:, i].copy_(op.apply(Bd[:, i]))
        g = to_numpy(gram(Bd, cross))
        return cls(cross, dense_cholesky(0.5 * (g + g.T)))

    def __call__(self, z):
        zd = as_vector(z, self.cross.device)
        return self.factor.solve_spd(to_numpy(gemv_t(self.cross, zd)))


@dataclass
class AugmentedPcgResult:
    """Outputs of one augmented-PCG run (krylov.py:159-178); ``x`` and ``V``
    are device tensors in the run's own coordinates."""

    k: int
    vhat: np.ndarray
    V: torch.Tensor
    gamma: np.ndarray
    residual_history: np.ndarray
    x: torch.Tensor
    converged: bool = True

    @property
    def final_residual(self) -> float:
        return float(self.residual_history[-1])


# ---------------------------------------------------------------------------
# device run buffers
# ---------------------------------------------------------------------------
class _Run:
    """Buffers and the rk_pcg_plan of one augmented-PCG run."""

    def __init__(self, n, device, mode_code, keep_av, m, vcap):
        self.n, self.device, self.mode_code, self.keep_av, self.m = n, device, mode_code, keep_av, m
        self.x = torch.zeros(n, dtype=F64, device=device)
        self.r = torch.empty(n, dtype=F64, device=device)
        self.r2 = torch.empty(n, dtype=F64, device=device)  # residual ping-pong buffer
        self.z = torch.empty(n, dtype=F64, device=device)
        self.mu = torch.zeros(max(m, 1), dtype=F64, device=device)
        self.st = torch.zeros(nat.STATE_BYTES, dtype=torch.uint8, device=device)
        self.tickets = torch.zeros(nat.PCG_TICKETS, dtype=torch.int32, device=device)
        self.st_host = torch.empty(nat.STATE_BYTES, dtype=torch.uint8, pin_memory=True)
        self.cstate = nat.RkPcgState.from_buffer(self.st_host.numpy())
        self.vcap = 0
        self.V = self.AV = self.ap = None
        self._alloc(vcap)
        self.plan = nat.RkPcgPlan()
        self._fill_plan()

    def _alloc(self, vcap):
        n, dev = self.n, self.device
        old = self.vcap
        V = empty_block(n, vcap, dev)
        AV = empty_block(n, vcap, dev) if self.keep_av else None
        hist = torch.zeros((4, vcap + 1), dtype=F64, device=dev)
        if old:
            V[:, :old].copy_(self.V)
            if self.keep_av:
                AV[:, :old].copy_(self.AV)
            hist[:, : old + 1].copy_(self.hist)
        self.V, self.AV, self.hist = V, AV, hist
        if not self.keep_av and self.ap is None:
            self.ap = torch.empty(n, dtype=F64, device=dev)
        self.coef = torch.empty(vcap + 1, dtype=F64, device=dev)
        need = nat.lib().rk_pcg_workspace_doubles(n, self.m, vcap)
        self.ws = torch.empty(max(need, 1), dtype=F64, device=dev)
        self.vcap = vcap

    def ensure(self, cols):
        if cols > self.vcap:
            self._alloc(max(cols, 2 * self.vcap))
            self._fill_plan()

    def _fill_plan(self):
        P = self.plan
        P.n = self.n
        P.x, P.r, P.r2, P.z = self.x.data_ptr(), self.r.data_ptr(), self.r2.data_ptr(), self.z.data_ptr()
        P.V, P.ldv, P.vcap = self.V.data_ptr(), block_ld(self.V), self.vcap
        if self.keep_av:
            P.AV, P.ldav = self.AV.data_ptr(), block_ld(self.AV)
        else:
            P.AV, P.ldav = self.ap.data_ptr(), 0
        P.mu, P.coef, P.st = self.mu.data_ptr(), self.coef.data_ptr(), self.st.data_ptr()
        h = self.hist
        P.alpha_h, P.gamma_h, P.rz_h, P.res_h = (h[i].data_ptr() for i in range(4))
        P.partials, P.partials_len, P.tickets = self.ws.data_ptr(), self.ws.numel(), self.tickets.data_ptr()
        P.mode = self.mode_code

    def set_projection(self, B, cross, factor_dev):
        P = self.plan
        if B is None:
            P.m, P.B, P.ldb, P.cross, P.ldc, P.L, P.ldl, P.wchol, P.sqd = 0, None, 0, None, 0, None, 0, 0, None
            P.linv_full = 0
            return
        self._keep = (B, cross, factor_dev)
        L, w, sqd = factor_dev[:3]
        P.linv_full = 1 if len(factor_dev) > 3 and factor_dev[3] else 0
        P.m = int(B.shape[1])
        P.B, P.ldb = B.data_ptr(), block_ld(B)
        P.cross, P.ldc = cross.data_ptr(), block_ld(cross)
        P.L, P.ldl, P.wchol = (L.data_ptr(), block_ld(L), w) if L is not None and w else (None, 0, 0)
        P.sqd = sqd.data_ptr() if sqd is not None else None

    def set_csr(self, A: SparseSpdMatrix | None):
        self.plan.A = A.csr if A is not None else nat.RkCsr()

    def set_precond(self, dinv):
        self.plan.dinv = dinv.data_ptr() if dinv is not None else None

    def write_state(self, threshold):
        ctypes_zero(self.cstate)
        self.cstate.threshold = float(threshold)
        self.st.copy_(self.st_host)

    def read_state(self):
        self.st_host.copy_(self.st)  # synchronising D2H of 96 bytes
        return self.cstate

    def histories(self, k):
        h = to_numpy(self.hist[:, : k + 1])
        return h[0, :k].copy(), h[1, :k].copy(), h[3, : k + 1].copy()

    def ap_column(self, k):
        return self.AV[:, k] if self.keep_av else self.ap


def ctypes_zero(s):
    import ctypes

    ctypes.memset(ctypes.addressof(s), 0, ctypes.sizeof(s))


_MODES = {"cg": 0, "fom": 1}


def _is_device(t) -> bool:
    return isinstance(t, torch.Tensor) and t.is_cuda


def _to_host_result(res: AugmentedPcgResult) -> AugmentedPcgResult:
    """x and V as numpy (V C-order N x k, np.column_stack's layout), as the
    reference's AugmentedPcgResult (krylov.py:159-178, 272-282)."""
    if res is None:
        return res
    if isinstance(res.x, torch.Tensor):
        res.x = to_numpy(res.x).copy()
    if isinstance(res.V, torch.Tensor):
        res.V = np.ascontiguousarray(to_numpy(res.V))
    return res


def augmented_pcg(
    op,
    b,
    yhat0=None,
    aug_basis=None,
    reduced_solver=None,
    precond=None,
    tol: float = 0.0,
    *,
    mode: str = "cg",
    paper_fom_beta: bool = False,
    relative: bool = False,
    max_iter: int | None = None,
    sink: InstrumentationSink | None = None,
    r0=None,
    monitor=None,
    batch: int | None = None,
    keep_products: bool = False,
    device_results: bool | None = None,
) -> AugmentedPcgResult:
    """Augmented PCG over the affine space Y yhat0 + directions (krylov.py:181-345).

    Same parameters, exceptions (``NotConverged`` with the partial result,
    ``Breakdown``, ``DimensionMismatch``, ``ValueError`` for an unknown mode)
    and sink accounting as the reference. ``batch`` caps the number of
    iterations launched between host checks on the fused path;
    ``keep_products`` keeps every A p_k as a column of ``result.AV`` (fom mode
    keeps them anyway) so a later POD truncation needs no SpMM. The result's
    ``x`` and ``V`` are numpy arrays when ``b`` is a host array (the
    reference's types) and device tensors when it is a device tensor;
    ``device_results`` forces either.
    """
    host = (not device_results) if device_results is not None else not _is_device(b)
    try:
        res = _augmented_pcg(op, b, yhat0, aug_basis, reduced_solver, precond, tol, mode=mode,
                             paper_fom_beta=paper_fom_beta, relative=relative, max_iter=max_iter, sink=sink,
                             r0=r0, monitor=monitor, batch=batch, keep_products=keep_products)
    except NotConverged as exc:
        if host:
            _to_host_result(exc.partial)
        raise
    return _to_host_result(res) if host else res


def _augmented_pcg(op, b, yhat0, aug_basis, reduced_solver, precond, tol, *, mode, paper_fom_beta, relative,
                   max_iter, sink, r0, monitor, batch, keep_products) -> AugmentedPcgResult:
    if isinstance(op, DenseReducedOperator):
        if precond is not None:
            raise NotImplementedError("a dense reduced operator runs unpreconditioned (as the reference's inner solves)")
        return _host_augmented_pcg(op, b, yhat0, aug_basis, reduced_solver, tol, mode, paper_fom_beta, relative,
                                   max_iter, r0, monitor)
    operator = _as_operator(op, sink)
    n = int(operator.dim)
    device = operator.device
    bd = as_vector(b, device)
    if bd.shape[0] != n:
        raise DimensionMismatch("augmented_pcg: rhs length mismatch")

    Y = None
    if aug_basis is not None:
        if isinstance(aug_basis, torch.Tensor):
            if aug_basis.dim() != 2 or aug_basis.shape[0] != n:
                raise DimensionMismatch("augmented_pcg: basis shape mismatch")
        else:
            arr = np.asarray(aug_basis)
            if arr.ndim != 2 or arr.shape[0] != n:
                raise DimensionMismatch("augmented_pcg: basis shape mismatch")
        Y = as_block(aug_basis, device)
        if Y.shape[1] == 0:
            Y = None
    if Y is not None:
        if yhat0 is None:
            raise DimensionMismatch("augmented_pcg: yhat0 required with a nonempty basis")
        yh = as_vector(yhat0, device)
        if yh.shape[0] != Y.shape[1]:
            raise DimensionMismatch("augmented_pcg: yhat0 length mismatch")
        if reduced_solver is None:
            reduced_solver = DirectReducedProjection.assemble(operator, Y)

    code = _MODES.get(mode, -1)
    if code == 1 and paper_fom_beta:
        code = 2
    direct = isinstance(reduced_solver, DirectReducedProjection)
    # SSOR runs inside the device-stepped loop (rk_pcg_*_ssor: the sweeps sit
    # between the two halves of the update kernel) when the loop needs no host
    # callback: its own matrix as the operator, a direct projection or none, no
    # monitor, a known mode.
    ssor = None
    if isinstance(precond, SsorPreconditioner):
        if (isinstance(operator, MatrixOperator) and operator.A is precond.A and (Y is None or direct)
                and monitor is None and code >= 0):
            ssor = precond
    if precond is not None and ssor is None and not isinstance(precond, (JacobiPreconditioner, IdentityPreconditioner)):
        # a preconditioner without a fused form here: the reference loop, step
        # by step, on device primitives
        return _augmented_pcg_generic(operator, bd, Y, yh if Y is not None else None, reduced_solver, precond,
                                      tol, mode, paper_fom_beta, relative, max_iter, sink, r0, monitor)

    m = int(Y.shape[1]) if Y is not None else 0
    keep_av = code == 1 or keep_products
    max_iter = n if max_iter is None else int(max_iter)
    hint_key = (n, device.index, keep_av)
    vcap = min(max_iter + 2, max(64, _CAP_HINT.get(hint_key, 0)))
    run = _Run(n, device, max(code, 0), keep_av, m if direct else 0, vcap=vcap)

    if Y is not None:
        gemv_n(Y, yh, out=run.x)
    if r0 is not None:
        r0d = as_vector(r0, device)
        if r0d.shape[0] != n:
            raise DimensionMismatch("augmented_pcg: r0 length mismatch")
        run.r.copy_(r0d)
    elif Y is not None and bool(torch.any(run.x != 0)):
        run.r.copy_(bd - operator.apply(run.x))
    else:
        run.r.copy_(bd)
    threshold = tol * norm(bd) if relative else tol

    if precond is None or ssor is not None:
        dinv = None
    elif isinstance(precond, (JacobiPreconditioner, IdentityPreconditioner)):
        dinv = precond.fused_inverse_diagonal()
    else:
        raise NotImplementedError(f"preconditioner {getattr(precond, 'kind', precond)!r} has no device form")
    run.set_precond(dinv)
    run.set_csr(operator.A if isinstance(operator, MatrixOperator) else None)
    if direct:
        run.set_projection(Y, reduced_solver.cross, reduced_solver.factor.device_form(device))
    else:
        run.set_projection(None, None, None)

    run.write_state(threshold)
    # entry: z = M^{-1} r, ||r0||, rz, mu, p_0 (krylov.py:268,290-292)
    if ssor is not None:
        nat.check(nat.lib().rk_pcg_entry_ssor(run.plan, ssor.device_plan(1), nat.stream_ptr(device)),
                  "augmented_pcg entry (ssor)")
    else:
        nat.check(nat.lib().rk_pcg_entry(run.plan, nat.stream_ptr(device)), "augmented_pcg entry")
    run.read_state()
    res0 = float(run.hist[3, 0].cpu())
    if monitor is not None:
        monitor(0, run.x.clone())
    if res0 <= threshold:  # krylov.py:284-285
        return _result(run, 0, True)
    if precond is not None and sink is not None:
        sink.add_precond()
    if Y is not None and not direct:
        _direction_with_callback(run, Y, reduced_solver, entry=True)
    # An unknown mode surfaces where the reference meets it (krylov.py:338-339):
    # at the first direction update, after iteration 0 has run in full -- its
    # matvec, the curvature check and the convergence test, which may still
    # return normally -- and after the next z = M^{-1} r. So run (as cg) one
    # iteration at most and raise then.
    loop_iter = max_iter if code >= 0 else min(max_iter, 1)

    fused = isinstance(operator, MatrixOperator) and (Y is None or direct) and monitor is None
    charge_precond = precond is not None and sink is not None
    if fused:
        k_final, status = _drive_fused(run, loop_iter, batch, ssor)
    else:
        # the stepped driver charges every application as it happens, so the
        # counters a monitor snapshots (threestage Checkpoint) are the reference's
        k_final, status = _drive_stepped(run, operator, Y, reduced_solver, direct, loop_iter, monitor,
                                         sink if charge_precond else None)
    if code < 0 and status == 0 and max_iter > 0:
        if fused:
            _count_matvecs(operator, 1)
            if charge_precond:
                sink.add_precond()
        raise ValueError(f"unknown mode {mode!r}")

    # cost accounting identical to the reference's call pattern (fused path:
    # charged here once the run is over)
    if status == 2:
        bd_iter = int(run.cstate.bd_iter)
        if fused:
            _count_matvecs(operator, bd_iter + 1)
            if charge_precond:
                sink.add_precond(bd_iter)
        raise Breakdown(f"direction curvature {run.cstate.gamma:.3e} at iteration {bd_iter}")
    if fused:
        _count_matvecs(operator, k_final)
    if status == 1:
        if fused and charge_precond:
            sink.add_precond(k_final - 1)
        return _result(run, k_final, True)
    if fused and charge_precond:
        sink.add_precond(max_iter)
    raise NotConverged(
        f"no convergence to {threshold:.3e} within {max_iter} iterations",
        partial=_result(run, max_iter, False),
    )


def _augmented_pcg_generic(operator, bd, Y, yh, reduced_solver, precond, tol, mode, paper_fom_beta, relative,
                           max_iter, sink, r0, monitor) -> AugmentedPcgResult:
    """krylov.py:234-345 line by line for a preconditioner applied by its own
    kernels (z = M^{-1} r between the residual update and the reductions):
    SpMV, deterministic dots, numpy-rounded axpys, GEMV-T/N for the
    projection; the scalars come to the host every iteration. The fom sweeps
    are modified Gram-Schmidt as in the reference."""
    from .linalg import axpby

    n = int(operator.dim)
    dev = operator.device
    hval = lambda t: float(t.cpu())  # noqa: E731
    x = gemv_n(Y, yh) if Y is not None else torch.zeros(n, dtype=torch.float64, device=dev)
    if r0 is not None:
        r = as_vector(r0, dev, copy=True)
        if r.shape[0] != n:
            raise DimensionMismatch("augmented_pcg: r0 length mismatch")
    elif Y is not None and bool(torch.any(x != 0)):
        r = bd - as_vector(operator.apply(x), dev)
    else:
        r = bd.clone()
    threshold = tol * norm(bd) if relative else tol
    history = [norm(r)]
    if monitor is not None:
        monitor(0, x.clone())

    def result(k, alphas, dirs, gammas, converged):
        V = torch.stack(dirs, dim=1) if dirs else torch.zeros((n, 0), dtype=torch.float64, device=dev)
        res = AugmentedPcgResult(k=k, vhat=np.asarray(alphas, dtype=np.float64), V=as_block(V, dev),
                                 gamma=np.asarray(gammas, dtype=np.float64),
                                 residual_history=np.asarray(history), x=x, converged=converged)
        res.AV = None
        return res

    if history[0] <= threshold:
        return result(0, [], [], [], True)
    if max_iter is None:
        max_iter = n

    def project(z):
        mu = reduced_solver(z)
        return gemv_n(Y, mu, z, op=2)  # z - Y mu

    z = precond.apply(r, sink)
    p = project(z) if Y is not None else z.clone()
    rz = hval(dot(r, z))
    alphas, dirs, gammas, a_dirs, rz_hist = [], [], [], [], []
    for k in range(max_iter):
        Ap = as_vector(operator.apply(p), dev)
        gamma = hval(dot(p, Ap))
        if not np.isfinite(gamma) or gamma <= _BREAKDOWN_RTOL * hval(dot(p, p)):
            raise Breakdown(f"direction curvature {gamma:.3e} at iteration {k}")
        alpha = rz / gamma
        x = axpby(alpha, p, 1.0, x)
        r = axpby(-alpha, Ap, 1.0, r)
        alphas.append(alpha)
        dirs.append(p)
        gammas.append(gamma)
        rz_hist.append(rz)
        if mode == "fom":
            a_dirs.append(Ap)
        history.append(norm(r))
        if monitor is not None:
            monitor(k + 1, x.clone())
        if history[-1] <= threshold:
            return result(k + 1, alphas, dirs, gammas, True)
        z = precond.apply(r, sink)
        rz_next = hval(dot(r, z))
        if mode == "cg":
            p = axpby(1.0, z, rz_next / rz, p.clone())
            if Y is not None:
                p = gemv_n(Y, reduced_solver(z), p, op=2)
        elif mode == "fom":
            p = project(z) if Y is not None else z.clone()
            if paper_fom_beta:
                for i in range(len(dirs)):
                    p = axpby(rz_next / rz_hist[i], dirs[i], 1.0, p)
            else:
                for _ in range(2):
                    for i in range(len(dirs)):
                        p = axpby(-(hval(dot(a_dirs[i], p)) / gammas[i]), dirs[i], 1.0, p)
        else:
            raise ValueError(f"unknown mode {mode!r}")
        rz = rz_next
    raise NotConverged(f"no convergence to {threshold:.3e} within {max_iter} iterations",
                       partial=result(max_iter, alphas, dirs, gammas, False))


def _count_matvecs(operator, count):
    if isinstance(operator, MatrixOperator) and operator.sink is not None and count:
        operator.sink.add_matvec(count)


# Direction-block capacity from the previous runs of the same size: a sequence's
# systems take similar iteration counts, so V / AV are allocated once at the
# right width instead of growing by doubling (a copy of both blocks per step).
_CAP_HINT: dict = {}


def _result(run: _Run, k: int, converged: bool) -> AugmentedPcgResult:
    key = (run.n, run.device.index, run.keep_av)
    _CAP_HINT[key] = max(_CAP_HINT.get(key, 0), min(int(1.25 * k) + 8, 1 << 16))
    alphas, gammas, hist = run.histories(k)
    res = AugmentedPcgResult(
        k=k, vhat=alphas, V=run.V[:, :k], gamma=gammas, residual_history=hist, x=run.x, converged=converged
    )
    res.AV = run.AV[:, :k] if run.keep_av else None  # A p_k columns (same operator as the run)
    return res


def _drive_cluster(run: _Run, max_iter: int):
    """Small systems: the persistent single-cluster solver (rk_pcg_run_cluster)
    runs to convergence in one launch; it is relaunched from the device state
    only when the direction block must grow first."""
    lib = nat.lib()
    k = 0
    while True:
        if run.vcap - 2 <= k:
            run.ensure(k + 66)  # doubles the block
        kend = min(max_iter, run.vcap - 2)
        nat.check(lib.rk_pcg_run_cluster(run.plan, kend, nat.stream_ptr(run.device)), "augmented_pcg cluster")
        st = run.read_state()
        if st.done or int(st.k) >= max_iter:
            return int(st.k), int(st.status)
        k = int(st.k)


def _drive_fused(run: _Run, max_iter: int, batch: int | None, ssor=None):
    """Batched device iterations; one 96-byte state read per batch. ``ssor``:
    the preconditioner whose sweeps run inside every step (rk_pcg_steps_ssor)."""
    if ssor is None and nat.lib().rk_pcg_cluster_eligible(run.plan):
        return _drive_cluster(run, max_iter)
    launched = 0
    step = 4
    cap = int(batch) if batch else 64
    st = run.cstate
    while launched < max_iter:
        nb = min(step, cap, max_iter - launched)
        run.ensure(launched + nb + 1)
        if ssor is not None:
            nat.check(nat.lib().rk_pcg_steps_ssor(run.plan, ssor.device_plan(nb), nb, launched + nb - 1,
                                                  nat.stream_ptr(run.device)), "augmented_pcg steps (ssor)")
        else:
            nat.check(nat.lib().rk_pcg_steps(run.plan, nb, launched + nb - 1, nat.stream_ptr(run.device)),
                      "augmented_pcg steps")
        launched += nb
        st = run.read_state()
        if st.done:
            return int(st.k), int(st.status)
        step = min(step * 2, cap)
    return int(st.k), int(st.status)


def _direction_with_callback(run: _Run, Y, reduced_solver, entry: bool):
    """mu from a Python reduced solver (e.g. the nested phi=1 projection), then
    the direction kernel with that mu (krylov.py:291,322-326)."""
    mu = as_vector(reduced_solver(run.z), run.device)
    P = run.plan
    saved = (P.m, P.B, P.ldb, P.mu)
    P.m, P.B, P.ldb, P.mu = int(Y.shape[1]), Y.data_ptr(), block_ld(Y), mu.data_ptr()
    try:
        if entry:  # p_0 = z - Y mu (the entry kernel wrote p_0 = z)
            nat.check(nat.lib().rk_gemv_n(run.n, P.m, P.B, P.ldb, P.mu, run.z.data_ptr(), run.V.data_ptr(), 2,
                                          nat.stream_ptr(run.device)), "entry direction")
        else:
            nat.check(nat.lib().rk_pcg_direction(P, int(run.cstate.k), nat.stream_ptr(run.device)),
                      "augmented_pcg direction")
    finally:
        P.m, P.B, P.ldb, P.mu = saved
        del mu


def _drive_stepped(run: _Run, operator, Y, reduced_solver, direct, max_iter, monitor, precond_sink=None):
    """One iteration at a time: operator callback, curvature, update, direction.
    Matvecs and (``precond_sink``) the z = M^{-1} r of every iteration that
    continues are charged as they happen (krylov.py:294-320)."""
    dev = run.device
    st = run.cstate
    for it in range(max_iter):
        run.ensure(it + 2)
        k = it
        p = run.V[:, k]
        dst = run.ap_column(k)
        if isinstance(operator, MatrixOperator):
            spmv_into(operator.A, p, dst)
            _count_matvecs(operator, 1)
        else:
            dst.copy_(as_vector(operator.apply(p), dev))
        nat.check(nat.lib().rk_pcg_curvature(run.plan, nat.stream_ptr(dev)), "curvature")
        nat.check(nat.lib().rk_pcg_update(run.plan, nat.stream_ptr(dev)), "update")
        st = run.read_state()
        if st.status == 2:
            return int(st.k), 2
        if monitor is not None:
            monitor(k + 1, run.x.clone())
        if st.done:
            return int(st.k), int(st.status)
        if precond_sink is not None:
            precond_sink.add_precond()
        if Y is not None and not direct:
            _direction_with_callback(run, Y, reduced_solver, entry=False)
        else:
            nat.check(nat.lib().rk_pcg_direction(run.plan, k, nat.stream_ptr(dev)), "direction")
    st = run.read_state()
    return int(st.k), int(st.status)


def pcg(A, b, x0=None, precond=None, tol: float = 0.0, max_iter: int | None = None, *, mode: str = "cg",
        relative: bool = False, sink: InstrumentationSink | None = None, monitor=None,
        device_results: bool | None = None) -> AugmentedPcgResult:
    """Plain PCG, the empty-basis case of augmented_pcg (krylov.py:348-386);
    host ``b`` gives numpy ``x``/``V`` as augmented_pcg."""
    host = (not device_results) if device_results is not None else not _is_device(b)
    try:
        res = _pcg(A, b, x0, precond, tol, max_iter, mode, relative, sink, monitor)
    except NotConverged as exc:
        if host:
            _to_host_result(exc.partial)
        raise
    return _to_host_result(res) if host else res


def _pcg(A, b, x0, precond, tol, max_iter, mode, relative, sink, monitor):
    operator = _as_operator(A, sink)
    bd = as_vector(b, operator.device)
    shift = None
    rhs = bd
    if x0 is not None:
        x0d = as_vector(x0, operator.device)
        if bool(torch.any(x0d != 0)):
            rhs = bd - operator.apply(x0d)
            shift = x0d
    try:
        res = augmented_pcg(operator, rhs, precond=precond, tol=tol, max_iter=max_iter, mode=mode,
                            relative=relative, sink=sink, monitor=monitor, device_results=True)
    except NotConverged as exc:
        if shift is not None and exc.partial is not None:
            exc.partial.x = exc.partial.x + shift
        raise
    if shift is not None:
        res.x = res.x + shift
    return res


@dataclass
class DirectSolveResult:
    what: np.ndarray
    rhat: DenseLowerTriangular
    aw: torch.Tensor  # cached A @ W on the device
    gram: np.ndarray | None = None  # W'AW as factored (host), for callers that extend it


def direct_reduced_solve(A, b, W, sink: InstrumentationSink | None = None, *,
                         aw_out=None, known=None, device_results: bool | None = None) -> DirectSolveResult:
    """See _direct_reduced_solve; for a host ``b`` the cached product ``aw``
    comes back as a C-order numpy array, as the reference's."""
    res = _direct_reduced_solve(A, b, W, sink, aw_out=aw_out, known=known)
    host = (not device_results) if device_results is not None else not _is_device(b)
    if host:
        res.aw = np.ascontiguousarray(to_numpy(res.aw))
    return res


def _direct_reduced_solve(A, b, W, sink: InstrumentationSink | None = None, *,
                          aw_out=None, known=None) -> DirectSolveResult:
    """Galerkin solve over range(W) by Cholesky of W'AW (krylov.py:396-411):
    SpMM + DMMA Gram on the device, dpotrf and the two triangular solves on
    the host (w x w). ``aw_out`` (N x w device block) receives A W.

    ``known = (w0, G0)``: the caller guarantees that ``aw_out[:, :w0]`` already
    holds A W[:, :w0] for this very matrix and G0 = W[:, :w0]' A W[:, :w0]
    (an invariant matrix with a snapshot grown in place, C1/C4). Only the new
    columns are multiplied and contracted -- A W[:, :w0] would come out of the
    SpMM bit for bit the same -- and the sink is charged exactly as the full
    assemble_gram (one gram, w matvecs)."""
    from .linalg import assemble_gram, gram as gram_xty, spmm

    A = as_matrix(A)
    Wd = as_block(W, A.device)
    bd = as_vector(b, A.device)
    w = int(Wd.shape[1])
    if known is not None and aw_out is not None and 0 < known[0] <= w:
        w0, G0 = known
        if sink is not None:
            sink.add_gram()
            sink.add_matvec(w)
        AW = aw_out
        g = np.empty((w, w))
        g[:w0, :w0] = G0
        if w > w0:
            spmm(A, Wd[:, w0:], out=AW[:, w0:])
            gn = to_numpy(gram_xty(Wd, AW[:, w0:]))       # W' A W_new, w x (w - w0)
            g[:, w0:] = gn
            g[w0:, :w0] = gn[:w0].T
    else:
        G, AW = assemble_gram(A, Wd, sink, out=aw_out)
        g = to_numpy(G)
    g = 0.5 * (g + g.T)
    rhat = _cholesky(g, A.device)
    what = rhat.solve_spd(to_numpy(gemv_t(Wd, bd)))
    return DirectSolveResult(what=what, rhat=rhat, aw=AW, gram=g)


DEVICE_CHOL_MIN = int(os.environ.get("RK_DEVICE_CHOL_MIN", "512"))


def _cholesky(g: np.ndarray, device) -> DenseLowerTriangular:
    """dense_cholesky (linalg.py:250-267) of the stage-1 Gram; from
    DEVICE_CHOL_MIN columns on by cuSOLVER potrf on the device (C4: w ~ 3000,
    seconds of host dpotrf per system), the factor kept on the device for the
    F^{-1} the fused kernels apply and copied back for the host solves. Same
    NotPositiveDefinite(pivot) on a failed leading minor."""
    w = int(g.shape[0])
    if w < DEVICE_CHOL_MIN:
        return dense_cholesky(g)
    Ld, info = torch.linalg.cholesky_ex(torch.from_numpy(np.ascontiguousarray(g)).to(device))
    info = int(info)
    if info > 0:
        raise NotPositiveDefinite(f"leading minor of order {info} is not positive definite", pivot=info - 1)
    rhat = DenseLowerTriangular.from_full(Ld.cpu().numpy())
    rhat._dev[(device.type, device.index)] = as_block(Ld, device)  # linalg.DenseLowerTriangular.device cache
    return rhat
