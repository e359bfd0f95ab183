"""Goal-oriented POD by the method of snapshots (``recykl/pod.py``).

The N-sized work (the A-weighted Gram S'AS and the reconstruction S @ coef)
runs in the DMMA kernels; the s x s eigenproblem runs in host LAPACK
(numpy.linalg.eigh = dsyevd), exactly the routine the reference calls, so the
spectrum and the energy truncation agree with the oracle to Gram rounding.
"""

from __future__ import annotations

import os
import warnings
from dataclasses import dataclass

import numpy as np
import torch

from . import _native as nat
from ._timing import phase as _phase
from .errors import DimensionMismatch, EmptyBasis, RankTruncatedWarning
from .linalg import (
    DenseBasis,
    SparseSpdMatrix,
    UpperGram,
    as_block,
    as_matrix,
    assemble_gram,
    block_ld,
    gemm_nn,
    gram,
    symmetric_evd,
    thin_svd,
    to_numpy,
)

_RANK_RTOL = 1e-12  # pod.py:30, on sigma^2 relative to the largest


@dataclass
class PodMetric:
    kind: str  # "explicit" | "factor"
    operand: object

    @classmethod
    def explicit(cls, theta) -> "PodMetric":
        return cls("explicit", theta)

    @classmethod
    def factor(cls, chalf) -> "PodMetric":
        return cls("factor", chalf)


@dataclass
class PodBasisResult:
    basis: DenseBasis
    singular_values: np.ndarray
    y: int
    snapshot_coef: np.ndarray | None = None

    @property
    def columns(self):
        return self.basis.columns


def energy_truncation_dim(sigma_sq, eps: float) -> int:
    """Smallest dimension whose cumulative energy reaches eps, never beyond the
    numerical rank (modes > 1e-12 sigma_1^2); pod.py:58-83."""
    s2 = np.asarray(sigma_sq, dtype=np.float64)
    if s2.size == 0:
        raise EmptyBasis("empty spectrum")
    if np.any(np.diff(s2) > 0) or np.any(s2 < -_RANK_RTOL * max(s2[0], 0.0)):
        raise DimensionMismatch("spectrum must be nonincreasing and nonnegative")
    total = float(np.sum(s2))
    if s2[0] <= 0.0 or total <= 0.0:
        raise EmptyBasis("all spectral energy is zero")
    rank = int(np.sum(s2 > _RANK_RTOL * s2[0]))
    reached = np.nonzero((np.cumsum(s2) / total)[:rank] >= eps)[0]
    if reached.size == 0:
        warnings.warn(
            "energy criterion unreachable within the numerical rank; truncating at the rank",
            RankTruncatedWarning,
        )
        return rank
    return int(reached[0]) + 1


def _finalize(S, gamma, sigma, V, eps, max_cols=None):
    """coef = V[:, :y] / sigma[:y] * gamma; basis = S @ coef (pod.py:86-97).
    ``max_cols`` reconstructs only a leading column prefix (columns are
    independent, so the prefix is identical to slicing the full basis)."""
    if np.all(gamma == 0.0):
        raise EmptyBasis("all snapshot weights are zero")
    sigma_sq = np.maximum(sigma, 0.0) ** 2
    y = energy_truncation_dim(sigma_sq, eps)
    coef = (V[:, :y] / sigma[:y]) * gamma[:, None]
    ncols = y if max_cols is None else min(y, int(max_cols))
    cols = gemm_nn(S, np.ascontiguousarray(coef[:, :ncols])) if isinstance(S, torch.Tensor) else S @ coef[:, :ncols]
    return PodBasisResult(
        basis=DenseBasis(cols, gram_diag=np.ones(ncols)),
        singular_values=np.maximum(sigma, 0.0),
        y=y,
        snapshot_coef=coef,
    )


DEVICE_EVD_MIN = int(os.environ.get("RK_DEVICE_EVD_MIN", "128"))


def pod_evd_from_gram(gram_sts, S, gamma, eps: float, *, max_cols: int | None = None) -> PodBasisResult:
    """Method of snapshots from a precomputed S'Theta S (pod.py:123-131).

    For m >= DEVICE_EVD_MIN (default 128) the reduced problem stays on the
    device: weighted Gram (rk_pod_weighted_gram), cuSOLVER syevd
    (torch.linalg.eigh, the K9 "small on-device eigensolver"), coefficients
    (rk_pod_coef); only the m eigenvalues come to the host for the energy
    criterion. Smaller problems use host LAPACK dsyevd exactly as the reference."""
    Sd = as_block(S)
    gamma = np.asarray(to_numpy(gamma), dtype=np.float64)
    m = gamma.shape[0]
    if m >= DEVICE_EVD_MIN and isinstance(Sd, torch.Tensor):
        return _pod_device(gram_sts, Sd, gamma, eps, max_cols)
    G = np.asarray(gram_sts, dtype=np.float64) if isinstance(gram_sts, UpperGram) else \
        np.asarray(to_numpy(gram_sts), dtype=np.float64)
    weighted = gamma[:, None] * G * gamma[None, :]
    with _phase("trunc_evd"):
        eigs, V = symmetric_evd(0.5 * (weighted + weighted.T))
    sigma = np.sqrt(np.maximum(eigs, 0.0))
    return _finalize(Sd, gamma, sigma, V, eps, max_cols=max_cols)


def _pod_device(gram_sts, Sd, gamma, eps, max_cols):
    dev = Sd.device
    m = gamma.shape[0]
    st = nat.stream_ptr(dev)
    gam_d = torch.from_numpy(np.ascontiguousarray(gamma)).to(dev)
    if isinstance(gram_sts, UpperGram):
        G, mode, scale = gram_sts.store, 1, gram_sts.scale
        ldg = m
    else:
        G = as_block(gram_sts, dev)
        mode, scale, ldg = 0, None, block_ld(G)
    Wt = torch.empty((m, m), dtype=torch.float64, device=dev)  # symmetric: layout-agnostic
    nat.check(nat.lib().rk_pod_weighted_gram(m, G.data_ptr(), ldg, mode, scale.data_ptr() if scale is not None
                                             else None, gam_d.data_ptr(), Wt.data_ptr(), m, st), "pod weighted gram")
    with _phase("trunc_evd"):
        evals, evecs = torch.linalg.eigh(Wt)  # ascending, like LAPACK
        eigs = evals.cpu().numpy()[::-1].copy()
    if np.all(gamma == 0.0):
        raise EmptyBasis("all snapshot weights are zero")
    sigma = np.sqrt(np.maximum(eigs, 0.0))
    y = energy_truncation_dim(np.maximum(sigma, 0.0) ** 2, eps)
    ncols = y if max_cols is None else min(y, int(max_cols))
    Vcm = evecs.t().contiguous()  # row i = eigenvector i -> column-major V with ld = m
    coef = torch.empty((max(ncols, 1), m), dtype=torch.float64, device=dev)  # column-major m x ncols
    sig_d = torch.from_numpy(np.ascontiguousarray(sigma[:ncols])).to(dev)
    nat.check(nat.lib().rk_pod_coef(m, ncols, Vcm.data_ptr(), m, sig_d.data_ptr(), gam_d.data_ptr(),
                                    coef.data_ptr(), m, st), "pod coef")
    coef_cm = coef[:ncols].t()  # (m, ncols) view, column-major
    cols = gemm_nn(Sd, coef_cm)
    return PodBasisResult(
        basis=DenseBasis(cols, gram_diag=np.ones(ncols)),
        singular_values=np.maximum(sigma, 0.0),
        y=y,
        snapshot_coef=coef_cm.cpu().numpy(),
    )


def pod_svd(S, gamma, chalf, eps: float, *, max_cols: int | None = None) -> PodBasisResult:
    """POD in the output metric Theta = F'F through the thin SVD of the factored
    weighted snapshots F (S diag(gamma)) (pod.py:134-157).

    F (``chalf``, q x N) usually has a handful of rows, so the N-sized
    contraction F S is the DMMA Gram S' F' (s x q) on the device; the q x s SVD
    runs in host LAPACK as in the reference, and the basis is the DMMA
    reconstruction S @ coef. Components beyond the factor rank carry zero
    energy (the spectrum is zero-padded to s)."""
    Sd = as_block(S)
    gamma = np.asarray(to_numpy(gamma), dtype=np.float64)
    F = chalf.detach() if isinstance(chalf, torch.Tensor) else np.atleast_2d(np.asarray(chalf, dtype=np.float64))
    if F.ndim == 1:
        F = F[None, :]
    if gamma.shape[0] != Sd.shape[1]:
        raise DimensionMismatch("one weight per snapshot required")
    if F.shape[1] != Sd.shape[0]:
        raise DimensionMismatch("metric factor columns must match snapshot length")
    Ft = as_block(F.t() if isinstance(F, torch.Tensor) else F.T, Sd.device)  # N x q
    factored = to_numpy(gram(Ft, Sd)) * gamma[None, :]                    # q x s = F S diag(gamma)
    _, sigma, V = thin_svd(factored)
    s = Sd.shape[1]
    if sigma.shape[0] < s:
        sigma = np.concatenate([sigma, np.zeros(s - sigma.shape[0])])
        Vfull = np.zeros((s, s))
        Vfull[:, : V.shape[1]] = V
        V = Vfull
    return _finalize(Sd, gamma, sigma, V, eps, max_cols=max_cols)


def pod_evd(S, gamma, theta, eps: float, *, max_cols: int | None = None) -> PodBasisResult:
    """POD with an explicit SPD metric (pod.py:100-120): device Gram S'(theta S)."""
    Sd = as_block(S)
    gamma = np.asarray(to_numpy(gamma), dtype=np.float64)
    if gamma.shape[0] != Sd.shape[1]:
        raise DimensionMismatch("one weight per snapshot required")
    G, _ = assemble_gram(as_matrix(theta), Sd, None)
    return pod_evd_from_gram(G, Sd, gamma, eps, max_cols=max_cols)
