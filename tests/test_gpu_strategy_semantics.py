"""Defining properties of the SURVEY 8f f3/f4 components on the device, the way
the reference's own unit tests state them (tests/test_truncation.py,
test_pod.py, test_preconditioners.py): harmonic-Ritz deflation, the explicit
A-orthonormalisation, output-metric POD, every compress strategy, SSOR."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pk():
    import paper_1512_05820_b200 as pk

    return pk


def _spd(pk, n, seed):
    """Sparse-ish SPD: a shifted random symmetric band, as a device matrix."""
    rng = np.random.default_rng(seed)
    B = np.zeros((n, n))
    for off in (1, 2, 5):
        v = rng.uniform(-1.0, 1.0, n - off)
        B += np.diag(v, off) + np.diag(v, -off)
    B += np.diag(np.abs(B).sum(axis=1) + rng.uniform(0.5, 2.0, n))
    return pk.SparseSpdMatrix.from_dense(B), B


def _basis(n, k, seed):
    return np.linalg.qr(np.random.default_rng(seed).standard_normal((n, k)))[0]


def _h(t):
    return t.cpu().numpy() if isinstance(t, torch.Tensor) else np.asarray(t)


def test_deflation_on_diagonal_keeps_smallest_eigenvectors(pk):
    A = pk.SparseSpdMatrix.from_diagonal(np.array([1.0, 2.0, 3.0]))
    out = pk.deflation_compress(np.eye(3), A, 2)
    np.testing.assert_allclose(out.spectrum, [1.0, 2.0], atol=1e-12)
    assert pk.principal_angle_distance(_h(out.Y_new), np.eye(3)[:, :2]) <= 1e-12


def test_deflation_properties(pk):
    A, Ad = _spd(pk, 40, 1)
    Z = _basis(40, 8, 2)
    out = pk.deflation_compress(Z, A, 4)
    Y = _h(out.Y_new)
    np.testing.assert_allclose(Y.T @ Ad @ Y, np.eye(4), atol=1e-10)        # A-orthonormal
    np.testing.assert_allclose(Z @ out.truncation_map, Y, atol=1e-10)       # Y = Z map
    AZ = Ad @ Z
    for i in range(4):                                                      # harmonic Ritz pairs
        y = Y[:, i]
        resid = Ad @ y - out.spectrum[i] * y
        assert np.linalg.norm(AZ.T @ resid) <= 1e-9 * np.linalg.norm(Ad @ y)
    full = pk.deflation_compress(Z, A, 8)                                   # full retention: same range
    assert pk.principal_angle_distance(_h(full.Y_new), Z) <= 1e-9


def test_enforce_a_orthogonality_properties(pk):
    A, Ad = _spd(pk, 30, 3)
    Yraw = _basis(30, 5, 4)
    Y, _ = pk.enforce_a_orthogonality(Yraw, A)
    Y = _h(Y)
    np.testing.assert_allclose(Y.T @ Ad @ Y, np.eye(5), atol=1e-10)
    assert pk.principal_angle_distance(Y, Yraw) <= 1e-10
    Y2, L2 = pk.enforce_a_orthogonality(Y, A)                               # idempotent
    np.testing.assert_allclose(L2.full(), np.eye(5), atol=1e-10)
    np.testing.assert_allclose(_h(Y2), Y, atol=1e-10)
    Y3, L3 = pk.enforce_a_orthogonality(2.0 * Y, A)                        # scale goes to the factor
    np.testing.assert_allclose(L3.full(), 2.0 * np.eye(5), atol=1e-10)
    np.testing.assert_allclose(_h(Y3), Y, atol=1e-10)


def test_pod_svd_identity_factor_is_plain_svd(pk):
    S = np.random.default_rng(5).standard_normal((25, 6))
    res = pk.pod_svd(S, np.ones(6), np.eye(25), 1.0)
    sv = np.linalg.svd(S, compute_uv=False)
    np.testing.assert_allclose(res.singular_values, sv, rtol=1e-12)


def test_pod_svd_matches_pod_evd_with_factored_metric(pk):
    """Cross-algorithm: Theta = F'F given as a factor (thin SVD) or explicitly
    (Gram + EVD) yields the same spectrum and basis range."""
    import scipy.sparse

    rng = np.random.default_rng(6)
    n, s = 30, 5
    F = rng.standard_normal((n, n)) / np.sqrt(n) + 2.0 * np.eye(n)
    S = rng.standard_normal((n, s))
    gam = rng.uniform(0.5, 1.5, s)
    a = pk.pod_svd(S, gam, F, 1.0)
    theta = pk.SparseSpdMatrix(n, *(lambda m: (m.indptr, m.indices, m.data))(scipy.sparse.csr_matrix(F.T @ F)))
    b = pk.pod_evd(S, gam, theta, 1.0)
    np.testing.assert_allclose(a.singular_values, b.singular_values, rtol=1e-9)
    assert pk.principal_angle_distance(_h(a.columns), _h(b.columns)) <= 1e-8


def test_pod_svd_semidefinite_metric(pk):
    """A one-row factor: one nonzero mode, the rest carry zero energy."""
    rng = np.random.default_rng(7)
    S = rng.standard_normal((20, 4))
    c = rng.standard_normal((1, 20))
    res = pk.pod_svd(S, np.ones(4), c, 1.0)
    assert res.y == 1
    np.testing.assert_allclose(res.singular_values[0], np.linalg.norm(c @ S), rtol=1e-12)
    assert np.all(res.singular_values[1:] == 0.0)


@pytest.mark.parametrize("strategy", ["pod-a-prev", "pod-a-rbf", "pod-ctc-prev", "pod-ctc-rbf", "deflate", "none"])
def test_every_strategy_keeps_range_inside_the_block(pk, strategy):
    A, Ad = _spd(pk, 36, 8)
    Z = _basis(36, 7, 9)
    C = np.random.default_rng(10).standard_normal((2, 36))
    cfg = pk.TruncationConfig(strategy=strategy, nu_y=1.0, nu_w=1.0, max_dim=4,
                              deflate_dim=4 if strategy == "deflate" else None)
    out = pk.compress(Z, cfg, weights=np.linspace(1.0, 2.0, 7), a_prev=A, chalf=C)
    Y = _h(out.Y_new)
    P = Z @ np.linalg.pinv(Z)
    assert np.linalg.norm(Y - P @ Y) <= 1e-9 * max(np.linalg.norm(Y), 1.0)
    if strategy != "none":
        np.testing.assert_allclose(Y.T @ Ad @ Y, np.eye(Y.shape[1]), atol=1e-9)  # enforced / A-metric


def test_ssor_matches_dense_factored_operator(pk):
    A, Ad = _spd(pk, 50, 11)
    r = np.random.default_rng(12).standard_normal(50)
    for omega in (0.7, 1.0, 1.6):
        M = pk.build_preconditioner(f"ssor:{omega}", A)
        D = np.diag(np.diag(Ad))
        T = np.tril(Ad, -1) + D / omega
        Mden = T @ np.linalg.inv(D) @ T.T
        np.testing.assert_allclose(_h(M.apply(r)), np.linalg.solve(Mden, r), rtol=1e-11, atol=1e-12)


def test_ssor_rejects_nonpositive_diagonal_and_bad_omega(pk):
    with pytest.raises(pk.NotPositiveDefinite):
        pk.build_preconditioner("ssor", pk.SparseSpdMatrix(2, np.array([0, 1, 2]), np.array([0, 1]),
                                                           np.array([1.0, 0.0]), validate=False))
    A = pk.SparseSpdMatrix.from_diagonal(np.ones(3))
    for bad in ("ssor:0", "ssor:2.5"):
        with pytest.raises(pk.RecyklError):
            pk.build_preconditioner(bad, A)
    with pytest.raises(pk.RecyklError):
        pk.build_preconditioner("ilu", A)


def test_ssor_pcg_equals_reference_loop_counts(pk):
    """The step-by-step loop with SSOR charges one preconditioner application
    per iteration plus the entry (krylov.py:288,319)."""
    A, _ = _spd(pk, 60, 13)
    b = np.random.default_rng(14).standard_normal(60)
    sink = pk.InstrumentationSink()
    M = pk.build_preconditioner("ssor", A)
    res = pk.pcg(A, b, precond=M, tol=1e-10, sink=sink)
    assert res.converged and sink.precond_applies == res.k and sink.matvecs == res.k
    x = _h(res.x)
    assert np.linalg.norm(b - A.to_scipy() @ x) <= 1e-10
