"""augmented_pcg / pcg / direct_reduced_solve on the device vs the reference's
goldens and the oracle (mirrors reference tests/test_krylov.py)."""

import numpy as np
import pytest

import golden_io as gio

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pk():
    import paper_1512_05820_b200 as pk

    return pk


def _np(t):
    return t.detach().cpu().numpy() if hasattr(t, "detach") else np.asarray(t)


@pytest.mark.parametrize("mode", ["cg", "fom"])
def test_augmented_pcg_matches_reference_golden(pk, mode):
    d = gio.load("kernels")
    A = pk.SparseSpdMatrix(len(d["rowptr"]) - 1, d["rowptr"], d["col"], d["val"])
    res = pk.augmented_pcg(A, d["b"], d["yhat0"], d["Y"], tol=1e-10, mode=mode, max_iter=400)
    assert res.k == int(d[f"{mode}_k"])
    x = _np(res.x)
    assert np.linalg.norm(x - d[f"{mode}_x"]) <= 1e-8 * np.linalg.norm(d[f"{mode}_x"])
    np.testing.assert_allclose(res.vhat, d[f"{mode}_vhat"], rtol=1e-6)
    np.testing.assert_allclose(res.gamma, d[f"{mode}_gamma"], rtol=1e-8)
    np.testing.assert_allclose(res.residual_history, d[f"{mode}_hist"], rtol=1e-5, atol=1e-14)
    # x = Y yhat0 + V vhat and gamma = p'Ap (reference test_krylov.py:71-82)
    rebuilt = d["Y"] @ d["yhat0"] + _np(res.V) @ res.vhat
    np.testing.assert_allclose(rebuilt, x, atol=1e-10)


def test_paper_fom_beta_matches_reference(pk):
    d = gio.load("kernels")
    A = pk.SparseSpdMatrix(len(d["rowptr"]) - 1, d["rowptr"], d["col"], d["val"])
    try:
        res = pk.augmented_pcg(A, d["b"], d["yhat0"], d["Y"], tol=1e-6, mode="fom", paper_fom_beta=True,
                               max_iter=25)
        conv = True
    except pk.NotConverged as exc:
        res, conv = exc.partial, False
    assert conv == bool(d["paper_conv"])
    assert res.k == int(d["paper_k"])
    np.testing.assert_allclose(res.residual_history, d["paper_hist"], rtol=1e-6)


def test_identity_system_one_iteration(pk):
    A = pk.SparseSpdMatrix.identity(3)
    res = pk.augmented_pcg(A, np.array([1.0, 2.0, 3.0]), tol=0.0)
    assert res.k == 1
    np.testing.assert_allclose(_np(res.x), [1.0, 2.0, 3.0])


def test_exact_solution_in_augmenting_subspace(pk):
    A = pk.SparseSpdMatrix.from_diagonal([1.0, 2.0])
    b = np.array([1.0, 2.0])
    Y = np.array([[1.0], [1.0]])
    yhat0 = np.linalg.solve(Y.T @ np.diag([1.0, 2.0]) @ Y, Y.T @ b)
    res = pk.augmented_pcg(A, b, yhat0, Y, tol=1e-14)
    assert res.k == 0
    np.testing.assert_allclose(_np(res.x), [1.0, 1.0])


def test_breakdown_on_indefinite_operator(pk):
    with pytest.raises(pk.Breakdown):
        # symmetric but indefinite (validation only checks symmetry and diagonal)
        A = pk.SparseSpdMatrix.from_dense(np.array([[1.0, 2.0], [2.0, 1.0]]))
        pk.augmented_pcg(A, np.array([1.0, -1.0]), tol=1e-12)


def test_not_converged_carries_partial(pk):
    rng = np.random.default_rng(18)
    Q, _ = np.linalg.qr(rng.standard_normal((30, 30)))
    M = (Q * np.logspace(0, 5, 30)) @ Q.T
    A = pk.SparseSpdMatrix.from_dense(0.5 * (M + M.T))
    sink = pk.InstrumentationSink()
    with pytest.raises(pk.NotConverged) as exc:
        pk.augmented_pcg(A, rng.standard_normal(30), tol=1e-14, max_iter=2, sink=sink)
    partial = exc.value.partial
    assert partial.k == 2 and not partial.converged
    assert tuple(partial.V.shape) == (30, 2)
    assert sink.matvecs == 2


def test_relative_tolerance(pk):
    d = gio.load("kernels")
    A = pk.SparseSpdMatrix(len(d["rowptr"]) - 1, d["rowptr"], d["col"], d["val"])
    b = 1e6 * d["b"]
    res = pk.augmented_pcg(A, b, tol=1e-8, relative=True, max_iter=300)
    assert res.final_residual <= 1e-8 * np.linalg.norm(b)


def test_monitor_sees_monotone_a_norm_error(pk):
    d = gio.load("kernels")
    A = pk.SparseSpdMatrix(len(d["rowptr"]) - 1, d["rowptr"], d["col"], d["val"])
    Ad = A.to_dense()
    xstar = np.linalg.solve(Ad, d["b"])
    errs = []

    def monitor(k, xk):
        e = xstar - xk.cpu().numpy()
        errs.append(np.sqrt(e @ Ad @ e))

    res = pk.augmented_pcg(A, d["b"], tol=1e-9 * np.linalg.norm(d["b"]), max_iter=250, monitor=monitor)
    assert len(errs) == res.k + 1
    assert np.all(np.diff(errs) <= 1e-10 * errs[0])


def test_precond_and_matvec_counts_match_oracle(pk):
    from oracle import recycle_oracle as O

    d = gio.load("kernels")
    n = len(d["rowptr"]) - 1
    A = pk.SparseSpdMatrix(n, d["rowptr"], d["col"], d["val"])
    M = pk.build_preconditioner("jacobi", A)
    sink = pk.InstrumentationSink()
    res = pk.augmented_pcg(A, d["b"], precond=M, tol=1e-9, sink=sink, mode="cg")
    As = O.as_csr(gio.sequence({"n": n, "p": 1, "A1_rowptr": d["rowptr"], "A1_col": d["col"],
                                "A1_val": d["val"], "b1": d["b"], "tol1": 1e-9})[0].A)
    t = O.Tally()
    ref = O.aug_pcg(lambda v: O.matvec(As, v, t), d["b"], dinv=1.0 / As.diagonal(), tol=1e-9, tally=t)
    assert res.k == ref.k
    assert sink.matvecs == t.matvecs and sink.precond_applies == t.precond


def test_pcg_with_initial_guess(pk):
    d = gio.load("kernels")
    A = pk.SparseSpdMatrix(len(d["rowptr"]) - 1, d["rowptr"], d["col"], d["val"])
    x0 = np.linalg.solve(A.to_dense(), d["b"]) + 1e-3
    res = pk.pcg(A, d["b"], x0=x0, tol=1e-10)
    xs = np.linalg.solve(A.to_dense(), d["b"])
    assert np.linalg.norm(_np(res.x) - xs) <= 1e-8 * np.linalg.norm(xs)


def test_direct_reduced_solve_known_answer(pk):
    A = pk.SparseSpdMatrix.from_diagonal([2.0, 3.0, 4.0])
    W = np.eye(3)[:, :2]
    sink = pk.InstrumentationSink()
    out = pk.direct_reduced_solve(A, np.array([2.0, 3.0, 4.0]), W, sink)
    np.testing.assert_allclose(out.what, [1.0, 1.0])
    assert sink.gram_assemblies == 1 and sink.matvecs == 2


def test_batching_does_not_change_results(pk):
    d = gio.load("kernels")
    A = pk.SparseSpdMatrix(len(d["rowptr"]) - 1, d["rowptr"], d["col"], d["val"])
    a = pk.augmented_pcg(A, d["b"], d["yhat0"], d["Y"], tol=1e-10, mode="fom", max_iter=400, batch=1)
    b = pk.augmented_pcg(A, d["b"], d["yhat0"], d["Y"], tol=1e-10, mode="fom", max_iter=400, batch=64)
    assert a.k == b.k
    assert np.array_equal(_np(a.x), _np(b.x))  # deterministic reductions: bitwise


@pytest.mark.parametrize("nx,width", [(64, 300), (96, 4500)])
def test_wide_projection_matches_oracle(pk, nx, width):
    """Projection width 300 (> the 256 above which mu = F^{-1} c is spread over
    the whole GPU by k_pcg_musolve instead of the finish kernel's last block)
    and 4500 (beyond the former 4096-column limit of the fused path; the
    reference has none): same iteration count and solution as the oracle on
    a 2-D Poisson matrix."""
    from oracle import recycle_oracle as O
    from paper_1512_05820_b200.problems import poisson2d_matrix

    L = poisson2d_matrix(nx)
    A = pk.SparseSpdMatrix(L.n, L.row_offsets, L.col_indices, L.values)
    As = O.as_csr(L)
    rng = np.random.default_rng(11)
    Y = np.linalg.qr(rng.standard_normal((L.n, width)))[0]
    b = rng.standard_normal(L.n)
    yhat0 = np.linalg.solve(Y.T @ (As @ Y), Y.T @ b)
    M = pk.build_preconditioner("jacobi", A)
    tol = 1e-8 * np.linalg.norm(b)
    res = pk.augmented_pcg(A, b, yhat0, Y, precond=M, tol=tol, mode="cg", max_iter=2000)
    t = O.Tally()
    proj = O.assembled_projection(lambda v: O.matvec(As, v, t), Y)
    ref = O.aug_pcg(lambda v: O.matvec(As, v, t), b, yhat0, Y, proj, 1.0 / As.diagonal(), tol, mode="cg",
                    max_iter=2000, tally=t)
    assert abs(res.k - ref.k) <= 2
    x = _np(res.x)
    assert np.linalg.norm(x - ref.x) <= 1e-8 * np.linalg.norm(ref.x)


def test_wide_stage1_cholesky_on_device(pk):
    """Stage-1 factors from 512 columns on come from cuSOLVER potrf: equal to
    the host dpotrf to rounding, and an indefinite Gram raises
    NotPositiveDefinite with the reference's pivot (first failing minor)."""
    import torch

    from paper_1512_05820_b200 import krylov

    rng = np.random.default_rng(4)
    w = 600
    M = rng.standard_normal((w, w))
    G = M @ M.T + w * np.eye(w)
    dev = torch.device("cuda", 0)
    L = krylov._cholesky(G, dev)
    np.testing.assert_allclose(L.full(), pk.dense_cholesky(G).full(), rtol=1e-10, atol=1e-12)
    Gbad = G.copy()
    Gbad[300, 300] = -1.0
    with pytest.raises(pk.NotPositiveDefinite) as e_dev:
        krylov._cholesky(Gbad, dev)
    with pytest.raises(pk.NotPositiveDefinite) as e_host:
        pk.dense_cholesky(Gbad)
    assert e_dev.value.pivot == e_host.value.pivot == 300


def test_reduced_spd_operator_matches_reference_statements(pk):
    """ReducedSpdOperator (krylov.py:60-83) on the device: p -> Y'(A(Yp)) by
    GEMV-N, SpMV, GEMV-T equals the reference's statements, charges one matvec
    per application and records the full products; augmented_pcg over it (the
    reference's stage-2 / phi=1 inner solve, threestage.py:143-220) takes the
    oracle's iterations and reaches its solution."""
    import torch

    from oracle import recycle_oracle as O
    from paper_1512_05820_b200.problems import poisson2d_matrix

    L = poisson2d_matrix(32)
    As = O.as_csr(L)
    A = pk.SparseSpdMatrix(L.n, L.row_offsets, L.col_indices, L.values)
    rng = np.random.default_rng(5)
    Y = np.linalg.qr(rng.standard_normal((L.n, 30)))[0]
    sink = pk.InstrumentationSink()
    op = pk.ReducedSpdOperator(A, Y, sink, record_products=True)
    p = rng.standard_normal(30)
    got = _np(op.apply(p))
    want = Y.T @ (As @ (Y @ p))
    assert np.linalg.norm(got - want) <= 1e-13 * np.linalg.norm(want)
    assert sink.matvecs == 1
    full = _np(op.full_products_block())
    assert full.shape == (L.n, 1)
    assert np.linalg.norm(full[:, 0] - As @ (Y @ p)) <= 1e-13 * np.linalg.norm(full[:, 0])
    assert isinstance(op.reduced_products[0], torch.Tensor)

    bhat = Y.T @ rng.standard_normal(L.n)
    sink2 = pk.InstrumentationSink()
    op2 = pk.ReducedSpdOperator(A, Y, sink2)
    res = pk.augmented_pcg(op2, bhat, tol=1e-10 * np.linalg.norm(bhat), mode="cg", max_iter=200)
    t = O.Tally()
    ref = O.aug_pcg(O.ReducedOp(As, Y, t), bhat, tol=1e-10 * np.linalg.norm(bhat), mode="cg", max_iter=200,
                    tally=t)
    assert res.k == ref.k
    assert sink2.matvecs == t.matvecs
    assert np.linalg.norm(_np(res.x) - ref.x) <= 1e-10 * np.linalg.norm(ref.x)
