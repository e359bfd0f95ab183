"""SURVEY 8f f3/f4 on the device: output-metric POD (pod-ctc-*, thin SVD of C S
plus the explicit A-orthonormalisation), harmonic-Ritz deflation and the SSOR
preconditioner (sync-free triangular sweeps), against runs of the reference
itself (tests/golden/next_strategies.npz) and the CPU oracle."""

import numpy as np
import pytest
import torch

import golden_io as gio
from test_gpu_sequence import EXACT_FLOOR, _check, _run


def _host(t):
    """numpy view of a result (host inputs give numpy, device inputs device tensors)."""
    return t.detach().cpu().numpy() if hasattr(t, "detach") else np.asarray(t)


pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pk():
    import paper_1512_05820_b200 as pk

    return pk


def _same_up_to_sign(got, ref, tol):
    for j in range(ref.shape[1]):
        s = np.sign(got[:, j] @ ref[:, j])
        assert np.linalg.norm(s * got[:, j] - ref[:, j]) <= tol * np.linalg.norm(ref[:, j]), j


@pytest.mark.parametrize("tag", list(gio.NEXT_CASES))
def test_next_strategy_sequences(pk, tag):
    d = gio.load("next_strategies")
    tr, mode, pc = gio.NEXT_CASES[tag]
    seq = gio.next_sequence(d)
    xs, reps, _ = _run(pk, seq, tr, mode, pc)
    first = _check(d, tag, xs, reps, strict=False, min_exact=EXACT_FLOOR[("next_strategies", tag)])
    assert all(r.converged for r in reps)
    assert [bool(r.truncated) for r in reps] == list(map(bool, d[f"{tag}truncated"]))
    for j, x in enumerate(xs, start=1):
        q = d["C"] @ _host(x)
        ref = d[f"{tag}q{j}"]
        tol = 1e-10 if j - 1 < first else 1e-4
        assert np.all(np.abs(q - ref) <= tol * np.abs(ref)), (tag, j)


def test_pod_svd_matches_reference(pk):
    d = gio.load("next_strategies")
    res = pk.pod_svd(d["k_S"], d["k_gamma"], d["C"], 1.0)
    sig = d["k_svd_sigma"]
    np.testing.assert_allclose(res.singular_values, sig, rtol=1e-12, atol=1e-13 * sig[0])
    assert res.y == int(d["k_svd_y"])
    _same_up_to_sign(res.columns.cpu().numpy(), d["k_svd_cols"], 1e-10)


def test_deflation_compress_matches_reference(pk):
    d = gio.load("next_strategies")
    A = pk.linalg.as_matrix(gio.next_sequence(d)[0].A)
    sink = pk.InstrumentationSink()
    out = pk.deflation_compress(d["k_S"], A, 6, sink=sink)
    np.testing.assert_allclose(out.spectrum, d["k_defl_mu"], rtol=1e-9)
    _same_up_to_sign(out.Y_new.cpu().numpy(), d["k_defl_Y"], 1e-8)
    assert out.stage1_width == 6 and out.enforced
    assert sink.gram_assemblies == 1 and sink.matvecs == d["k_S"].shape[1]  # one assemble_gram


def test_enforce_a_orthogonality(pk):
    d = gio.load("next_strategies")
    A = pk.linalg.as_matrix(gio.next_sequence(d)[0].A)
    Y, L = pk.enforce_a_orthogonality(d["k_S"][:, :5], A)
    G, _ = pk.assemble_gram(A, Y)
    np.testing.assert_allclose(G.cpu().numpy(), np.eye(5), atol=1e-12)
    # same range: Y L' reproduces the input
    np.testing.assert_allclose(Y.cpu().numpy() @ L.full().T, d["k_S"][:, :5], rtol=1e-12, atol=1e-12)


def test_ssor_apply_matches_reference(pk):
    d = gio.load("next_strategies")
    A = pk.linalg.as_matrix(gio.next_sequence(d)[0].A)
    M = pk.build_preconditioner("ssor:1.3", A)
    sink = pk.InstrumentationSink()
    z = M.apply(d["k_ssor_r"], sink).cpu().numpy()
    ref = d["k_ssor_z"]
    np.testing.assert_allclose(z, ref, rtol=1e-12, atol=1e-14 * np.abs(ref).max())
    assert sink.precond_applies == 1
    with pytest.raises(pk.RecyklError):
        pk.build_preconditioner("ssor:2.0", A)


def test_ssor_on_elasticity_vs_oracle_and_deterministic(pk):
    """Block-structured 3-D operator (Q1 elasticity, 1,944 rows): the sweeps
    agree with the oracle's triangular solves and repeat bit for bit."""
    from oracle import recycle_oracle as O
    from paper_1512_05820_b200.problems import elasticity_sequence

    H = next(iter(elasticity_sequence((8, 8, 8), p=1))).A
    A = pk.SparseSpdMatrix(H.n, H.row_offsets, H.col_indices, H.values)
    r = np.random.default_rng(2).standard_normal(H.n)
    M = pk.build_preconditioner("ssor", A)
    z1 = M.apply(r).cpu().numpy()
    z2 = M.apply(torch.from_numpy(r).cuda()).cpu().numpy()
    assert np.array_equal(z1, z2)
    ref = O.Ssor(H.to_scipy(), 1.0)(r)
    np.testing.assert_allclose(z1, ref, rtol=1e-11, atol=1e-13 * np.abs(ref).max())


def test_ssor_level_order_respects_dependencies(pk):
    """rk_ssor_levels: the hand-out order of each sweep is a permutation in
    which every row comes after the rows it depends on (strictly lower entries
    forward, strictly upper backward) and levels are non-decreasing; the depth
    of a 3-D 7-point stencil in natural order is nx + ny + nz - 2."""
    from paper_1512_05820_b200.problems import laplacian3d

    nx, ny, nz = 9, 7, 5
    H = laplacian3d(nx, ny, nz)
    A = pk.SparseSpdMatrix(H.n, H.row_offsets, H.col_indices, H.values)
    M = pk.build_preconditioner("ssor:1.2", A)
    assert M.depth == nx + ny + nz - 2
    rp, ci = np.asarray(H.row_offsets), np.asarray(H.col_indices)
    for order, upper in zip(M._order, (False, True)):
        o = order.cpu().numpy()
        assert sorted(o.tolist()) == list(range(H.n))
        pos = np.empty(H.n, dtype=np.int64)
        pos[o] = np.arange(H.n)
        for i in range(H.n):
            deps = ci[rp[i]:rp[i + 1]]
            deps = deps[deps > i] if upper else deps[deps < i]
            assert np.all(pos[deps] < pos[i])


@pytest.mark.parametrize("mode", ["cg", "fom"])
def test_ssor_device_stepped_loop_matches_stepwise_loop(pk, mode):
    """SSOR inside the device-stepped PCG loop (rk_pcg_steps_ssor: update of x
    and r, forward and backward sweep, r'z and cross'z, direction, no host
    round trip per iteration) against the reference loop taken step by step
    with every scalar on the host (the path a monitor forces): plain and with a
    direct projection onto a recycled basis; same iteration count, x within
    1e-11, identical sink counters."""
    from paper_1512_05820_b200.linalg import InstrumentationSink, scale_columns
    from paper_1512_05820_b200.problems import elasticity_sequence

    spec = next(iter(elasticity_sequence((10, 9, 8), p=1, seed=5)))
    A = pk.SparseSpdMatrix.from_host(spec.A)
    b = torch.from_numpy(spec.b).cuda()
    tol = 1e-8 * float(np.linalg.norm(spec.b))

    def run(stepwise, **kw):
        sink = InstrumentationSink()
        M = pk.build_preconditioner("ssor:1.3", A)
        mon = (lambda k, x: None) if stepwise else None
        res = pk.augmented_pcg(A, b, precond=M, tol=tol, mode=mode, sink=sink, monitor=mon, **kw)
        return res, sink.snapshot()

    f, cf = run(False)
    g, cg_ = run(True)
    assert f.converged and f.k == g.k and cf == cg_
    assert torch.linalg.norm(f.x - g.x) <= 1e-11 * torch.linalg.norm(g.x)
    # recycle 12 directions: stage-1 projection, then the augmented loop
    Y = scale_columns(f.V[:, :12], np.sqrt(f.gamma[:12]))
    b2 = b + 0.05 * torch.roll(b, 7)
    st1 = pk.direct_reduced_solve(A, b2, Y)
    fac = pk.BlockDiagFactor()
    fac.append_cholesky(st1.rhat)
    proj = pk.DirectReducedProjection(st1.aw, fac)

    def run2(stepwise):
        sink = InstrumentationSink()
        M = pk.build_preconditioner("ssor:1.3", A)
        mon = (lambda k, x: None) if stepwise else None
        return pk.augmented_pcg(A, b2, st1.what, Y, proj, M, tol, mode=mode, sink=sink, monitor=mon), sink.snapshot()

    f2, c2 = run2(False)
    g2, d2 = run2(True)
    assert f2.converged and f2.k == g2.k and c2 == d2 and f2.k < f.k
    assert torch.linalg.norm(f2.x - g2.x) <= 1e-11 * torch.linalg.norm(g2.x)


def test_manifest_sequence_on_device(pk):
    """f1: a reference-written manifest, loaded lazily (parse + upload of system
    j+1 on the helper thread while j solves), gives bit-identical solutions to
    the same arrays handed over in memory."""
    import os

    from paper_1512_05820_b200.problems import load_sequence_manifest

    d = gio.load("manifest")
    tr = dict(strategy="pod-a-rbf", nu_y=1.0, nu_w=1.0, storage_cap=8, max_dim=6)
    lazy = load_sequence_manifest(os.path.join(gio.GOLDEN, "manifest_small", "manifest.json"), lazy=True)
    xs1, reps1, _ = _run(pk, lazy, tr, "cg", "jacobi")
    mem = gio.sequence(d)
    mem.systems[1].xbar = d["xbar2"]
    xs2, reps2, _ = _run(pk, mem, tr, "cg", "jacobi")
    assert [r.stage3_iters for r in reps1] == [r.stage3_iters for r in reps2]
    for a, b in zip(xs1, xs2):
        assert np.array_equal(a, b)
