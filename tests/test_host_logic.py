"""Host-side logic of the drop-in (no GPU): weights, energy truncation,
configuration validation, block factors, and the synthetic generators."""

import math
import warnings

import numpy as np
import pytest

from paper_1512_05820_b200 import errors
from paper_1512_05820_b200.krylov import BlockDiagFactor
from paper_1512_05820_b200.linalg import DenseLowerTriangular, InstrumentationSink, dense_cholesky, symmetric_evd
from paper_1512_05820_b200.pod import energy_truncation_dim
from paper_1512_05820_b200.problems import (
    elasticity_sequence,
    laplacian3d,
    poisson2d_sequence,
    q1_element_stiffness,
    diffusion3d_sequence,
)
from paper_1512_05820_b200.threestage import StageTolerances
from paper_1512_05820_b200.truncation import TruncationConfig
from paper_1512_05820_b200.weights import WeightHistory, idw_weight, weights_previous, weights_rbf


def test_stage_tolerance_defaults():
    eps, eps_hat, eps_inner = StageTolerances(eps=1e-6).resolved()
    assert eps == 1e-6 and eps_hat == pytest.approx(1e-10) and eps_inner == pytest.approx(1e-8)
    assert StageTolerances(1e-4, 1e-9, 1e-5).resolved() == (1e-4, 1e-9, 1e-5)


def test_truncation_config_validation():
    with pytest.raises(errors.RecyklError):
        TruncationConfig(strategy="bogus")
    with pytest.raises(errors.RecyklError):
        TruncationConfig(nu_w=0.9, nu_y=0.5)
    with pytest.raises(errors.RecyklError):
        TruncationConfig(storage_cap=0)
    with pytest.raises(errors.RecyklError):
        TruncationConfig(strategy="deflate")
    assert TruncationConfig(strategy="pod-a-prev").weight_kind == "prev"
    assert TruncationConfig().storage_cap == math.inf


def test_energy_truncation_known_answers():
    assert energy_truncation_dim(np.array([4.0, 3.0, 2.0, 1.0]), 0.7) == 2
    assert energy_truncation_dim(np.array([4.0, 3.0, 2.0, 1.0]), 0.75) == 3
    assert energy_truncation_dim(np.array([4.0, 3.0, 2.0, 1.0]), 0.0) == 1
    with warnings.catch_warnings(record=True) as w:
        warnings.simplefilter("always")
        assert energy_truncation_dim(np.array([1.0, 1e-13]), 1.0) == 1
        assert any(issubclass(x.category, errors.RankTruncatedWarning) for x in w)
    with pytest.raises(errors.EmptyBasis):
        energy_truncation_dim(np.zeros(3), 0.5)
    with pytest.raises(errors.DimensionMismatch):
        energy_truncation_dim(np.array([1.0, 2.0]), 0.5)


def test_rbf_weights_arithmetic():
    h = WeightHistory()
    h.push([1.0, 2.0])
    h.push([1.0, 1.0, 4.0])
    np.testing.assert_allclose(weights_rbf(h, 2), [1.0 + 0.5, 1.0 + 1.0, 4.0])
    np.testing.assert_allclose(weights_previous(h), [1.0, 1.0, 4.0])
    assert idw_weight(3) == 0.25
    with pytest.raises(errors.NoHistory):
        weights_rbf(WeightHistory(), 1)


def test_block_diag_factor_host_solve():
    rng = np.random.default_rng(0)
    M = rng.standard_normal((4, 4))
    G = M @ M.T + 4 * np.eye(4)
    f = BlockDiagFactor()
    f.append_cholesky(dense_cholesky(G))
    f.append_sqrt_diag(np.array([2.0, 3.0]))
    rhs = rng.standard_normal(6)
    out = f.solve_spd(rhs)
    np.testing.assert_allclose(out[:4], np.linalg.solve(G, rhs[:4]), rtol=1e-12)
    np.testing.assert_allclose(out[4:], rhs[4:] / np.array([4.0, 9.0]))


def test_dense_cholesky_pivot_and_evd_order():
    with pytest.raises(errors.NotPositiveDefinite) as exc:
        dense_cholesky(np.diag([1.0, -1.0, 1.0]))
    assert exc.value.pivot == 1
    w, V = symmetric_evd(np.diag([1.0, 3.0, 2.0]))
    assert list(w) == [3.0, 2.0, 1.0]
    L = DenseLowerTriangular.from_full(np.array([[2.0, 0.0], [1.0, 3.0]]))
    np.testing.assert_allclose(L.solve_spd(np.array([4.0, 11.0])), np.linalg.solve(L.full() @ L.full().T, [4.0, 11.0]))


def test_sink_counts_threadsafe():
    import threading

    s = InstrumentationSink()
    ts = [threading.Thread(target=lambda: [s.add_matvec() for _ in range(1000)]) for _ in range(4)]
    [t.start() for t in ts]
    [t.join() for t in ts]
    assert s.snapshot()["matvecs"] == 4000


def test_c1_generator_matches_recipe():
    seq = poisson2d_sequence(8, p=3, rtol=1e-6, seed=0)
    A = seq[0].A.to_scipy().toarray()
    assert A.shape == (64, 64) and np.allclose(A, A.T) and A[0, 0] == 4.0 and A[0, 1] == -1.0 and A[0, 8] == -1.0
    rng = np.random.default_rng(0)
    b0 = rng.standard_normal(64)
    c = rng.standard_normal(64)
    xi1 = rng.standard_normal(64)
    np.testing.assert_array_equal(seq[0].b, b0 + 0.1 * xi1)
    np.testing.assert_array_equal(seq.C[0], c)
    assert seq[0].tol == pytest.approx(1e-6 * np.linalg.norm(seq[0].b))


def test_q1_element_stiffness_properties():
    K = q1_element_stiffness(0.3, 1.0, 1.0)
    assert np.allclose(K, K.T)
    w = np.linalg.eigvalsh(K)
    # six rigid-body modes, the rest positive
    assert np.sum(np.abs(w) < 1e-10 * w.max()) == 6 and w.min() > -1e-10


def test_elasticity_generator_sizes_and_spd():
    seq = elasticity_sequence((3, 2, 2), p=2, rtol=1e-5, seed=1)
    spec = seq[0]
    A = spec.A.to_scipy()
    assert A.shape[0] == 3 * 3 * 3 * 3  # free nodes (ix >= 1): 3 x 3 x 3, 3 dofs each
    assert abs(A - A.T).max() == 0.0
    assert np.linalg.eigvalsh(A.toarray()).min() > 0
    assert np.all(np.diff(spec.A.col_indices[spec.A.row_offsets[0]:spec.A.row_offsets[1]]) > 0)
    # the sequence drifts: system 2 differs from system 1
    assert not np.array_equal(seq[0].A.values, seq[1].A.values)
    # ... as base + i * delta on a fixed pattern (what the device path uploads once)
    base, delta, coef = seq[1].A.affine
    assert coef == 2.0 and np.array_equal(seq[1].A.values, base + 2 * delta)
    assert seq[1].A.affine[0] is seq[0].A.affine[0] and seq[1].A.nnz == base.size


def test_c3_shape_constants():
    """C3 (64^3 elements) has the BASELINE/SURVEY sizes; checked on the pattern
    formula at a smaller size, then the closed form for 64^3."""
    from paper_1512_05820_b200.problems import ElasticityAssembler

    asm = ElasticityAssembler(4, 4, 4)
    assert asm.n == 3 * 4 * 5 * 5
    # closed form of free dofs for 64^3: 3 * 64 * 65 * 65
    assert 3 * 64 * 65 * 65 == 811200


def test_laplacian_and_diffusion_generators():
    L = laplacian3d(4, 3, 2).to_scipy().toarray()
    assert L.shape == (24, 24) and np.allclose(L, L.T) and np.all(np.diag(L) == 6.0)
    seq = diffusion3d_sequence(6, p=2, rtol=1e-4, seed=2, corr_len=2.0)
    A = seq[0].A.to_scipy()
    assert abs(A - A.T).max() < 1e-14 and np.linalg.eigvalsh(A.toarray()).min() > 0


@pytest.mark.parametrize("mode", ["cg", "fom"])
def test_dense_reduced_pcg_matches_oracle(mode):
    """The y-dimensional nested solves (stage 2, phi = 1) run augmented PCG on
    a DenseReducedOperator in host numpy: same iterates, vhat, gamma and the
    same one-matvec-per-application charging as the oracle's restatement of
    krylov.py:181-345 with the operator p -> G p."""
    from oracle import recycle_oracle as O
    from paper_1512_05820_b200.krylov import DenseReducedOperator, augmented_pcg

    rng = np.random.default_rng(5)
    y = 40
    M = rng.standard_normal((y, y))
    G = M @ M.T + y * np.eye(y)
    B = np.linalg.qr(rng.standard_normal((y, 6)))[0]
    b = rng.standard_normal(y)
    yh = np.linalg.solve(B.T @ G @ B, B.T @ b)
    cross = G @ B
    L = dense_cholesky(B.T @ cross)
    sink = InstrumentationSink()
    op = DenseReducedOperator(G, sink=sink, record_products=True)
    res = augmented_pcg(op, b, yh, B, lambda z: L.solve_spd(cross.T @ z), None, 1e-10, mode=mode,
                        r0=b - cross @ yh)
    t = O.Tally()
    proj = O.Projection(cross, O.Factor())
    proj.factor.add_dense(O.cholesky_lower(B.T @ cross))
    ref = O.aug_pcg(lambda v: (t.__setattr__("matvecs", t.matvecs + 1), G @ v)[1], b, yh, B, proj, None, 1e-10,
                    mode=mode, r0=b - cross @ yh, tally=t)
    assert res.k == ref.k and sink.matvecs == res.k == len(op.reduced_products)
    np.testing.assert_allclose(res.x, ref.x, rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(res.gamma, ref.gamma, rtol=1e-12)
