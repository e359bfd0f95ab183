"""Kernel-level parity of libpodcg.so against the reference's goldens and numpy
(fp64; bit-level where the op is elementwise, 1e-12-relative for reductions)."""

import numpy as np
import pytest
import scipy.sparse
import torch

import golden_io as gio

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pk():
    import paper_1512_05820_b200 as pk

    return pk


def _dev_matrix(pk, rowptr, col, val):
    return pk.SparseSpdMatrix(len(rowptr) - 1, rowptr, col, val)


def test_library_reports_sm_count(pk):
    from paper_1512_05820_b200 import _native as nat

    assert nat.lib().rk_device_sm_count() >= 100


def test_spmv_matches_reference_golden(pk):
    d = gio.load("kernels")
    A = _dev_matrix(pk, d["rowptr"], d["col"], d["val"])
    y = pk.spmv(A, d["x"]).cpu().numpy()
    # linalg test: SpMV vs dense to 1e-12 (reference tests/test_linalg.py:52-64)
    np.testing.assert_allclose(y, d["Ax"], rtol=1e-12, atol=1e-12 * np.abs(d["Ax"]).max())


@pytest.mark.parametrize("lanes", [0, 1, 2, 4, 8, 16, 32])
def test_spmv_all_lane_widths(pk, lanes):
    from paper_1512_05820_b200.problems import elasticity_sequence, laplacian3d

    for H in (laplacian3d(9, 7, 5), next(iter(elasticity_sequence((3, 4, 5), p=1))).A):
        A = pk.SparseSpdMatrix(H.n, H.row_offsets, H.col_indices, H.values, lanes=lanes)
        x = np.random.default_rng(lanes).standard_normal(H.n)
        ref = H.to_scipy() @ x
        got = pk.spmv(A, x).cpu().numpy()
        np.testing.assert_allclose(got, ref, rtol=1e-13, atol=1e-13 * np.abs(ref).max())


def test_bsr3_view_for_vector_problems(pk):
    """Q1 elasticity has exact 3x3 blocks: the SpMV streams the BSR view and
    matches scipy's CSR product; the fused PCG SpMV agrees with the plain one."""
    from paper_1512_05820_b200.problems import elasticity_sequence

    H = next(iter(elasticity_sequence((5, 4, 3), p=1))).A
    A = pk.SparseSpdMatrix(H.n, H.row_offsets, H.col_indices, H.values)
    bsr = A._pattern.bsr
    assert A.bval is not None and bsr.nreal * 9 == A.nnz and bsr.nblk >= bsr.nreal and bsr.nblk % 32 == 0
    x = np.random.default_rng(9).standard_normal(H.n)
    ref = H.to_scipy() @ x
    np.testing.assert_allclose(pk.spmv(A, x).cpu().numpy(), ref, rtol=1e-13, atol=1e-13 * np.abs(ref).max())
    # values refreshed on the same pattern are gathered again
    A2 = A.with_values(torch.from_numpy(2.0 * H.values).cuda())
    np.testing.assert_allclose(pk.spmv(A2, x).cpu().numpy(), 2.0 * ref, rtol=1e-13, atol=1e-13 * np.abs(ref).max())
    # a scalar problem has no block view
    B = pk.SparseSpdMatrix.from_diagonal(np.arange(1.0, 8.0))
    assert B.bval is None


def _csr_chain_rows(H, x, rows):
    """scipy's csr_matvec arithmetic for the given rows: s = 0; for each stored
    entry in CSR order, s = s + v * x[col] with the product and the sum each
    rounded (Python floats round exactly like that)."""
    out = []
    for i in rows:
        s = 0.0
        lo, hi = int(H.row_offsets[i]), int(H.row_offsets[i + 1])
        for q in range(lo, hi):
            s = s + float(H.values[q]) * float(x[H.col_indices[q]])
        out.append(s)
    return np.array(out)


def _scipy_rows(H, x, rows):
    import scipy.sparse

    return (scipy.sparse.csr_matrix((H.values, H.col_indices, H.row_offsets), shape=(H.n, H.n)) @ x)[rows]


def test_sell_spmv_is_scipy_csr_matvec_bitwise(pk):
    """Bitwise: the 3x3-block SpMV (tiled slot-row layout) computes each row as
    scipy's csr_matvec does (separately rounded multiply and add over the row's
    entries in CSR order, padding slots contributing exactly nothing); the
    fused PCG SpMV uses the same row routine."""
    from paper_1512_05820_b200.problems import elasticity_sequence

    H = next(iter(elasticity_sequence((6, 5, 4), p=1))).A
    A = pk.SparseSpdMatrix(H.n, H.row_offsets, H.col_indices, H.values)
    assert A.bval is not None
    x = np.random.default_rng(3).standard_normal(H.n)
    got = pk.spmv(A, x).cpu().numpy()
    rows = np.arange(H.n)
    assert np.array_equal(got, _csr_chain_rows(H, x, rows))
    assert np.array_equal(got, _scipy_rows(H, x, rows))


def test_sell_spmv_scipy_bitwise_at_c3_size(pk):
    """The same bitwise check on sampled rows of the full C3 matrix (64^3 Q1
    elasticity, 811,200 rows), for the plain and the fused PCG SpMV."""
    from paper_1512_05820_b200.problems import elasticity_sequence

    H = next(iter(elasticity_sequence((64, 64, 64), p=1))).A
    A = pk.SparseSpdMatrix(H.n, H.row_offsets, H.col_indices, H.values)
    assert A.bval is not None
    x = np.random.default_rng(23).standard_normal(H.n)
    rows = np.unique(np.concatenate([np.arange(96), H.n - 1 - np.arange(96),
                                     np.random.default_rng(5).integers(0, H.n, 1500)]))
    want = _csr_chain_rows(H, x, rows)
    got = pk.spmv(A, x).cpu().numpy()
    assert np.array_equal(got[rows], want)
    assert np.array_equal(got, _scipy_rows(H, x, np.arange(H.n)))
    # fused: one stepped PCG iteration stores A p_0 with p_0 = z = D^{-1} b
    M = pk.build_preconditioner("jacobi", A)
    b = torch.from_numpy(x).cuda()
    try:
        res = pk.augmented_pcg(A, b, precond=M, tol=0.0, max_iter=1, keep_products=True)
    except pk.NotConverged as exc:
        res = exc.partial
    p0 = res.V[:, 0].cpu().numpy()  # V holds the directions p_k as iterated
    assert np.array_equal(res.AV[:, 0].cpu().numpy()[rows], _csr_chain_rows(H, p0, rows))


def test_sell_spmm_columns_are_bitwise_spmv(pk):
    """K2 on the 3x3 SELL view: every column of A X is bitwise the SpMV of that
    column (same row chain), for widths that exercise full and ragged tiles."""
    from paper_1512_05820_b200.linalg import as_block, spmm
    from paper_1512_05820_b200.problems import elasticity_sequence

    H = next(iter(elasticity_sequence((7, 5, 6), p=1))).A
    A = pk.SparseSpdMatrix(H.n, H.row_offsets, H.col_indices, H.values)
    assert A.bval is not None
    for m in (1, 5, 8, 13):
        X = np.random.default_rng(m).standard_normal((H.n, m))
        Y = spmm(A, as_block(X)).cpu().numpy()
        for j in range(m):
            assert np.array_equal(Y[:, j], pk.spmv(A, X[:, j]).cpu().numpy()), (m, j)


def test_spmv_sink_counts_one_matvec(pk):
    A = pk.SparseSpdMatrix.identity(5)
    sink = pk.InstrumentationSink()
    pk.spmv(A, np.ones(5), sink)
    assert sink.matvecs == 1


def test_assemble_gram_matches_golden_and_counts(pk):
    d = gio.load("kernels")
    A = _dev_matrix(pk, d["rowptr"], d["col"], d["val"])
    sink = pk.InstrumentationSink()
    G, AS = pk.assemble_gram(A, d["S"], sink)
    np.testing.assert_allclose(AS.cpu().numpy(), d["AS"], rtol=1e-12, atol=1e-12 * np.abs(d["AS"]).max())
    np.testing.assert_allclose(G.cpu().numpy(), d["G"], rtol=1e-12, atol=1e-12 * np.abs(d["G"]).max())
    assert sink.gram_assemblies == 1 and sink.matvecs == d["S"].shape[1]


@pytest.mark.parametrize("n,m1,m2", [(1, 1, 1), (37, 3, 5), (1000, 64, 64), (4099, 65, 130), (70001, 20, 20),
                                     (20000, 200, 7)])
def test_dmma_gram_shapes(pk, n, m1, m2):
    from paper_1512_05820_b200.linalg import as_block, gram

    rng = np.random.default_rng(n + m1)
    X = rng.standard_normal((n, m1))
    Y = rng.standard_normal((n, m2))
    G = gram(as_block(X), as_block(Y)).cpu().numpy()
    ref = X.T @ Y
    np.testing.assert_allclose(G, ref, rtol=1e-11, atol=1e-12 * np.sqrt(n))


@pytest.mark.parametrize("n,m,y_old", [(5000, 7, 3), (3001, 130, 60), (20011, 386, 40), (9000, 700, 60),
                                       (40000, 129, 0), (1200, 257, 256), (700, 130, 60), (513, 64, 0),
                                       (100, 200, 64), (70000, 640, 64)])
@pytest.mark.parametrize("single", [True, False])
def test_dmma_symmetric_gram_upper_shapes(pk, n, m, y_old, single):
    """K7 in upper mode over balanced, fragment-masked units: widths that are
    not tile multiples (386 = 3 x 128 + 2), the two-segment right operand
    (stage-1 A W + the run's A p_k, one TMA box per buffer and a two-box
    straddling tile) and the per-block col_off path, diagonal tiles split by
    fragment-row pairs, few rows (tiles written straight to G) and many
    (split-K partials); every entry of the upper triangle matches numpy, and
    repeated calls are bitwise identical (fixed-order split reduction)."""
    from paper_1512_05820_b200.linalg import as_block, symmetric_gram_from_products

    rng = np.random.default_rng(n + m)
    Z = rng.standard_normal((n, m))
    AZ = rng.standard_normal((n, m))
    segs = [(as_block(AZ[:, :y_old]), 0)] if y_old else []
    segs.append((as_block(AZ[:, y_old:]), y_old))
    Zd = as_block(Z)
    U1 = symmetric_gram_from_products(Zd, segs, single_launch=single)
    U2 = symmetric_gram_from_products(Zd, segs, single_launch=single)
    assert torch.equal(U1.store, U2.store)
    G = np.asarray(U1)
    ref = Z.T @ AZ
    iu = np.triu_indices(m)
    np.testing.assert_allclose(G[iu], ref[iu], rtol=1e-11, atol=1e-12 * np.sqrt(n))


@pytest.mark.parametrize("n,m1,m2", [(811200, 60, 60), (100000, 3000, 110), (4096, 20, 20), (300000, 386, 386)])
def test_dmma_gram_workload_shapes(pk, n, m1, m2):
    """The Gram shapes the sequences issue: stage-1 W'(AW) (C3), the new
    columns of an accumulated C4 snapshot (w x k_new), C1, and a C2-width
    square; against a torch fp64 reference on the device."""
    from paper_1512_05820_b200.linalg import empty_block, gram

    gen = torch.Generator(device="cuda").manual_seed(m1 + m2)
    X, Y = empty_block(n, m1, "cuda"), empty_block(n, m2, "cuda")
    X.copy_(torch.randn(n, m1, generator=gen, device="cuda", dtype=torch.float64))
    Y.copy_(torch.randn(n, m2, generator=gen, device="cuda", dtype=torch.float64))
    G = gram(X, Y)
    ref = X.t() @ Y
    assert float((G - ref).abs().max()) <= 1e-12 * n ** 0.5 * 10


@pytest.mark.parametrize("n,s,y", [(1, 1, 1), (33, 17, 3), (4096, 100, 60), (9999, 300, 70)])
def test_dmma_gemm_nn_shapes(pk, n, s, y):
    from paper_1512_05820_b200.linalg import as_block, gemm_nn

    rng = np.random.default_rng(n + s)
    S = rng.standard_normal((n, s))
    C = rng.standard_normal((s, y))
    out = gemm_nn(as_block(S), C).cpu().numpy()
    np.testing.assert_allclose(out, S @ C, rtol=1e-11, atol=1e-12 * np.sqrt(s))


def test_gemv_pair(pk):
    from paper_1512_05820_b200.linalg import as_block, as_vector, gemv_n, gemv_t

    rng = np.random.default_rng(7)
    n, m = 5003, 41
    B = rng.standard_normal((n, m))
    x = rng.standard_normal(n)
    c = rng.standard_normal(m)
    Bd = as_block(B)
    np.testing.assert_allclose(gemv_t(Bd, as_vector(x)).cpu().numpy(), B.T @ x, rtol=1e-12, atol=1e-11)
    np.testing.assert_allclose(gemv_n(Bd, c).cpu().numpy(), B @ c, rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(gemv_n(Bd, c, as_vector(x), op=2).cpu().numpy(), x - B @ c, rtol=1e-12, atol=1e-12)


def test_spmm_matches_scipy(pk):
    from paper_1512_05820_b200.linalg import as_block, spmm
    from paper_1512_05820_b200.problems import elasticity_sequence

    H = next(iter(elasticity_sequence((4, 3, 3), p=1))).A
    A = pk.SparseSpdMatrix(H.n, H.row_offsets, H.col_indices, H.values)
    X = np.random.default_rng(3).standard_normal((H.n, 19))
    got = spmm(A, as_block(X)).cpu().numpy()
    ref = H.to_scipy() @ X
    np.testing.assert_allclose(got, ref, rtol=1e-12, atol=1e-12 * np.abs(ref).max())


def test_pod_from_gram_matches_reference(pk):
    d = gio.load("kernels")
    res = pk.pod_evd_from_gram(d["G"], d["S"], d["gamma"], 0.999)
    assert res.y == int(d["pod_y"])
    sig = d["pod_sigma"]
    lead = sig > 1e-6 * sig[0]
    np.testing.assert_allclose(res.singular_values[lead], sig[lead], rtol=1e-10)
    got = res.columns.cpu().numpy()
    ref = d["pod_basis"]
    for j in range(res.y):
        s = np.sign(got[:, j] @ ref[:, j])
        np.testing.assert_allclose(s * got[:, j], ref[:, j], rtol=1e-8, atol=1e-10 * np.abs(ref[:, j]).max())


def test_validation_errors(pk):
    with pytest.raises(pk.NotSymmetric):
        pk.SparseSpdMatrix.from_dense(np.array([[2.0, 1.0], [0.0, 2.0]]))
    with pytest.raises(pk.NotPositiveDefinite) as exc:
        pk.SparseSpdMatrix.from_dense(np.array([[2.0, 0.0, 0.0], [0.0, -1.0, 0.0], [0.0, 0.0, 1.0]]))
    assert exc.value.pivot == 1
    with pytest.raises(pk.DimensionMismatch):
        pk.SparseSpdMatrix(3, np.array([0, 1]), np.array([0]), np.array([1.0]))


def test_jacobi_inverse_diagonal_bitwise(pk):
    d = gio.load("kernels")
    A = _dev_matrix(pk, d["rowptr"], d["col"], d["val"])
    M = pk.build_preconditioner("jacobi", A)
    ref = 1.0 / scipy.sparse.csr_matrix((d["val"], d["col"], d["rowptr"])).diagonal()
    assert np.array_equal(M.fused_inverse_diagonal().cpu().numpy(), ref)
    r = np.random.default_rng(1).standard_normal(A.n)
    assert np.array_equal(M.apply(r).cpu().numpy(), r * ref)


def test_unsorted_input_is_canonicalised(pk):
    rowptr = np.array([0, 2, 4])
    col = np.array([1, 0, 1, 0])
    val = np.array([1.0, 4.0, 3.0, 1.0])
    A = pk.SparseSpdMatrix(2, rowptr, col, val)
    np.testing.assert_allclose(pk.spmv(A, np.array([1.0, 2.0])).cpu().numpy(), [6.0, 7.0])


def test_c5_small_pod_matches_reference(pk):
    """C5 at reduced size (Laplacian 16x16x32, 256 Gaussian snapshots): device
    Gram + on-device reduced eigenproblem vs the reference's LAPACK result."""
    import warnings

    from paper_1512_05820_b200.problems import laplacian3d, snapshot_matrix

    d = gio.load("c5_small")
    L = laplacian3d(16, 16, 32)
    A = pk.SparseSpdMatrix(L.n, L.row_offsets, L.col_indices, L.values)
    S = snapshot_matrix(L.n, 256, seed=5)
    G, _ = pk.assemble_gram(A, S)
    np.testing.assert_allclose(np.diag(G.cpu().numpy()), d["G_diag"], rtol=1e-12)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        res = pk.pod_evd_from_gram(G, S, np.ones(256), 1.0)
    assert res.y == int(d["y"])
    sig = d["sigma"]
    np.testing.assert_allclose(res.singular_values[:200], sig[:200], rtol=1e-10)
    got = res.columns[:, :20].cpu().numpy()
    ref = d["basis20"]
    for j in range(20):
        s = np.sign(got[:, j] @ ref[:, j])
        assert np.linalg.norm(s * got[:, j] - ref[:, j]) <= 1e-8 * np.linalg.norm(ref[:, j])


def test_c5_small_blocked_gram_matches_reference(pk):
    """The column-blocked Gram (A S never materialised, upper triangle only)
    gives the reference's POD on the C5-small golden: blocks of 96 columns so
    the diagonal blocks straddle the 64-row tiles."""
    import warnings

    from paper_1512_05820_b200.problems import laplacian3d, snapshot_matrix

    d = gio.load("c5_small")
    L = laplacian3d(16, 16, 32)
    A = pk.SparseSpdMatrix(L.n, L.row_offsets, L.col_indices, L.values)
    S = snapshot_matrix(L.n, 256, seed=5)
    sink = pk.InstrumentationSink()
    G = pk.assemble_gram_blocked(A, S, sink=sink, block=96)
    assert sink.snapshot()["matvecs"] == 256 and sink.snapshot()["gram_assemblies"] == 1
    Gh = np.asarray(G)
    np.testing.assert_allclose(np.diag(Gh), d["G_diag"], rtol=1e-12)
    Gf, _ = pk.assemble_gram(A, S)
    np.testing.assert_allclose(Gh, Gf.cpu().numpy(), rtol=0, atol=1e-12 * np.abs(Gh).max())
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        res = pk.pod_evd_from_gram(G, S, np.ones(256), 1.0)
    assert res.y == int(d["y"])
    np.testing.assert_allclose(res.singular_values[:200], d["sigma"][:200], rtol=1e-10)
    got = res.columns[:, :20].cpu().numpy()
    ref = d["basis20"]
    for j in range(20):
        s = np.sign(got[:, j] @ ref[:, j])
        assert np.linalg.norm(s * got[:, j] - ref[:, j]) <= 1e-8 * np.linalg.norm(ref[:, j])


def test_scalar_sell_spmv_and_spmm(pk):
    """7-point stencil (C2/C5 shape, reduced): the scalar SELL-32 view is chosen,
    SpMV equals scipy's csr_matvec bitwise, SpMM (lanes-per-row CSR kernel
    unless RK_SELL1_SPMM=1) agrees with it, and a forced lanes-per-row CSR agrees."""
    import scipy.sparse

    from paper_1512_05820_b200.linalg import as_block, spmm
    from paper_1512_05820_b200.problems import laplacian3d

    L = laplacian3d(24, 20, 36)
    A = pk.SparseSpdMatrix(L.n, L.row_offsets, L.col_indices, L.values)
    assert A.csr.bdim == 1 and A.bval is not None
    rng = np.random.default_rng(7)
    X = rng.standard_normal((L.n, 11))
    ref = scipy.sparse.csr_matrix((L.values, L.col_indices, L.row_offsets), shape=(L.n, L.n)) @ X
    Y = spmm(A, as_block(X)).cpu().numpy()
    for j in range(11):
        y = pk.spmv(A, X[:, j]).cpu().numpy()
        np.testing.assert_allclose(Y[:, j], y, rtol=1e-14, atol=1e-14 * np.abs(y).max())
        assert np.array_equal(y, ref[:, j])  # one row per lane in CSR order: scipy's arithmetic
    B = pk.SparseSpdMatrix(L.n, L.row_offsets, L.col_indices, L.values, lanes=2)
    assert B.csr.bdim == 0 and B.bval is None
    np.testing.assert_allclose(pk.spmv(B, X[:, 0]).cpu().numpy(), Y[:, 0], rtol=1e-14, atol=1e-13)


def test_device_spd_inverse_wide_factor(pk):
    """F^{-1} of a wide dense factor (>= 256 columns) comes from cuSOLVER potri
    on the device; it equals the host dtrtri route to rounding."""
    import scipy.linalg

    rng = np.random.default_rng(9)
    w = 300
    M = rng.standard_normal((w, w))
    G = M @ M.T + w * np.eye(w)
    L = pk.dense_cholesky(G)
    F = L.device_spd_inverse(torch.device("cuda", 0)).cpu().numpy()
    Li = np.tril(scipy.linalg.lapack.dtrtri(L.full(), lower=1)[0])
    np.testing.assert_allclose(F, Li.T @ Li, rtol=1e-11, atol=1e-13 * np.abs(F).max())


@pytest.mark.parametrize("case", ["elasticity", "stencil7", "poisson2d", "ragged", "long_rows"])
def test_device_pattern_views_equal_host_builders(pk, case):
    """the SELL-32 views built on the device (rk_sell_plan /
    rk_sell_fill) are bitwise the host builders' arrays (slice offsets, slot
    columns, value permutation), and both decline the same patterns."""
    import scipy.sparse as sp

    from paper_1512_05820_b200 import linalg as L
    from paper_1512_05820_b200.problems import elasticity_sequence, laplacian3d, poisson2d_matrix

    if case == "elasticity":
        H = next(iter(elasticity_sequence((7, 5, 4), p=1))).A
        rp, ci, n = np.asarray(H.row_offsets), np.asarray(H.col_indices), H.n
    elif case == "stencil7":
        H = laplacian3d(13, 9, 7)
        rp, ci, n = np.asarray(H.row_offsets), np.asarray(H.col_indices), H.n
    elif case == "poisson2d":
        H = poisson2d_matrix(33)
        rp, ci, n = np.asarray(H.row_offsets), np.asarray(H.col_indices), H.n
    else:
        rng = np.random.default_rng(4)
        n = 301
        dens = 0.01 if case == "ragged" else 0.08
        M = sp.random(n, n, density=dens, random_state=5, format="csr") + sp.eye(n, format="csr")
        M = (M + M.T).tocsr()
        M.sort_indices()
        rp, ci = M.indptr, M.indices
    dev = torch.device("cuda", 0)
    dr = torch.from_numpy(np.ascontiguousarray(rp, dtype=np.int32)).to(dev)
    dc = torch.from_numpy(np.ascontiguousarray(ci, dtype=np.int32)).to(dev)
    hb, db = L._bsr3_from_host(rp, ci, n, dev), L._bsr3_on_device(dr, dc, n, int(ci.size), dev)
    assert (hb is None) == (db is None)
    if hb is not None:
        assert hb.nblk == db.nblk and hb.nreal == db.nreal
        for a, b in ((hb.browptr, db.browptr), (hb.bcol, db.bcol), (hb.perm, db.perm)):
            assert torch.equal(a, b)
        return
    hs, ds = L._sell1_from_host(rp, ci, n, dev), L._sell1_on_device(dr, dc, n, int(ci.size), dev)
    assert (hs is None) == (ds is None), case
    if hs is not None:
        assert hs.nslot == ds.nslot
        for a, b in ((hs.sptr, ds.sptr), (hs.scol, ds.scol), (hs.perm, ds.perm)):
            assert torch.equal(a, b)
    if case == "long_rows":
        assert hs is None  # rows beyond SELL1_MAX_ROW keep the lanes-per-row CSR kernel
