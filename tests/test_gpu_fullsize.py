"""Size-independent properties at BASELINE's full sizes, where the oracle
would take minutes per system: the solver's exit residual is the true
residual, every run converged within the reference's tolerance, the
truncated POD basis is A-orthonormal (Phi' A Phi = I), and the C5 POD
basis reconstructs the snapshot energy."""

import os

import numpy as np
import pytest
import torch


def _host(t):
    """numpy view of a result (host inputs give numpy, device inputs device tensors)."""
    return t.detach().cpu().numpy() if hasattr(t, "detach") else np.asarray(t)


pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pk():
    import paper_1512_05820_b200 as pk

    return pk


def _true_residual(A_host, b, x):
    import scipy.sparse

    As = scipy.sparse.csr_matrix((A_host.values, A_host.col_indices, A_host.row_offsets), shape=(A_host.n,) * 2)
    return float(np.linalg.norm(b - As @ x))


@pytest.mark.parametrize("workload", ["c3", "c2"])
def test_full_size_sequence_residuals_and_basis(pk, workload):
    """C3 (811,200 DOF Q1 elasticity, 3x3-block SELL) and C2 (2.1M-row
    diffusion, scalar SELL), first 3 systems at full size: each x meets
    ||b - A x|| <= tol (checked on the host with scipy, independent of the
    device residual recurrence, allowing the recurrence/true-residual drift
    of 1e-3 relative the reference also has), and after every truncation the
    new basis is A-orthonormal (leading 10 modes) to 1e-9."""
    from paper_1512_05820_b200.problems import diffusion3d_sequence, elasticity_sequence
    from paper_1512_05820_b200.linalg import assemble_gram

    if workload == "c3":
        seq, cap = elasticity_sequence((64, 64, 64), p=3, rtol=1e-5, seed=3), 60
    else:
        seq, cap = diffusion3d_sequence(128, p=3, rtol=1e-4, seed=2), 40
    specs = list(seq)
    cfg = pk.SolverConfig(truncation=pk.TruncationConfig(strategy="pod-a-rbf", nu_y=1.0, nu_w=1.0,
                                                         storage_cap=cap, max_dim=cap), mode="cg")
    state = pk.RecycleState.empty(seq.n, torch.device("cuda", 0))
    for j, s in enumerate(specs):
        A = pk.SparseSpdMatrix.from_host(s.A)
        M = pk.build_preconditioner("jacobi", A)
        x, rep, state = pk.solve_system(A, s.b, None, state, pk.StageTolerances(eps=s.tol), cfg, M=M)
        assert rep.converged and rep.stage3_iters > 0
        res = _true_residual(s.A, s.b, _host(x))
        assert res <= s.tol * (1 + 1e-3), (j, res, s.tol)
        if rep.truncated:
            # leading modes (the trailing ones carry sigma_1 / sigma_i rounding amplification)
            G, _ = assemble_gram(A, state.Y[:, :10])
            G = G.cpu().numpy()
            assert np.abs(G - np.eye(G.shape[0])).max() <= 1e-9


def test_c5_full_size_pod_properties(pk):
    """C5 shape (7-point Laplacian on 128x128x256, N = 4,194,304) with 64
    Gaussian snapshots: the column-blocked Gram is symmetric positive, the POD
    basis is A-orthonormal and reproduces S in the A-norm (sum of sigma^2 =
    trace of the Gram)."""
    from paper_1512_05820_b200.linalg import assemble_gram, empty_block
    from paper_1512_05820_b200.problems import laplacian3d

    L = laplacian3d(128, 128, 256)
    A = pk.SparseSpdMatrix(L.n, L.row_offsets, L.col_indices, L.values)
    S = empty_block(L.n, 64, "cuda")
    S.normal_(generator=torch.Generator(device="cuda").manual_seed(5))
    G = pk.assemble_gram_blocked(A, S, block=40)
    Gh = np.asarray(G)
    Gf, _ = assemble_gram(A, S)
    np.testing.assert_allclose(Gh, Gf.cpu().numpy(), rtol=0, atol=1e-11 * np.abs(Gh).max())
    import warnings

    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        res = pk.pod_evd_from_gram(G, S, np.ones(64), 1.0)
    Phi = res.columns
    P, _ = assemble_gram(A, Phi)
    assert np.abs(P.cpu().numpy() - np.eye(Phi.shape[1])).max() <= 1e-12
    np.testing.assert_allclose(np.sum(res.singular_values ** 2), np.trace(Gh), rtol=1e-12)


def test_c3_full_size_prefix_matches_reference(pk):
    """The bench's own C3 workload at full size (N = 811,200): its first two
    systems against the reference itself (tests/golden/c3_full.npz, made by
    oracle/make_golden.py run_c3_full). At this size the algorithm is
    rounding-chaotic: the reference, with every right-hand side scaled by
    (1 + 1e-15), keeps system 1 (748 iterations, x moves 6.4e-10) but takes
    669 instead of 670 iterations on system 2 (x moves 5.4e-8, q 1.2e-8). The
    bar: stage-3 counts within +-2 of the reference, and x / q = c'x within
    the north-star's 1e-8 / 1e-10 or, where the reference's own envelope is
    wider, within 5x that envelope. Measured (scipy-exact SpMV): system 1 748
    iterations, x 1.3e-9, q 7.1e-10; system 2 669, x 5.9e-8, q 1.3e-8."""
    import warnings

    import golden_io as gio
    from paper_1512_05820_b200.problems import elasticity_sequence

    d = gio.load("c3_full")
    p = int(d["p"])
    seq = elasticity_sequence((64, 64, 64), p=p, rtol=1e-5, seed=3)
    cfg = pk.SolverConfig(truncation=pk.TruncationConfig(strategy="pod-a-rbf", nu_y=1.0, nu_w=1.0,
                                                         storage_cap=60, max_dim=60), mode="cg")
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        xs, reps, _ = pk.run_sequence(seq, cfg, precond_factory=lambda A: pk.build_preconditioner("jacobi", A))
    idx = d["idx"]
    for j, (x, r) in enumerate(zip(xs, reps), start=1):
        assert abs(r.stage3_iters - int(d["cg_stage3_iters"][j - 1])) <= 2
        xh = _host(x)
        q, qref = float(seq.C[0] @ xh), float(d[f"cg_q{j}"])
        env_q = abs(float(d[f"pert_q{j}"]) - qref) / abs(qref)
        assert abs(q - qref) / abs(qref) <= max(1e-10, 5 * env_q), (j, q, qref, env_q)
        ref = d[f"cg_xs{j}"]
        env_x = float(d[f"pert_xrel{j}"])
        assert np.linalg.norm(xh[idx] - ref) / np.linalg.norm(ref) <= max(1e-8, 5 * env_x)
    # the first system (plain Jacobi PCG) is not chaotic at the 1e-15 level: exact counters
    assert reps[0].stage3_iters == int(d["cg_stage3_iters"][0])
    assert reps[0].matvecs == int(d["cg_matvecs"][0])


def test_c2_full_size_prefix_matches_oracle(pk):
    """C2 at full size (128^3 diffusion, N = 2,097,152, the scalar SELL-32
    path): its first two systems through the pinned oracle on the host and
    through the device path give identical iteration counts and counters and
    x / q = c'x within 1e-12 (measured: 1e-14 -- the SELL rows are scipy's
    csr_matvec bit for bit, only the dot-product order differs)."""
    import warnings

    from oracle import recycle_oracle as O
    from paper_1512_05820_b200.problems import diffusion3d_sequence

    tr = dict(strategy="pod-a-rbf", nu_y=1.0, nu_w=1.0, storage_cap=40, max_dim=40)
    seq = diffusion3d_sequence(128, p=2, rtol=1e-4, seed=2)
    specs = list(seq)
    oxs, oreps, _ = O.run_sequence(specs, O.Config(mode="cg", **tr), precond="jacobi")
    cfg = pk.SolverConfig(truncation=pk.TruncationConfig(**tr), mode="cg")
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        xs, reps, _ = pk.run_sequence(pk.SystemSequence(seq.n, specs, C=seq.C), cfg,
                                      precond_factory=lambda A: pk.build_preconditioner("jacobi", A))
    assert [r.stage3_iters for r in reps] == [r.stage3_iters for r in oreps]
    assert [r.matvecs for r in reps] == [r.matvecs for r in oreps]
    for x, ox in zip(xs, oxs):
        xh = _host(x)
        assert np.linalg.norm(xh - ox) <= 1e-12 * np.linalg.norm(ox)
        assert abs(seq.C[0] @ xh - seq.C[0] @ ox) <= 1e-12 * abs(seq.C[0] @ ox)


def test_c3_sequence_within_reference_envelope(pk):
    """The bench's 40-system C3 sequence against the reference's own run of it
    (tests/golden/c3_seq.npz, oracle/run_reference_c3.py) and the reference's
    rounding envelope: recykl's own runs of the same sequence with every
    right-hand side scaled by 1 + 1e-15 and by 1 - 1e-15, all 40 systems each
    (c3_seq_pert_p40.npz, c3_seq_pert_m40.npz, oracle/run_reference_seq.py
    --pert, ~100 minutes per run; the shorter earlier runs, made with other
    BLAS thread counts, are used too where they reach).
    The reference is chaotic at this size in CG mode: a 1e-15 perturbation
    moves system 4 by 6 iterations, system 9 by 26, system 18 by 44 (7.3%) and
    systems 34-36 by 110 (26%: the drop to ~430 iterations arrives four
    systems later or earlier), the 40-system total from 22,513 to 23,534 /
    23,256 (ours: 23,258). So, per system: systems 1-3
    (reference swing <= 2) within +-2; every system within twice the largest
    relative swing any perturbed reference run has shown up to that system,
    plus 1%; q and x within 5x the reference's own envelope on the systems a
    perturbed run covers; and the 40-system iteration total within 5% of the
    reference's. (FOM mode, recykl's default, is not chaotic and is held to
    the plain north-star bar in test_c3_fom_matches_reference_full_size.)"""
    import os
    import warnings

    from paper_1512_05820_b200.problems import elasticity_sequence

    gdir = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
    d = np.load(os.path.join(gdir, "c3_seq.npz"))
    p = int(d["p_done"])
    ref = d["iters"][:p].astype(float)
    swing = np.zeros(p)          # largest relative swing of any perturbed run, per system
    covered = np.zeros(p, bool)
    env_q = env_x = 0.0
    for name in ("c3_seq_pert", "c3_seq_pert_m", "c3_seq_pert_p", "c3_seq_pert_m40", "c3_seq_pert_p40"):
        path = os.path.join(gdir, name + ".npz")
        if not os.path.exists(path):
            continue
        e = np.load(path)
        pe = min(int(e["p_done"]), p)
        swing[:pe] = np.maximum(swing[:pe], np.abs(e["iters"][:pe] - ref[:pe]) / ref[:pe])
        covered[:pe] = True
        env_q = max(env_q, float(np.max(np.abs(e["q"][:pe] - d["q"][:pe]) / np.abs(d["q"][:pe]))))
        env_x = max(env_x, float(np.max(np.linalg.norm(e["xs"][:pe] - d["xs"][:pe], axis=1)
                                        / np.linalg.norm(d["xs"][:pe], axis=1))))
    env_rel = np.maximum.accumulate(swing)
    assert covered[:18].all()
    seq = elasticity_sequence((64, 64, 64), p=p, rtol=1e-5, seed=3)
    cfg = pk.SolverConfig(truncation=pk.TruncationConfig(strategy="pod-a-rbf", nu_y=1.0, nu_w=1.0,
                                                         storage_cap=60, max_dim=60), mode="cg")
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        xs, reps, _ = pk.run_sequence(seq, cfg, precond_factory=lambda A: pk.build_preconditioner("jacobi", A))
    its = np.array([r.stage3_iters for r in reps])
    assert all(r.converged for r in reps)
    assert np.abs(its[:3] - ref[:3]).max() <= 2
    pc = int(covered.sum())      # perturbed runs cover a prefix
    assert covered[:pc].all()
    rel = np.abs(its[:pc] - ref[:pc]) / ref[:pc]
    assert np.all(rel <= 2 * env_rel[:pc] + 0.01), (rel, env_rel)
    assert abs(int(its.sum()) - int(ref.sum())) <= 0.05 * int(ref.sum())
    idx = d["idx"]
    for j in range(pc):
        xh = _host(xs[j])
        q = float(seq.C[0] @ xh)
        assert abs(q - d["q"][j]) / abs(d["q"][j]) <= max(1e-10, 5 * env_q)
        assert np.linalg.norm(xh[idx] - d["xs"][j]) / np.linalg.norm(d["xs"][j]) <= max(1e-8, 5 * env_x)


def test_c2_sequence_matches_reference_run(pk):
    """The bench's C2 sequence (128^3 diffusion, 30 systems, N = 2,097,152)
    against the reference's own run of it (tests/golden/c2_seq.npz,
    oracle/run_reference_c2.py): the north-star bar on every system --
    identical stage-3 iterations and counters, q = c'x within 1e-10 and x
    (at 2000 fixed indices) within 1e-8 (measured: q <= 1e-12, x <= 6e-13)."""
    import os
    import warnings

    from paper_1512_05820_b200.problems import diffusion3d_sequence

    d = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "c2_seq.npz"))
    p = int(d["p_done"])
    seq = diffusion3d_sequence(128, p=p, rtol=1e-4, seed=2)
    cfg = pk.SolverConfig(truncation=pk.TruncationConfig(strategy="pod-a-rbf", nu_y=1.0, nu_w=1.0,
                                                         storage_cap=40, max_dim=40), mode="cg")
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        xs, reps, _ = pk.run_sequence(seq, cfg, precond_factory=lambda A: pk.build_preconditioner("jacobi", A))
    assert [r.stage3_iters for r in reps] == d["iters"][:p].tolist()
    assert [r.matvecs for r in reps] == d["matvecs"][:p].tolist()
    idx = d["idx"]
    for j, x in enumerate(xs):
        xh = _host(x)
        q = float(seq.C[0] @ xh)
        assert abs(q - d["q"][j]) <= 1e-10 * abs(d["q"][j])
        assert np.linalg.norm(xh[idx] - d["xs"][j]) <= 1e-8 * np.linalg.norm(d["xs"][j])


def _reference_run(name):
    import os

    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", f"{name}.npz")
    if not os.path.exists(path):
        pytest.skip(f"{name}.npz not generated (oracle/run_reference_seq.py)")
    return np.load(path)


def _run_prefix(pk, seq, cfg):
    import warnings

    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        return pk.run_sequence(seq, cfg, precond_factory=lambda A: pk.build_preconditioner("jacobi", A))


def test_c3_fom_matches_reference_full_size(pk):
    """The north-star configuration (C3: 64^3 Q1 elasticity, N = 811,200) in
    the reference's DEFAULT mode, fom (threestage.py:68; two re-orthogonalisation
    sweeps per iteration, krylov.py:327-337), against recykl's own run of its
    first systems (tests/golden/c3_fom.npz, oracle/run_reference_seq.py
    --mode fom). Full re-orthogonalisation is not rounding-chaotic, so the
    plain north-star bar holds on every system: identical stage-3 iterations
    and matvecs, x (at 2000 fixed indices) within 1e-8, q = c'x within 1e-10."""
    from paper_1512_05820_b200.problems import elasticity_sequence

    d = _reference_run("c3_fom")
    p = int(d["p_done"])
    seq = elasticity_sequence((64, 64, 64), p=p, rtol=1e-5, seed=3)
    cfg = pk.SolverConfig(truncation=pk.TruncationConfig(strategy="pod-a-rbf", nu_y=1.0, nu_w=1.0,
                                                         storage_cap=60, max_dim=60), mode="fom")
    xs, reps, _ = _run_prefix(pk, seq, cfg)
    assert [r.stage3_iters for r in reps] == d["iters"][:p].tolist()
    assert [r.matvecs for r in reps] == d["matvecs"][:p].tolist()
    idx = d["idx"]
    for j, x in enumerate(xs):
        xh = _host(x)
        q = float(seq.C[0] @ xh)
        assert abs(q - d["q"][j]) <= 1e-10 * abs(d["q"][j]), (j, q, d["q"][j])
        assert np.linalg.norm(xh[idx] - d["xs"][j]) <= 1e-8 * np.linalg.norm(d["xs"][j]), j


def test_c4_prefix_matches_reference(pk):
    """C4 (BASELINE configs[3]: 128x128x64 Q1 elasticity, K + M/dt^2, N =
    3,219,840, one invariant matrix, rtol 1e-6, pod-a-rbf cap 3000) against
    recykl's own runs of its first systems (tests/golden/c4_prefix*.npz,
    oracle/run_reference_seq.py --workload c4). System 1 is plain Jacobi PCG,
    the later ones the stage-1 direct projection onto all stored directions
    (125, 241, ... columns) followed by augmented CG. The north-star bar on
    every system: identical stage-3 iterations, matvecs, preconditioner
    applications and basis dimensions, x (at 2000 fixed indices) within 1e-8,
    q = c'x within 1e-10 -- or, where the reference does not reproduce itself
    to that bar, within twice its own run-to-run difference: recykl runs with
    8, 6 and 5 BLAS threads differ from each other by 1.1e-9 / 3.7e-8 in q
    and 2.8e-10 / 2.3e-8 in x on systems 1 / 2 at identical counters (rtol
    1e-6 stops the iteration long before 1e-10, and numpy's dot order follows
    the threads). Measured on the first two systems: q within 1.7e-9 /
    8.6e-12 of the 6-thread run, 2.8e-9 / 3.7e-8 of the 8-thread one --
    inside the reference's own scatter."""
    from paper_1512_05820_b200.problems import elasticity_sequence

    runs = []
    for name in ("c4_prefix4", "c4_prefix4b", "c4_prefix", "c4_prefix3"):
        path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", name + ".npz")
        if os.path.exists(path):
            runs.append(np.load(path))
    if not runs:
        pytest.skip("c4_prefix*.npz not generated (oracle/run_reference_seq.py)")
    runs.sort(key=lambda r: -int(r["p_done"]))
    d = runs[0]
    p = int(d["p_done"])
    # the reference's own scatter per system: the largest pairwise difference of its runs,
    # carried forward (it only grows along a recycled sequence) to systems one run covers
    env_q, env_x = np.zeros(p), np.zeros(p)
    for o in runs[1:]:
        po = min(int(o["p_done"]), p)
        assert o["iters"][:po].tolist() == d["iters"][:po].tolist()
        env_q[:po] = np.maximum(env_q[:po], np.abs(o["q"][:po] - d["q"][:po]) / np.abs(d["q"][:po]))
        env_x[:po] = np.maximum(env_x[:po], np.linalg.norm(o["xs"][:po] - d["xs"][:po], axis=1)
                                / np.linalg.norm(d["xs"][:po], axis=1))
    env_q, env_x = np.maximum.accumulate(env_q), np.maximum.accumulate(env_x)
    seq = elasticity_sequence((128, 128, 64), p=p, rtol=1e-6, seed=4, dynamic=True)
    cfg = pk.SolverConfig(truncation=pk.TruncationConfig(strategy="pod-a-rbf", nu_y=1.0, nu_w=1.0,
                                                         storage_cap=3000, max_dim=60), mode="cg")
    xs, reps, _ = _run_prefix(pk, seq, cfg)
    assert [r.stage3_iters for r in reps] == d["iters"][:p].tolist()
    assert [r.matvecs for r in reps] == d["matvecs"][:p].tolist()
    assert [r.precond_applies for r in reps] == d["precond"][:p].tolist()
    assert [r.basis_dim for r in reps] == d["basis_dim"][:p].tolist()
    idx = d["idx"]
    for j, x in enumerate(xs):
        xh = _host(x)
        q = float(seq.C[0] @ xh)
        tol_q, tol_x = max(1e-10, 2 * env_q[j]), max(1e-8, 2 * env_x[j])
        assert abs(q - d["q"][j]) <= tol_q * abs(d["q"][j]), (j, q, d["q"][j])
        assert np.linalg.norm(xh[idx] - d["xs"][j]) <= tol_x * np.linalg.norm(d["xs"][j]), j


def test_c5_full_size_matches_reference(pk):
    """C5 (BASELINE configs[4]) at full size: A = 7-point Laplacian on
    128 x 128 x 256 (N = 4,194,304), S = 256 N(0,1) snapshots from the same
    seeded host generator, G = assemble_gram(A, S) and pod_evd_from_gram(G, S,
    1, 1.0) on the device against recykl's own run (tests/golden/
    c5_full_m256.npz, oracle/run_reference_c5.py; linalg.py:160-174,
    pod.py:123-131). Bar: G's diagonal and sampled entries within 1e-12
    relative, sigma within 1e-10, the same retained dimension y, Phi at 2000
    rows within 1e-8 (column signs are LAPACK's choice: aligned first)."""
    from paper_1512_05820_b200.linalg import as_block, assemble_gram
    from paper_1512_05820_b200.problems import laplacian3d, snapshot_matrix

    d = _reference_run("c5_full_m256")
    m = int(d["m"])
    L = laplacian3d(128, 128, 256)
    A = pk.SparseSpdMatrix(L.n, L.row_offsets, L.col_indices, L.values)
    S = as_block(snapshot_matrix(L.n, m, seed=int(d["seed"])))
    G, AS = assemble_gram(A, S)
    del AS
    Gh = _host(G)
    np.testing.assert_allclose(np.diag(Gh), d["G_diag"], rtol=1e-12)
    ij = d["G_ij"]
    np.testing.assert_allclose(Gh[ij[:, 0], ij[:, 1]], d["G_ij_val"], rtol=1e-12,
                               atol=1e-12 * np.abs(d["G_diag"]).max())
    import warnings

    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        res = pk.pod_evd_from_gram(G, S, np.ones(m), 1.0)
    assert res.y == int(d["y"])
    np.testing.assert_allclose(res.singular_values, d["sigma"], rtol=1e-10)
    rows = torch.from_numpy(d["rows"]).to("cuda")
    phi = res.columns[rows].cpu().numpy()
    ref = d["phi_rows"][:, :phi.shape[1]]
    sign = np.sign(np.sum(phi * ref, axis=0))
    assert np.all(sign != 0)
    phi = phi * sign
    assert np.linalg.norm(phi - ref) <= 1e-8 * np.linalg.norm(ref)
    colerr = np.linalg.norm(phi - ref, axis=0) / np.linalg.norm(ref, axis=0)
    assert colerr.max() <= 1e-8, colerr.max()
