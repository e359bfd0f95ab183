"""Whole-path parity: run_sequence on the device vs the reference's frozen
fixtures and golden runs (counters exact, x to 1e-8, q = c'x to 1e-10)."""

import json
import os
import warnings

import numpy as np
import torch
import pytest

import golden_io as gio


def _host(t):
    """numpy view of a result (host inputs give numpy, device inputs device tensors)."""
    return t.detach().cpu().numpy() if hasattr(t, "detach") else np.asarray(t)


pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pk():
    import paper_1512_05820_b200 as pk

    return pk


def _run(pk, seq, tr, mode, precond):
    cfg = pk.SolverConfig(truncation=pk.TruncationConfig(**tr), mode=mode)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        return pk.run_sequence(seq, cfg, precond_factory=lambda A: pk.build_preconditioner(precond, A))


def _sensitivity(make_seq, ocfg, c):
    """Per-system response of the reference algorithm (oracle) to scaling every
    right-hand side by (1 + 1e-15): relative change of q = c'x and of x."""
    from oracle import recycle_oracle as O

    xa, _, _ = O.run_sequence(make_seq(), ocfg)
    seq = make_seq()
    for s in seq.systems:
        s.b = s.b * (1 + 1e-15)
    xb, _, _ = O.run_sequence(seq, ocfg)
    dq = np.array([abs(c @ u - c @ v) / abs(c @ u) for u, v in zip(xa, xb)])
    dx = np.array([np.linalg.norm(u - v) / np.linalg.norm(u) for u, v in zip(xa, xb)])
    return dq, dx


def _log_exact(tag, first, total):
    """Record how many leading systems matched the reference exactly (set
    RK_EXACT_LOG=path to collect them; the floors below come from such a run)."""
    path = os.environ.get("RK_EXACT_LOG")
    if path:
        with open(path, "a") as fh:
            fh.write(json.dumps({"case": os.environ.get("PYTEST_CURRENT_TEST", "").split(" ")[0], "tag": tag,
                                 "exact": first, "systems": total}) + "\n")


def _check(d, tag, xs, reps, strict=True, c=None, sensitive=False, envelope=None, min_exact=None):
    """Parity policy (BASELINE north_star): iterations within +-2 per system,
    x to 1e-8 and q = c'x to 1e-10.

    A recycled sequence is chaotic in the last bit: the reference itself flips
    an exit test when its input is perturbed by 1e-15 (tests/test_oracle.py::
    test_reference_is_rounding_sensitive_on_c1_s5). So up to the first system
    whose iteration count differs, every counter must match exactly and x, q
    meet 1e-8 / 1e-10; from that system on (only allowed when ``strict`` is
    False) counts stay within +-2 and solutions agree at the forcing level."""
    cnt = gio.counters(d, tag)
    got = [r.stage3_iters for r in reps]
    want = list(map(int, cnt["stage3_iters"]))
    assert len(got) == len(want)
    first = next((j for j, (a, b) in enumerate(zip(got, want)) if a != b), len(got))
    _log_exact(tag, first, len(got))
    if strict:
        assert first == len(got), (tag, got, want)
    else:
        # a non-strict case still has a floor on the systems that match exactly
        # (counters, x to 1e-8, q to 1e-10): a change that breaks parity from
        # system 2 on fails here, however close the later counts stay
        assert min_exact is not None, "non-strict parity needs a floor of exactly-matched systems"
        assert first >= min_exact, (tag, f"{first} of {len(got)} systems exact, floor {min_exact}", got, want)
    assert all(abs(a - b) <= 2 for a, b in zip(got, want)), (tag, got, want)
    exact = slice(0, first)
    for key, attr in (("matvecs", "matvecs"), ("precond_applies", "precond_applies"),
                      ("stage2_iters", "stage2_iters"), ("stage1_dim", "stage1_dim")):
        assert [getattr(r, attr) for r in reps][exact] == list(map(int, cnt[key]))[exact], (tag, key)
    # ``sensitive``: a configuration in which the reference itself moves x by
    # up to ~3e-8 and q by ~1e-7 under a 1e-15 input perturbation
    # (test_oracle.py::test_reference_is_rounding_sensitive_on_c1_s5)
    # ``envelope`` = (dq, dx) from _sensitivity: the reference's own response to
    # a 1e-15 input perturbation; we allow 50x that (GPU reductions perturb
    # every dot product, not just the input), never less than 1e-10 / 1e-8.
    base_x, base_q = (1e-6, 1e-6) if sensitive else (1e-8, 1e-10)
    for j, x in enumerate(xs, start=1):
        xh = _host(x)
        if envelope is not None:
            base_q = max(1e-10, 50 * envelope[0][j - 1])
            base_x = max(1e-8, 50 * envelope[1][j - 1])
        tol_x = base_x if j - 1 < first else 1e-4
        key = f"{tag}x{j}"
        if key in d:
            ref = d[key]
            assert np.linalg.norm(xh - ref) <= tol_x * np.linalg.norm(ref), (tag, j)
        qkey = f"{tag}q{j}"
        if c is not None and qkey in d:
            q_ref = float(d[qkey])
            tol_q = base_q if j - 1 < first else 1e-4
            assert abs(float(c @ xh) - q_ref) <= tol_q * abs(q_ref), (tag, j)
    return first


# Leading systems that must match the reference exactly (counters, x to 1e-8,
# q to 1e-10) in each non-strict case: measured with RK_EXACT_LOG on a B200
# (deterministic kernels, so the count is reproducible; profiles/r02/
# exact_matches.jsonl), never lowered. Every case currently matches on every
# system, so each floor is the case's full length.
EXACT_FLOOR = {
    ("stage_variants", "s2_"): 5, ("stage_variants", "s2cg_"): 5, ("stage_variants", "phi1_"): 5,
    ("stage_variants", "prev_"): 5, ("stage_variants", "none_"): 5,
    ("elasticity", "cg_"): 4, ("elasticity", "fom_"): 4,
    ("c1", "fom_"): 20, ("c1", "cg_"): 20, ("c1", "s5_"): 20,
    ("c2_small", "cg_"): 4, ("c2_small", "fom_"): 4, ("c3_mid", "cg_"): 3, ("c3_mid", "fom_"): 3,
    ("next_strategies", "ctcr_"): 6, ("next_strategies", "ctcp_"): 6, ("next_strategies", "defl_"): 6,
    ("next_strategies", "defs_"): 6, ("next_strategies", "ssor_"): 6, ("next_strategies", "ssor15_"): 6,
}


FIXTURES = {
    "identity_like": (dict(strategy="none"), "identity"),
    "invariant_matrix": (dict(strategy="none", nu_w=1.0), "identity"),
    "drifting_pod": (dict(strategy="pod-a-rbf", nu_y=1.0, nu_w=1.0, storage_cap=30, max_dim=20), "jacobi"),
}


@pytest.mark.parametrize("name", list(FIXTURES))
def test_reference_fixture_counters(pk, name):
    d = gio.load(name)
    tr, pc = FIXTURES[name]
    xs, reps, _ = _run(pk, gio.sequence(d), tr, "fom", pc)
    frozen = gio.frozen(d)["frozen"]
    assert [r.stage3_iters for r in reps] == frozen["stage3_iters"]
    assert [r.stage2_iters for r in reps] == frozen["stage2_iters"]
    assert [r.stage1_dim for r in reps] == frozen["stage1_dims"]
    assert [r.matvecs for r in reps] == frozen["matvecs"]
    np.testing.assert_allclose([r.final_residual for r in reps], frozen["final_residuals"], rtol=1e-6, atol=1e-12)
    _check(d, "", xs, reps)


def test_drifting_pod_cg_mode(pk):
    d = gio.load("drifting_pod")
    tr, pc = FIXTURES["drifting_pod"]
    xs, reps, _ = _run(pk, gio.sequence(d), tr, "cg", pc)
    _check(d, "cg_", xs, reps)


STAGE = {
    "s2_": (dict(strategy="pod-a-rbf", nu_y=1.0, nu_w=1.0, stage1_dim=4, storage_cap=30, max_dim=20), "fom"),
    "s2cg_": (dict(strategy="pod-a-rbf", nu_y=1.0, nu_w=1.0, stage1_dim=4, storage_cap=30, max_dim=20), "cg"),
    "phi1_": (dict(strategy="pod-a-rbf", nu_y=1.0, nu_w=1.0, stage1_dim=4, full_orth=True, storage_cap=30,
                   max_dim=20), "fom"),
    "prev_": (dict(strategy="pod-a-prev", nu_y=0.999, nu_w=0.9, storage_cap=25, max_dim=12), "cg"),
    "none_": (dict(strategy="none", nu_w=1.0), "fom"),
}


@pytest.mark.parametrize("tag", list(STAGE))
def test_stage_variants(pk, tag):
    d = gio.load("stage_variants")
    tr, mode = STAGE[tag]
    xs, reps, _ = _run(pk, gio.sequence(d), tr, mode, "jacobi")
    _check(d, tag, xs, reps, strict=False, min_exact=EXACT_FLOOR[("stage_variants", tag)])


@pytest.mark.parametrize("tag,mode", [("cg_", "cg"), ("fom_", "fom")])
def test_elasticity_q1_sequence(pk, tag, mode):
    d = gio.load("elasticity")
    tr = dict(strategy="pod-a-rbf", nu_y=1.0, nu_w=1.0, storage_cap=12, max_dim=12)
    xs, reps, _ = _run(pk, gio.elasticity_sequence(d), tr, mode, "jacobi")
    _check(d, tag, xs, reps, strict=False, min_exact=EXACT_FLOOR[("elasticity", tag)])


@pytest.mark.parametrize("tag,mode,extra", [("fom_", "fom", {}), ("cg_", "cg", {}), ("s5_", "fom", {"stage1_dim": 5})])
def test_c1_poisson_sequence(pk, tag, mode, extra):
    from paper_1512_05820_b200.problems import poisson2d_sequence

    d = gio.load("c1")
    seq = poisson2d_sequence(64, p=int(d["p"]))
    tr = dict(strategy="pod-a-rbf", nu_y=1.0, nu_w=1.0, storage_cap=20, max_dim=20, **extra)
    xs, reps, _ = _run(pk, seq, tr, mode, "jacobi")
    first = _check(d, tag, xs, reps, strict=False, c=d["c"], sensitive=(tag == "s5_"),
                   min_exact=EXACT_FLOOR[("c1", tag)])
    # the fom and cg recipes are not rounding-sensitive: all 20 systems exact
    if tag in ("fom_", "cg_"):
        assert first == len(reps)


def test_reference_matrix_objects_are_accepted(pk):
    """Drop-in: host CSR objects with the reference's field names upload as-is."""
    d = gio.load("drifting_pod")
    seq = gio.sequence(d)
    A = pk.linalg.as_matrix(seq[0].A)
    assert A.n == seq.n and A.nnz == len(seq[0].A.values)


def test_affine_sequence_values_formed_on_device(pk):
    """a drifting sequence given as values = base + i * delta
    (problems.AffineHostCsr, the C3 generator) uploads base and delta once and
    forms every system's values on the GPU -- bitwise numpy's `base + i *
    delta`, in CSR order and in the SELL slots the SpMV streams -- and the
    sequence solves exactly as from materialised host matrices."""
    from paper_1512_05820_b200 import linalg as L
    from paper_1512_05820_b200.problems import HostCsr, LinearSystemSpec, SystemSequence, elasticity_sequence

    seq = elasticity_sequence((6, 5, 4), p=4, rtol=1e-6, seed=11)
    specs = list(seq)
    L.clear_upload_caches()
    for s in specs:
        A = pk.linalg.as_matrix(s.A)
        assert np.array_equal(A.values.cpu().numpy(), s.A.values)
        x = np.random.default_rng(0).standard_normal(seq.n)
        assert np.array_equal(A.matvec(x).cpu().numpy(), s.A.to_scipy() @ x) or \
            np.allclose(A.matvec(x).cpu().numpy(), s.A.to_scipy() @ x, rtol=1e-13, atol=1e-13)
    assert len(L._affine_cache) == 1                      # one upload of (base, delta) for the whole sequence
    plain = SystemSequence(seq.n, [LinearSystemSpec(A=HostCsr(s.A.n, s.A.row_offsets, s.A.col_indices, s.A.values),
                                                    b=s.b, xbar=None, tol=s.tol) for s in specs], C=seq.C)
    cfg = pk.SolverConfig(truncation=pk.TruncationConfig(strategy="pod-a-rbf", nu_y=1.0, nu_w=1.0, storage_cap=20,
                                                         max_dim=10), mode="cg")
    jac = lambda A: pk.build_preconditioner("jacobi", A)  # noqa: E731
    xs_a, reps_a, _ = pk.run_sequence(seq, cfg, precond_factory=jac)
    xs_p, reps_p, _ = pk.run_sequence(plain, cfg, precond_factory=jac)
    assert [r.stage3_iters for r in reps_a] == [r.stage3_iters for r in reps_p]
    for a, b in zip(xs_a, xs_p):
        assert np.array_equal(np.asarray(a), np.asarray(b))


@pytest.mark.parametrize("name,tag,mode,cap", [("c2_small", "cg_", "cg", 12), ("c2_small", "fom_", "fom", 12),
                                               ("c3_mid", "cg_", "cg", 30), ("c3_mid", "fom_", "fom", 30)])
def test_c2_c3_like_sequences(pk, name, tag, mode, cap):
    """Variable-coefficient 3-D diffusion (C2 shape) and Q1 elasticity (C3 shape,
    3x3-block SpMV path) against runs of the reference itself."""
    from oracle import recycle_oracle as O

    d = gio.load(name)
    tr = dict(strategy="pod-a-rbf", nu_y=1.0, nu_w=1.0, storage_cap=cap, max_dim=cap)
    xs, reps, _ = _run(pk, gio.pattern_sequence(d), tr, mode, "jacobi")
    env = _sensitivity(lambda: gio.pattern_sequence(d), O.Config(mode=mode, **tr), d["c"])
    first = _check(d, tag, xs, reps, strict=False, c=d["c"], envelope=env, min_exact=EXACT_FLOOR[(name, tag)])
    assert first >= 2  # at least the first two systems are bitwise-faithful in their counters
    if mode == "fom":  # full re-orthogonalisation is not rounding-chaotic: the plain bar holds
        assert env[0].max() < 1e-12


def test_concurrent_sequences_match_serial(pk):
    """The reference runs method configurations in threads (bench.py:160-205);
    the C-ABI is re-entrant, so concurrent sequences equal serial ones."""
    import concurrent.futures

    d = gio.load("drifting_pod")
    tr, pc = FIXTURES["drifting_pod"]
    serial = [_run(pk, gio.sequence(d), tr, mode, pc) for mode in ("fom", "cg")]
    with concurrent.futures.ThreadPoolExecutor(max_workers=2) as ex:
        futs = [ex.submit(_run, pk, gio.sequence(d), tr, mode, pc) for mode in ("fom", "cg")]
        conc = [f.result() for f in futs]
    for (xs_s, rep_s, _), (xs_c, rep_c, _) in zip(serial, conc):
        assert [r.stage3_iters for r in rep_s] == [r.stage3_iters for r in rep_c]
        assert [r.matvecs for r in rep_s] == [r.matvecs for r in rep_c]
        for a, b in zip(xs_s, xs_c):
            assert np.array_equal(a, b)  # deterministic kernels: bitwise identical


def test_not_converged_stage3_continues_and_stops(pk):
    """threestage.py:388-390,594-595: a starved stage 3 is reported, not raised;
    run_sequence stops at it unless stop_on_failure=False."""
    d = gio.load("drifting_pod")
    tr, pc = FIXTURES["drifting_pod"]
    cfg = pk.SolverConfig(truncation=pk.TruncationConfig(**tr), mode="fom", max_iter=5)
    jac = lambda A: pk.build_preconditioner(pc, A)  # noqa: E731
    xs, reps, _ = pk.run_sequence(gio.sequence(d), cfg, precond_factory=jac)
    assert len(reps) == 1 and not reps[0].converged and reps[0].stage3_iters == 5
    xs, reps, _ = pk.run_sequence(gio.sequence(d), cfg, precond_factory=jac, stop_on_failure=False)
    assert len(reps) == int(d["p"]) and not any(r.converged for r in reps)


def test_invariant_matrix_stage1_reuses_products(pk):
    """Invariant matrix, snapshot accumulating without truncation (C4 pattern):
    with one shared device matrix object stage 1 multiplies only the new
    columns of W (the cached A W columns are what the SpMM would give bit for
    bit); the run matches one with a fresh matrix object per system (full
    stage-1 SpMM + Gram every time) with identical counters."""
    from paper_1512_05820_b200.problems import poisson2d_sequence

    seq = poisson2d_sequence(32, p=6)
    specs = list(seq)
    A0 = pk.SparseSpdMatrix.from_host(specs[0].A)
    shared = pk.SystemSequence(seq.n, [pk.LinearSystemSpec(A=A0, b=s.b, xbar=None, tol=s.tol) for s in specs],
                               C=seq.C)
    fresh = pk.SystemSequence(seq.n, [pk.LinearSystemSpec(A=A0.with_values(A0.values.clone()), b=s.b, xbar=None,
                                                          tol=s.tol) for s in specs], C=seq.C)
    tr = dict(strategy="pod-a-rbf", nu_y=1.0, nu_w=1.0, storage_cap=1000, max_dim=60)
    xs_a, rep_a, _ = _run(pk, shared, tr, "cg", "jacobi")
    xs_b, rep_b, _ = _run(pk, fresh, tr, "cg", "jacobi")
    assert rep_a[-1].basis_dim > 0 and not any(r.truncated for r in rep_a)
    assert [r.matvecs for r in rep_a] == [r.matvecs for r in rep_b]
    assert [r.stage3_iters for r in rep_a] == [r.stage3_iters for r in rep_b]
    for a, b in zip(xs_a, xs_b):
        a, b = _host(a), _host(b)
        assert np.linalg.norm(a - b) <= 1e-10 * np.linalg.norm(b)


def test_copied_state_never_writes_into_shared_storage(pk):
    """RecycleState grows Y and reuses A W storage in place; a shallow copy
    (copy.copy) shares those tensors but must not write into them: two
    branches continued from a copy give bitwise the results of branches
    continued from a deep copy."""
    import copy

    from paper_1512_05820_b200.problems import poisson2d_sequence

    specs = list(poisson2d_sequence(32, p=6))
    A = pk.SparseSpdMatrix.from_host(specs[0].A)
    M = pk.build_preconditioner("jacobi", A)
    cfg = pk.SolverConfig(truncation=pk.TruncationConfig(strategy="pod-a-rbf", nu_y=1.0, nu_w=1.0,
                                                         storage_cap=1000, max_dim=60), mode="cg")
    tol = pk.StageTolerances(eps=specs[0].tol)

    def branch_pair(shallow):
        st = pk.RecycleState.empty(A.n, A.device)
        for s in specs[:2]:
            _, _, st = pk.solve_system(A, s.b, None, st, tol, cfg, M=M)
        if shallow:
            other = copy.copy(st)
        else:
            other = pk.RecycleState(n=st.n, Y=st.Y.clone(), stage1_idx=list(st.stage1_idx),
                                    last_trunc_index=st.last_trunc_index, systems_seen=st.systems_seen)
        other.history = copy.deepcopy(st.history)
        other.stage1_idx = list(st.stage1_idx)
        xs = []
        for a, b in ((specs[2], specs[3]), (specs[4], specs[5])):
            xa, _, st = pk.solve_system(A, a.b, None, st, tol, cfg, M=M)
            xb, _, other = pk.solve_system(A, b.b, None, other, tol, cfg, M=M)
            xs += [_host(xa), _host(xb)]
        return xs

    deep = branch_pair(False)
    shallow = branch_pair(True)
    for u, v in zip(deep, shallow):
        assert np.array_equal(u, v)
