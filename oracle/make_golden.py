"""Generate golden vectors by running the REFERENCE itself (test infrastructure).

Imports ``recykl`` from /root/reference/pkg/src (read-only, in this container
only), runs its public API on seeded inputs and writes small compressed
fixtures to tests/golden/. The GPU box never reads /root/reference: the tests
there only read these committed fixtures.

    python oracle/make_golden.py            # rewrites tests/golden/*.npz
    python oracle/make_golden.py run_next_strategies   # one generator only
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

REF_SRC = "/root/reference/pkg/src"
REF_FIX = "/root/reference/pkg/tests/fixtures"
HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(os.path.dirname(HERE), "tests", "golden")
sys.path.insert(0, os.path.dirname(HERE))


def _ref():
    if REF_SRC not in sys.path:
        sys.path.insert(0, REF_SRC)
    import recykl  # noqa: F401

    return recykl


def _pack_sequence(seq, prefix):
    d = {}
    for j, spec in enumerate(seq, start=1):
        A = spec.A
        d[f"{prefix}A{j}_rowptr"] = np.asarray(A.row_offsets, dtype=np.int64)
        d[f"{prefix}A{j}_col"] = np.asarray(A.col_indices, dtype=np.int64)
        d[f"{prefix}A{j}_val"] = np.asarray(A.values, dtype=np.float64)
        d[f"{prefix}b{j}"] = np.asarray(spec.b, dtype=np.float64)
        d[f"{prefix}tol{j}"] = np.float64(spec.tol)
    d[f"{prefix}p"] = np.int64(len(list(seq)))
    d[f"{prefix}n"] = np.int64(seq.n)
    return d


def _pack_run(solutions, reports, prefix):
    d = {}
    for key in ("stage3_iters", "stage2_iters", "stage1_dim", "matvecs", "precond_applies", "final_residual",
                "truncated", "converged"):
        d[f"{prefix}{key}"] = np.asarray([getattr(r, key) for r in reports])
    for j, x in enumerate(solutions, start=1):
        d[f"{prefix}x{j}"] = np.asarray(x, dtype=np.float64)
    return d


def run_fixture_cases(rk):
    """Replay the reference's frozen fixture cases with the reference and keep
    the inputs (its xorshift generator is not part of the product)."""
    from recykl import preconditioners
    from recykl.problems import gen_diffusion_sequence
    from recykl.threestage import SolverConfig, run_sequence
    from recykl.truncation import TruncationConfig

    out = {}
    for name in ("identity_like", "invariant_matrix", "drifting_pod"):
        with open(os.path.join(REF_FIX, f"{name}.json")) as fh:
            payload = json.load(fh)
        case = payload["case"]
        gen = dict(case["generator"])
        gen["grid"] = tuple(gen["grid"])
        seq = gen_diffusion_sequence(**gen)
        variants = {"": dict(mode="fom")}
        if name == "drifting_pod":
            variants.update({
                "cg_": dict(mode="cg"),
                "paper_": dict(mode="fom", paper=True),
            })
        d = _pack_sequence(seq, "")
        d["frozen_json"] = np.asarray(json.dumps(payload))
        for tag, v in variants.items():
            cfg = SolverConfig(truncation=TruncationConfig(**case["config"]), mode=v["mode"])
            pf = None
            if case["precond"] != "identity":
                pf = lambda A, kind=case["precond"]: preconditioners.build(kind, A)
            else:
                pf = lambda A: preconditioners.build("identity", A)
            if v.get("paper"):
                continue  # paper_fom_beta is not reachable through run_sequence
            xs, reps, _ = run_sequence(seq, cfg, precond_factory=pf)
            d.update(_pack_run(xs, reps, tag))
        out[name] = d
    return out


def run_stage_variants(rk):
    """drifting-like sequences that exercise stage 2 (stage1_dim < y) and phi = 1."""
    from recykl import preconditioners
    from recykl.problems import gen_diffusion_sequence
    from recykl.threestage import SolverConfig, run_sequence
    from recykl.truncation import TruncationConfig

    seq = gen_diffusion_sequence((10, 10), p=5, delta=0.05, seed=37, tol=1e-9)
    d = _pack_sequence(seq, "")
    pf = lambda A: preconditioners.build("jacobi", A)  # noqa: E731
    cases = {
        "s2_": dict(tr=dict(strategy="pod-a-rbf", nu_y=1.0, nu_w=1.0, stage1_dim=4, storage_cap=30, max_dim=20),
                    mode="fom"),
        "s2cg_": dict(tr=dict(strategy="pod-a-rbf", nu_y=1.0, nu_w=1.0, stage1_dim=4, storage_cap=30, max_dim=20),
                      mode="cg"),
        "phi1_": dict(tr=dict(strategy="pod-a-rbf", nu_y=1.0, nu_w=1.0, stage1_dim=4, full_orth=True,
                              storage_cap=30, max_dim=20), mode="fom"),
        "prev_": dict(tr=dict(strategy="pod-a-prev", nu_y=0.999, nu_w=0.9, storage_cap=25, max_dim=12),
                      mode="cg"),
        "none_": dict(tr=dict(strategy="none", nu_w=1.0), mode="fom"),
    }
    for tag, c in cases.items():
        cfg = SolverConfig(truncation=TruncationConfig(**c["tr"]), mode=c["mode"])
        xs, reps, _ = run_sequence(seq, cfg, precond_factory=pf)
        d.update(_pack_run(xs, reps, tag))
    return {"stage_variants": d}


def run_c1(rk, p=20):
    """C1 recipe through the reference, both modes."""
    from recykl import preconditioners
    from recykl.linalg import SparseSpdMatrix
    from recykl.problems import LinearSystemSpec, SystemSequence
    from recykl.threestage import SolverConfig, run_sequence
    from recykl.truncation import TruncationConfig

    from paper_1512_05820_b200.problems import poisson2d_sequence

    mine = poisson2d_sequence(64, p=p)
    A0 = mine[0].A
    A = SparseSpdMatrix(A0.n, A0.row_offsets, A0.col_indices, A0.values)
    seq = SystemSequence(n=mine.n, systems=[LinearSystemSpec(A=A, b=s.b, xbar=None, tol=s.tol) for s in mine])
    pf = lambda M: preconditioners.build("jacobi", M)  # noqa: E731
    d = {"c": mine.C[0], "p": np.int64(p)}
    for tag, mode, extra in (("fom_", "fom", {}), ("cg_", "cg", {}), ("s5_", "fom", {"stage1_dim": 5})):
        tr = dict(strategy="pod-a-rbf", nu_y=1.0, nu_w=1.0, storage_cap=20, max_dim=20, **extra)
        cfg = SolverConfig(truncation=TruncationConfig(**tr), mode=mode)
        xs, reps, _ = run_sequence(seq, cfg, precond_factory=pf)
        r = _pack_run(xs, reps, tag)
        for j in range(1, len(xs) + 1):
            r[f"{tag}q{j}"] = np.float64(mine.C[0] @ xs[j - 1])
            if j > 3:
                del r[f"{tag}x{j}"]   # keep the fixture small: x for the first 3 systems, q for all
        d.update(r)
    return {"c1": d}


def run_elasticity(rk):
    """A 4x4x4-element C3-like elasticity sequence through the reference."""
    from recykl import preconditioners
    from recykl.linalg import SparseSpdMatrix
    from recykl.problems import LinearSystemSpec, SystemSequence
    from recykl.threestage import SolverConfig, run_sequence
    from recykl.truncation import TruncationConfig

    from paper_1512_05820_b200.problems import elasticity_sequence

    mine = elasticity_sequence((4, 4, 4), p=4, rtol=1e-8, seed=11)
    specs = list(mine)
    seq = SystemSequence(n=mine.n, systems=[
        LinearSystemSpec(A=SparseSpdMatrix(s.A.n, s.A.row_offsets, s.A.col_indices, s.A.values), b=s.b,
                         xbar=None, tol=s.tol) for s in specs])
    pf = lambda M: preconditioners.build("jacobi", M)  # noqa: E731
    d = {"n": np.int64(mine.n), "c": mine.C[0]}
    for j, s in enumerate(specs, start=1):
        d[f"val{j}"] = s.A.values
        d[f"b{j}"] = s.b
        d[f"tol{j}"] = np.float64(s.tol)
    d["rowptr"] = specs[0].A.row_offsets
    d["col"] = specs[0].A.col_indices
    for tag, mode in (("cg_", "cg"), ("fom_", "fom")):
        cfg = SolverConfig(truncation=TruncationConfig(strategy="pod-a-rbf", nu_y=1.0, nu_w=1.0, storage_cap=12,
                                                       max_dim=12), mode=mode)
        xs, reps, _ = run_sequence(seq, cfg, precond_factory=pf)
        d.update(_pack_run(xs, reps, tag))
    return {"elasticity": d}


def _ref_sequence(mine):
    from recykl.linalg import SparseSpdMatrix
    from recykl.problems import LinearSystemSpec, SystemSequence

    specs = list(mine)
    return specs, SystemSequence(n=mine.n, systems=[
        LinearSystemSpec(A=SparseSpdMatrix(s.A.n, s.A.row_offsets, s.A.col_indices, s.A.values), b=s.b,
                         xbar=None, tol=s.tol) for s in specs])


def run_c2_small(rk):
    """A 10^3 C2-like variable-coefficient diffusion sequence (drifting matrix)."""
    from recykl import preconditioners
    from recykl.threestage import SolverConfig, run_sequence
    from recykl.truncation import TruncationConfig

    from paper_1512_05820_b200.problems import diffusion3d_sequence

    mine = diffusion3d_sequence(10, p=4, rtol=1e-8, seed=4, corr_len=3.0)
    specs, seq = _ref_sequence(mine)
    d = {"n": np.int64(mine.n), "c": mine.C[0], "rowptr": specs[0].A.row_offsets, "col": specs[0].A.col_indices}
    for j, s in enumerate(specs, start=1):
        d[f"val{j}"], d[f"b{j}"], d[f"tol{j}"] = s.A.values, s.b, np.float64(s.tol)
    pf = lambda M: preconditioners.build("jacobi", M)  # noqa: E731
    for tag, mode in (("cg_", "cg"), ("fom_", "fom")):
        cfg = SolverConfig(truncation=TruncationConfig(strategy="pod-a-rbf", nu_y=1.0, nu_w=1.0, storage_cap=12,
                                                       max_dim=12), mode=mode)
        xs, reps, _ = run_sequence(seq, cfg, precond_factory=pf)
        d.update(_pack_run(xs, reps, tag))
        for j, x in enumerate(xs, start=1):
            d[f"{tag}q{j}"] = np.float64(mine.C[0] @ x)
    return {"c2_small": d}


def run_c3_mid(rk):
    """A 10^3-element C3-like Q1 elasticity prefix (N = 3630), CG and FOM."""
    from recykl import preconditioners
    from recykl.threestage import SolverConfig, run_sequence
    from recykl.truncation import TruncationConfig

    from paper_1512_05820_b200.problems import elasticity_sequence

    mine = elasticity_sequence((10, 10, 10), p=3, rtol=1e-6, seed=3)
    specs, seq = _ref_sequence(mine)
    d = {"n": np.int64(mine.n), "c": mine.C[0], "rowptr": specs[0].A.row_offsets, "col": specs[0].A.col_indices}
    for j, s in enumerate(specs, start=1):
        d[f"val{j}"], d[f"b{j}"], d[f"tol{j}"] = s.A.values, s.b, np.float64(s.tol)
    pf = lambda M: preconditioners.build("jacobi", M)  # noqa: E731
    for tag, mode in (("cg_", "cg"), ("fom_", "fom")):
        cfg = SolverConfig(truncation=TruncationConfig(strategy="pod-a-rbf", nu_y=1.0, nu_w=1.0, storage_cap=30,
                                                       max_dim=30), mode=mode)
        xs, reps, _ = run_sequence(seq, cfg, precond_factory=pf)
        d.update(_pack_run(xs, reps, tag))
        for j, x in enumerate(xs, start=1):
            d[f"{tag}q{j}"] = np.float64(mine.C[0] @ x)
    return {"c3_mid": d}


def run_c3_full(rk, p=2):
    """The bench's own C3 workload at full size (64^3 Q1 elasticity, N =
    811,200), its first p systems through the reference itself (CG, cap =
    max_dim = 60): counters, q = c'x, ||x|| and x at 2000 fixed indices (the
    full vectors would be 6.5 MB each; the test regenerates the inputs from
    the seeded generator)."""
    from recykl import preconditioners
    from recykl.threestage import SolverConfig, run_sequence
    from recykl.truncation import TruncationConfig

    from paper_1512_05820_b200.problems import elasticity_sequence

    mine = elasticity_sequence((64, 64, 64), p=p, rtol=1e-5, seed=3)
    specs, seq = _ref_sequence(mine)
    idx = np.sort(np.random.default_rng(0).choice(mine.n, 2000, replace=False))
    d = {"n": np.int64(mine.n), "p": np.int64(p), "idx": idx}
    cfg = SolverConfig(truncation=TruncationConfig(strategy="pod-a-rbf", nu_y=1.0, nu_w=1.0, storage_cap=60,
                                                   max_dim=60), mode="cg")
    xs, reps, _ = run_sequence(seq, cfg, precond_factory=lambda M: preconditioners.build("jacobi", M))
    for key in ("stage3_iters", "matvecs", "precond_applies", "final_residual", "truncated", "converged"):
        d[f"cg_{key}"] = np.asarray([getattr(r, key) for r in reps])
    for j, x in enumerate(xs, start=1):
        d[f"cg_q{j}"] = np.float64(mine.C[0] @ x)
        d[f"cg_xnorm{j}"] = np.float64(np.linalg.norm(x))
        d[f"cg_xs{j}"] = np.asarray(x, dtype=np.float64)[idx]
    # the reference's own rounding envelope at this size: every right-hand side
    # scaled by (1 + 1e-15), same everything else
    for s in seq.systems:
        s.b = s.b * (1 + 1e-15)
    xs2, reps2, _ = run_sequence(seq, cfg, precond_factory=lambda M: preconditioners.build("jacobi", M))
    d["pert_stage3_iters"] = np.asarray([r.stage3_iters for r in reps2])
    for j, (x, x2) in enumerate(zip(xs, xs2), start=1):
        d[f"pert_q{j}"] = np.float64(mine.C[0] @ x2)
        d[f"pert_xrel{j}"] = np.float64(np.linalg.norm(x2 - x) / np.linalg.norm(x))
    return {"c3_full": d}


def run_c5_small(rk):
    """C5 microbench at reduced size: Laplacian 16x16x32, Gaussian S with 256
    columns, gamma = 1: assemble_gram + pod_evd_from_gram (nu = 1)."""
    import warnings

    from recykl.linalg import SparseSpdMatrix, assemble_gram
    from recykl.pod import pod_evd_from_gram

    from paper_1512_05820_b200.problems import laplacian3d, snapshot_matrix

    L = laplacian3d(16, 16, 32)
    A = SparseSpdMatrix(L.n, L.row_offsets, L.col_indices, L.values)
    S = snapshot_matrix(L.n, 256, seed=5)
    G, _ = assemble_gram(A, S)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        res = pod_evd_from_gram(G, S, np.ones(256), 1.0)
    return {"c5_small": {"n": np.int64(L.n), "m": np.int64(256), "sigma": res.singular_values,
                         "y": np.int64(res.y), "basis20": res.columns[:, :20].copy(), "G_diag": np.diag(G).copy()}}


def run_kernels(rk):
    """Kernel-level goldens: spmv, assemble_gram, pod_evd_from_gram, augmented_pcg."""
    from recykl.krylov import augmented_pcg
    from recykl.linalg import SparseSpdMatrix, assemble_gram, spmv
    from recykl.pod import pod_evd_from_gram

    rng = np.random.default_rng(123)
    n = 300
    M = np.where(rng.random((n, n)) < 0.04, rng.standard_normal((n, n)), 0.0)
    M = 0.5 * (M + M.T)
    np.fill_diagonal(M, np.abs(M).sum(axis=1) + 1.0)
    A = SparseSpdMatrix.from_dense(M)
    x = rng.standard_normal(n)
    S = rng.standard_normal((n, 24))
    G, AS = assemble_gram(A, S)
    gamma = 0.5 + rng.random(24)
    pod = pod_evd_from_gram(G, S, gamma, 0.999)
    b = rng.standard_normal(n)
    Y = rng.standard_normal((n, 5))
    Ad = A.to_dense()
    yhat0 = np.linalg.solve(Y.T @ Ad @ Y, Y.T @ b)
    out = {"rowptr": A.row_offsets, "col": A.col_indices, "val": A.values, "x": x, "Ax": spmv(A, x), "S": S,
           "G": G, "AS": AS, "gamma": gamma, "pod_sigma": pod.singular_values, "pod_y": np.int64(pod.y),
           "pod_basis": pod.columns, "b": b, "Y": Y, "yhat0": yhat0}
    for mode in ("cg", "fom"):
        res = augmented_pcg(A, b, yhat0, Y, tol=1e-10, mode=mode, max_iter=400)
        out[f"{mode}_k"] = np.int64(res.k)
        out[f"{mode}_x"] = res.x
        out[f"{mode}_vhat"] = res.vhat
        out[f"{mode}_gamma"] = res.gamma
        out[f"{mode}_hist"] = res.residual_history
    from recykl.errors import NotConverged

    try:
        res = augmented_pcg(A, b, yhat0, Y, tol=1e-6, mode="fom", paper_fom_beta=True, max_iter=25)
        conv = True
    except NotConverged as exc:
        res, conv = exc.partial, False
    out["paper_k"], out["paper_x"], out["paper_conv"] = np.int64(res.k), res.x, np.bool_(conv)
    out["paper_hist"] = res.residual_history
    return {"kernels": out}


NEXT_CASES = {
    "ctcr_": (dict(strategy="pod-ctc-rbf", nu_y=1.0, nu_w=1.0, storage_cap=25, max_dim=10), "cg", "jacobi"),
    "ctcp_": (dict(strategy="pod-ctc-prev", nu_y=0.999, nu_w=0.9, storage_cap=25, max_dim=10), "fom", "jacobi"),
    "defl_": (dict(strategy="deflate", deflate_dim=8, storage_cap=25), "cg", "jacobi"),
    "defs_": (dict(strategy="deflate", deflate_dim=8, stage1_dim=4, storage_cap=25), "fom", "jacobi"),
    "ssor_": (dict(strategy="pod-a-rbf", nu_y=1.0, nu_w=1.0, storage_cap=20, max_dim=12), "cg", "ssor"),
    "ssor15_": (dict(strategy="pod-a-rbf", nu_y=1.0, nu_w=1.0, storage_cap=20, max_dim=12), "fom", "ssor:1.5"),
}


def run_next_strategies(rk):
    """SURVEY 8f f3/f4 through the reference: output-metric POD (pod-ctc-*, with
    the A-orthonormalisation), harmonic-Ritz deflation and SSOR preconditioning
    on a drifting diffusion sequence with a 2-row output matrix; plus kernel-level
    vectors for pod_svd, deflation_compress and one SSOR application."""
    from recykl import preconditioners
    from recykl.linalg import SparseSpdMatrix
    from recykl.pod import pod_svd
    from recykl.problems import gen_diffusion_sequence, gen_output_matrix
    from recykl.threestage import SolverConfig, run_sequence
    from recykl.truncation import TruncationConfig, deflation_compress

    seq = gen_diffusion_sequence((10, 10), p=6, delta=0.05, seed=41, tol=1e-9)
    seq.C = gen_output_matrix(2, seq.n, seed=3)
    d = _pack_sequence(seq, "")
    d["C"] = seq.C
    for tag, (tr, mode, pc) in NEXT_CASES.items():
        kind, omega = (pc.split(":") + ["1.0"])[:2] if pc.startswith("ssor") else (pc, "1.0")
        pf = lambda A, kind=kind, omega=float(omega): preconditioners.build(kind, A, omega)  # noqa: E731
        cfg = SolverConfig(truncation=TruncationConfig(**tr), mode=mode)
        xs, reps, _ = run_sequence(seq, cfg, precond_factory=pf)
        d.update(_pack_run(xs, reps, tag))
        for j, x in enumerate(xs, start=1):
            d[f"{tag}q{j}"] = seq.C @ x
    # kernel level
    rng = np.random.default_rng(11)
    A = seq[0].A
    S = rng.standard_normal((seq.n, 14))
    gam = rng.uniform(0.5, 2.0, 14)
    r = pod_svd(S, gam, seq.C, 1.0)
    d["k_S"], d["k_gamma"] = S, gam
    d["k_svd_sigma"], d["k_svd_y"], d["k_svd_cols"] = r.singular_values, np.int64(r.y), r.columns
    out = deflation_compress(S, A, 6, stage1_dim=None)
    d["k_defl_Y"], d["k_defl_mu"], d["k_defl_map"] = out.Y_new, out.spectrum, out.truncation_map
    M = preconditioners.build("ssor", A, 1.3)
    v = rng.standard_normal(seq.n)
    d["k_ssor_r"], d["k_ssor_z"] = v, M.apply(v)
    assert isinstance(A, SparseSpdMatrix)
    return {"next_strategies": d}


BAD_MM = {
    "bad_header.mtx": "%%MatrixMarket matrix coordinate complex symmetric\n2 2 1\n1 1 1.0\n",
    "not_square.mtx": "%%MatrixMarket matrix coordinate real symmetric\n2 3 1\n1 1 1.0\n",
    "too_many.mtx": "%%MatrixMarket matrix coordinate real symmetric\n2 2 1\n1 1 1.0\n2 2 1.0\n",
    "too_few.mtx": "%%MatrixMarket matrix coordinate real symmetric\n2 2 3\n1 1 1.0\n2 2 1.0\n",
    "out_of_range.mtx": "%%MatrixMarket matrix coordinate real symmetric\n2 2 2\n1 1 1.0\n3 2 1.0\n",
    "malformed_entry.mtx": "%%MatrixMarket matrix coordinate real symmetric\n2 2 2\n1 1 1.0\n2 x 1.0\n",
    "comments.mtx": "%%MatrixMarket matrix coordinate real symmetric\n% a comment\n\n2 2 3\n1 1 4.0\n"
                    "% inner\n2 1 -1.0\n2 2 4.0\n",
    "general_asym.mtx": "%%MatrixMarket matrix coordinate real general\n2 2 3\n1 1 4.0\n2 1 -1.0\n2 2 4.0\n",
    "array_bad.mtx": "%%MatrixMarket matrix array real general\n3 1\n1.0\n2.0\n",
    "array_ok.mtx": "%%MatrixMarket matrix array real general\n3 2\n1.0\n2.0\n3.0\n4.0\n5.0\n6.0\n",
}


def run_manifest(rk):
    """a sequence written by the reference (write_sequence: JSON
    manifest + Matrix Market files, kept under tests/golden/manifest_small/) with
    the arrays the reference reads back, plus the reference's verdict (exception
    type and message, paths relative) on malformed files (tests/golden/mm_cases/)."""
    from recykl import mmio
    from recykl.problems import gen_diffusion_sequence, gen_output_matrix, load_sequence_manifest, write_sequence

    seq = gen_diffusion_sequence((6, 5), p=3, delta=0.1, seed=5, tol=1e-9)
    seq.C = gen_output_matrix(2, seq.n, seed=7)
    seq.systems[1].xbar = np.linspace(0.0, 1.0, seq.n)
    mdir = os.path.join(OUT, "manifest_small")
    write_sequence(seq, mdir, name="golden")
    back = load_sequence_manifest(os.path.join(mdir, "manifest.json"))
    d = _pack_sequence(back, "")
    d["C"] = back.C
    d["xbar2"] = back.systems[1].xbar
    cdir = os.path.join(OUT, "mm_cases")
    os.makedirs(cdir, exist_ok=True)
    verdicts = {}
    for name, text in BAD_MM.items():
        path = os.path.join(cdir, name)
        with open(path, "w") as fh:
            fh.write(text)
        reader = mmio.read_array if name.startswith("array") else mmio.read_matrix
        try:
            out = reader(path)
            verdicts[name] = {"ok": True, "value": np.asarray(out.to_scipy().toarray() if hasattr(out, "to_scipy")
                                                               else out).tolist()}
        except Exception as exc:  # noqa: BLE001 - recording the reference's verdict
            verdicts[name] = {"ok": False, "type": type(exc).__name__,
                              "message": str(exc).replace(cdir + os.sep, "")}
    d["verdicts_json"] = np.array(json.dumps(verdicts))
    return {"manifest": d}


def main():
    rk = _ref()
    os.makedirs(OUT, exist_ok=True)
    blobs = {}
    only = sys.argv[1:]
    runs = [run_fixture_cases, run_stage_variants, run_kernels, run_elasticity, run_c1, run_c2_small, run_c3_mid,
            run_c5_small, run_next_strategies, run_manifest, run_c3_full]
    for fn in runs:
        if (not only and fn is not run_c3_full) or fn.__name__ in only:  # c3_full (minutes) only by name
            blobs.update(fn(rk))
    for name, d in blobs.items():
        path = os.path.join(OUT, f"{name}.npz")
        np.savez_compressed(path, **d)
        print(f"wrote {path} ({os.path.getsize(path) / 1024:.0f} KiB)")


if __name__ == "__main__":
    main()
