"""The drop-in boundary exercised by the reference's OWN front-end.

recykl (the unmodified reference, installed into baseline/_ref by
``pip install --target baseline/_ref``) keeps its fixture
checker, benchmark runners and report writers; only ``run_sequence`` --
imported by name into ``recykl.fixtures`` and ``recykl.bench``
(fixtures.py:20, bench.py:26-34) -- is swapped for the B200 one, exactly the
two-line patch INTEGRATION.md shows. Everything the reference does with the
results (counter diffs, ``seq.C @ (xstar - cp.x)`` on checkpoints, CSV
rows) must keep working and give the reference's numbers:

* ``fixtures.verify_fixture`` on the three frozen fixtures
  (pkg/tests/fixtures/*.json, copied to tests/golden/recykl_fixtures/): no
  mismatch;
* ``fixtures.write_calibration_record`` (SSOR omega = 1.7 on the 50x50
  acceptance sequence, fixtures.py:72-109): the per-system stage-3 counts of
  pcg / no-trunc / POD(40,0) equal acceptance_calibration.json's frozen ones
  (sums 323 / 56 / 65);
* ``bench.run_methods(threads=2)`` over the default roster and
  ``bench.write_run_outputs``: identical CSV counter columns to the
  reference's own run;
* ``bench.output_error_run``: identical per-tau matvec / precond averages.
"""

import csv
import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")
FIXTURES = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "recykl_fixtures")

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def recykl():
    if not os.path.isdir(os.path.join(REF, "recykl")):
        pytest.skip("reference not installed in baseline/_ref (see DESIGN.md, reference arm)")
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import recykl
    import recykl.bench
    import recykl.fixtures

    return recykl


@pytest.fixture
def swapped(recykl, monkeypatch):
    """recykl with the B200 run_sequence patched in where its front-end looks it up."""
    import paper_1512_05820_b200 as pk

    monkeypatch.setattr(recykl.fixtures, "run_sequence", pk.run_sequence)
    monkeypatch.setattr(recykl.bench, "run_sequence", pk.run_sequence)
    return recykl


@pytest.mark.parametrize("name", ["identity_like", "invariant_matrix", "drifting_pod"])
def test_verify_fixture_through_reference_frontend(swapped, name):
    assert swapped.fixtures.verify_fixture(os.path.join(FIXTURES, f"{name}.json")) == {}


def test_acceptance_calibration_ssor_replay(swapped, tmp_path):
    """SSOR omega = 1.7 through the reference's own precond factory
    (``lambda A: preconditioners.build("ssor", A, omega=1.7)``), adopted as
    the device SSOR by run_sequence."""
    path = swapped.fixtures.write_calibration_record(str(tmp_path))
    got = json.load(open(path))["measured"]
    want = json.load(open(os.path.join(FIXTURES, "acceptance_calibration.json")))["measured"]
    for key in ("pcg_stage3", "notrunc_stage3", "pod_stage3"):
        assert got[key] == want[key], (key, got[key], want[key])
    assert (sum(got["pcg_stage3"]), sum(got["notrunc_stage3"]), sum(got["pod_stage3"])) == (323, 56, 65)
    assert got["pod_vs_notrunc_ratio"] == pytest.approx(want["pod_vs_notrunc_ratio"], rel=1e-12)


def _roster(recykl, precond):
    return recykl.bench.default_methods(storage_cap=16, precond=precond, mode="fom")


def _small_sequence(recykl):
    from recykl.problems import gen_diffusion_sequence

    return gen_diffusion_sequence((12, 12), 6, 0.05, seed=7, tol=1e-8)


def _csv_rows(path):
    with open(path) as fh:
        return list(csv.DictReader(fh))


@pytest.mark.parametrize("precond", ["identity", "jacobi"])
def test_run_methods_csv_counters_match_reference(recykl, monkeypatch, tmp_path, precond):
    import paper_1512_05820_b200 as pk

    seq = _small_sequence(recykl)
    ref_runs = recykl.bench.run_methods(seq, _roster(recykl, precond), threads=2, keep_solutions=True)
    ref_out = recykl.bench.write_run_outputs(ref_runs, str(tmp_path / "ref"))
    monkeypatch.setattr(recykl.bench, "run_sequence", pk.run_sequence)
    runs = recykl.bench.run_methods(seq, _roster(recykl, precond), threads=2, keep_solutions=True)
    out = recykl.bench.write_run_outputs(runs, str(tmp_path / "b200"))
    got, want = _csv_rows(out["systems"]), _csv_rows(ref_out["systems"])
    assert len(got) == len(want)
    counters = ("method", "j", "matvecs", "precond_apps", "stage1_dim", "stage2_iters", "stage3_iters")
    for g, w in zip(got, want):
        assert {k: g[k] for k in counters} == {k: w[k] for k in counters}, (g, w)
        assert float(g["final_residual"]) == pytest.approx(float(w["final_residual"]), rel=1e-6, abs=1e-14)
    for run, ref in zip(runs, ref_runs):
        for x, xr in zip(run.solutions, ref.solutions):
            assert isinstance(x, np.ndarray)
            assert np.linalg.norm(x - xr) <= 1e-8 * np.linalg.norm(xr), run.method.name


def test_output_error_run_matches_reference(recykl, monkeypatch):
    """output_error_run evaluates ``seq.C @ (xstar - cp.x)`` on every checkpoint
    (bench.py:286): the checkpoints must be host arrays on the reference's
    path, and the per-tau costs the reference's."""
    import paper_1512_05820_b200 as pk

    seq = _small_sequence(recykl)
    seq.C = np.random.default_rng(3).standard_normal((2, seq.n))
    taus = (1e-2, 1e-4, 1e-6)
    methods = _roster(recykl, "jacobi")
    want = recykl.bench.output_error_run(seq, methods, taus, threads=1)
    monkeypatch.setattr(recykl.bench, "run_sequence", pk.run_sequence)
    got = recykl.bench.output_error_run(seq, methods, taus, threads=2)
    assert len(got) == len(want)
    for g, w in zip(got, want):
        for k in ("method", "tau", "avg_matvecs", "avg_precond_apps", "systems_met", "systems"):
            assert g[k] == w[k], (k, g, w)
