"""SURVEY 8f f1, host side: Matrix Market + JSON manifest I/O against files and
verdicts produced by the reference itself (oracle/make_golden.py run_manifest):
same arrays back, byte-identical files written, same errors (type, file:line
message) on malformed input. CPU only."""

import filecmp
import json
import os

import numpy as np
import pytest

import golden_io as gio
from paper_1512_05820_b200 import mmio
from paper_1512_05820_b200.errors import ManifestError, NotSymmetric
from paper_1512_05820_b200.problems import load_sequence_manifest, write_sequence

MDIR = os.path.join(gio.GOLDEN, "manifest_small")
CDIR = os.path.join(gio.GOLDEN, "mm_cases")


@pytest.mark.parametrize("lazy", [False, True])
def test_load_reference_written_manifest(lazy):
    d = gio.load("manifest")
    seq = load_sequence_manifest(os.path.join(MDIR, "manifest.json"), lazy=lazy)
    assert seq.n == int(d["n"]) and seq.p == int(d["p"])
    assert np.array_equal(seq.C, d["C"])
    for j, spec in enumerate(seq, start=1):
        assert np.array_equal(spec.A.row_offsets, d[f"A{j}_rowptr"])
        assert np.array_equal(spec.A.col_indices, d[f"A{j}_col"])
        assert np.array_equal(spec.A.values, d[f"A{j}_val"])  # bit exact (repr round trip)
        assert np.array_equal(spec.b, d[f"b{j}"])
        assert spec.tol == float(d[f"tol{j}"])
        if j == 2:
            assert np.array_equal(spec.xbar, d["xbar2"])
        else:
            assert spec.xbar is None
    assert seq.metadata["name"].startswith("diffusion")


def test_written_files_are_byte_identical_to_the_reference(tmp_path):
    seq = load_sequence_manifest(os.path.join(MDIR, "manifest.json"))
    path = write_sequence(seq, tmp_path, name="golden")
    for name in sorted(os.listdir(MDIR)):
        assert filecmp.cmp(os.path.join(MDIR, name), os.path.join(tmp_path, name), shallow=False), name
    assert json.load(open(path)) == json.load(open(os.path.join(MDIR, "manifest.json")))


@pytest.mark.parametrize("name", sorted(os.listdir(CDIR)))
def test_malformed_files_same_verdict_as_reference(name):
    want = json.loads(str(gio.load("manifest")["verdicts_json"]))[name]
    path = os.path.join(CDIR, name)
    reader = mmio.read_array if name.startswith("array") else mmio.read_matrix
    if want["ok"]:
        out = reader(path)
        got = out.to_scipy().toarray() if hasattr(out, "to_scipy") else out
        assert np.array_equal(np.asarray(got), np.asarray(want["value"]))
        return
    exc_type = {"ManifestError": ManifestError, "NotSymmetric": NotSymmetric}[want["type"]]
    with pytest.raises(exc_type) as exc:
        reader(path)
    assert str(exc.value).replace(CDIR + os.sep, "") == want["message"]


def test_manifest_errors(tmp_path):
    bad = tmp_path / "m.json"
    bad.write_text("{not json")
    with pytest.raises(ManifestError, match=r"m.json:1: invalid JSON"):
        load_sequence_manifest(bad)
    bad.write_text(json.dumps({"systems": []}))
    with pytest.raises(ManifestError, match="must carry 'n' and 'systems'"):
        load_sequence_manifest(bad)
    bad.write_text(json.dumps({"n": 3, "systems": [{"rhs": "b.mtx"}]}))
    with pytest.raises(ManifestError, match="system 1 entry malformed"):
        load_sequence_manifest(bad)
    # dimension mismatch between the manifest and its files
    m = json.load(open(os.path.join(MDIR, "manifest.json")))
    m["n"] = 7
    for f in os.listdir(MDIR):
        if f.endswith(".mtx"):
            (tmp_path / f).write_bytes(open(os.path.join(MDIR, f), "rb").read())
    (tmp_path / "manifest.json").write_text(json.dumps(m))
    with pytest.raises(ManifestError, match="system 1 dimension mismatch"):
        load_sequence_manifest(tmp_path / "manifest.json")


def test_round_trip_large_values_bit_exact(tmp_path):
    from paper_1512_05820_b200.problems import elasticity_sequence

    H = next(iter(elasticity_sequence((3, 3, 2), p=1))).A
    mmio.write_symmetric_matrix(tmp_path / "A.mtx", H)
    back = mmio.read_matrix(tmp_path / "A.mtx")
    assert np.array_equal(back.row_offsets, H.row_offsets)
    assert np.array_equal(back.col_indices, H.col_indices)
    assert np.array_equal(back.values, H.values)
    v = np.random.default_rng(0).standard_normal((5, 3)) * 1e-300
    mmio.write_array(tmp_path / "v.mtx", v)
    assert np.array_equal(mmio.read_array(tmp_path / "v.mtx"), v)
