"""Loaders for the committed golden fixtures (tests/golden/*.npz)."""

import json
import os

import numpy as np

from paper_1512_05820_b200.problems import HostCsr, LinearSystemSpec, SystemSequence

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name):
    return dict(np.load(os.path.join(GOLDEN, f"{name}.npz"), allow_pickle=False))


def sequence(d, prefix=""):
    n = int(d[f"{prefix}n"])
    p = int(d[f"{prefix}p"])
    specs = []
    for j in range(1, p + 1):
        A = HostCsr(n, d[f"{prefix}A{j}_rowptr"], d[f"{prefix}A{j}_col"], d[f"{prefix}A{j}_val"])
        specs.append(LinearSystemSpec(A=A, b=d[f"{prefix}b{j}"], xbar=None, tol=float(d[f"{prefix}tol{j}"])))
    return SystemSequence(n, specs)


def elasticity_sequence(d):
    n = int(d["n"])
    specs = []
    j = 1
    while f"val{j}" in d:
        A = HostCsr(n, d["rowptr"], d["col"], d[f"val{j}"])
        specs.append(LinearSystemSpec(A=A, b=d[f"b{j}"], xbar=None, tol=float(d[f"tol{j}"])))
        j += 1
    return SystemSequence(n, specs, C=d["c"][None, :])


def frozen(d):
    return json.loads(str(d["frozen_json"]))


def counters(d, prefix):
    keys = ("stage3_iters", "stage2_iters", "stage1_dim", "matvecs", "precond_applies", "final_residual",
            "truncated", "converged")
    return {k: d[f"{prefix}{k}"] for k in keys}


pattern_sequence = elasticity_sequence  # same layout: rowptr, col, val{j}, b{j}, tol{j}, c


# SURVEY 8f f3/f4 cases (oracle/make_golden.py NEXT_CASES): truncation config,
# mode, preconditioner
NEXT_CASES = {
    "ctcr_": (dict(strategy="pod-ctc-rbf", nu_y=1.0, nu_w=1.0, storage_cap=25, max_dim=10), "cg", "jacobi"),
    "ctcp_": (dict(strategy="pod-ctc-prev", nu_y=0.999, nu_w=0.9, storage_cap=25, max_dim=10), "fom", "jacobi"),
    "defl_": (dict(strategy="deflate", deflate_dim=8, storage_cap=25), "cg", "jacobi"),
    "defs_": (dict(strategy="deflate", deflate_dim=8, stage1_dim=4, storage_cap=25), "fom", "jacobi"),
    "ssor_": (dict(strategy="pod-a-rbf", nu_y=1.0, nu_w=1.0, storage_cap=20, max_dim=12), "cg", "ssor"),
    "ssor15_": (dict(strategy="pod-a-rbf", nu_y=1.0, nu_w=1.0, storage_cap=20, max_dim=12), "fom", "ssor:1.5"),
}


def next_sequence(d):
    seq = sequence(d)
    seq.C = d["C"]
    return seq
