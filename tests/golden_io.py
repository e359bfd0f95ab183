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
