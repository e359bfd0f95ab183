"""Run the reference itself (recykl, imported from /root/reference in this
container) on one of the bench's full-size sequences and save per-system
counters, q = c'x, ||x||, x at 2000 fixed indices and wall times to
tests/golden/<out>.npz (rewritten after every system, so a prefix is usable
while the run continues). Test infrastructure only: the GPU tests read the
.npz, never the reference.

    python oracle/run_reference_seq.py --workload c3 --mode fom --systems 2 --out c3_fom
    python oracle/run_reference_seq.py --workload c3 --pert 1e-15 --out c3_seq_pert_p
    python oracle/run_reference_seq.py --workload c4 --systems 3 --out c4_prefix

Workloads (the same generators and solver configurations as bench.py):
  c3  64^3 Q1 elasticity, 40 systems, rtol 1e-5, pod-a-rbf cap = max_dim = 60
  c4  128x128x64 Q1 elasticity K + M/dt^2 (dt 0.05), rtol 1e-6, pod-a-rbf
      cap 3000, max_dim 60

With --pert e every right-hand side (and so the absolute tolerance, which the
generator derives from ||b||) is scaled by (1 + e): the reference's own
rounding envelope on the same sequence. The per-system call pattern is
recykl.threestage.run_sequence's (threestage.py:550-596): a fresh
InstrumentationSink and Jacobi preconditioner per system, solve_system with
the carried RecycleState.
"""
import argparse
import os
import sys
import time
import warnings

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
warnings.simplefilter("ignore")

WORKLOADS = {
    "c3": dict(ne=(64, 64, 64), p=40, rtol=1e-5, seed=3, dynamic=False, cap=60, max_dim=60),
    "c4": dict(ne=(128, 128, 64), p=60, rtol=1e-6, seed=4, dynamic=True, cap=3000, max_dim=60),
}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="c3", choices=sorted(WORKLOADS))
    ap.add_argument("--mode", default="cg", choices=["cg", "fom"])
    ap.add_argument("--systems", type=int, default=None)
    ap.add_argument("--pert", type=float, default=0.0)
    ap.add_argument("--out", required=True)
    args = ap.parse_args()

    from recykl import preconditioners
    from recykl.linalg import InstrumentationSink, SparseSpdMatrix
    from recykl.threestage import RecycleState, SolverConfig, StageTolerances, solve_system
    from recykl.truncation import TruncationConfig

    from paper_1512_05820_b200.problems import elasticity_sequence

    w = WORKLOADS[args.workload]
    p = args.systems or w["p"]
    seq = elasticity_sequence(w["ne"], p=p, rtol=w["rtol"], seed=w["seed"], dynamic=w["dynamic"])
    idx = np.sort(np.random.default_rng(0).choice(seq.n, 2000, replace=False))
    cfg = SolverConfig(truncation=TruncationConfig(strategy="pod-a-rbf", nu_y=1.0, nu_w=1.0,
                                                   storage_cap=w["cap"], max_dim=w["max_dim"]), mode=args.mode)
    out = {"n": np.int64(seq.n), "idx": idx, "iters": [], "matvecs": [], "precond": [], "grams": [],
           "q": [], "xnorm": [], "wall": [], "basis_dim": [], "truncated": []}
    xs_s = []
    state = RecycleState.empty(seq.n)
    A, host_vals = None, None
    path = os.path.join(os.path.dirname(HERE), "tests", "golden", args.out + ".npz")
    for j, s in enumerate(seq, start=1):
        if s.A.values is not host_vals:  # C4: one invariant matrix object for the whole sequence
            host_vals = s.A.values
            A = SparseSpdMatrix(s.A.n, s.A.row_offsets, s.A.col_indices, s.A.values)
        b = s.b * (1 + args.pert) if args.pert else s.b
        tol = s.tol * (1 + args.pert) if args.pert else s.tol
        sink = InstrumentationSink()
        t0 = time.perf_counter()
        x, rep, state = solve_system(A, b, None, state, StageTolerances(eps=tol), cfg,
                                     M=preconditioners.build("jacobi", A), sink=sink)
        out["wall"].append(time.perf_counter() - t0)
        out["iters"].append(rep.stage3_iters)
        out["matvecs"].append(rep.matvecs)
        out["precond"].append(rep.precond_applies)
        out["grams"].append(sink.gram_assemblies)
        out["basis_dim"].append(rep.basis_dim)
        out["truncated"].append(bool(rep.truncated))
        out["q"].append(float(seq.C[0] @ x))
        out["xnorm"].append(float(np.linalg.norm(x)))
        xs_s.append(np.asarray(x)[idx])
        d = {k: np.asarray(v) for k, v in out.items()}
        d["xs"] = np.stack(xs_s)
        d["p_done"] = np.int64(j)
        d["perturbation"] = np.float64(args.pert)
        d["mode"] = np.array(args.mode)
        d["workload"] = np.array(args.workload)
        np.savez_compressed(path + ".tmp.npz", **d)
        os.replace(path + ".tmp.npz", path)
        print(j, rep.stage3_iters, rep.matvecs, round(out["wall"][-1], 1), flush=True)


if __name__ == "__main__":
    main()
