"""phi = 1 (full_orth: stage 3 against all of Y through nested reduced solves)
and stage 2 (stage1_dim < y) on a C3-shaped sequence: wall time per system
and the counters, for the paper's POD(5, nu)it style configurations (f2).

python scripts/phi1_probe.py [--grid 64] [--systems 6]     (GPU box) -> JSON lines
"""
import argparse
import json
import os
import sys
import time
import warnings

import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
warnings.simplefilter("ignore")
import paper_1512_05820_b200 as pk  # noqa: E402
from paper_1512_05820_b200.problems import elasticity_sequence  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--grid", type=int, default=64)
    ap.add_argument("--systems", type=int, default=6)
    args = ap.parse_args()
    seq = elasticity_sequence((args.grid,) * 3, p=args.systems, rtol=1e-5, seed=3)
    specs = list(seq)
    A = {}
    dev_specs = []
    for s in specs:
        dev_specs.append(pk.LinearSystemSpec(A=pk.SparseSpdMatrix.from_host(s.A), b=torch.from_numpy(s.b).cuda(),
                                             xbar=None, tol=s.tol))
    dseq = pk.SystemSequence(seq.n, dev_specs, C=seq.C)
    jac = lambda M: pk.build_preconditioner("jacobi", M)  # noqa: E731
    for name, tr in (("phi0_cap60", dict(nu_y=1.0, nu_w=1.0, storage_cap=60, max_dim=60)),
                     ("phi0_s5", dict(nu_y=1.0, nu_w=1.0, storage_cap=60, max_dim=60, stage1_dim=5)),
                     ("phi1_s5", dict(nu_y=1.0, nu_w=1.0, storage_cap=60, max_dim=60, stage1_dim=5, full_orth=True)),
                     ("phi1_cap60", dict(nu_y=1.0, nu_w=1.0, storage_cap=60, max_dim=60, full_orth=True))):
        cfg = pk.SolverConfig(truncation=pk.TruncationConfig(strategy="pod-a-rbf", **tr), mode="cg")
        pk.run_sequence(dseq, cfg, precond_factory=jac)  # warm-up
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        xs, reps, _ = pk.run_sequence(dseq, cfg, precond_factory=jac)
        torch.cuda.synchronize()
        t = time.perf_counter() - t0
        print(json.dumps({"config": name, "seconds": round(t, 3), "stage3_iters": [r.stage3_iters for r in reps],
                          "stage2_iters": [r.stage2_iters for r in reps], "matvecs": [r.matvecs for r in reps],
                          "wall_per_system": [round(r.wall_time, 3) for r in reps]}), flush=True)


if __name__ == "__main__":
    main()
