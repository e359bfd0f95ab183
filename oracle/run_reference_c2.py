"""Run the reference itself (recykl, from /root/reference in this container)
on the bench's full C2 sequence (128^3 variable-coefficient diffusion, 30
systems, CG, Jacobi, pod-a-rbf cap = max_dim = 40) and save per-system
counters, q = c'x, ||x||, x at 2000 fixed indices and wall times to
tests/golden/c2_seq.npz.
Test infrastructure only (the GPU tests read the .npz, never the reference).

python oracle/run_reference_c2.py [systems] [perturbation]   (CPU, ~2 min per system here)

With a perturbation e, every right-hand side is scaled by (1 + e) and the
result goes to tests/golden/c2_seq_pert.npz: the reference's own rounding
envelope on the same sequence.
"""
import os
import sys
import time
import warnings

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
warnings.simplefilter("ignore")


def main(p=30, pert=0.0):
    from recykl import preconditioners
    from recykl.linalg import InstrumentationSink, SparseSpdMatrix
    from recykl.threestage import RecycleState, SolverConfig, StageTolerances, solve_system
    from recykl.truncation import TruncationConfig

    from paper_1512_05820_b200.problems import diffusion3d_sequence

    mine = diffusion3d_sequence(128, p=p, rtol=1e-4, seed=2)
    idx = np.sort(np.random.default_rng(0).choice(mine.n, 2000, replace=False))
    cfg = SolverConfig(truncation=TruncationConfig(strategy="pod-a-rbf", nu_y=1.0, nu_w=1.0, storage_cap=40,
                                                   max_dim=40), mode="cg")
    out = {"n": np.int64(mine.n), "idx": idx, "iters": [], "matvecs": [], "q": [], "xnorm": [], "wall": []}
    xs_s = []
    state = None
    for j, s in enumerate(mine, start=1):
        A = SparseSpdMatrix(s.A.n, s.A.row_offsets, s.A.col_indices, s.A.values)
        b = s.b * (1 + pert) if pert else s.b
        if state is None:
            state = RecycleState.empty(mine.n)
        t0 = time.perf_counter()
        x, rep, state = solve_system(A, b, None, state, StageTolerances(eps=s.tol), cfg,
                                     M=preconditioners.build("jacobi", A), sink=InstrumentationSink())
        out["wall"].append(time.perf_counter() - t0)
        out["iters"].append(rep.stage3_iters)
        out["matvecs"].append(rep.matvecs)
        out["q"].append(float(mine.C[0] @ x))
        out["xnorm"].append(float(np.linalg.norm(x)))
        xs_s.append(np.asarray(x)[idx])
        d = {k: np.asarray(v) for k, v in out.items()}
        d["xs"] = np.stack(xs_s)
        d["p_done"] = np.int64(j)
        d["perturbation"] = np.float64(pert)
        name = "c2_seq_pert.npz" if pert else "c2_seq.npz"
        np.savez_compressed(os.path.join(os.path.dirname(HERE), "tests", "golden", name), **d)
        print(j, rep.stage3_iters, round(out["wall"][-1], 1), flush=True)


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 30, float(sys.argv[2]) if len(sys.argv) > 2 else 0.0)
