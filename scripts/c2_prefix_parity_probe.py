"""C2 at full size (128^3 variable-coefficient diffusion, N = 2,097,152,
scalar SELL-32 path): the first systems through the oracle (the pinned numpy
restatement of the reference, on the box's host cores) and through the
device path; per-system iterations, matvecs, q = c'x and x."""
import json
import os
import sys
import time
import warnings

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
warnings.simplefilter("ignore")
import paper_1512_05820_b200 as pk  # noqa: E402
from oracle import recycle_oracle as O  # noqa: E402
from paper_1512_05820_b200.problems import diffusion3d_sequence  # noqa: E402

p = int(sys.argv[1]) if len(sys.argv) > 1 else 3
tr = dict(strategy="pod-a-rbf", nu_y=1.0, nu_w=1.0, storage_cap=40, max_dim=40)
seq = diffusion3d_sequence(128, p=p, rtol=1e-4, seed=2)
specs = list(seq)
t0 = time.perf_counter()
oxs, oreps, _ = O.run_sequence(specs, O.Config(mode="cg", **tr), precond="jacobi")
t_cpu = time.perf_counter() - t0
cfg = pk.SolverConfig(truncation=pk.TruncationConfig(**tr), mode="cg")
xs, reps, _ = pk.run_sequence(pk.SystemSequence(seq.n, specs, C=seq.C), cfg,
                              precond_factory=lambda A: pk.build_preconditioner("jacobi", A))
for j, (x, r, ox, orp) in enumerate(zip(xs, reps, oxs, oreps), start=1):
    xh = x.cpu().numpy()
    q, oq = float(seq.C[0] @ xh), float(seq.C[0] @ ox)
    print(json.dumps({"system": j, "iters": r.stage3_iters, "oracle_iters": orp.stage3_iters, "matvecs": r.matvecs,
                      "oracle_matvecs": orp.matvecs, "q_rel": abs(q - oq) / abs(oq),
                      "x_rel": float(np.linalg.norm(xh - ox) / np.linalg.norm(ox))}), flush=True)
print(json.dumps({"oracle_cpu_s": round(t_cpu, 1), "cores": len(os.sched_getaffinity(0))}))
