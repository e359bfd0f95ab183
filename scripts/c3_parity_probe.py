"""Deviation of the device C3 run from the reference at full size
(tests/golden/c3_full.npz): iterations, q = c'x and x (sampled) per system,
next to the reference's own envelope under a 1e-15 RHS perturbation."""
import json
import os
import sys
import warnings

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests"))
warnings.simplefilter("ignore")
import golden_io as gio  # noqa: E402
import paper_1512_05820_b200 as pk  # noqa: E402
from paper_1512_05820_b200.problems import elasticity_sequence  # noqa: E402

d = gio.load("c3_full")
p = int(d["p"])
seq = elasticity_sequence((64, 64, 64), p=p, rtol=1e-5, seed=3)
cfg = pk.SolverConfig(truncation=pk.TruncationConfig(strategy="pod-a-rbf", nu_y=1.0, nu_w=1.0, storage_cap=60,
                                                     max_dim=60), mode="cg")
xs, reps, _ = pk.run_sequence(seq, cfg, precond_factory=lambda A: pk.build_preconditioner("jacobi", A))
idx = d["idx"]
for j, (x, r) in enumerate(zip(xs, reps), start=1):
    xh = x.cpu().numpy()
    q = float(seq.C[0] @ xh)
    ref = d[f"cg_xs{j}"]
    print(json.dumps({"system": j, "iters": r.stage3_iters, "ref_iters": int(d["cg_stage3_iters"][j - 1]),
                      "ref_pert_iters": int(d["pert_stage3_iters"][j - 1]),
                      "q_rel": abs(q - float(d[f"cg_q{j}"])) / abs(float(d[f"cg_q{j}"])),
                      "ref_pert_q_rel": abs(float(d[f"pert_q{j}"]) - float(d[f"cg_q{j}"])) / abs(float(d[f"cg_q{j}"])),
                      "x_rel_sampled": float(np.linalg.norm(xh[idx] - ref) / np.linalg.norm(ref)),
                      "ref_pert_x_rel": float(d[f"pert_xrel{j}"])}))
