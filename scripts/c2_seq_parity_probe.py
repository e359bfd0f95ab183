"""The device C2 sequence against the reference's own run of it
(tests/golden/c2_seq.npz from oracle/run_reference_c2.py): per-system
stage-3 iterations, matvecs, q = c'x and x at 2000 fixed indices."""
import json
import os
import sys
import warnings

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
warnings.simplefilter("ignore")
import paper_1512_05820_b200 as pk  # noqa: E402
from paper_1512_05820_b200.problems import diffusion3d_sequence  # noqa: E402

if os.environ.get("RK_PROBE_FRESH_GRAM") == "1":  # truncation Gram by a fresh SpMM, as the reference
    from paper_1512_05820_b200 import threestage

    threestage._keep_products = lambda cfg: False
d = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests", "golden", "c2_seq.npz"))
p = int(d["p_done"])
seq = diffusion3d_sequence(128, p=p, rtol=1e-4, seed=2)
cfg = pk.SolverConfig(truncation=pk.TruncationConfig(strategy="pod-a-rbf", nu_y=1.0, nu_w=1.0, storage_cap=40,
                                                     max_dim=40), mode="cg")
xs, reps, _ = pk.run_sequence(seq, cfg, precond_factory=lambda A: pk.build_preconditioner("jacobi", A))
idx = d["idx"]
rows = []
for j, (x, r) in enumerate(zip(xs, reps)):
    xh = x.cpu().numpy()
    q = float(seq.C[0] @ xh)
    rows.append({"system": j + 1, "iters": r.stage3_iters, "ref_iters": int(d["iters"][j]),
                 "matvecs": r.matvecs, "ref_matvecs": int(d["matvecs"][j]),
                 "q_rel": abs(q - float(d["q"][j])) / abs(float(d["q"][j])),
                 "x_rel": float(np.linalg.norm(xh[idx] - d["xs"][j]) / np.linalg.norm(d["xs"][j]))})
    print(json.dumps(rows[-1]), flush=True)
di = np.array([r["iters"] - r["ref_iters"] for r in rows])
print(json.dumps({"systems": p, "total_iters": int(sum(r["iters"] for r in rows)),
                  "ref_total_iters": int(d["iters"][:p].sum()), "max_abs_iter_diff": int(np.abs(di).max()),
                  "max_q_rel": max(r["q_rel"] for r in rows), "max_x_rel": max(r["x_rel"] for r in rows),
                  "ref_wall_s": float(d["wall"][:p].sum())}))
