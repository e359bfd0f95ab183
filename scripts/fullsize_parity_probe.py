"""Per-system comparison of the device path with a reference run of a full-size
sequence (tests/golden/<name>.npz from oracle/run_reference_seq.py):
python scripts/fullsize_parity_probe.py c3_fom|c3_seq|c4_prefix  -> JSON lines"""
import json
import os
import sys
import warnings

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "oracle"))
warnings.simplefilter("ignore")
import paper_1512_05820_b200 as pk  # noqa: E402
from paper_1512_05820_b200.problems import elasticity_sequence  # noqa: E402
from run_reference_seq import WORKLOADS  # noqa: E402

name = sys.argv[1]
d = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests", "golden", f"{name}.npz"))
w = WORKLOADS[str(d["workload"])]
mode = str(d["mode"])
p = int(d["p_done"])
seq = elasticity_sequence(w["ne"], p=p, rtol=w["rtol"], seed=w["seed"], dynamic=w["dynamic"])
cfg = pk.SolverConfig(truncation=pk.TruncationConfig(strategy="pod-a-rbf", nu_y=1.0, nu_w=1.0,
                                                     storage_cap=w["cap"], max_dim=w["max_dim"]), mode=mode)
xs, reps, _ = pk.run_sequence(seq, cfg, precond_factory=lambda A: pk.build_preconditioner("jacobi", A))
idx = d["idx"]
for j, (x, r) in enumerate(zip(xs, reps)):
    q = float(seq.C[0] @ x)
    print(json.dumps({"case": name, "system": j + 1, "iters": r.stage3_iters, "ref_iters": int(d["iters"][j]),
                      "matvecs": r.matvecs, "ref_matvecs": int(d["matvecs"][j]),
                      "q_rel": abs(q - float(d["q"][j])) / abs(float(d["q"][j])),
                      "x_rel": float(np.linalg.norm(x[idx] - d["xs"][j]) / np.linalg.norm(d["xs"][j])),
                      "wall_s": round(r.wall_time, 3), "ref_wall_s": round(float(d["wall"][j]), 1)}), flush=True)
