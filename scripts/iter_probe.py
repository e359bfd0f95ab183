"""Per-iteration wall time of the fused stage-3 loop (C3, 60-column basis) vs the
sum of its kernels: python scripts/iter_probe.py [iters] [batch]."""
import ctypes
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1512_05820_b200 as pk  # noqa: E402
from paper_1512_05820_b200 import _native as nat  # noqa: E402
from paper_1512_05820_b200.linalg import scale_columns  # noqa: E402
from paper_1512_05820_b200.problems import elasticity_sequence  # noqa: E402

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 400
batch = int(sys.argv[2]) if len(sys.argv) > 2 else None
spec = next(iter(elasticity_sequence((64, 64, 64), p=1)))
A = pk.SparseSpdMatrix.from_host(spec.A)
M = pk.build_preconditioner("jacobi", A)
b = torch.from_numpy(spec.b).cuda()
try:
    res = pk.augmented_pcg(A, b, precond=M, tol=0.0, max_iter=60)
except pk.NotConverged as exc:
    res = exc.partial
Y = scale_columns(res.V, np.sqrt(res.gamma))
st1 = pk.direct_reduced_solve(A, b, Y)
f = pk.BlockDiagFactor()
f.append_cholesky(st1.rhat)
proj = pk.DirectReducedProjection(st1.aw, f)
out = {}
for label, prof in (("wall", False), ("kernels", True)):
    torch.cuda.synchronize()
    if prof:
        nat.lib().rk_profile_begin()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    try:
        pk.augmented_pcg(A, b, st1.what, Y, proj, M, 0.0, max_iter=iters, batch=batch, keep_products=True)
    except pk.NotConverged:
        pass
    e1.record()
    torch.cuda.synchronize()
    out[label + "_ms_per_iter"] = round(e0.elapsed_time(e1) / iters, 4)
    if prof:
        ms = (ctypes.c_double * 4)()
        cnt = (ctypes.c_int64 * 4)()
        nat.lib().rk_profile_end(ms, cnt)
        out["kernel_avg_ms"] = [round(ms[i] / max(cnt[i], 1), 4) for i in range(4)]
        out["kernel_sum_ms"] = round(sum(out["kernel_avg_ms"]), 4)
print(json.dumps(out))
