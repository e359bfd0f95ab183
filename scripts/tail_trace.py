"""Timeline of the direction kernel's combine prologue (needs a -DRK_TAIL_TRACE build, e.g.
make -C paper_1512_05820_b200/csrc OUT=$PWD/gpurun_trace FLAGS="... -DRK_TAIL_TRACE";
then RK_LIB=gpurun_trace/libpodcg.so python scripts/tail_trace.py)."""
import ctypes
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1512_05820_b200 as pk  # noqa: E402
from paper_1512_05820_b200 import _native as nat  # noqa: E402
from paper_1512_05820_b200.linalg import scale_columns  # noqa: E402
from paper_1512_05820_b200.problems import elasticity_sequence  # noqa: E402

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
try:
    pk.augmented_pcg(A, b, st1.what, Y, proj, M, 0.0, max_iter=70)
except pk.NotConverged:
    pass
torch.cuda.synchronize()
buf = (ctypes.c_uint64 * 512)()
nat.lib().rk_debug_trace(buf, 512)
t = np.array(list(buf), dtype=np.float64).reshape(64, 8)
t = t[t[:, 3] > 0]
# stamps of block 0 of k_pcg_direction (globaltimer, ns): 0 after griddepcontrol.wait,
# 1 after the group sums, 2 after the mu solve, 3 at the end of the row loop
d = np.diff(t[:, :4], axis=1) / 1e3
names = ["group_sums", "mu_solve", "row_loop"]
print(json.dumps({"rows": int(len(t)), "block0_step_us(median)": dict(zip(names, np.round(np.median(d, axis=0), 3).tolist())),
                  "block0_total_us": round(float(np.median((t[:, 3] - t[:, 0]) / 1e3)), 3)}))
