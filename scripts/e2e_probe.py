"""Where the e2e time goes: run_sequence over host CSR (as bench.py's e2e leg)
with only the host-side prefetch timers on (no device synchronisation added).
python scripts/e2e_probe.py [systems]"""
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1512_05820_b200 as pk  # noqa: E402
from paper_1512_05820_b200 import _timing  # noqa: E402
from paper_1512_05820_b200.problems import elasticity_sequence  # noqa: E402

p = int(sys.argv[1]) if len(sys.argv) > 1 else 40
if os.environ.get("SWITCH"):
    sys.setswitchinterval(float(os.environ["SWITCH"]))
seq = elasticity_sequence((64, 64, 64), p=p)
specs = list(seq)
cfg = pk.SolverConfig(truncation=pk.TruncationConfig(strategy="pod-a-rbf", nu_y=1.0, nu_w=1.0, storage_cap=60,
                                                     max_dim=60), mode="cg")
jac = lambda A: pk.build_preconditioner("jacobi", A)  # noqa: E731
hseq = pk.SystemSequence(seq.n, specs, C=seq.C)
pk.run_sequence(pk.SystemSequence(seq.n, specs[:3], C=seq.C), cfg, precond_factory=jac)  # warm caches
_timing.ENABLED = True
_timing.phase.__enter__ = lambda self: self
_timing.phase.__exit__ = lambda self, *a: False
_timing.reset()
torch.cuda.synchronize()
ms0 = torch.cuda.memory_stats()
t0 = time.perf_counter()
xs, reps, _ = pk.run_sequence(hseq, cfg, precond_factory=jac)
assert all(not hasattr(x, 'is_cuda') for x in xs)  # host inputs -> numpy solutions
torch.cuda.synchronize()
t = time.perf_counter() - t0
ms1 = torch.cuda.memory_stats()
alloc = {k: ms1[k] - ms0[k] for k in ("num_device_alloc", "num_device_free", "num_alloc_retries", "num_sync_all_streams")
         if k in ms1}
dspecs = [pk.LinearSystemSpec(A=pk.SparseSpdMatrix.from_host(s.A), b=torch.from_numpy(s.b).cuda(), xbar=None, tol=s.tol)
          for s in specs]
dseq = pk.SystemSequence(seq.n, dspecs, C=seq.C)
torch.cuda.synchronize()
t0 = time.perf_counter()
_, dreps, _ = pk.run_sequence(dseq, cfg, precond_factory=jac)
torch.cuda.synchronize()
td = time.perf_counter() - t0
print(json.dumps({"systems": p, "e2e_s": round(t, 3), "device_inputs_s": round(td, 3),
                  "device_solve_wall_sum_s": round(sum(r.wall_time for r in dreps), 3), "allocator": alloc,
                  "per_system_wall_ms_host_inputs": [round(1e3 * r.wall_time, 1) for r in reps[:8]],
                  "per_system_wall_ms_device_inputs": [round(1e3 * r.wall_time, 1) for r in dreps[:8]], "solve_wall_sum_s": round(sum(r.wall_time for r in reps), 3),
                  "iters": int(sum(r.stage3_iters for r in reps)),
                  "host_timers_s": {k: round(v, 3) for k, v in _timing.TIMES.items()}}))
