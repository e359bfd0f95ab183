"""SSOR-preconditioned CG on a 64^3 7-point diffusion matrix (N = 262,144): the
device-stepped loop (rk_pcg_steps_ssor) against the stepwise loop that brings
every scalar to the host (forced by a monitor). python scripts/ssor_probe.py"""
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1512_05820_b200 as pk  # noqa: E402
from paper_1512_05820_b200.problems import diffusion3d_sequence  # noqa: E402

spec = next(iter(diffusion3d_sequence(64, p=1, rtol=1e-8, seed=2)))
A = pk.SparseSpdMatrix.from_host(spec.A)
b = torch.from_numpy(spec.b).cuda()
out = {}
for name, mon in (("device_stepped", None), ("stepwise_host_scalars", lambda k, x: None)):
    for rep in range(2):
        M = pk.build_preconditioner("ssor:1.5", A)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        res = pk.augmented_pcg(A, b, precond=M, tol=spec.tol, monitor=mon)
        torch.cuda.synchronize()
        t = time.perf_counter() - t0
    out[name] = {"iters": int(res.k), "s": round(t, 4), "us_per_iteration": round(1e6 * t / res.k, 1)}
print(json.dumps({"n": A.n, **out}))
