"""Probe: host LAPACK eigh vs on-device cuSOLVER eigh for the POD Gram sizes."""
import time

import numpy as np
import torch

rng = np.random.default_rng(0)
for m in (200, 500, 760, 1060):
    Z = rng.standard_normal((m, m))
    G = Z @ Z.T / m + np.diag(np.logspace(0, -14, m))
    t = time.perf_counter()
    for _ in range(3):
        w, V = np.linalg.eigh(G)
    th = (time.perf_counter() - t) / 3
    Gd = torch.from_numpy(G).cuda()
    torch.linalg.eigh(Gd)
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(3):
        wd, Vd = torch.linalg.eigh(Gd)
    torch.cuda.synchronize()
    tg = (time.perf_counter() - t) / 3
    err = np.max(np.abs(wd.cpu().numpy() - w)) / w[-1]
    print(f"m={m} host {th*1e3:.1f} ms  cusolver {tg*1e3:.1f} ms  max rel eig diff {err:.2e}")
