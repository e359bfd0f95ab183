"""Exploratory GPU measurements (not the bench): C3 prefix timing, per-kernel
event times, DMMA Gram vs cuBLAS DGEMM."""

import ctypes
import json
import os
import sys
import time
import warnings

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
warnings.simplefilter("ignore")

import paper_1512_05820_b200 as pk  # noqa: E402
from paper_1512_05820_b200 import _native as nat  # noqa: E402
from paper_1512_05820_b200.linalg import as_block, empty_block, gram, gemm_nn  # noqa: E402
from paper_1512_05820_b200.problems import elasticity_sequence  # noqa: E402

out = {"host_cores": len(os.sched_getaffinity(0))}
try:
    out["mem_gb"] = os.sysconf("SC_PAGE_SIZE") * os.sysconf("SC_PHYS_PAGES") / 1e9
except Exception:
    pass
dev = torch.device("cuda", 0)
import argparse
ap = argparse.ArgumentParser()
ap.add_argument("--systems", type=int, default=3)
ap.add_argument("--mode", default="cg")
ap.add_argument("--no-micro", action="store_true")
args = ap.parse_args()
P = args.systems
mode = args.mode
t = time.time()
seq = elasticity_sequence((64, 64, 64), p=P)
out["gen_s"] = time.time() - t
specs = list(seq)
t = time.time()
dspecs = [pk.LinearSystemSpec(A=pk.SparseSpdMatrix.from_host(s.A), b=torch.from_numpy(s.b).to(dev), xbar=None,
                              tol=s.tol) for s in specs]
torch.cuda.synchronize()
out["upload_s"] = time.time() - t
dseq = pk.SystemSequence(seq.n, dspecs)
cfg = pk.SolverConfig(truncation=pk.TruncationConfig(strategy="pod-a-rbf", nu_y=1.0, nu_w=1.0, storage_cap=60,
                                                     max_dim=60), mode=mode)
lib = nat.lib()
lib.rk_profile_begin()
t = time.time()
xs, reps, _ = pk.run_sequence(dseq, cfg, precond_factory=lambda A: pk.build_preconditioner("jacobi", A))
torch.cuda.synchronize()
out["seq_s"] = time.time() - t
ms = (ctypes.c_double * 4)()
cnt = (ctypes.c_int64 * 4)()
lib.rk_profile_end(ms, cnt)
out["reports"] = [dict(iters=r.stage3_iters, wall=r.wall_time, matvecs=r.matvecs, trunc=r.truncated,
                       res=r.final_residual) for r in reps]
A = dspecs[0].A
spmv_bytes = 12 * A.nnz + 4 * (A.n + 1) + 16 * A.n
avg = [ms[i] / max(cnt[i], 1) for i in range(4)]
out["kernel_avg_ms"] = avg
out["kernel_counts"] = list(cnt)
out["spmv_GBps"] = spmv_bytes / (avg[0] * 1e-3) / 1e9
out["update_GBps(m=60)"] = (64 * A.n + 60 * 8 * A.n) / (avg[1] * 1e-3) / 1e9
out["direction_GBps(m=60)"] = (3 * 8 * A.n + 60 * 8 * A.n) / (avg[3] * 1e-3) / 1e9

if args.no_micro:
    print(json.dumps(out, indent=1))
    sys.exit(0)


# DMMA Gram vs cuBLAS DGEMM
def timeit(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps

for n, m in ((811200, 1060), (4194304, 256), (811200, 60)):
    X = empty_block(n, m, dev)
    X.normal_()
    Y = empty_block(n, m, dev)
    Y.normal_()
    t_ms = timeit(lambda: gram(X, Y))
    out[f"gram_{n}x{m}_ms"] = t_ms
    out[f"gram_{n}x{m}_TFs"] = 2 * n * m * m / (t_ms * 1e-3) / 1e12
    C = torch.randn(m, 60, dtype=torch.float64, device=dev)
    t2 = timeit(lambda: gemm_nn(X, C))
    out[f"gemmnn_{n}x{m}x60_TFs"] = 2 * n * m * 60 / (t2 * 1e-3) / 1e12
    del X, Y
a = torch.randn(8192, 8192, dtype=torch.float64, device=dev)
b = torch.randn(8192, 8192, dtype=torch.float64, device=dev)
tm = timeit(lambda: a @ b, 3)
out["cublas_dgemm_8192_TFs"] = 2 * 8192 ** 3 / (tm * 1e-3) / 1e12
Xt = torch.randn(811200, 1060, dtype=torch.float64, device=dev)
tm = timeit(lambda: Xt.t() @ Xt, 3)
out["cublas_gram_811200x1060_TFs"] = 2 * 811200 * 1060 ** 2 / (tm * 1e-3) / 1e12
print(json.dumps(out, indent=1))
os.makedirs("gpurun_out", exist_ok=True)
with open("gpurun_out/explore_c3.json", "w") as fh:
    json.dump(out, fh, indent=1)
