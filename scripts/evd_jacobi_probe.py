"""Probe: cuSOLVER syevd (what torch.linalg.eigh runs) vs syevj (Jacobi) on the
weighted POD Grams of a real C3 run (captured from pod._pod_device), with the
eigenvalue / eigenvector agreement the parity bar needs.

python scripts/evd_jacobi_probe.py      (GPU box) -> JSON lines
"""
import ctypes
import json
import os
import sys
import warnings

import numpy as np
import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
warnings.simplefilter("ignore")
import paper_1512_05820_b200 as pk  # noqa: E402
from paper_1512_05820_b200.problems import elasticity_sequence  # noqa: E402

cs = ctypes.CDLL("libcusolver.so.11")
vp, i32 = ctypes.c_void_p, ctypes.c_int


def capture(nsys=4):
    mats = []
    real = torch.linalg.eigh

    def spy(W):
        mats.append(W.detach().clone())
        return real(W)

    torch.linalg.eigh = spy
    try:
        seq = elasticity_sequence((64, 64, 64), p=nsys, rtol=1e-5, seed=3)
        cfg = pk.SolverConfig(truncation=pk.TruncationConfig(strategy="pod-a-rbf", nu_y=1.0, nu_w=1.0,
                                                             storage_cap=60, max_dim=60), mode="cg")
        pk.run_sequence(seq, cfg, precond_factory=lambda A: pk.build_preconditioner("jacobi", A))
    finally:
        torch.linalg.eigh = real
    return mats


def main():
    h = vp()
    assert cs.cusolverDnCreate(ctypes.byref(h)) == 0
    cs.cusolverDnSetStream(h, vp(torch.cuda.current_stream().cuda_stream))
    params = vp()
    assert cs.cusolverDnCreateSyevjInfo(ctypes.byref(params)) == 0
    cs.cusolverDnXsyevjSetTolerance(params, ctypes.c_double(0.0))   # machine precision
    cs.cusolverDnXsyevjSetMaxSweeps(params, i32(100))
    info = torch.zeros(1, dtype=torch.int32, device="cuda")
    for W in capture():
        m = W.shape[0]
        # syevd via torch
        for _ in range(2):
            w_ref, V_ref = torch.linalg.eigh(W)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            w_ref, V_ref = torch.linalg.eigh(W)
        e1.record()
        torch.cuda.synchronize()
        t_evd = e0.elapsed_time(e1) / 5
        # syevj
        A = W.clone()
        wj = torch.empty(m, dtype=torch.float64, device="cuda")
        lw = i32()
        assert cs.cusolverDnDsyevj_bufferSize(h, 1, 0, m, vp(A.data_ptr()), m, vp(wj.data_ptr()), ctypes.byref(lw),
                                              params) == 0
        work = torch.empty(max(lw.value, 1), dtype=torch.float64, device="cuda")
        times = []
        for rep in range(4):
            A.copy_(W)
            torch.cuda.synchronize()
            e0.record()
            st = cs.cusolverDnDsyevj(h, 1, 0, m, vp(A.data_ptr()), m, vp(wj.data_ptr()), vp(work.data_ptr()), lw,
                                     vp(info.data_ptr()), params)
            e1.record()
            torch.cuda.synchronize()
            assert st == 0 and int(info.item()) == 0, (st, int(info.item()))
            times.append(e0.elapsed_time(e1))
        sweeps = i32()
        cs.cusolverDnXsyevjGetSweeps(h, params, ctypes.byref(sweeps))
        wr, wjh = w_ref.cpu().numpy(), wj.cpu().numpy()
        lead = slice(m - 60, m)
        rel = np.max(np.abs(wjh[lead] - wr[lead]) / np.abs(wr[lead]))
        Vr = V_ref.cpu().numpy()[:, lead]
        Vj = A.cpu().numpy().T[:, lead] if False else A.cpu().numpy()[:, lead]
        # A holds eigenvectors column-major = rows of the row-major torch view -> transpose
        Vj = A.t().cpu().numpy()[:, lead]
        dots = np.abs(np.sum(Vr * Vj, axis=0))
        print(json.dumps({"m": m, "syevd_ms": round(t_evd, 3), "syevj_ms": round(min(times[1:]), 3),
                          "sweeps": sweeps.value, "lead60_eig_rel": float(rel),
                          "lead60_vec_min_abs_dot": float(dots.min()),
                          "offdiag_frac": float((W - torch.diag(torch.diag(W))).norm() / W.norm())}), flush=True)


if __name__ == "__main__":
    main()
