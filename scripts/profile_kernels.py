"""Short, deterministic C3 kernel workload for ncu (a few hundred launches):
plain PCG iterations, stage-1 assemble_gram + augmented PCG against a
60-column A-orthogonal basis (the stage-3 shape of every system j >= 2), and
one truncation (SpMM + DMMA Gram at the grown width, DMMA reconstruction)."""

import argparse
import os
import sys
import warnings

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
warnings.simplefilter("ignore")

import paper_1512_05820_b200 as pk  # noqa: E402
from paper_1512_05820_b200.linalg import (  # noqa: E402
    empty_block, gemm_nn, gram, scale_columns, spmm, symmetric_gram_from_products)
from paper_1512_05820_b200.problems import elasticity_sequence  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--grid", type=int, default=64)
ap.add_argument("--iters", type=int, default=40)
ap.add_argument("--grown", type=int, default=760)
ap.add_argument("--mode", default="cg")
args = ap.parse_args()

dev = torch.device("cuda", 0)
spec = next(iter(elasticity_sequence((args.grid,) * 3, p=1)))
A = pk.SparseSpdMatrix.from_host(spec.A)
M = pk.build_preconditioner("jacobi", A)
b = torch.from_numpy(spec.b).to(dev)

# plain PCG (system 1 shape); 60 directions become the recycled basis
try:
    res = pk.augmented_pcg(A, b, precond=M, tol=0.0, max_iter=60, mode=args.mode)
except pk.NotConverged as exc:
    res = exc.partial
Y = scale_columns(res.V, np.sqrt(res.gamma))

# stage 1 + stage 3 against the 60-column basis (system j >= 2 shape)
st1 = pk.direct_reduced_solve(A, b, Y)
f = pk.BlockDiagFactor()
f.append_cholesky(st1.rhat)
proj = pk.DirectReducedProjection(st1.aw, f)
try:
    pk.augmented_pcg(A, b, st1.what, Y, proj, M, 0.0, mode=args.mode, max_iter=args.iters)
except pk.NotConverged:
    pass

# truncation at the grown width: the sequence's Z'AZ from the cached products
# A Y (stage 1) and A V (stage 3) -- one upper-triangle launch over both segments
Z = empty_block(A.n, args.grown, dev)
Z.normal_()
AZ = spmm(A, Z)
U = symmetric_gram_from_products(Z, [(AZ[:, :60], 0), (AZ[:, 60:], 60)])
G = gram(Z[:, :256], AZ[:, :256])  # full Gram tile path (128 x 64 tiles)
C = torch.randn(args.grown, 60, dtype=torch.float64, device=dev)
Phi = gemm_nn(Z, C)
torch.cuda.synchronize()
print("ok", float(G[0, 0]), float(Phi[0, 0]))
