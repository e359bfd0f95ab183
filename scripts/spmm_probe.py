"""C5 SpMM A S on the 7-point Laplacian (128x128x256) for a block of columns:
CUDA-event time and GB/s (bytes: matrix once per 8-column pass + S read + AS
written). RK_SELL1_SPMM=1 selects the scalar SELL SpMM, else the CSR kernel.

python scripts/spmm_probe.py [--cols 256]     (GPU box)
"""
import argparse
import json
import math
import os
import sys

import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import paper_1512_05820_b200 as pk  # noqa: E402
from paper_1512_05820_b200.linalg import empty_block, spmm  # noqa: E402
from paper_1512_05820_b200.problems import laplacian3d  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cols", type=int, default=256)
    ap.add_argument("--reps", type=int, default=5)
    args = ap.parse_args()
    L = laplacian3d(128, 128, 256)
    A = pk.SparseSpdMatrix(L.n, L.row_offsets, L.col_indices, L.values)
    S = empty_block(L.n, args.cols, "cuda")
    S.normal_()
    out = empty_block(L.n, args.cols, "cuda")
    spmm(A, S, out=out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.reps):
        spmm(A, S, out=out)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.reps
    mat = 12 * L.nnz + 4 * (L.n + 1)
    ideal = mat + 16 * L.n * args.cols
    passes = mat * math.ceil(args.cols / 8) + 16 * L.n * args.cols
    print(json.dumps({"variant": os.environ.get("RK_SELL1_SPMM", "0"), "cols": args.cols, "ms": round(ms, 3),
                      "GB_s_matrix_once": round(ideal / ms / 1e6, 1), "GB_s_per_pass": round(passes / ms / 1e6, 1)}))


if __name__ == "__main__":
    main()
