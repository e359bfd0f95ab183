"""Time the DMMA Gram kernels at the shapes the C3 truncation and C5 use.

python scripts/gram_probe.py [--c5-max 2048]     (GPU box) -> one JSON line per shape

The tile variant is chosen per shape by dmma.cu (RK_GRAM_TILE=0/1/2 forces
64x64 / 128x64 / 128x128; it is read once per process, so sweep variants with
one process each). Every shape is also checked against cuBLAS (torch.mm).
"""
import argparse
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
from paper_1512_05820_b200.linalg import as_block, empty_block, gemm_nn, gram, symmetric_gram_from_products  # noqa: E402

DMMA_PEAK = 37.1


def _time(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def _rel(G, R):
    return float((G - R).abs().max() / R.abs().max())


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--c5-max", type=int, default=2048)
    ap.add_argument("--skip-c3", action="store_true")
    args = ap.parse_args()
    dev = torch.device("cuda:0")
    g = torch.Generator(device=dev).manual_seed(0)
    tile = os.environ.get("RK_GRAM_TILE", "auto")
    out = []
    if not args.skip_c3:
        # C3 truncation: Z = [Y_old (60) | V (k)], products (AY, 0), (AV, 60)
        for n, y_old, k in ((2097152, 40, 346), (811200, 60, 578), (811200, 60, 440), (811200, 60, 740)):
            m = y_old + k
            Z = empty_block(n, m, dev)
            Z.copy_(torch.randn(n, m, generator=g, device=dev, dtype=torch.float64))
            AY = empty_block(n, y_old, dev)
            AY.copy_(torch.randn(n, y_old, generator=g, device=dev, dtype=torch.float64))
            AV = empty_block(n, k, dev)
            AV.copy_(torch.randn(n, k, generator=g, device=dev, dtype=torch.float64))
            ms = _time(lambda: symmetric_gram_from_products(Z, [(AY, 0), (AV, y_old)]))
            # the same triangle as two rk_gram_upper launches (one per product block)
            ms2 = _time(lambda: symmetric_gram_from_products(Z, [(AY, 0), (AV, y_old)], single_launch=False))
            U = symmetric_gram_from_products(Z, [(AY, 0), (AV, y_old)])
            ref = Z[:, :m].t() @ AV[:, :k]
            got = U.store[y_old:m, :m]  # rows of the row-major store = columns of G
            upper = torch.triu(torch.ones(m, k, dtype=torch.bool, device=dev), diagonal=-y_old)
            err = float(((got.t() - ref).abs() * upper).max() / ref.abs().max())
            flops = n * m * (m + 1)  # one triangle
            tf = flops / ms / 1e9
            out.append({"op": "gram_upper_c2" if n == 2097152 else "gram_upper_c3", "tile": tile, "n": n, "m": m, "ms": round(ms, 3),
                        "ms_two_launches": round(ms2, 3),
                        "tflops_triangle": round(tf, 2), "frac": round(tf / DMMA_PEAK, 3), "rel_err_vs_cublas": err})
            coef = torch.randn(m, 60, generator=g, device=dev, dtype=torch.float64)
            ms = _time(lambda: gemm_nn(Z, coef))
            out.append({"op": "gemm_nn_c3", "n": n, "s": m, "y": 60, "ms": round(ms, 3),
                        "tflops": round(2 * n * m * 60 / ms / 1e9, 2)})
            del Z, AY, AV, U, ref
    n = 4194304
    for m in (256, 1024, 2048):
        if m > args.c5_max:
            continue
        S = as_block(torch.randn(n, m, generator=g, device=dev, dtype=torch.float64))
        ms = _time(lambda: gram(S, S), reps=3)
        G = gram(S, S)
        idx = torch.arange(0, n, 64, device=dev)
        err = None
        if m <= 1024:
            R = S.t() @ S
            err = _rel(G, R)
            del R
        tf = 2 * n * m * m / ms / 1e9
        out.append({"op": "gram_full_c5", "tile": tile, "n": n, "m": m, "ms": round(ms, 3), "tflops": round(tf, 2),
                    "frac": round(tf / DMMA_PEAK, 3), "rel_err_vs_cublas": err})
        del S, G, idx
        torch.cuda.empty_cache()
    for o in out:
        print(json.dumps(o), flush=True)


if __name__ == "__main__":
    t = time.time()
    main()
    print(json.dumps({"wall_s": round(time.time() - t, 1)}))
