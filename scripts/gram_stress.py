"""Race hunt for the DMMA Gram: every shape is computed `reps` times; each
repeat must equal the first one bitwise (fixed-order split combine) and match
cuBLAS. python scripts/gram_stress.py [--reps 30]  (GPU box) -> one JSON line per shape."""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
from paper_1512_05820_b200.linalg import empty_block, gram, symmetric_gram_from_products  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=30)
    args = ap.parse_args()
    dev = torch.device("cuda:0")
    g = torch.Generator(device=dev).manual_seed(0)
    for n, y_old, k in ((811200, 60, 578), (811200, 60, 440), (811200, 64, 574), (2097152, 40, 346), (300000, 0, 638)):
        m = y_old + k
        Z, AY, AV = empty_block(n, m, dev), empty_block(n, max(y_old, 1), dev), empty_block(n, k, dev)
        for t in (Z, AY, AV):
            t.copy_(torch.randn(t.shape, generator=g, device=dev, dtype=torch.float64))
        segs = ([(AY[:, :y_old], 0)] if y_old else []) + [(AV, y_old)]
        ref = torch.cat([Z.t() @ AY[:, :y_old], Z.t() @ AV], dim=1)
        upper = torch.triu(torch.ones(m, m, dtype=torch.bool, device=dev))
        first, bad, worst, cols = None, 0, 0.0, set()
        for r in range(args.reps):
            U = symmetric_gram_from_products(Z, segs)
            G = U.store[:m, :m].t().clone()  # rows of the row-major store = columns of G
            E = ((G - ref).abs() * upper) / ref.abs().max()
            err = float(E.max())
            worst = max(worst, err)
            cols |= set(torch.nonzero(E.max(dim=0).values > 1e-9).flatten().tolist())
            if first is None:
                first = G
            elif not torch.equal(G * upper, first * upper):
                bad += 1
        print(json.dumps({"n": n, "m": m, "c1": y_old, "reps": args.reps, "repeats_differing": bad, "worst_rel_err": worst,
                          "wrong_columns": sorted(cols)}), flush=True)
        del Z, AY, AV, ref, first
    n, m = 2097152, 256
    S = empty_block(n, m, dev)
    S.copy_(torch.randn(n, m, generator=g, device=dev, dtype=torch.float64))
    ref = S.t() @ S
    first, bad, worst = None, 0, 0.0
    for r in range(args.reps):
        G = gram(S, S)
        worst = max(worst, float((G - ref).abs().max() / ref.abs().max()))
        if first is None:
            first = G.clone()
        elif not torch.equal(G, first):
            bad += 1
    print(json.dumps({"n": n, "m": m, "full": True, "reps": args.reps, "repeats_differing": bad, "worst_rel_err": worst}))


if __name__ == "__main__":
    main()
