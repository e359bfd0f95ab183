"""Where a wrong Gram entry sits (debug aid for scripts/gram_stress.py)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
from paper_1512_05820_b200.linalg import empty_block, symmetric_gram_from_products  # noqa: E402

dev = torch.device("cuda:0")
g = torch.Generator(device=dev).manual_seed(0)
n, y_old, k = (int(v) for v in (sys.argv[1:4] if len(sys.argv) > 3 else (2097152, 40, 346)))
m = y_old + k
Z, AY, AV = empty_block(n, m, dev), empty_block(n, max(y_old, 1), dev), empty_block(n, k, dev)
for t in (Z, AY, AV):
    t.copy_(torch.randn(t.shape, generator=g, device=dev, dtype=torch.float64))
segs = ([(AY[:, :y_old], 0)] if y_old else []) + [(AV, y_old)]
ref = torch.cat([Z.t() @ AY[:, :y_old], Z.t() @ AV], dim=1)
upper = torch.triu(torch.ones(m, m, dtype=torch.bool, device=dev))
for r in range(6):
    U = symmetric_gram_from_products(Z, segs)
    G = U.store[:m, :m].t().clone()
    E = ((G - ref).abs() * upper)
    bad = torch.nonzero(E > 1e-6)
    rows = sorted(set(bad[:, 0].tolist()))
    cols = sorted(set(bad[:, 1].tolist()))
    def rng(v):
        out, s = [], None
        for x in v:
            if s is None:
                s = p = x
            elif x == p + 1:
                p = x
            else:
                out.append((s, p)); s = p = x
        if s is not None:
            out.append((s, p))
        return out
    print(json.dumps({"rep": r, "tile": os.environ.get("RK_GRAM_TILE", "auto"), "nbad": int(bad.shape[0]), "rows": rng(rows), "cols": rng(cols),
                      "max_abs_err": float(E.max()), "median_bad_err": float(E[E > 1e-6].median()) if bad.shape[0] else 0.0}), flush=True)
