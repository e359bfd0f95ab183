"""Time K2 (A X, m columns) on the C3 matrix: python scripts/spmm_probe.py [m ...]."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1512_05820_b200 as pk  # noqa: E402
from paper_1512_05820_b200.linalg import empty_block, spmm  # noqa: E402
from paper_1512_05820_b200.problems import elasticity_sequence  # noqa: E402

spec = next(iter(elasticity_sequence((64, 64, 64), p=1)))
A = pk.SparseSpdMatrix.from_host(spec.A)
dev = A.device
for m in [int(a) for a in sys.argv[1:]] or [60]:
    X = empty_block(A.n, m, dev)
    X.normal_()
    Y = empty_block(A.n, m, dev)
    spmm(A, X, out=Y) if "out" in spmm.__code__.co_varnames else spmm(A, X)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        spmm(A, X)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    print(json.dumps({"m": m, "ms": round(ms, 3), "bsr": A.bval is not None, "ct": os.environ.get("RK_SPMM_CT", "8")}))
