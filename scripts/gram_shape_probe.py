"""One Gram shape, timed (CUDA events) and optionally profiled:
python scripts/gram_shape_probe.py --n 811200 --m 638 --y-old 60 [--full] [--reps 5]
Upper mode = the truncation Gram Z'AZ from two product segments (as
threestage.update_basis); --full = the plain X'Y of the same width."""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
from paper_1512_05820_b200.linalg import empty_block, gram, symmetric_gram_from_products  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=811200)
ap.add_argument("--m", type=int, default=638)
ap.add_argument("--y-old", type=int, default=60)
ap.add_argument("--full", action="store_true")
ap.add_argument("--reps", type=int, default=5)
a = ap.parse_args()
dev = torch.device("cuda:0")
g = torch.Generator(device=dev).manual_seed(0)
Z, AZ = empty_block(a.n, a.m, dev), empty_block(a.n, a.m, dev)
Z.copy_(torch.randn(a.n, a.m, generator=g, device=dev, dtype=torch.float64))
AZ.copy_(torch.randn(a.n, a.m, generator=g, device=dev, dtype=torch.float64))
AY, AV = AZ[:, : a.y_old], AZ[:, a.y_old:]
fn = (lambda: gram(Z, AZ)) if a.full else (lambda: symmetric_gram_from_products(Z, [(AY, 0), (AV, a.y_old)]))
fn()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(a.reps):
    fn()
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / a.reps
flops = 2 * a.n * a.m * a.m if a.full else a.n * a.m * (a.m + 1)
print(json.dumps({"n": a.n, "m": a.m, "full": a.full, "tile": os.environ.get("RK_GRAM_TILE", "auto"), "ms": round(ms, 3),
                  "tflops": round(flops / ms / 1e9, 2), "frac": round(flops / ms / 1e9 / 37.1, 3)}))
