"""Time the DMMA Gram kernels at the shapes the C3 truncation and C5 use.

python scripts/gram_probe.py   (GPU box) -> one JSON line per shape
"""
import json
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_1512_05820_b200.linalg import as_block, empty_block, gemm_nn, gram, symmetric_gram_from_products  # noqa: E402


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


def main():
    dev = torch.device("cuda:0")
    g = torch.Generator(device=dev).manual_seed(0)
    out = []
    # C3 truncation: Z = [Y_old (60) | V (k)], products (AY, 0), (AV, 60)
    for n, y_old, k in ((811200, 60, 640), (811200, 60, 440), (811200, 60, 740)):
        m = y_old + k
        Z = empty_block(n, m, dev)
        Z.copy_(torch.randn(n, m, generator=g, device=dev, dtype=torch.float64))
        AY = empty_block(n, y_old, dev)
        AY.copy_(torch.randn(n, y_old, generator=g, device=dev, dtype=torch.float64))
        AV = empty_block(n, k, dev)
        AV.copy_(torch.randn(n, k, generator=g, device=dev, dtype=torch.float64))
        ms = _time(lambda: symmetric_gram_from_products(Z, [(AY, 0), (AV, y_old)]))
        flops = n * m * (m + 1)  # one triangle
        out.append({"op": "gram_upper_c3", "n": n, "m": m, "ms": round(ms, 3), "tflops_triangle": round(flops / ms / 1e9, 2)})
        coef = torch.randn(m, 60, generator=g, device=dev, dtype=torch.float64)
        ms = _time(lambda: gemm_nn(Z, coef))
        out.append({"op": "gemm_nn_c3", "n": n, "s": m, "y": 60, "ms": round(ms, 3),
                    "tflops": round(2 * n * m * 60 / ms / 1e9, 2)})
        del Z, AY, AV
    for n, m in ((4194304, 256), (4194304, 1024)):
        S = as_block(torch.randn(n, m, generator=g, device=dev, dtype=torch.float64))
        ms = _time(lambda: gram(S, S), reps=3)
        out.append({"op": "gram_full_c5", "n": n, "m": m, "ms": round(ms, 3), "tflops": round(2 * n * m * m / ms / 1e9, 2)})
        del S
    for o in out:
        print(json.dumps(o))


if __name__ == "__main__":
    t = time.time()
    main()
    print(json.dumps({"wall_s": round(time.time() - t, 1)}))
