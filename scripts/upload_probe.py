"""Probe: host-side cost of uploading one C3 system (pageable H2D + gather + validation)."""
import sys, time, os
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1512_05820_b200 as pk
from paper_1512_05820_b200.problems import elasticity_sequence
specs = list(elasticity_sequence((64, 64, 64), p=3))
for s in specs:
    torch.cuda.synchronize(); t = time.perf_counter()
    A = pk.SparseSpdMatrix.from_host(s.A); torch.cuda.synchronize()
    t1 = time.perf_counter()
    v = torch.from_numpy(s.A.values).to('cuda'); torch.cuda.synchronize(); t2 = time.perf_counter()
    pin = torch.empty(s.A.values.shape, dtype=torch.float64, pin_memory=True)
    t3 = time.perf_counter(); pin.numpy()[:] = s.A.values; t4 = time.perf_counter()
    v2 = pin.to('cuda', non_blocking=True); torch.cuda.synchronize(); t5 = time.perf_counter()
    print(f"from_host {1e3*(t1-t):.1f} ms | pageable H2D {1e3*(t2-t1):.1f} ms | host->pinned memcpy {1e3*(t4-t3):.1f} ms | pinned H2D {1e3*(t5-t4):.1f} ms", flush=True)
