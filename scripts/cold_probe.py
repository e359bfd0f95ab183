"""Where a cold first upload of a C3 system goes (the `cold_value` leg of
bench.py): host sortedness check, int32 pattern upload, device SELL build,
the two affine value arrays, value formation + gather + validation.
python scripts/cold_probe.py   (GPU box)"""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1512_05820_b200 as pk  # noqa: E402
from paper_1512_05820_b200 import linalg as L  # noqa: E402
from paper_1512_05820_b200.problems import elasticity_sequence  # noqa: E402

specs = list(elasticity_sequence((64, 64, 64), p=2))
torch.zeros(1, device="cuda")
out = {}


def timed(name, fn):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = fn()
    torch.cuda.synchronize()
    out[name] = round(time.perf_counter() - t0, 4)
    return r


A0 = specs[0].A
timed("rows_sorted_host", lambda: L._rows_sorted(np.asarray(A0.row_offsets), np.asarray(A0.col_indices)))
L.clear_upload_caches()
timed("first_system_cold_total", lambda: pk.SparseSpdMatrix.from_host(A0))
timed("second_system_warm_total", lambda: pk.SparseSpdMatrix.from_host(specs[1].A))
L.clear_upload_caches()
timed("pattern_only_cold", lambda: L._device_pattern(np.asarray(A0.row_offsets), np.asarray(A0.col_indices), torch.device("cuda", 0), A0.n))
timed("affine_parts_upload", lambda: L._affine_device_parts(A0.affine[0], A0.affine[1], torch.device("cuda", 0)))
print(json.dumps(out))
