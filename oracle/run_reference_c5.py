"""Run the reference itself (recykl, from /root/reference in this container)
on the full-size C5 truncation step (BASELINE configs[4]): A = 7-point
Laplacian on 128 x 128 x 256 (N = 4,194,304), S = N(0,1) snapshots of m
columns from numpy's default_rng(seed) (problems.snapshot_matrix, the same
host generator the GPU test uses), G, AS = assemble_gram(A, S)
(linalg.py:160-174), then pod_evd_from_gram(G, S, gamma = 1, eps = 1)
(pod.py:123-131). Saves sigma, y, G's diagonal and 8 sampled entries, and
Phi at 2000 fixed rows to tests/golden/c5_full_m<m>.npz. Test
infrastructure only (the GPU test reads the .npz, never the reference).

    python oracle/run_reference_c5.py [m=256]     (~30 GB of host memory at m = 256)
"""
import os
import sys
import time
import warnings

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
warnings.simplefilter("ignore")


def main(m=256, seed=5):
    from recykl.linalg import SparseSpdMatrix, assemble_gram
    from recykl.pod import pod_evd_from_gram

    from paper_1512_05820_b200.problems import laplacian3d, snapshot_matrix

    H = laplacian3d(128, 128, 256)
    A = SparseSpdMatrix(H.n, H.row_offsets, H.col_indices, H.values)
    t0 = time.perf_counter()
    S = snapshot_matrix(H.n, m, seed=seed)
    t_gen = time.perf_counter() - t0
    t0 = time.perf_counter()
    G, AS = assemble_gram(A, S)
    t_gram = time.perf_counter() - t0
    del AS
    t0 = time.perf_counter()
    res = pod_evd_from_gram(G, S, np.ones(m), 1.0)
    t_pod = time.perf_counter() - t0
    rows = np.sort(np.random.default_rng(1).choice(H.n, 2000, replace=False))
    ij = np.random.default_rng(2).integers(0, m, size=(8, 2))
    out = {
        "n": np.int64(H.n), "m": np.int64(m), "seed": np.int64(seed), "sigma": res.singular_values,
        "y": np.int64(res.y), "G_diag": np.diag(G).copy(), "G_ij": ij, "G_ij_val": G[ij[:, 0], ij[:, 1]],
        "rows": rows, "phi_rows": np.asarray(res.basis.columns)[rows], "coef": res.snapshot_coef,
        "wall": np.array([t_gen, t_gram, t_pod]),
    }
    path = os.path.join(os.path.dirname(HERE), "tests", "golden", f"c5_full_m{m}.npz")
    np.savez_compressed(path, **out)
    print(path, res.y, [round(t, 1) for t in out["wall"]], flush=True)


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 256)
