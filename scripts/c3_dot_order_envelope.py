"""The reference algorithm's own reduction-order envelope at full C3 size:
plain Jacobi PCG on C3 system 1 (the reference's statements, krylov.py:181-345
with x0 = 0) with the dot products taken as BLAS ddot (numpy `@`, what the
reference does), numpy's pairwise np.sum(a * b), or math.fsum. Measured here
(8-core container): BLAS 748 iterations, pairwise 747, and the solutions differ
by 1.9e-8 relative -- a summation order alone moves the count by one.

python scripts/c3_dot_order_envelope.py blas pairwise exact      (CPU, ~80 s each)
"""
import math, sys, time
import numpy as np, scipy.sparse
sys.path.insert(0, "/root/repo")
from paper_1512_05820_b200.problems import elasticity_sequence
s = next(iter(elasticity_sequence((64, 64, 64), p=1, rtol=1e-5, seed=3)))
A = scipy.sparse.csr_matrix((s.A.values, s.A.col_indices, s.A.row_offsets), shape=(s.A.n,) * 2)
b = s.b; tol = s.tol; dinv = 1.0 / A.diagonal()
dots = {"blas": lambda a, c: float(a @ c), "pairwise": lambda a, c: float(np.sum(a * c)),
        "exact": lambda a, c: math.fsum(a * c)}
for name in sys.argv[1:]:
    dot = dots[name]
    t0 = time.time()
    x = np.zeros_like(b); r = b.copy(); z = dinv * r; p = z.copy(); rz = dot(r, z)
    for k in range(5000):
        Ap = A @ p
        gamma = dot(p, Ap); alpha = rz / gamma
        x = x + alpha * p; r = r - alpha * Ap
        if math.sqrt(dot(r, r)) <= tol:
            break
        z = dinv * r; rzn = dot(r, z); p = z + (rzn / rz) * p; rz = rzn
    print(name, k + 1, round(time.time() - t0, 1), flush=True)
    np.save(f"/tmp/cg_x_{name}.npy", x)
