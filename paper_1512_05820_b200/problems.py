"""Seeded synthetic SPD system sequences with the BASELINE.json shapes (C1-C5).

BASELINE names no public suite and the paper's Sierra matrices are not
available, so these generators stand in for them:

* C1 ``poisson2d_sequence``: 2-D 5-point Poisson on a 64 x 64 interior grid,
  invariant matrix, b_i = b_0 + 0.1 xi_i (numpy default_rng(0), drawn in the
  order b_0, c, xi_1..xi_p).
* C2 ``diffusion3d_sequence``: 3-D 7-point variable-coefficient diffusion on
  128^3, kappa_i = exp(g + 0.05 i h) with g, h Gaussian random fields of
  correlation length 8 cells; face coefficient (kappa_p + kappa_q)/2 and
  boundary faces add kappa_p to the diagonal (as problems.py:75-89 of the
  reference does in 2-D); b_i white noise smoothed by 3 damped-Jacobi sweeps.
* C3/C4 ``elasticity_sequence``: trilinear Q1 hexahedral linear elasticity
  (nu = 0.3, 2x2x2 Gauss), clamped at x = 0, E_e = 1 + 0.5 U_e; system i
  scales element e by (1 + 0.02 i U'_e) and loads the x = 1 face with a
  traction whose direction rotates 2 degrees per system. The dynamic variant
  (C4) adds the lumped mass M / dt^2 and uses a seeded smooth load history.
* C5 ``laplacian3d`` + ``snapshot_matrix``: constant 7-point Laplacian and a
  Gaussian snapshot block.

Systems are emitted as host CSR (``HostCsr``) sharing one pattern per
sequence, so the device layer uploads the pattern once and only values per
system; tolerances are absolute, tol_i = rtol * ||b_i||, following the
forcing condition ||b - A x|| <= eps (reference krylov.py:267).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
import scipy.sparse


@dataclass
class HostCsr:
    """Host CSR (both triangles) with the reference SparseSpdMatrix's field names."""

    n: int
    row_offsets: np.ndarray
    col_indices: np.ndarray
    values: np.ndarray

    @property
    def nnz(self) -> int:
        return int(self.values.shape[0])

    def to_scipy(self) -> scipy.sparse.csr_matrix:
        return scipy.sparse.csr_matrix((self.values, self.col_indices, self.row_offsets), shape=(self.n, self.n))

    def diagonal(self) -> np.ndarray:
        return self.to_scipy().diagonal()


class AffineHostCsr:
    """Host CSR whose values are ``base + coef * delta`` on a fixed pattern: the
    form in which a drifting sequence changes its matrix (C3: element e scaled
    by 1 + 0.02 i U_e is ``vals_E + i * vals_D``). It has the reference
    SparseSpdMatrix's field names, so every host consumer (the reference
    itself, scipy) sees an ordinary matrix -- ``values`` materialises
    ``base + coef * delta`` with numpy on first use. The device path
    (``SparseSpdMatrix.from_host``) instead uploads ``base`` and ``delta`` once
    per sequence and forms each system's values on the GPU with the same two
    roundings (no per-system upload of the 0.5-2 GB of values)."""

    def __init__(self, n: int, row_offsets: np.ndarray, col_indices: np.ndarray, base: np.ndarray,
                 delta: np.ndarray, coef: float):
        self.n = int(n)
        self.row_offsets = row_offsets
        self.col_indices = col_indices
        self.affine = (base, delta, float(coef))
        self._values = None

    @property
    def values(self) -> np.ndarray:
        if self._values is None:
            base, delta, coef = self.affine
            self._values = base + coef * delta
        return self._values

    @property
    def nnz(self) -> int:
        return int(self.affine[0].shape[0])

    def to_scipy(self) -> scipy.sparse.csr_matrix:
        return scipy.sparse.csr_matrix((self.values, self.col_indices, self.row_offsets), shape=(self.n, self.n))

    def diagonal(self) -> np.ndarray:
        return self.to_scipy().diagonal()


@dataclass
class LinearSystemSpec:
    A: object
    b: np.ndarray
    xbar: np.ndarray | None
    tol: float


@dataclass
class SystemSequence:
    """Sequence of systems (problems.py:43-58 of the reference); ``systems``
    may be a list or a zero-argument factory of an iterator (lazy)."""

    n: int
    systems: object
    C: np.ndarray | None = None
    metadata: dict = field(default_factory=dict)
    p_hint: int | None = None

    @property
    def p(self) -> int:
        return len(self.systems) if isinstance(self.systems, list) else int(self.p_hint or 0)

    def __iter__(self):
        if isinstance(self.systems, list):
            return iter(self.systems)
        return iter(self.systems())

    def __getitem__(self, j):
        if isinstance(self.systems, list):
            return self.systems[j]
        for i, s in enumerate(self):
            if i == j:
                return s
        raise IndexError(j)

    def take(self, count: int) -> "SystemSequence":
        """Prefix of the sequence (the sequence is causal, so prefix parity is exact)."""
        items = []
        for i, s in enumerate(self):
            if i >= count:
                break
            items.append(s)
        return SystemSequence(self.n, items, self.C, dict(self.metadata, prefix=count))


def _from_scipy(M) -> HostCsr:
    csr = scipy.sparse.csr_matrix(M).astype(np.float64)
    csr.sum_duplicates()
    csr.sort_indices()
    return HostCsr(csr.shape[0], csr.indptr.astype(np.int64), csr.indices.astype(np.int32), csr.data)


# ---------------------------------------------------------------------------
# C1: 2-D Poisson
# ---------------------------------------------------------------------------
def poisson2d_matrix(nx: int) -> HostCsr:
    """kron(I, T) + kron(S, I), T = tridiag(-1, 4, -1), S = offdiag(-1)."""
    T = scipy.sparse.diags([-np.ones(nx - 1), 4.0 * np.ones(nx), -np.ones(nx - 1)], [-1, 0, 1])
    S = scipy.sparse.diags([-np.ones(nx - 1), -np.ones(nx - 1)], [-1, 1])
    I = scipy.sparse.identity(nx)
    return _from_scipy(scipy.sparse.kron(I, T) + scipy.sparse.kron(S, I))


def poisson2d_sequence(nx: int = 64, p: int = 20, rtol: float = 1e-6, seed: int = 0) -> SystemSequence:
    A = poisson2d_matrix(nx)
    n = A.n
    rng = np.random.default_rng(seed)
    b0 = rng.standard_normal(n)
    c = rng.standard_normal(n)
    systems = []
    for _ in range(p):
        b = b0 + 0.1 * rng.standard_normal(n)
        systems.append(LinearSystemSpec(A=A, b=b, xbar=None, tol=rtol * float(np.linalg.norm(b))))
    return SystemSequence(n, systems, C=c[None, :], metadata={"name": f"C1-poisson2d-{nx}", "rtol": rtol,
                                                              "seed": seed, "qoi": "c'x"})


# ---------------------------------------------------------------------------
# C2: 3-D variable-coefficient diffusion
# ---------------------------------------------------------------------------
def gaussian_field(shape, corr_len: float, rng) -> np.ndarray:
    """Unit-variance Gaussian random field: white noise filtered by a Gaussian
    kernel of correlation length ``corr_len`` cells (FFT)."""
    noise = rng.standard_normal(shape)
    ks = np.meshgrid(*[np.fft.fftfreq(s) for s in shape], indexing="ij", sparse=True)
    k2 = sum(k * k for k in ks)
    filt = np.exp(-0.5 * (2.0 * np.pi * corr_len) ** 2 * k2)
    f = np.real(np.fft.ifftn(np.fft.fftn(noise) * filt))
    f -= f.mean()
    return f / max(f.std(), 1e-300)


def _stencil7_pattern(nx, ny, nz):
    """CSR pattern of the 7-point stencil on an nx*ny*nz grid (x fastest)."""
    n = nx * ny * nz
    idx = np.arange(n).reshape(nz, ny, nx)
    offs = [(-1, 0, 0), (0, -1, 0), (0, 0, -1), (0, 0, 0), (0, 0, 1), (0, 1, 0), (1, 0, 0)]  # (dz, dy, dx) sorted
    valid = []
    for dz, dy, dx in offs:
        v = np.ones((nz, ny, nx), dtype=bool)
        if dz == -1: v[0, :, :] = False
        if dz == 1: v[-1, :, :] = False
        if dy == -1: v[:, 0, :] = False
        if dy == 1: v[:, -1, :] = False
        if dx == -1: v[:, :, 0] = False
        if dx == 1: v[:, :, -1] = False
        valid.append(v.reshape(-1))
    valid = np.stack(valid)
    cnt = valid.sum(0)
    rowptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(cnt, out=rowptr[1:])
    pos = np.cumsum(valid, axis=0) - valid
    col = np.empty(int(rowptr[-1]), dtype=np.int32)
    flat = idx.reshape(-1)
    slots = []
    for d, (dz, dy, dx) in enumerate(offs):
        rows = flat[valid[d]]
        where = rowptr[rows] + pos[d, valid[d]]
        col[where] = rows + dx + nx * (dy + ny * dz)
        slots.append(where)
    return rowptr, col, valid, slots, offs


def diffusion3d_values(kappa: np.ndarray, pattern) -> np.ndarray:
    """Values of the variable-coefficient operator on a fixed 7-point pattern."""
    rowptr, col, valid, slots, offs = pattern
    nz, ny, nx = kappa.shape
    k = kappa
    vals = np.empty(col.shape[0], dtype=np.float64)
    diag = np.zeros_like(k)
    for d, (dz, dy, dx) in enumerate(offs):
        if (dz, dy, dx) == (0, 0, 0):
            continue
        # neighbour coefficient, boundary faces contribute kappa_p to the diagonal
        nb = np.roll(k, shift=(-dz, -dy, -dx), axis=(0, 1, 2))
        edge = 0.5 * (k + nb)
        v = valid[d].reshape(k.shape)
        diag += np.where(v, edge, k)
        vals[slots[d]] = -edge.reshape(-1)[valid[d]]
    d0 = offs.index((0, 0, 0))
    vals[slots[d0]] = diag.reshape(-1)
    return vals


def diffusion3d_sequence(n: int = 128, p: int = 30, rtol: float = 1e-4, seed: int = 2,
                         corr_len: float = 8.0) -> SystemSequence:
    rng = np.random.default_rng(seed)
    shape = (n, n, n)
    g = gaussian_field(shape, corr_len, rng)
    h = gaussian_field(shape, corr_len, rng)
    c = rng.standard_normal(n ** 3)
    pattern = _stencil7_pattern(n, n, n)
    rowptr, col = pattern[0], pattern[1]
    N = n ** 3
    lap = HostCsr(N, rowptr, col, diffusion3d_values(np.ones(shape), pattern))
    lap_s = lap.to_scipy()
    lap_dinv = 1.0 / lap_s.diagonal()
    rhs_seed = int(rng.integers(2**31))

    def gen():
        r = np.random.default_rng(rhs_seed)
        for i in range(1, p + 1):
            kappa = np.exp(g + 0.05 * i * h)
            A = HostCsr(N, rowptr, col, diffusion3d_values(kappa, pattern))
            b = r.standard_normal(N)
            for _ in range(3):  # damped Jacobi smoothing with the unit-coefficient Laplacian
                b = b - (2.0 / 3.0) * lap_dinv * (lap_s @ b)
            yield LinearSystemSpec(A=A, b=b, xbar=None, tol=rtol * float(np.linalg.norm(b)))

    return SystemSequence(N, gen, C=c[None, :], p_hint=p,
                          metadata={"name": f"C2-diffusion3d-{n}", "rtol": rtol, "seed": seed})


# ---------------------------------------------------------------------------
# C3/C4: Q1 hexahedral linear elasticity
# ---------------------------------------------------------------------------
def q1_element_stiffness(nu: float = 0.3, E: float = 1.0, h: float = 1.0) -> np.ndarray:
    """24 x 24 stiffness of a cube element of side h (2x2x2 Gauss); local node
    a = lx + 2 ly + 4 lz, dof 3a + c."""
    lam = E * nu / ((1 + nu) * (1 - 2 * nu))
    mu = E / (2 * (1 + nu))
    D = np.zeros((6, 6))
    D[:3, :3] = lam
    D[np.arange(3), np.arange(3)] += 2 * mu
    D[3:, 3:] = mu * np.eye(3)
    corners = np.array([[(a >> 0) & 1, (a >> 1) & 1, (a >> 2) & 1] for a in range(8)]) * 2.0 - 1.0
    gp = np.array([-1.0, 1.0]) / math.sqrt(3.0)
    K = np.zeros((24, 24))
    jac = h / 2.0
    for xi in gp:
        for eta in gp:
            for zeta in gp:
                q = np.array([xi, eta, zeta])
                dN = np.zeros((8, 3))
                for a in range(8):
                    s = corners[a]
                    f = 1.0 + s * q
                    dN[a, 0] = 0.125 * s[0] * f[1] * f[2]
                    dN[a, 1] = 0.125 * s[1] * f[0] * f[2]
                    dN[a, 2] = 0.125 * s[2] * f[0] * f[1]
                dN /= jac
                B = np.zeros((6, 24))
                for a in range(8):
                    bx, by, bz = dN[a]
                    c = 3 * a
                    B[0, c] = bx
                    B[1, c + 1] = by
                    B[2, c + 2] = bz
                    B[3, c + 1], B[3, c + 2] = bz, by
                    B[4, c], B[4, c + 2] = bz, bx
                    B[5, c], B[5, c + 1] = by, bx
                K += B.T @ D @ B * jac ** 3
    return 0.5 * (K + K.T)


class ElasticityAssembler:
    """Fixed CSR pattern of the clamped Q1 mesh plus fast value assembly.

    Free nodes are those with ix >= 1 (x = 0 clamped), numbered x fastest;
    dof = 3 * node + component (3 x 3 blocks). Row entries are sorted by
    column, so the pattern is valid CSR for the device kernels.
    """

    OFFS = [(dz, dy, dx) for dz in (-1, 0, 1) for dy in (-1, 0, 1) for dx in (-1, 0, 1)]

    def __init__(self, nex: int, ney: int, nez: int, nu: float = 0.3):
        self.ne = (nex, ney, nez)
        self.h = 1.0 / nex
        self.K0 = q1_element_stiffness(nu, 1.0, self.h)
        fx, fy, fz = nex, ney + 1, nez + 1          # free-node grid (ix = 1..nex)
        self.fshape = (fz, fy, fx)
        nf = fx * fy * fz
        self.nfree = nf
        self.n = 3 * nf
        IZ, IY, IX = np.meshgrid(np.arange(fz), np.arange(fy), np.arange(1, nex + 1), indexing="ij")
        valid = []
        for dz, dy, dx in self.OFFS:
            v = ((IX + dx >= 1) & (IX + dx <= nex) & (IY + dy >= 0) & (IY + dy <= ney)
                 & (IZ + dz >= 0) & (IZ + dz <= nez))
            valid.append(v.reshape(-1))
        valid = np.stack(valid)
        cnt = valid.sum(0)
        rowlen = np.repeat(3 * cnt, 3)
        rowptr = np.zeros(self.n + 1, dtype=np.int64)
        np.cumsum(rowlen, out=rowptr[1:])
        pos = np.cumsum(valid, axis=0) - valid
        nnz = int(rowptr[-1])
        col = np.empty(nnz, dtype=np.int32)
        self.slots = {}
        fa_all = np.arange(nf)
        for d, (dz, dy, dx) in enumerate(self.OFFS):
            fa = fa_all[valid[d]]
            fb = fa + dx + fx * (dy + fy * dz)
            for ci in range(3):
                base = rowptr[3 * fa + ci] + 3 * pos[d, valid[d]]
                for cj in range(3):
                    col[base + cj] = 3 * fb + cj
                    self.slots[(d, ci, cj)] = base + cj
        self.valid = valid
        self.rowptr, self.col, self.nnz = rowptr, col, nnz

    def values(self, elem_scale: np.ndarray) -> np.ndarray:
        """Assembled values of sum_e s_e K0 on the fixed pattern."""
        nex, ney, nez = self.ne
        s = np.asarray(elem_scale, dtype=np.float64).reshape(nez, ney, nex)
        spad = np.zeros((nez + 2, ney + 2, nex + 2))
        spad[1:-1, 1:-1, 1:-1] = s
        fz, fy, fx = self.fshape
        shifted = {}
        for lz in (0, 1):
            for ly in (0, 1):
                for lx in (0, 1):
                    # element (ix - lx, iy - ly, iz - lz) of free node (ix >= 1), padded +1
                    shifted[(lx, ly, lz)] = spad[1 - lz : 1 - lz + fz, 1 - ly : 1 - ly + fy,
                                                 2 - lx : 2 - lx + fx].reshape(-1)
        vals = np.empty(self.nnz, dtype=np.float64)
        K0 = self.K0
        for d, (dz, dy, dx) in enumerate(self.OFFS):
            v = self.valid[d]
            terms = []
            for (lx, ly, lz), sh in shifted.items():
                mx, my, mz = lx + dx, ly + dy, lz + dz
                if 0 <= mx <= 1 and 0 <= my <= 1 and 0 <= mz <= 1:
                    terms.append((lx + 2 * ly + 4 * lz, mx + 2 * my + 4 * mz, sh[v]))
            for ci in range(3):
                for cj in range(3):
                    acc = np.zeros(int(v.sum()))
                    for la, lb, sh in terms:
                        acc += K0[3 * la + ci, 3 * lb + cj] * sh
                    vals[self.slots[(d, ci, cj)]] = acc
        return vals

    def lumped_mass_diagonal(self, rho: float = 1.0) -> np.ndarray:
        """Row-sum lumped mass per dof: each element's rho h^3 split over 8 nodes."""
        nex, ney, nez = self.ne
        ones = np.ones(nex * ney * nez)
        fz, fy, fx = self.fshape
        spad = np.zeros((nez + 2, ney + 2, nex + 2))
        spad[1:-1, 1:-1, 1:-1] = ones.reshape(nez, ney, nex)
        m = np.zeros(self.nfree)
        for lz in (0, 1):
            for ly in (0, 1):
                for lx in (0, 1):
                    m += spad[1 - lz : 1 - lz + fz, 1 - ly : 1 - ly + fy, 2 - lx : 2 - lx + fx].reshape(-1)
        return np.repeat(m * rho * self.h ** 3 / 8.0, 3)

    def diagonal_slots(self) -> np.ndarray:
        d0 = self.OFFS.index((0, 0, 0))
        return np.concatenate([self.slots[(d0, c, c)][None, :] for c in range(3)]).T.reshape(-1)

    def face_load(self, traction) -> np.ndarray:
        """Consistent-area nodal forces of a traction on the x = 1 face: a
        uniform 3-vector, or a nodal field of shape (nez + 1, ney + 1, 3)."""
        nex, ney, nez = self.ne
        fz, fy, fx = self.fshape
        wy = np.full(fy, self.h)
        wy[[0, -1]] *= 0.5
        wz = np.full(fz, self.h)
        wz[[0, -1]] *= 0.5
        b = np.zeros((fz, fy, fx, 3))
        b[:, :, -1, :] = (wz[:, None] * wy[None, :])[..., None] * np.asarray(traction, dtype=np.float64)
        return b.reshape(-1)


def elasticity_sequence(ne=(64, 64, 64), p: int = 40, rtol: float = 1e-5, seed: int = 3,
                        dynamic: bool = False, dt: float = 0.05) -> SystemSequence:
    """C3 (static, drifting moduli, rotating traction) or C4 (dynamic: K + M/dt^2,
    seeded smooth load history)."""
    nex, ney, nez = ne
    asm = ElasticityAssembler(nex, ney, nez)
    rng = np.random.default_rng(seed)
    ne_tot = nex * ney * nez
    E = 1.0 + 0.5 * rng.random(ne_tot)
    U = rng.random(ne_tot)
    c = rng.standard_normal(asm.n)
    vals_E = asm.values(E)
    rowptr, col, N = asm.rowptr, asm.col, asm.n
    meta = {"name": f"C{'4' if dynamic else '3'}-elasticity-{nex}x{ney}x{nez}", "rtol": rtol, "seed": seed,
            "nnz": asm.nnz}
    if not dynamic:
        vals_D = asm.values(0.02 * E * U)

        def gen():
            for i in range(1, p + 1):
                # element e scaled by (1 + 0.02 i U_e): values vals_E + i * vals_D
                th = math.radians(2.0 * i)
                b = asm.face_load((0.5, math.cos(th), math.sin(th)))
                yield LinearSystemSpec(A=AffineHostCsr(N, rowptr, col, vals_E, vals_D, i), b=b, xbar=None,
                                       tol=rtol * float(np.linalg.norm(b)))
    else:
        vals = vals_E.copy()
        vals[asm.diagonal_slots()] += asm.lumped_mass_diagonal() / dt ** 2
        A = HostCsr(N, rowptr, col, vals)
        fz, fy, _ = asm.fshape
        # seeded load history: a smooth random traction field on the x = 1 face
        # that drifts by a fresh smooth random increment every step (each system
        # brings one new load direction) plus a slowly rotating uniform part
        load_seed = int(rng.integers(2**31))
        base = rng.standard_normal(3)

        def gen():
            r = np.random.default_rng(load_seed)
            trac = np.zeros((fz, fy, 3))
            for i in range(1, p + 1):
                t = i * dt
                inc = np.stack([gaussian_field((fz, fy), 4.0, r) for _ in range(3)], axis=-1)
                trac = trac + 0.5 * inc
                th = 2 * math.pi * 0.5 * t
                b = asm.face_load(trac + base * math.cos(th))
                yield LinearSystemSpec(A=A, b=b, xbar=None, tol=rtol * float(np.linalg.norm(b)))

    return SystemSequence(N, gen, C=c[None, :], p_hint=p, metadata=meta)


# ---------------------------------------------------------------------------
# C5: Laplacian + snapshot block
# ---------------------------------------------------------------------------
def laplacian3d(nx: int, ny: int, nz: int) -> HostCsr:
    """Constant-coefficient 7-point Laplacian (diag 6, off-diagonals -1, Dirichlet)."""
    pattern = _stencil7_pattern(nx, ny, nz)
    rowptr, col, valid, slots, offs = pattern
    vals = np.full(col.shape[0], -1.0)
    vals[slots[offs.index((0, 0, 0))]] = 6.0
    return HostCsr(nx * ny * nz, rowptr, col, vals)


def snapshot_matrix(n: int, m: int, seed: int = 5) -> np.ndarray:
    """N(0,1) snapshot block S (n x m), host (for small parity sizes)."""
    return np.random.default_rng(seed).standard_normal((n, m))


# ---------------------------------------------------------------------------
# On-disk sequences: JSON manifest + Matrix Market files (problems.py:160-230)
# ---------------------------------------------------------------------------
def write_sequence(seq: SystemSequence, out_dir, name: str = "sequence") -> str:
    """Matrix Market files plus a JSON manifest, the reference's layout and
    file names (problems.py:160-187); returns the manifest path."""
    import json
    import os

    from . import mmio

    os.makedirs(out_dir, exist_ok=True)
    entries = []
    for j, spec in enumerate(seq, start=1):
        mat_name, rhs_name = f"A_{j:03d}.mtx", f"b_{j:03d}.mtx"
        mmio.write_symmetric_matrix(os.path.join(out_dir, mat_name), spec.A)
        mmio.write_array(os.path.join(out_dir, rhs_name), np.asarray(spec.b))
        entry = {"matrix": mat_name, "rhs": rhs_name, "tol": spec.tol}
        if spec.xbar is not None:
            guess_name = f"x_{j:03d}.mtx"
            mmio.write_array(os.path.join(out_dir, guess_name), np.asarray(spec.xbar))
            entry["guess"] = guess_name
        entries.append(entry)
    manifest = {"n": seq.n, "name": name, "systems": entries, "metadata": seq.metadata}
    if seq.C is not None:
        mmio.write_array(os.path.join(out_dir, "C.mtx"), seq.C)
        manifest["output_matrix"] = "C.mtx"
    path = os.path.join(out_dir, "manifest.json")
    with open(path, "w") as fh:
        json.dump(manifest, fh, indent=2)
        fh.write("\n")
    return path


def load_sequence_manifest(path, *, lazy: bool = False) -> SystemSequence:
    """A sequence described by a JSON manifest (problems.py:190-230), same
    checks and ManifestError messages. ``lazy`` defers reading each system's
    files to iteration time, so ``run_sequence`` parses and uploads system j+1
    on its helper thread while system j solves (nothing but the current and
    the next system is held in host memory)."""
    import json
    import os

    from . import mmio
    from .errors import ManifestError

    try:
        with open(path) as fh:
            manifest = json.load(fh)
    except json.JSONDecodeError as exc:
        raise ManifestError(f"{path}:{exc.lineno}: invalid JSON ({exc.msg})") from exc
    base = os.path.dirname(os.path.abspath(path))
    try:
        n = int(manifest["n"])
        raw_systems = manifest["systems"]
    except (KeyError, TypeError, ValueError) as exc:
        raise ManifestError(f"{path}: manifest must carry 'n' and 'systems'") from exc
    parsed = []
    for idx, entry in enumerate(raw_systems, start=1):
        try:
            parsed.append((entry["matrix"], entry["rhs"], float(entry.get("tol", 1e-8)), entry.get("guess")))
        except (KeyError, TypeError, ValueError) as exc:
            raise ManifestError(f"{path}: system {idx} entry malformed") from exc

    def load(idx, mat_file, rhs_file, tol, guess):
        A = mmio.read_matrix(os.path.join(base, mat_file))
        b = mmio.read_array(os.path.join(base, rhs_file))
        if A.n != n or b.shape[0] != n:
            raise ManifestError(
                f"{path}: system {idx} dimension mismatch (matrix {A.n}, rhs {b.shape[0]}, manifest {n})")
        xbar = None
        if guess is not None:
            xbar = mmio.read_array(os.path.join(base, guess))
            if xbar.shape[0] != n:
                raise ManifestError(f"{path}: system {idx} guess has wrong length")
        return LinearSystemSpec(A=A, b=np.asarray(b), xbar=xbar, tol=tol)

    if lazy:
        def systems():
            for idx, item in enumerate(parsed, start=1):
                yield load(idx, *item)
    else:
        systems = [load(idx, *item) for idx, item in enumerate(parsed, start=1)]
    C = None
    if manifest.get("output_matrix"):
        C = np.atleast_2d(mmio.read_array(os.path.join(base, manifest["output_matrix"])))
        if C.shape[1] != n:
            raise ManifestError(f"{path}: output matrix has {C.shape[1]} columns, expected {n}")
    meta = manifest.get("metadata", {"name": manifest.get("name")})
    return SystemSequence(n=n, systems=systems, C=C, metadata=meta, p_hint=len(parsed))
