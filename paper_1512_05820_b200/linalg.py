"""Device-resident sparse and dense kernels behind the reference's ``linalg`` API.

Mirrors ``recykl/linalg.py``: ``InstrumentationSink`` (linalg.py:29-60),
``SparseSpdMatrix`` (63-135), ``spmv`` (138-148), ``weighted_inner`` (151-157),
``assemble_gram`` (160-174), ``DenseBasis`` (177-205),
``DenseLowerTriangular`` (217-247), ``dense_cholesky`` (250-267),
``symmetric_evd`` (270-280), ``thin_svd`` (283-290),
``principal_angle_distance`` (319-337).

Vectors and N x m blocks live on the GPU as float64 torch tensors; blocks are
column-major (``stride(0) == 1``) with a leading dimension padded to a
multiple of 32 rows so every column is 256-byte aligned. The small dense
factorizations (Cholesky of w x w, eigh of m x m) run on the host through the
same LAPACK routines the reference calls (dpotrf, dsyevd), which keeps the
reduced problems bit-compatible with the oracle; everything of size N runs in
``libpodcg.so``.
"""

from __future__ import annotations

import os
import threading
from dataclasses import dataclass

import numpy as np
import scipy.linalg
import scipy.sparse
import torch

from . import _native as nat
from .errors import DimensionMismatch, IterationLimit, NotPositiveDefinite, NotSymmetric, RankDeficient

_SYMMETRY_RTOL = 1e-12
LD_ALIGN = 32
F64 = torch.float64


class InstrumentationSink:
    """Lock-protected cost counters, same semantics as linalg.py:29-60."""

    def __init__(self):
        self._lock = threading.Lock()
        self.matvecs = 0
        self.precond_applies = 0
        self.gram_assemblies = 0

    def add_matvec(self, count: int = 1) -> None:
        with self._lock:
            self.matvecs += count

    def add_precond(self, count: int = 1) -> None:
        with self._lock:
            self.precond_applies += count

    def add_gram(self) -> None:
        with self._lock:
            self.gram_assemblies += 1

    def snapshot(self) -> dict:
        with self._lock:
            return {
                "matvecs": self.matvecs,
                "precond_applies": self.precond_applies,
                "gram_assemblies": self.gram_assemblies,
            }


# ---------------------------------------------------------------------------
# device buffers
# ---------------------------------------------------------------------------
def padded_ld(n: int) -> int:
    return max(LD_ALIGN, (int(n) + LD_ALIGN - 1) // LD_ALIGN * LD_ALIGN)


def empty_block(n: int, m: int, device, cap: int | None = None) -> torch.Tensor:
    """Uninitialised column-major n x m block (capacity ``cap`` columns)."""
    cap = max(int(m), int(cap or 0), 1)
    store = torch.empty((cap, padded_ld(n)), dtype=F64, device=device)
    return store[: int(m), : int(n)].t()


def block_capacity(B: torch.Tensor) -> int:
    """Columns the storage behind a block view can hold starting at its first
    column (0 when it is not a column-0 view of an empty_block store)."""
    base = B._base if B._base is not None else None
    if base is None or base.dim() != 2 or B.dim() != 2 or B.storage_offset() != base.storage_offset():
        return 0
    if int(B.shape[1]) > 1 and int(B.stride(1)) != int(base.shape[1]):
        return 0
    if int(B.shape[0]) > int(base.shape[1]):
        return 0
    return int(base.shape[0])


def grow_block(B: torch.Tensor, m: int) -> torch.Tensor | None:
    """View of the first ``m`` columns of B's storage (B's columns unchanged,
    columns beyond them uninitialised), or None when the capacity is short."""
    if block_capacity(B) < m:
        return None
    return B._base[: int(m), : int(B.shape[0])].t()


def zeros_block(n: int, m: int, device, cap: int | None = None) -> torch.Tensor:
    b = empty_block(n, m, device, cap)
    if m:
        b.zero_()
    return b


def block_ld(t: torch.Tensor) -> int:
    """Leading dimension of a column-major device block (n x m); for a single
    column any even value >= n is valid (it is never used for addressing)."""
    if t.dim() != 2:
        raise DimensionMismatch("expected a 2-D block")
    n, m = int(t.shape[0]), int(t.shape[1])
    if m > 1:
        return int(t.stride(1))
    ld = max(int(t.stride(1)), n, 1)
    return ld + (ld % 2)


def _is_device_block(t) -> bool:
    if not (isinstance(t, torch.Tensor) and t.is_cuda and t.dtype == F64 and t.dim() == 2):
        return False
    n, m = int(t.shape[0]), int(t.shape[1])
    if n > 1 and t.stride(0) != 1:
        return False
    if m > 1 and (t.stride(1) < n or t.stride(1) % 2 != 0):
        return False
    return t.data_ptr() % 16 == 0


def as_block(B, device=None) -> torch.Tensor:
    """Column-major, 16-byte aligned float64 device block view of ``B`` (n x m)."""
    if device is None:
        device = nat.require_device()
    if _is_device_block(B):
        return B
    if isinstance(B, torch.Tensor):
        src = B.detach()
        if src.dim() == 1:
            src = src[:, None]
    else:
        src = torch.from_numpy(np.atleast_2d(np.asarray(B, dtype=np.float64)))
        if np.asarray(B).ndim == 1:
            src = src.reshape(-1, 1)
    n, m = src.shape
    out = empty_block(n, m, device)
    if m and n:
        out.copy_(src.to(device=device, dtype=F64))
    return out


_STAGE_MIN_BYTES = 1 << 22
_STAGE_CHUNK = 32 << 20  # bytes per staging chunk of large uploads
_stage_pool = None
_stage_pool_lock = threading.Lock()


def _staging_pool():
    global _stage_pool
    with _stage_pool_lock:
        if _stage_pool is None:
            import concurrent.futures

            _stage_pool = concurrent.futures.ThreadPoolExecutor(max_workers=4, thread_name_prefix="rk-stage")
        return _stage_pool


def host_to_device(arr: np.ndarray, device, dtype=np.float64) -> torch.Tensor:
    """H2D copy of a host array. Large arrays are staged through pinned memory
    in 32 MB chunks copied by a small thread pool (np.copyto releases the GIL)
    and each chunk's asynchronous DMA is queued as soon as it is staged, so the
    host copy, the DMA and the device work of the launching thread overlap; the
    torch host allocator keeps the pinned block alive until the copies are done."""
    a = np.ascontiguousarray(np.asarray(arr, dtype=dtype))
    if a.nbytes < _STAGE_MIN_BYTES:
        return torch.from_numpy(a).to(device)
    tdtype = torch.from_numpy(a[:0]).dtype
    stage = torch.empty(a.shape, dtype=tdtype, pin_memory=True)
    out = torch.empty(a.shape, dtype=tdtype, device=device)
    flat_a, flat_s, flat_o = a.reshape(-1), stage.reshape(-1), out.reshape(-1)
    step = max(1, _STAGE_CHUNK // a.itemsize)
    bounds = [(i, min(i + step, flat_a.size)) for i in range(0, flat_a.size, step)]
    sv = flat_s.numpy()
    pool = _staging_pool()
    futures = [pool.submit(np.copyto, sv[lo:hi], flat_a[lo:hi]) for lo, hi in bounds]
    for (lo, hi), fut in zip(bounds, futures):
        fut.result()
        flat_o[lo:hi].copy_(flat_s[lo:hi], non_blocking=True)
    return out


def as_vector(x, device=None, copy: bool = False) -> torch.Tensor:
    """Contiguous float64 device vector."""
    if device is None:
        device = nat.require_device()
    if isinstance(x, torch.Tensor):
        t = x.detach().to(device=device, dtype=F64)
        if t.dim() != 1:
            t = t.reshape(-1)
        t = t.contiguous()
        return t.clone() if copy and t.data_ptr() == x.data_ptr() else t
    return host_to_device(np.asarray(x, dtype=np.float64).reshape(-1), device)


def to_numpy(t) -> np.ndarray:
    """Host copy of a device tensor (or passthrough for arrays)."""
    if isinstance(t, torch.Tensor):
        return t.detach().cpu().numpy()
    return np.asarray(t)


def column(B: torch.Tensor, j: int) -> torch.Tensor:
    return B[:, j]


def hstack_blocks(blocks, n: int, device, cap_extra: int = 0) -> torch.Tensor:
    """Column concatenation into a fresh block (np.hstack of threestage.py:365)."""
    m = sum(int(b.shape[1]) for b in blocks)
    out = empty_block(n, m, device, cap=m + cap_extra)
    at = 0
    for b in blocks:
        w = int(b.shape[1])
        if w:
            out[:, at : at + w].copy_(b)
        at += w
    return out


# ---------------------------------------------------------------------------
# CSR matrix
# ---------------------------------------------------------------------------
_pattern_cache_lock = threading.Lock()
_pattern_cache: list = []  # [(host rowptr, host col, _Pattern)]
_affine_cache_lock = threading.Lock()
_affine_cache: list = []  # [(host base, host delta, device, device base, device delta)]


def clear_upload_caches() -> None:
    """Forget the uploaded patterns and affine value parts (a first call in a fresh process)."""
    with _pattern_cache_lock:
        _pattern_cache.clear()
    with _affine_cache_lock:
        _affine_cache.clear()


def _affine_device_parts(base: np.ndarray, delta: np.ndarray, device):
    """Device copies of the two value arrays of an affine sequence
    (problems.AffineHostCsr), uploaded once per (base, delta) pair: every
    system's values are then formed on the GPU. The host arrays
    are kept referenced, so the identity test stays valid."""
    with _affine_cache_lock:
        for hb, hd, dv, db, dd in _affine_cache:
            if hb is base and hd is delta and dv == device:
                return db, dd
    db = host_to_device(base, device)
    dd = host_to_device(delta, device)
    torch.cuda.current_stream(device).synchronize()  # later systems read them from other streams
    with _affine_cache_lock:
        _affine_cache.insert(0, (base, delta, device, db, dd))
        del _affine_cache[2:]
    return db, dd
USE_BSR3 = os.environ.get("RK_BSR", "1") != "0"
DEVICE_SPDINV_MIN = int(os.environ.get("RK_DEVICE_SPDINV_MIN", "256"))
USE_SELL1 = os.environ.get("RK_SELL1", "1") != "0"
SELL1_MAX_ROW = 16      # scalar SELL for short rows (7-point stencils); longer rows keep lanes-per-row CSR
SELL1_MAX_PAD = 1.25    # ... and only when slices pad the pattern by at most 25%


SELL_SLICE = 32  # block rows per slice (one warp, one block row per lane)


class _Bsr3:
    """Sliced-ELL view of a 3x3-block pattern (SELL-32 of 3x3 blocks): slice
    offsets (in slots), the block column of every slot and the permutation that
    gathers CSR values into the slot-row value tiles (-1 = padding).
    ``nblk`` is the number of slots (real blocks + padding)."""

    def __init__(self, browptr, bcol, perm, nblk, nreal):
        self.browptr, self.bcol, self.perm, self.nblk = browptr, bcol, perm, int(nblk)
        self.nreal = int(nreal)


class _Sell1:
    """Scalar sliced-ELL view (SELL-32, one row per lane): slice offsets (in
    slots), the column of every slot and the permutation that gathers CSR
    values into slot order (-1 = padding)."""

    def __init__(self, sptr, scol, perm, nslot):
        self.sptr, self.scol, self.perm, self.nslot = sptr, scol, perm, int(nslot)


class _Pattern:
    def __init__(self, rowptr: torch.Tensor, col: torch.Tensor, bsr: _Bsr3 | None, sell: _Sell1 | None = None):
        self.rowptr, self.col, self.bsr, self.sell = rowptr, col, bsr, sell


def _sell1_from_host(rp: np.ndarray, ci: np.ndarray, n: int, device) -> _Sell1 | None:
    """Scalar SELL-32 view of a pattern with short rows: slot (s, t, lane) =
    sptr[s] + 32 t + lane holds entry t of row 32 s + lane; slices are padded
    to their widest row with value 0 and the lane's own row as column."""
    if n == 0 or ci.size == 0:
        return None
    rp = np.asarray(rp, dtype=np.int64)
    lens = np.diff(rp)
    if lens.max() > SELL1_MAX_ROW:
        return None
    nsl = (n + SELL_SLICE - 1) // SELL_SLICE
    lp = np.zeros(nsl * SELL_SLICE, dtype=np.int64)
    lp[:n] = lens
    width = lp.reshape(nsl, SELL_SLICE).max(axis=1)
    sptr = np.zeros(nsl + 1, dtype=np.int64)
    np.cumsum(width * SELL_SLICE, out=sptr[1:])
    nslot = int(sptr[-1])
    if nslot > SELL1_MAX_PAD * ci.size or nslot >= 2**31:
        return None
    row = np.repeat(np.arange(n, dtype=np.int64), lens)
    t_loc = np.arange(ci.size, dtype=np.int64) - rp[row]
    slot = sptr[row // SELL_SLICE] + t_loc * SELL_SLICE + row % SELL_SLICE
    sl_of = np.repeat(np.arange(nsl, dtype=np.int64), width * SELL_SLICE)
    pos = np.arange(nslot, dtype=np.int64) - sptr[sl_of]
    scol = np.minimum(sl_of * SELL_SLICE + pos % SELL_SLICE, n - 1)
    scol[slot] = np.asarray(ci, dtype=np.int64)
    perm = np.full(nslot, -1, dtype=np.int64)
    perm[slot] = np.arange(ci.size, dtype=np.int64)
    to = lambda arr: torch.from_numpy(np.ascontiguousarray(arr, dtype=np.int32)).to(device)  # noqa: E731
    return _Sell1(to(sptr), to(scol), to(perm), nslot)


def _bsr3_from_host(rp: np.ndarray, ci: np.ndarray, n: int, device) -> _Bsr3 | None:
    """Detect an exact 3x3 block structure (rows 3i..3i+2 share block columns,
    columns come in aligned triples) and build its device view; None if not."""
    if n == 0 or n % 3 or ci.size == 0 or ci.size % 9:
        return None
    rp = np.asarray(rp, dtype=np.int64)
    lens = np.diff(rp)
    if np.any(lens % 3):
        return None
    lr = lens.reshape(-1, 3)
    if not (np.array_equal(lr[:, 0], lr[:, 1]) and np.array_equal(lr[:, 0], lr[:, 2])):
        return None
    t = np.asarray(ci, dtype=np.int64).reshape(-1, 3)
    if not (np.all(t[:, 0] % 3 == 0) and np.all(t[:, 1] == t[:, 0] + 1) and np.all(t[:, 2] == t[:, 0] + 2)):
        return None
    nbr = n // 3
    nb_per = lr[:, 0] // 3
    browptr = np.zeros(nbr + 1, dtype=np.int64)
    np.cumsum(nb_per, out=browptr[1:])
    nblk = int(browptr[-1])
    b_row = np.repeat(np.arange(nbr, dtype=np.int64), nb_per)
    t_loc = np.arange(nblk, dtype=np.int64) - browptr[b_row]
    first = [rp[3 * b_row + a] for a in range(3)]            # CSR start of rows 3i+a
    bcol = t[first[0] // 3 + t_loc, 0] // 3
    for a in (1, 2):
        if not np.array_equal(t[first[a] // 3 + t_loc, 0] // 3, bcol):
            return None
    # slices of 32 block rows, each padded to its widest row; slot (s, t, lane)
    nsl = (nbr + SELL_SLICE - 1) // SELL_SLICE
    nb_pad = np.zeros(nsl * SELL_SLICE, dtype=np.int64)
    nb_pad[:nbr] = nb_per
    width = nb_pad.reshape(nsl, SELL_SLICE).max(axis=1)
    sptr = np.zeros(nsl + 1, dtype=np.int64)
    np.cumsum(width * SELL_SLICE, out=sptr[1:])
    nslot = int(sptr[-1])
    slot = sptr[b_row // SELL_SLICE] + t_loc * SELL_SLICE + (b_row % SELL_SLICE)
    scol = np.empty(nslot, dtype=np.int64)
    # padding slots point at a valid block column (the lane's own row, clamped)
    sl_of = np.repeat(np.arange(nsl, dtype=np.int64), width * SELL_SLICE)
    pos = np.arange(nslot, dtype=np.int64) - sptr[sl_of]
    scol[:] = np.minimum(sl_of * SELL_SLICE + pos % SELL_SLICE, nbr - 1)
    scol[slot] = bcol
    # values: per slot row (32 lanes) a contiguous 9 x 32 tile, entry e of slot s
    # at 9 * (s - s % 32) + 32 e + s % 32 (one 2304-byte stream per warp step)
    perm = np.full(9 * nslot, -1, dtype=np.int64)
    tile = 9 * (slot - slot % SELL_SLICE) + slot % SELL_SLICE
    for a in range(3):
        for c in range(3):
            perm[tile + SELL_SLICE * (3 * a + c)] = first[a] + 3 * t_loc + c
    to = lambda arr: torch.from_numpy(np.ascontiguousarray(arr, dtype=np.int32)).to(device)  # noqa: E731
    return _Bsr3(to(sptr), to(scol), to(perm), nslot, nblk)


PATTERN_ON_DEVICE = os.environ.get("RK_PATTERN", "device") != "host"


def _sell_view_on_device(dr: torch.Tensor, dc: torch.Tensor, n: int, nnz: int, bdim: int, device):
    """rk_sell_plan + rk_sell_fill: the (3x3-block or scalar) SELL-32 arrays of
    the uploaded pattern, bitwise those of _bsr3_from_host / _sell1_from_host;
    None when the pattern does not qualify (two scalar reads in between)."""
    rows = n // bdim
    nsl = (rows + SELL_SLICE - 1) // SELL_SLICE
    i32 = torch.int32
    len_ws = torch.empty(max(rows, 1), dtype=i32, device=device)
    sptr = torch.empty(nsl + 1, dtype=i32, device=device)
    flags = torch.zeros(2, dtype=torch.int64, device=device)  # [nslot, bad]
    bad = flags[1:].view(torch.int32)[:1]
    s = nat.stream_ptr(device)
    nat.check(nat.lib().rk_sell_plan(n, dr.data_ptr(), dc.data_ptr(), bdim, SELL1_MAX_ROW, len_ws.data_ptr(),
                                     sptr.data_ptr(), flags.data_ptr(), bad.data_ptr(), s), "sell plan")
    nslot, bad_flag = flags.tolist()
    if bad_flag & 0xFFFFFFFF:
        return None
    if bdim == 1 and (nslot > SELL1_MAX_PAD * nnz or nslot >= 2**31):
        return None
    scol = torch.empty(max(nslot, 1), dtype=i32, device=device)
    perm = torch.empty(max(bdim * bdim * nslot, 1), dtype=i32, device=device)
    nat.check(nat.lib().rk_sell_fill(n, dr.data_ptr(), dc.data_ptr(), bdim, len_ws.data_ptr(), sptr.data_ptr(),
                                     nslot, scol.data_ptr(), perm.data_ptr(), s), "sell fill")
    return sptr, scol, perm, nslot


def _bsr3_on_device(dr: torch.Tensor, dc: torch.Tensor, n: int, nnz: int, device) -> _Bsr3 | None:
    if n == 0 or n % 3 or nnz == 0 or nnz % 9:
        return None
    v = _sell_view_on_device(dr, dc, n, nnz, 3, device)
    return None if v is None else _Bsr3(v[0], v[1], v[2], v[3], nnz // 9)


def _sell1_on_device(dr: torch.Tensor, dc: torch.Tensor, n: int, nnz: int, device) -> _Sell1 | None:
    if n == 0 or nnz == 0:
        return None
    v = _sell_view_on_device(dr, dc, n, nnz, 1, device)
    return None if v is None else _Sell1(v[0], v[1], v[2], v[3])


def _pattern_known(rowptr: np.ndarray, col: np.ndarray, device) -> bool:
    """Same host pattern objects already uploaded (and checked) for this device."""
    with _pattern_cache_lock:
        return any(p.rowptr.device == device and hr is rowptr and hc is col for hr, hc, p in _pattern_cache)


def _device_pattern(rowptr: np.ndarray, col: np.ndarray, device, n: int) -> _Pattern:
    with _pattern_cache_lock:
        for hr, hc, p in _pattern_cache:
            if p.rowptr.device == device and (hr is rowptr or np.array_equal(hr, rowptr)) and (
                hc is col or (hc.shape == col.shape and np.array_equal(hc, col))
            ):
                return p
    dr = torch.from_numpy(np.ascontiguousarray(rowptr, dtype=np.int32)).to(device)
    dc = torch.from_numpy(np.ascontiguousarray(col, dtype=np.int32)).to(device)
    nnz = int(col.size)
    if PATTERN_ON_DEVICE:  # ms on the device instead of seconds of numpy per pattern
        bsr = _bsr3_on_device(dr, dc, n, nnz, device) if USE_BSR3 else None
        sell = _sell1_on_device(dr, dc, n, nnz, device) if (USE_SELL1 and bsr is None) else None
    else:
        bsr = _bsr3_from_host(rowptr, col, n, device) if USE_BSR3 else None
        sell = _sell1_from_host(rowptr, col, n, device) if (USE_SELL1 and bsr is None) else None
    p = _Pattern(dr, dc, bsr, sell)
    with _pattern_cache_lock:
        _pattern_cache.insert(0, (rowptr, col, p))
        del _pattern_cache[2:]
    return p


class SparseSpdMatrix:
    """SPD CSR matrix resident on the GPU (linalg.py:63-135).

    Both triangles are stored; indices are int32, values float64.
    Construction validates numerical symmetry to 1e-12 relative and a strictly
    positive diagonal on the device (linalg.py:105-119), raising
    ``NotSymmetric`` / ``NotPositiveDefinite(pivot)`` like the reference.
    Instances are immutable and safe to share across threads.
    """

    def __init__(self, n, row_offsets, col_indices, values, *, device=None, validate: bool = True,
                 lanes: int = 0, _pattern: "_Pattern | None" = None):
        self.n = int(n)
        dev = device if device is not None else nat.require_device()
        self.device = torch.device(dev)
        if _pattern is not None:
            pattern = _pattern
        elif isinstance(row_offsets, torch.Tensor) and isinstance(col_indices, torch.Tensor):
            rp = row_offsets.to(self.device, torch.int32).contiguous()
            ci = col_indices.to(self.device, torch.int32).contiguous()
            if rp.shape != (self.n + 1,):
                raise DimensionMismatch(
                    f"row_offsets must have length n+1={self.n + 1}, got {tuple(rp.shape)}"
                )
            pattern = _Pattern(rp, ci, None)
        else:
            rp_h = np.asarray(row_offsets)
            ci_h = np.asarray(col_indices)
            if rp_h.shape != (self.n + 1,):
                raise DimensionMismatch(
                    f"row_offsets must have length n+1={self.n + 1}, got {rp_h.shape}"
                )
            if ci_h.size and not _pattern_known(rp_h, ci_h, self.device) and not _rows_sorted(rp_h, ci_h):
                csr = scipy.sparse.csr_matrix(
                    (np.asarray(values, dtype=np.float64), ci_h, rp_h), shape=(self.n, self.n)
                )
                csr.sum_duplicates()
                rp_h, ci_h, values = csr.indptr, csr.indices, csr.data
            if rp_h.size and int(rp_h[-1]) >= 2**31:
                raise DimensionMismatch("nnz must be < 2^31 for the int32 device layout")
            pattern = _device_pattern(rp_h, ci_h, self.device, self.n)
        if isinstance(values, torch.Tensor):
            vals = values.to(self.device, F64).contiguous()
        else:
            vals = host_to_device(values, self.device)
        rp, ci = pattern.rowptr, pattern.col
        self._pattern = pattern
        self.rowptr = rp
        self.col = ci
        self.values = vals
        self.nnz = int(vals.numel())
        self.lanes = int(lanes)
        self._csr = nat.RkCsr(self.n, self.nnz, rp.data_ptr(), ci.data_ptr(), vals.data_ptr(), self.lanes, 0)
        self.bval = None
        bsr = pattern.bsr
        if bsr is not None and bsr.nreal * 9 == self.nnz:
            # 3x3 block values for the SpMV kernels (one gather per matrix)
            self.bval = torch.empty(9 * bsr.nblk, dtype=F64, device=self.device)
            nat.check(nat.lib().rk_bsr3_gather(bsr.nblk, bsr.perm.data_ptr(), vals.data_ptr(), self.bval.data_ptr(),
                                               nat.stream_ptr(self.device)), "bsr3 gather")
            c = self._csr
            c.nblk, c.browptr, c.bcol, c.bval = bsr.nblk, bsr.browptr.data_ptr(), bsr.bcol.data_ptr(), \
                self.bval.data_ptr()
            c.bdim = 3
        sell = getattr(pattern, "sell", None)
        if self.bval is None and sell is not None and self.lanes == 0:
            # scalar SELL-32 values for the SpMV / SpMM kernels (one gather per matrix)
            self.bval = torch.empty(sell.nslot, dtype=F64, device=self.device)
            nat.check(nat.lib().rk_sell_gather(sell.nslot, sell.perm.data_ptr(), vals.data_ptr(),
                                               self.bval.data_ptr(), nat.stream_ptr(self.device)), "sell gather")
            c = self._csr
            c.nblk, c.browptr, c.bcol, c.bval = sell.nslot, sell.sptr.data_ptr(), sell.scol.data_ptr(), \
                self.bval.data_ptr()
            c.bdim = 1
        self._diag = None
        self._dinv = None
        self._bad_diag = None
        if validate:
            self._validate()

    # -- construction helpers (linalg.py:86-103) ---------------------------
    @classmethod
    def from_scipy(cls, mat, **kw) -> "SparseSpdMatrix":
        csr = scipy.sparse.csr_matrix(mat).astype(np.float64)
        csr.sum_duplicates()
        return cls(csr.shape[0], csr.indptr, csr.indices, csr.data, **kw)

    @classmethod
    def from_dense(cls, mat, **kw) -> "SparseSpdMatrix":
        if isinstance(mat, torch.Tensor):
            mat = mat.detach().cpu().numpy()
        csr = scipy.sparse.csr_matrix(np.asarray(mat, dtype=np.float64))
        return cls(csr.shape[0], csr.indptr, csr.indices, csr.data, **kw)

    @classmethod
    def identity(cls, n: int, **kw) -> "SparseSpdMatrix":
        return cls.from_scipy(scipy.sparse.identity(n, format="csr"), **kw)

    @classmethod
    def from_diagonal(cls, diag, **kw) -> "SparseSpdMatrix":
        return cls.from_scipy(scipy.sparse.diags(np.asarray(diag, dtype=np.float64), format="csr"), **kw)

    @classmethod
    def from_host(cls, A, **kw) -> "SparseSpdMatrix":
        """Upload any CSR-like host matrix: this class, the reference's
        SparseSpdMatrix (n, row_offsets, col_indices, values), or scipy."""
        if isinstance(A, SparseSpdMatrix):
            return A
        affine = getattr(A, "affine", None)
        if affine is not None:
            # values = base + coef * delta formed on the device with numpy's two
            # roundings (rk_axpby: fl(fl(coef * delta) + base)); only the two
            # parts ever cross PCIe, once per sequence
            base, delta, coef = affine
            dev = torch.device(kw["device"]) if kw.get("device") is not None else nat.require_device()
            db, dd = _affine_device_parts(base, delta, dev)
            vals = db.clone()
            axpby(float(coef), dd, 1.0, vals)
            return cls(A.n, A.row_offsets, A.col_indices, vals, **kw)
        if all(hasattr(A, a) for a in ("n", "row_offsets", "col_indices", "values")):
            return cls(A.n, A.row_offsets, A.col_indices, A.values, **kw)
        if scipy.sparse.issparse(A):
            return cls.from_scipy(A, **kw)
        return cls.from_dense(A, **kw)

    def with_values(self, values, validate: bool = True) -> "SparseSpdMatrix":
        """Same sparsity pattern, new values (per-system refresh of a sequence)."""
        return SparseSpdMatrix(self.n, self.rowptr, self.col, values, device=self.device, validate=validate,
                               lanes=self.lanes, _pattern=self._pattern)

    def _validate(self) -> None:
        s = nat.scratch(self.device)
        ws = s.workspace(nat.lib().rk_reduce_workspace_doubles(max(self.n, 1), 8))
        out = torch.zeros(2, dtype=F64, device=self.device)
        bad = torch.empty(1, dtype=torch.int64, device=self.device)
        diag = torch.empty(self.n, dtype=F64, device=self.device)
        dinv = torch.empty(self.n, dtype=F64, device=self.device)
        st = nat.stream_ptr(self.device)
        if self.nnz:
            nat.check(nat.lib().rk_csr_asymmetry(self._csr, out.data_ptr(), ws.data_ptr(), ws.numel(),
                                                 s.tickets.data_ptr(), st), "SparseSpdMatrix validate")
        nat.check(nat.lib().rk_csr_diagonal(self._csr, diag.data_ptr(), dinv.data_ptr(), bad.data_ptr(), st),
                  "SparseSpdMatrix diagonal")
        worst, scale = (float(v) for v in out.cpu())
        if scale > 0 and worst > _SYMMETRY_RTOL * scale:
            raise NotSymmetric(f"matrix asymmetry {worst:.3e} exceeds {_SYMMETRY_RTOL:.0e} * {scale:.3e}")
        b = int(bad.cpu())
        self._diag, self._dinv = diag, dinv
        self._bad_diag = b if 0 <= b < self.n else -1
        if self._bad_diag >= 0:
            d = float(diag[self._bad_diag].cpu())
            raise NotPositiveDefinite(f"diagonal entry {self._bad_diag} is {d!r}, must be > 0",
                                      pivot=self._bad_diag)

    def _diagonals(self):
        if self._diag is None:
            bad = torch.empty(1, dtype=torch.int64, device=self.device)
            diag = torch.empty(self.n, dtype=F64, device=self.device)
            dinv = torch.empty(self.n, dtype=F64, device=self.device)
            nat.check(nat.lib().rk_csr_diagonal(self._csr, diag.data_ptr(), dinv.data_ptr(), bad.data_ptr(),
                                                nat.stream_ptr(self.device)), "diagonal")
            b = int(bad.cpu())
            self._diag, self._dinv = diag, dinv
            self._bad_diag = b if 0 <= b < self.n else -1
        return self._diag, self._dinv, self._bad_diag

    @property
    def shape(self):
        return (self.n, self.n)

    @property
    def csr(self) -> nat.RkCsr:
        return self._csr

    def diagonal(self) -> torch.Tensor:
        return self._diagonals()[0]

    def to_scipy(self) -> scipy.sparse.csr_matrix:
        return scipy.sparse.csr_matrix(
            (self.values.cpu().numpy(), self.col.cpu().numpy(), self.rowptr.cpu().numpy()),
            shape=(self.n, self.n),
        )

    def to_dense(self) -> np.ndarray:
        return self.to_scipy().toarray()

    def matvec(self, x, sink: InstrumentationSink | None = None) -> torch.Tensor:
        return spmv(self, x, sink)


def _rows_sorted(rp: np.ndarray, ci: np.ndarray) -> bool:
    if ci.size < 2:
        return True
    inc = ci[1:] > ci[:-1]  # one pass, no widened copy (0.32 s -> 0.06 s for the 63.7M entries of C3)
    # a descent is allowed only where a new row starts
    rs = np.asarray(rp[1:-1], dtype=np.int64) - 1
    rs = rs[(rs >= 0) & (rs < ci.size - 1)]
    inc[rs] = True
    return bool(inc.all())


def as_matrix(A) -> SparseSpdMatrix:
    return A if isinstance(A, SparseSpdMatrix) else SparseSpdMatrix.from_host(A)


# ---------------------------------------------------------------------------
# kernels (linalg.py:138-174)
# ---------------------------------------------------------------------------
def spmv_into(A: SparseSpdMatrix, x: torch.Tensor, y: torch.Tensor) -> torch.Tensor:
    nat.check(nat.lib().rk_spmv(A.csr, x.data_ptr(), y.data_ptr(), nat.stream_ptr(A.device)), "spmv")
    return y


def spmv(A: SparseSpdMatrix, x, sink: InstrumentationSink | None = None) -> torch.Tensor:
    """y = A x on the device (linalg.py:138-148); counts one matvec."""
    A = as_matrix(A)
    xd = as_vector(x, A.device)
    if xd.shape[0] != A.n:
        raise DimensionMismatch(f"matvec: matrix is {A.n}x{A.n}, vector has length {xd.shape[0]}")
    if sink is not None:
        sink.add_matvec()
    y = torch.empty(A.n, dtype=F64, device=A.device)
    return spmv_into(A, xd, y)


def spmm(A: SparseSpdMatrix, B: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
    """A B for a column-major block (scipy csr_matvecs, linalg.py:173); no counting."""
    m = int(B.shape[1])
    if out is None:
        out = empty_block(A.n, m, A.device)
    if m:
        nat.check(nat.lib().rk_spmm(A.csr, m, B.data_ptr(), block_ld(B), out.data_ptr(), block_ld(out),
                                    nat.stream_ptr(A.device)), "spmm")
    return out


def gram(X: torch.Tensor, Y: torch.Tensor) -> torch.Tensor:
    """X' Y (m1 x m2) with the DMMA split-K kernel; returned as an (m1, m2) view."""
    n, m1 = X.shape
    n2, m2 = Y.shape
    if n != n2:
        raise DimensionMismatch("gram: row counts differ")
    dev = X.device
    store = torch.empty((max(m2, 1), max(m1, 1)), dtype=F64, device=dev)
    G = store[:m2, :m1].t()
    if m1 and m2:
        s = nat.scratch(dev)
        need = nat.lib().rk_gram_workspace_doubles(n, m1, m2)
        ws = s.workspace(max(need, 1))
        nat.check(nat.lib().rk_gram(n, m1, X.data_ptr(), block_ld(X), m2, Y.data_ptr(), block_ld(Y),
                                    G.data_ptr(), max(m1, 1), ws.data_ptr(), ws.numel(), nat.stream_ptr(dev)),
                  "gram")
    return G


class UpperGram:
    """Symmetric Gram Z'AZ kept on the device as its upper triangle.

    ``store`` is an (m, m) tensor read as a column-major matrix (ld = m) whose
    upper tiles were produced by rk_gram_upper(_split); ``scale`` (device vector
    or None) multiplies column b of the triangle. ``np.asarray`` gives the full
    mirrored host matrix (the reference's ``gram_zz``)."""

    def __init__(self, store: torch.Tensor, scale: torch.Tensor | None):
        self.store = store
        self.scale = scale
        self.m = int(store.shape[0])

    def __array__(self, dtype=None, copy=None):
        G = self.store.cpu().numpy().T.copy()  # G[a, b], a row, b column
        if self.scale is not None:
            G = G * self.scale.cpu().numpy()[None, :]
        iu = np.triu_indices(self.m, 1)
        G[(iu[1], iu[0])] = G[iu]
        return G if dtype is None else G.astype(dtype)

    @property
    def shape(self):
        return (self.m, self.m)


def symmetric_gram_from_products(Z: torch.Tensor, products, col_scale=None, single_launch: bool = True) -> UpperGram:
    """Z'AZ from cached products A Z (no SpMM).

    ``products`` is a list of (AZ_block, col_off): AZ_block holds A applied to
    columns [col_off, col_off + w) of Z (the stage-1 product A W and the stored
    A p_k of the PCG run); two contiguous segments covering Z go to one
    rk_gram_upper_split launch. Only the upper tiles are computed
    (rk_gram_upper, half the flops of the reference's full B'(AB));
    ``col_scale`` (length m or None) rescales column j (products of unscaled
    directions)."""
    n, m = Z.shape
    dev = Z.device
    store = torch.zeros((max(m, 1), max(m, 1)), dtype=F64, device=dev)  # column-major m x m (ld = m)
    s = nat.scratch(dev)
    scale = as_vector(col_scale, dev) if col_scale is not None else None
    segs = [(AB, off) for AB, off in products if int(AB.shape[1])]
    if single_launch and len(segs) <= 2 and segs and segs[0][1] == 0 and sum(int(AB.shape[1]) for AB, _ in segs) == m and \
            (len(segs) == 1 or segs[1][1] == int(segs[0][0].shape[1])):
        # A Z covered by at most two contiguous segments: one launch whose tiles
        # sit on the diagonal of the whole m x m triangle
        Y1 = segs[0][0]
        Y2 = segs[1][0] if len(segs) == 2 else Y1
        c1 = int(Y1.shape[1])
        ws = s.workspace(max(nat.lib().rk_gram_upper_workspace_doubles(n, m, m, 0), 1))
        nat.check(nat.lib().rk_gram_upper_split(n, m, Z.data_ptr(), block_ld(Z), c1, Y1.data_ptr(), block_ld(Y1),
                                                Y2.data_ptr(), block_ld(Y2), store.data_ptr(), m, ws.data_ptr(),
                                                ws.numel(), nat.stream_ptr(dev)), "gram_upper_split")
        return UpperGram(store[:m, :m], scale)
    for AB, off in products:
        w = int(AB.shape[1])
        if w == 0:
            continue
        ws = s.workspace(max(nat.lib().rk_gram_upper_workspace_doubles(n, m, w, off), 1))
        Gblk = store[off : off + w]  # rows of the row-major store = columns of G
        nat.check(nat.lib().rk_gram_upper(n, m, Z.data_ptr(), block_ld(Z), w, AB.data_ptr(), block_ld(AB), off,
                                          Gblk.data_ptr(), m, ws.data_ptr(), ws.numel(), nat.stream_ptr(dev)),
                  "gram_upper")
    return UpperGram(store[:m, :m], scale)


def gemm_nn(S: torch.Tensor, C, out: torch.Tensor | None = None) -> torch.Tensor:
    """S (N x s) @ C (s x y) with the DMMA kernel (pod.py:91-93)."""
    n, s = S.shape
    Cd = as_block(C, S.device)
    if Cd.shape[0] != s:
        raise DimensionMismatch("gemm_nn: inner dimensions differ")
    y = int(Cd.shape[1])
    if out is None:
        out = empty_block(n, y, S.device)
    if y and n:
        if s == 0:
            out.zero_()
        else:
            nat.check(nat.lib().rk_gemm_nn(n, s, y, S.data_ptr(), block_ld(S), Cd.data_ptr(), block_ld(Cd),
                                           out.data_ptr(), block_ld(out), nat.stream_ptr(S.device)), "gemm_nn")
    return out


def gemv_t(B: torch.Tensor, x: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
    """B' x (krylov.py:156 `cross.T @ z`), deterministic split reduction."""
    n, m = B.shape
    dev = B.device
    if out is None:
        out = torch.empty(m, dtype=F64, device=dev)
    if m:
        s = nat.scratch(dev)
        ws = s.workspace(nat.lib().rk_reduce_workspace_doubles(max(n, 1), m))
        nat.check(nat.lib().rk_gemv_t(n, m, B.data_ptr(), block_ld(B), x.data_ptr(), out.data_ptr(),
                                      ws.data_ptr(), ws.numel(), nat.stream_ptr(dev)), "gemv_t")
    return out


def gemv_n(B: torch.Tensor, c, y0: torch.Tensor | None = None, op: int = 0,
           out: torch.Tensor | None = None) -> torch.Tensor:
    """B c (op 0), y0 + B c (op 1), y0 - B c (op 2) (krylov.py:291,326)."""
    n, m = B.shape
    dev = B.device
    cd = as_vector(c, dev)
    if out is None:
        out = torch.empty(n, dtype=F64, device=dev)
    if n:
        nat.check(nat.lib().rk_gemv_n(n, m, B.data_ptr(), block_ld(B), cd.data_ptr() if m else None,
                                      y0.data_ptr() if y0 is not None else None, out.data_ptr(), op,
                                      nat.stream_ptr(dev)), "gemv_n")
    return out


def axpby(a: float, x: torch.Tensor, b: float, y: torch.Tensor) -> torch.Tensor:
    """y <- fl(fl(a x) + fl(b y)) in place (numpy's `y + a * x` when b = 1)."""
    if y.numel():
        nat.check(nat.lib().rk_axpby(int(y.numel()), float(a), x.data_ptr(), float(b), y.data_ptr(),
                                     nat.stream_ptr(y.device)), "axpby")
    return y


def dot(x: torch.Tensor, y: torch.Tensor) -> torch.Tensor:
    """x'y as a 1-element device tensor (deterministic)."""
    dev = x.device
    s = nat.scratch(dev)
    ws = s.workspace(nat.lib().rk_reduce_workspace_doubles(max(int(x.numel()), 1), 1))
    out = torch.empty(1, dtype=F64, device=dev)
    nat.check(nat.lib().rk_dot(int(x.numel()), x.data_ptr(), y.data_ptr(), out.data_ptr(), ws.data_ptr(),
                               ws.numel(), s.tickets.data_ptr(), nat.stream_ptr(dev)), "dot")
    return out


def norm(x: torch.Tensor) -> float:
    """||x||_2 = sqrt(x'x) (numpy.linalg.norm for 1-D input)."""
    return float(np.sqrt(float(dot(x, x).cpu())))


def scale_columns(V: torch.Tensor, s, out: torch.Tensor | None = None) -> torch.Tensor:
    """V[:, j] / s[j] (threestage.py:483)."""
    n, m = V.shape
    dev = V.device
    sd = as_vector(s, dev)
    if out is None:
        out = empty_block(n, m, dev)
    if n and m:
        nat.check(nat.lib().rk_scale_columns(n, m, V.data_ptr(), block_ld(V), sd.data_ptr(), out.data_ptr(),
                                             block_ld(out), nat.stream_ptr(dev)), "scale_columns")
    return out


def weighted_inner(A: SparseSpdMatrix, x, y) -> float:
    """A-weighted inner product x'Ay (linalg.py:151-157)."""
    A = as_matrix(A)
    xd = as_vector(x, A.device)
    yd = as_vector(y, A.device)
    if xd.shape[0] != A.n or yd.shape[0] != A.n:
        raise DimensionMismatch("weighted_inner: dimension mismatch")
    Ay = spmv(A, yd)
    return float(dot(xd, Ay).cpu())


def assemble_gram(A: SparseSpdMatrix, B, sink: InstrumentationSink | None = None, out: torch.Tensor | None = None):
    """(B'AB, AB) (linalg.py:160-174): SpMM then the DMMA Gram; counts one gram
    assembly plus one matvec per column, exactly like the reference. ``out``
    (N x m device block) receives AB instead of a fresh allocation."""
    A = as_matrix(A)
    Bd = as_block(B, A.device)
    if Bd.shape[0] != A.n:
        raise DimensionMismatch("assemble_gram: basis rows must match matrix dimension")
    if sink is not None:
        sink.add_gram()
        sink.add_matvec(int(Bd.shape[1]))
    AB = spmm(A, Bd, out=out)
    return gram(Bd, AB), AB


def assemble_gram_blocked(A: SparseSpdMatrix, B, sink: InstrumentationSink | None = None,
                          block: int = 256, events: list | None = None) -> UpperGram:
    """B'AB (linalg.py:160-174) without materialising AB: A B is formed ``block``
    columns at a time (SpMM into one reusable N x block buffer) and each column
    block of the Gram's upper triangle is contracted against the leading columns
    of B it needs (rk_gram_upper). Peak extra memory is N x block instead of
    N x m (C5 at m = 2048: 8.6 GB instead of 68.7 GB), and only the triangle is
    computed (the reference symmetrises anyway, pod.py:129). Charged exactly as
    assemble_gram: one gram assembly plus one matvec per column. ``events``
    (measurement only) collects (spmm_start, gram_start, gram_end) CUDA events
    per column block on the launching stream."""
    A = as_matrix(A)
    Bd = as_block(B, A.device)
    n, m = int(Bd.shape[0]), int(Bd.shape[1])
    if n != A.n:
        raise DimensionMismatch("assemble_gram: basis rows must match matrix dimension")
    if sink is not None:
        sink.add_gram()
        sink.add_matvec(m)
    dev = A.device
    store = torch.zeros((max(m, 1), max(m, 1)), dtype=F64, device=dev)  # column-major m x m (ld = m)
    if m == 0:
        return UpperGram(store[:0, :0], None)
    block = max(1, min(int(block), m))
    AB = empty_block(n, block, dev)
    s = nat.scratch(dev)
    lib = nat.lib()
    for j0 in range(0, m, block):
        w = min(block, m - j0)
        ABj = AB[:, :w]
        if events is not None:
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
            events.append(ev)
            ev[0].record()
        spmm(A, Bd[:, j0 : j0 + w], out=ABj)
        if events is not None:
            ev[1].record()
        rows = j0 + w  # rows of G at or above the diagonal of this column block
        ws = s.workspace(max(lib.rk_gram_upper_workspace_doubles(n, rows, w, j0), 1))
        Gblk = store[j0 : j0 + w]  # rows of the row-major store = columns of G
        nat.check(lib.rk_gram_upper(n, rows, Bd.data_ptr(), block_ld(Bd), w, ABj.data_ptr(), block_ld(ABj), j0,
                                    Gblk.data_ptr(), m, ws.data_ptr(), ws.numel(), nat.stream_ptr(dev)),
                  "gram_upper")
        if events is not None:
            ev[2].record()
    return UpperGram(store[:m, :m], None)


# ---------------------------------------------------------------------------
# small dense algebra (host LAPACK, as the reference)
# ---------------------------------------------------------------------------
@dataclass
class DenseBasis:
    """Block of length-n columns with optional Gram metadata (linalg.py:177-205)."""

    columns: object
    gram_diag: np.ndarray | None = None

    def __post_init__(self):
        if not isinstance(self.columns, torch.Tensor):
            self.columns = np.atleast_2d(np.asarray(self.columns, dtype=np.float64))
        if self.gram_diag is not None:
            self.gram_diag = np.asarray(self.gram_diag, dtype=np.float64)
            if self.gram_diag.shape != (self.columns.shape[1],):
                raise DimensionMismatch("gram_diag length must equal column count")

    @property
    def n(self) -> int:
        return int(self.columns.shape[0])

    @property
    def m(self) -> int:
        return int(self.columns.shape[1])

    @classmethod
    def empty(cls, n: int) -> "DenseBasis":
        return cls(np.zeros((n, 0)))


def as_columns(basis):
    if basis is None:
        raise DimensionMismatch("expected a basis, got None")
    if isinstance(basis, DenseBasis):
        return basis.columns
    return basis


class DenseLowerTriangular:
    """Packed lower-triangular Cholesky factor L with G = L L' (linalg.py:217-247).

    Kept on the host (it is w x w); ``device()`` returns a cached column-major
    device copy for the fused PCG kernels."""

    def __init__(self, entries_packed, m: int):
        self.m = int(m)
        self.entries = np.asarray(entries_packed, dtype=np.float64)
        if self.entries.shape != (self.m * (self.m + 1) // 2,):
            raise DimensionMismatch("packed entry count must be m(m+1)/2")
        self._full = np.zeros((self.m, self.m))
        self._full[np.tril_indices(self.m)] = self.entries
        if self.m and np.any(np.diag(self._full) <= 0.0):
            raise NotPositiveDefinite("lower-triangular factor must have positive diagonal")
        self._dev = {}

    @classmethod
    def from_full(cls, L) -> "DenseLowerTriangular":
        L = np.asarray(L, dtype=np.float64)
        return cls(L[np.tril_indices(L.shape[0])], L.shape[0])

    def full(self) -> np.ndarray:
        return self._full.copy()

    def device(self, device) -> torch.Tensor:
        key = (device.type, device.index)
        t = self._dev.get(key)
        if t is None:
            t = self._dev[key] = as_block(self._full, device)
        return t

    def device_inverse(self, device) -> torch.Tensor:
        """Column-major device copy of L^{-1} (LAPACK dtrtri): the fused PCG
        kernels apply F^{-1} = L^{-T} L^{-1} as two triangular mat-vecs."""
        key = ("inv", device.type, device.index)
        t = self._dev.get(key)
        if t is None:
            Linv, info = scipy.linalg.lapack.dtrtri(self._full, lower=1)
            if info != 0:
                raise NotPositiveDefinite("singular Cholesky factor", pivot=int(info - 1) if info > 0 else None)
            t = self._dev[key] = as_block(np.tril(Linv), device)
        return t

    def device_spd_inverse(self, device) -> torch.Tensor:
        """Column-major device copy of F^{-1} = L^{-T} L^{-1} (host dtrtri, then a
        w x w product; from DEVICE_SPDINV_MIN columns on, cuSOLVER potri on the
        device -- at C4's w ~ 3000 the host route takes seconds per system):
        the fused kernels apply it as one symmetric mat-vec."""
        key = ("spdinv", device.type, device.index)
        t = self._dev.get(key)
        if t is None and self.m >= DEVICE_SPDINV_MIN:
            L = self.device(device)  # column-major, lower
            F = torch.cholesky_inverse(L, upper=False)
            if not bool(torch.isfinite(F).all()):
                raise NotPositiveDefinite("singular Cholesky factor")
            t = self._dev[key] = as_block(F, device)
        if t is None:
            Linv, info = scipy.linalg.lapack.dtrtri(self._full, lower=1)
            if info != 0:
                raise NotPositiveDefinite("singular Cholesky factor", pivot=int(info - 1) if info > 0 else None)
            Linv = np.tril(Linv)
            t = self._dev[key] = as_block(Linv.T @ Linv, device)
        return t

    def device_form(self, device):
        """(F^{-1}, w, sqd=None, full=True) in the form the fused PCG kernels take."""
        return (self.device_spd_inverse(device) if self.m else None, self.m, None, True)

    def solve_lower(self, rhs):
        return scipy.linalg.solve_triangular(self._full, np.asarray(rhs, dtype=np.float64), lower=True)

    def solve_upper(self, rhs):
        return scipy.linalg.solve_triangular(self._full, np.asarray(rhs, dtype=np.float64), lower=True, trans="T")

    def solve_spd(self, rhs):
        return self.solve_upper(self.solve_lower(rhs))


def _host(G) -> np.ndarray:
    return to_numpy(G) if isinstance(G, torch.Tensor) else np.asarray(G, dtype=np.float64)


def dense_cholesky(G) -> DenseLowerTriangular:
    """LAPACK dpotrf of a (host copy of a) small SPD matrix (linalg.py:250-267)."""
    G = np.asarray(_host(G), dtype=np.float64)
    if G.ndim != 2 or G.shape[0] != G.shape[1]:
        raise DimensionMismatch("dense_cholesky: matrix must be square")
    if G.shape[0] == 0:
        return DenseLowerTriangular(np.zeros(0), 0)
    L, info = scipy.linalg.lapack.dpotrf(G, lower=1, clean=1, overwrite_a=0)
    if info > 0:
        raise NotPositiveDefinite(f"leading minor of order {info} is not positive definite", pivot=int(info - 1))
    if info < 0:
        raise DimensionMismatch(f"dpotrf: illegal argument {-info}")
    return DenseLowerTriangular.from_full(L)


def symmetric_evd(G):
    """eigh with eigenvalues descending (linalg.py:270-280), host LAPACK dsyevd."""
    G = np.asarray(_host(G), dtype=np.float64)
    try:
        w, V = np.linalg.eigh(G)
    except np.linalg.LinAlgError as exc:
        raise IterationLimit(f"symmetric EVD did not converge: {exc}") from exc
    return w[::-1].copy(), V[:, ::-1].copy()


def generalized_symmetric_evd(K, Mmat):
    """K G = Mmat G diag(w) for symmetric K and SPD Mmat (linalg.py:293-307):
    host LAPACK (scipy eigh, dsygvd) on the small z x z pair, eigenvalues
    descending, eigenvectors Mmat-orthonormal."""
    K = np.asarray(_host(K), dtype=np.float64)
    Mmat = np.asarray(_host(Mmat), dtype=np.float64)
    if K.shape != Mmat.shape:
        raise DimensionMismatch("generalized EVD: operand shapes differ")
    try:
        w, G = scipy.linalg.eigh(K, Mmat)
    except (np.linalg.LinAlgError, scipy.linalg.LinAlgError) as exc:
        raise NotPositiveDefinite(f"mass matrix is not SPD: {exc}") from exc
    return w[::-1].copy(), G[:, ::-1].copy()


def thin_svd(B):
    B = np.atleast_2d(_host(B))
    try:
        U, s, Vt = np.linalg.svd(B, full_matrices=False)
    except np.linalg.LinAlgError as exc:
        raise IterationLimit(f"SVD did not converge: {exc}") from exc
    return U, s, Vt.T


def _orthonormal_basis(B: np.ndarray, label: str) -> np.ndarray:
    if B.shape[1] == 0:
        return B
    U, s, _ = np.linalg.svd(B, full_matrices=False)
    if s[0] == 0.0 or s[-1] <= max(B.shape) * np.finfo(float).eps * s[0]:
        raise RankDeficient(f"{label} basis is rank deficient")
    return U


def principal_angle_distance(U, V) -> float:
    """sin of the largest principal angle between range(U) and range(V)."""
    Qu = _orthonormal_basis(np.atleast_2d(_host(as_columns(U))), "first")
    Qv = _orthonormal_basis(np.atleast_2d(_host(as_columns(V))), "second")
    if Qu.shape[0] != Qv.shape[0]:
        raise DimensionMismatch("principal_angle_distance: ambient dimensions differ")
    if Qu.shape[1] == 0:
        return 0.0
    if Qv.shape[1] == 0:
        return 1.0
    d = float(np.linalg.norm(Qu - Qv @ (Qv.T @ Qu), 2))
    return min(max(d, 0.0), 1.0)
