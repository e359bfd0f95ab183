"""ctypes binding of the C-ABI library ``libpodcg.so`` (include/podcg.h).

The product path has no CPU fallback: if the shared library is missing or no
CUDA device is present, every device entry point raises ``NativeUnavailable``.
Pointers handed to the library are ``torch.Tensor.data_ptr()`` of CUDA
tensors; the stream is torch's current stream on the tensor's device.
"""

from __future__ import annotations

import ctypes
import os
import threading

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("RK_LIB") or os.path.join(_HERE, "_lib", "libpodcg.so")

c_i64 = ctypes.c_int64
c_i32 = ctypes.c_int32
c_dbl = ctypes.c_double
c_vp = ctypes.c_void_p


class NativeUnavailable(RuntimeError):
    """The CUDA extension (libpodcg.so) or a CUDA device is unavailable."""


class RkCsr(ctypes.Structure):
    _fields_ = [
        ("n", c_i64),
        ("nnz", c_i64),
        ("rowptr", c_vp),
        ("col", c_vp),
        ("val", c_vp),
        ("lanes", c_i32),
        ("bdim", c_i32),
        ("nblk", c_i64),
        ("browptr", c_vp),
        ("bcol", c_vp),
        ("bval", c_vp),
    ]


class RkPcgState(ctypes.Structure):
    _fields_ = [
        ("k", c_i64),
        ("done", c_i64),
        ("status", c_i64),
        ("bd_iter", c_i64),
        ("rz", c_dbl),
        ("gamma", c_dbl),
        ("pp", c_dbl),
        ("alpha", c_dbl),
        ("rr", c_dbl),
        ("beta", c_dbl),
        ("threshold", c_dbl),
        ("rz_next", c_dbl),
    ]


class RkSsorPlan(ctypes.Structure):
    _fields_ = [
        ("dw", c_vp),
        ("d", c_vp),
        ("work", c_vp),
        ("flags", c_vp),
        ("counters", c_vp),
        ("order_fwd", c_vp),
        ("order_bwd", c_vp),
        ("epoch", c_i32),
    ]


class RkPcgPlan(ctypes.Structure):
    _fields_ = [
        ("n", c_i64),
        ("A", RkCsr),
        ("x", c_vp),
        ("r", c_vp),
        ("r2", c_vp),
        ("z", c_vp),
        ("V", c_vp),
        ("ldv", c_i64),
        ("vcap", c_i64),
        ("AV", c_vp),
        ("ldav", c_i64),
        ("dinv", c_vp),
        ("m", c_i64),
        ("B", c_vp),
        ("ldb", c_i64),
        ("cross", c_vp),
        ("ldc", c_i64),
        ("L", c_vp),
        ("ldl", c_i64),
        ("wchol", c_i64),
        ("sqd", c_vp),
        ("mu", c_vp),
        ("coef", c_vp),
        ("st", c_vp),
        ("alpha_h", c_vp),
        ("gamma_h", c_vp),
        ("rz_h", c_vp),
        ("res_h", c_vp),
        ("partials", c_vp),
        ("partials_len", c_i64),
        ("tickets", c_vp),
        ("mode", c_i32),
        ("linv_full", c_i32),
    ]


STATE_BYTES = ctypes.sizeof(RkPcgState)
PCG_TICKETS = 272  # RK_PCG_TICKETS (include/podcg.h)

_SIGNATURES = {
    "rk_last_error": (ctypes.c_char_p, []),
    "rk_device_sm_count": (c_i32, []),
    "rk_pcg_workspace_doubles": (c_i64, [c_i64, c_i64, c_i64]),
    "rk_reduce_workspace_doubles": (c_i64, [c_i64, c_i64]),
    "rk_gram_workspace_doubles": (c_i64, [c_i64, c_i64, c_i64]),
    "rk_gram_upper_workspace_doubles": (c_i64, [c_i64, c_i64, c_i64, c_i64]),
    "rk_pcg_entry": (c_i32, [ctypes.POINTER(RkPcgPlan), c_vp]),
    "rk_pcg_steps": (c_i32, [ctypes.POINTER(RkPcgPlan), c_i32, c_i64, c_vp]),
    "rk_pcg_entry_ssor": (c_i32, [ctypes.POINTER(RkPcgPlan), ctypes.POINTER(RkSsorPlan), c_vp]),
    "rk_pcg_steps_ssor": (c_i32, [ctypes.POINTER(RkPcgPlan), ctypes.POINTER(RkSsorPlan), c_i32, c_i64, c_vp]),
    "rk_pcg_cluster_eligible": (c_i32, [ctypes.POINTER(RkPcgPlan)]),
    "rk_pcg_cluster_max_rows": (c_i64, []),
    "rk_pcg_run_cluster": (c_i32, [ctypes.POINTER(RkPcgPlan), c_i64, c_vp]),
    "rk_pcg_curvature": (c_i32, [ctypes.POINTER(RkPcgPlan), c_vp]),
    "rk_pcg_update": (c_i32, [ctypes.POINTER(RkPcgPlan), c_vp]),
    "rk_pcg_direction": (c_i32, [ctypes.POINTER(RkPcgPlan), c_i64, c_vp]),
    "rk_spmv": (c_i32, [ctypes.POINTER(RkCsr), c_vp, c_vp, c_vp]),
    "rk_spmm": (c_i32, [ctypes.POINTER(RkCsr), c_i64, c_vp, c_i64, c_vp, c_i64, c_vp]),
    "rk_csr_diagonal": (c_i32, [ctypes.POINTER(RkCsr), c_vp, c_vp, c_vp, c_vp]),
    "rk_csr_asymmetry": (c_i32, [ctypes.POINTER(RkCsr), c_vp, c_vp, c_i64, c_vp, c_vp]),
    "rk_sell_gather": (c_i32, [c_i64, c_vp, c_vp, c_vp, c_vp]),
    "rk_bsr3_gather": (c_i32, [c_i64, c_vp, c_vp, c_vp, c_vp]),
    "rk_sell_plan": (c_i32, [c_i64, c_vp, c_vp, c_i32, c_i32, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "rk_sell_fill": (c_i32, [c_i64, c_vp, c_vp, c_i32, c_vp, c_vp, c_i64, c_vp, c_vp, c_vp]),
    "rk_gemv_t": (c_i32, [c_i64, c_i64, c_vp, c_i64, c_vp, c_vp, c_vp, c_i64, c_vp]),
    "rk_gemv_n": (c_i32, [c_i64, c_i64, c_vp, c_i64, c_vp, c_vp, c_vp, c_i32, c_vp]),
    "rk_dot": (c_i32, [c_i64, c_vp, c_vp, c_vp, c_vp, c_i64, c_vp, c_vp]),
    "rk_scale_columns": (c_i32, [c_i64, c_i64, c_vp, c_i64, c_vp, c_vp, c_i64, c_vp]),
    "rk_axpby": (c_i32, [c_i64, c_dbl, c_vp, c_dbl, c_vp, c_vp]),
    "rk_sub_from": (c_i32, [c_i64, c_vp, c_vp, c_vp]),
    "rk_gram": (c_i32, [c_i64, c_i64, c_vp, c_i64, c_i64, c_vp, c_i64, c_vp, c_i64, c_vp, c_i64, c_vp]),
    "rk_gram_upper": (c_i32, [c_i64, c_i64, c_vp, c_i64, c_i64, c_vp, c_i64, c_i64, c_vp, c_i64, c_vp, c_i64,
                              c_vp]),
    "rk_gram_upper_split": (c_i32, [c_i64, c_i64, c_vp, c_i64, c_i64, c_vp, c_i64, c_vp, c_i64, c_vp, c_i64, c_vp,
                                    c_i64, c_vp]),
    "rk_gemm_nn": (c_i32, [c_i64, c_i64, c_i64, c_vp, c_i64, c_vp, c_i64, c_vp, c_i64, c_vp]),
    "rk_pod_weighted_gram": (c_i32, [c_i64, c_vp, c_i64, c_i32, c_vp, c_vp, c_vp, c_i64, c_vp]),
    "rk_pod_coef": (c_i32, [c_i64, c_i64, c_vp, c_i64, c_vp, c_vp, c_vp, c_i64, c_vp]),
    "rk_profile_begin": (c_i32, []),
    "rk_launch_count": (c_i64, []),
    "rk_debug_trace": (c_i32, [ctypes.POINTER(ctypes.c_uint64), c_i64]),
    "rk_ssor_apply": (c_i32, [ctypes.POINTER(RkCsr), c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_i32, c_vp, c_vp,
                              c_vp]),
    "rk_ssor_levels": (c_i32, [ctypes.POINTER(RkCsr), c_i32, c_vp, c_vp, c_vp, c_i32, c_vp]),
    "rk_profile_end": (c_i32, [ctypes.POINTER(c_dbl), ctypes.POINTER(c_i64)]),
    "rk_profile_cluster": (c_i32, [ctypes.POINTER(c_dbl), ctypes.POINTER(c_i64)]),
}

EXPORTED_SYMBOLS = tuple(_SIGNATURES)

_lib = None
_lib_lock = threading.Lock()


def load_library(path: str | None = None):
    """Load and type the shared library (no CUDA device needed to load it)."""
    global _lib
    with _lib_lock:
        if _lib is not None and path is None:
            return _lib
        p = path or LIB_PATH
        if not os.path.exists(p):
            raise NativeUnavailable(
                f"{p} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
            )
        lib = ctypes.CDLL(p)
        for name, (res, args) in _SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        if path is None:
            _lib = lib
        return lib


def lib():
    if _lib is None:
        load_library()
    return _lib


_ERRS = {-1: "DimensionMismatch", -2: "NotPositiveDefinite", -3: "CUDA", -4: "argument"}


def check(rc: int, what: str) -> None:
    if rc != 0:
        from .errors import DimensionMismatch, NotPositiveDefinite, RecyklError

        msg = lib().rk_last_error().decode(errors="replace")
        if rc == -1:
            raise DimensionMismatch(f"{what}: {msg}")
        if rc == -2:
            raise NotPositiveDefinite(f"{what}: {msg}")
        raise RecyklError(f"{what} failed ({_ERRS.get(rc, rc)}): {msg}")


def require_device() -> torch.device:
    if not torch.cuda.is_available():
        raise NativeUnavailable("no CUDA device: the B200 path has no CPU fallback")
    lib()
    return torch.device("cuda", torch.cuda.current_device())


def stream_ptr(device: torch.device | None = None) -> int:
    return torch.cuda.current_stream(device).cuda_stream


def ptr(t: torch.Tensor | None) -> int | None:
    if t is None:
        return None
    return t.data_ptr()


# ---------------------------------------------------------------------------
# per-thread scratch (re-entrant: each host thread owns its reduction workspace)
# ---------------------------------------------------------------------------
_tls = threading.local()


class Scratch:
    """Reduction workspace + zeroed tickets owned by one host thread."""

    def __init__(self, device):
        self.device = device
        self.ws = torch.empty(0, dtype=torch.float64, device=device)
        self.tickets = torch.zeros(PCG_TICKETS, dtype=torch.int32, device=device)
        self.out = torch.zeros(8, dtype=torch.float64, device=device)

    def workspace(self, ndoubles: int) -> torch.Tensor:
        if self.ws.numel() < ndoubles:
            self.ws = torch.empty(max(int(ndoubles), 2 * self.ws.numel(), 4096), dtype=torch.float64,
                                  device=self.device)
        return self.ws


def scratch(device) -> Scratch:
    key = (device.type, device.index)
    cache = getattr(_tls, "cache", None)
    if cache is None:
        cache = _tls.cache = {}
    s = cache.get(key)
    if s is None:
        s = cache[key] = Scratch(device)
    return s
