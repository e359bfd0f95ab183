"""Opt-in host-side phase timing (RK_PHASE_TIMING=1): synchronises the device
around each phase of solve_system/update_basis and accumulates wall seconds.
Off by default (no synchronisation is added to the product path)."""

import os
import time

import torch

ENABLED = os.environ.get("RK_PHASE_TIMING") == "1"
TIMES: dict = {}


class phase:
    def __init__(self, name: str):
        self.name = name

    def __enter__(self):
        if ENABLED:
            torch.cuda.synchronize()
            self.t0 = time.perf_counter()
        return self

    def __exit__(self, *exc):
        if ENABLED:
            torch.cuda.synchronize()
            TIMES[self.name] = TIMES.get(self.name, 0.0) + time.perf_counter() - self.t0
        return False


def add(name: str, seconds: float) -> None:
    """Accumulate a host-side wall interval (no device synchronisation)."""
    if ENABLED:
        TIMES[name] = TIMES.get(name, 0.0) + seconds


def reset():
    TIMES.clear()
