"""Snapshot weights for goal-oriented truncation (``recykl/weights.py``).

Host-side bookkeeping of m-vectors (m <= a few thousand): the coefficient
history of previous solutions in the accumulated block and the
inverse-distance (RBF) blend rho(r) = 2^{-(r-1)} over a window
(weights.py:32-34, 53-90, 112-128). Shorter entries are zero-padded on the
right, which is exact because the block only grows by appending columns.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .errors import NoHistory


def idw_weight(r: int) -> float:
    """Weight of the solution r systems back (r >= 1): 1 / 2^(r-1)."""
    return 1.0 / 2.0 ** (r - 1)


@dataclass
class WeightScheme:
    kind: str
    window: int | None = None

    def __post_init__(self):
        if self.kind not in ("ideal", "prev", "rbf"):
            raise ValueError(f"unknown weight scheme {self.kind!r}")


class WeightHistory:
    """Coefficient vectors of earlier solutions, each in the block coordinates
    of its own time; reads pad them to the current width."""

    def __init__(self):
        self._entries: list[np.ndarray] = []

    def __len__(self) -> int:
        return len(self._entries)

    def push(self, eta) -> None:
        self._entries.append(np.array(eta, dtype=np.float64, copy=True).reshape(-1))

    def reset(self) -> None:
        self._entries.clear()

    def width(self) -> int:
        return max((e.shape[0] for e in self._entries), default=0)

    def padded(self, index: int) -> np.ndarray:
        e = self._entries[index]
        out = np.zeros(self.width())
        out[: e.shape[0]] = e
        return out

    def reexpress(self, trunc_map, gram) -> None:
        """Project every entry onto the post-truncation basis: map' gram eta."""
        g = gram.detach().cpu().numpy() if hasattr(gram, "detach") else np.asarray(gram)
        proj = np.asarray(trunc_map).T @ g
        self._entries = [proj @ self.padded(i) for i in range(len(self._entries))]


def weights_previous(history: WeightHistory) -> np.ndarray:
    """Most recent solution's coefficients in the current block."""
    if len(history) == 0:
        raise NoHistory("no previous solve recorded")
    return history.padded(len(history) - 1)


def weights_rbf(history: WeightHistory, omega: int) -> np.ndarray:
    """sum_{i=1..omega} 2^{-(i-1)} eta_{last-i+1}, accumulated newest first."""
    if len(history) == 0:
        raise NoHistory("no previous solve recorded")
    omega = max(1, min(int(omega), len(history)))
    out = np.zeros(history.width())
    last = len(history) - 1
    for i in range(1, omega + 1):
        out += idw_weight(i) * history.padded(last - (i - 1))
    return out
