"""Token routing counts (moesim dispatch.py:27-104), computed by the C++ planner.

`build_dispatch` returns the reference's route tensor route[s, e, d]; the device
dispatch kernel (K4) then executes it token by token: the slots of one
(source, expert) cell, in (t, j) order, fill the destinations in ascending device
order with exactly route[s, e, d] tokens each.
"""

from __future__ import annotations

import numpy as np

from . import _native as N
from .costmodel import TrafficMatrix
from .errors import DimensionError
from .placement import ChunkPlacement


class DispatchPlan:
    """route[s, e, d]: tokens of expert e sent from device s to device d (dispatch.py:27-46)."""

    __slots__ = ("route",)

    def __init__(self, route) -> None:
        self.route = np.asarray(route, dtype=np.int64)

    @property
    def num_devices(self) -> int:
        return self.route.shape[0]

    @property
    def num_experts(self) -> int:
        return self.route.shape[1]

    def tokens_to_device(self) -> np.ndarray:
        return self.route.sum(axis=(0, 1))

    def max_device_tokens(self) -> int:
        return int(self.tokens_to_device().max())


def _integral_counts(tokens) -> np.ndarray:
    counts = np.asarray(tokens)
    if counts.ndim != 2:
        raise DimensionError(f"token matrix must be 2-D, got shape {counts.shape}")
    if np.any(counts < 0):
        raise DimensionError("token counts must be non-negative")
    if not np.all(np.equal(np.mod(counts, 1), 0)):
        raise DimensionError("token counts must be integral")
    return np.ascontiguousarray(counts.astype(np.int64))


def build_dispatch(tokens, placement: ChunkPlacement, topology) -> DispatchPlan:
    """Route a (devices × experts) integral count matrix onto a placement (dispatch.py:49-97):
    local replica first, else split evenly over same-node holders, else over all holders;
    remainders to the least-assigned destination, lowest index on ties."""
    counts = np.asarray(tokens)
    if counts.ndim != 2:
        raise DimensionError(f"token matrix must be 2-D, got shape {counts.shape}")
    D, E = counts.shape
    if D != placement.num_devices or E != placement.num_chunks:
        raise DimensionError(
            f"token matrix {counts.shape} does not match placement "
            f"{placement.num_devices} devices x {placement.num_chunks} experts")
    if D != topology.num_devices:
        raise DimensionError("token matrix and topology disagree on device count")
    counts = _integral_counts(counts)
    route = np.zeros((D, E, D), dtype=np.int64)
    topo = topology.native()
    N.check(N.LIB.fssdp_build_dispatch(D, E, counts.ctypes.data_as(N.P_i64),
                                       placement.mask.ctypes.data_as(N.P_u8), N.C.byref(topo),
                                       route.ctypes.data_as(N.P_i64)), "build_dispatch")
    return DispatchPlan(route)


def dispatch_traffic(plan: DispatchPlan, token_bytes: int) -> TrafficMatrix:
    """A2A byte matrix of a dispatch; local tokens are free (dispatch.py:100-104)."""
    moved = plan.route.sum(axis=1).astype(np.float64) * token_bytes
    np.fill_diagonal(moved, 0.0)
    return TrafficMatrix(moved)
