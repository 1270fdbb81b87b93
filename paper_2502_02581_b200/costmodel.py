"""Traffic accounting of the sparse collectives (moesim costmodel.py:21-194).

These are the SpAG/SpRS *message schedules* the device kernels execute (each added
replica = one owner->holder copy of the expert; each replica gradient = one
holder->owner transfer) and the alpha-beta latency the placement decisions price.
Computation is in the C++ planner (csrc/planner.cpp), float64 bit-exact.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _native as N
from .errors import DimensionMismatchError, InvalidPairError
from .placement import ChunkPlacement, _same_dims


class TrafficMatrix:
    """Square, non-negative, zero-diagonal byte matrix; [s, r] = bytes s -> r (costmodel.py:21-57)."""

    __slots__ = ("data",)

    def __init__(self, data) -> None:
        arr = np.array(data, dtype=np.float64, copy=True)
        if arr.ndim != 2 or arr.shape[0] != arr.shape[1]:
            raise DimensionMismatchError(f"traffic matrix must be square, got {arr.shape}")
        if (arr < 0).any():
            raise DimensionMismatchError("traffic matrix entries must be non-negative")
        if (np.diagonal(arr) != 0).any():
            raise DimensionMismatchError(
                "traffic matrix diagonal must be zero (local moves are free)")
        self.data = arr

    @classmethod
    def zeros(cls, num_devices: int) -> "TrafficMatrix":
        return cls(np.zeros((num_devices, num_devices)))

    @property
    def num_devices(self) -> int:
        return self.data.shape[0]

    def total(self) -> float:
        return float(self.data.sum())

    def inbound(self) -> np.ndarray:
        return self.data.sum(axis=0)

    def outbound(self) -> np.ndarray:
        return self.data.sum(axis=1)

    def transpose(self) -> "TrafficMatrix":
        return TrafficMatrix(self.data.T)

    def is_zero(self) -> bool:
        return not self.data.any()


@dataclass(frozen=True)
class SparsityReport:
    """(costmodel.py:60-72) fraction of chunks moved, total bytes, bottleneck device/bytes."""

    sparsity: float
    total_interdevice_bytes: float
    bottleneck_device: int
    bottleneck_bytes: float


def _traffic(fn, pre: ChunkPlacement, post: ChunkPlacement, chunk_bytes, what: str):
    _same_dims(pre, post)
    D = pre.num_devices
    mat = np.zeros((D, D), dtype=np.float64)
    rep = np.zeros(4, dtype=np.float64)
    rc = fn(pre.num_chunks, D, pre.mask.ctypes.data_as(N.P_u8), post.mask.ctypes.data_as(N.P_u8),
            float(chunk_bytes), mat.ctypes.data_as(N.P_f64), rep.ctypes.data_as(N.P_f64))
    if rc == -2:
        raise InvalidPairError(N.last_error())
    N.check(rc, what)
    return TrafficMatrix(mat), SparsityReport(float(rep[0]), float(rep[1]), int(rep[2]),
                                              float(rep[3]))


def spag_traffic(pre: ChunkPlacement, post: ChunkPlacement, chunk_bytes: int):
    """SparseAllGather byte flow: owner unicasts to every added holder (costmodel.py:87-108)."""
    return _traffic(N.LIB.fssdp_spag_traffic, pre, post, chunk_bytes, "spag_traffic")


def sprs_traffic(pre: ChunkPlacement, post: ChunkPlacement, chunk_bytes: int):
    """SparseReduceScatter byte flow: replicas send to the final owner (costmodel.py:111-132)."""
    return _traffic(N.LIB.fssdp_sprs_traffic, pre, post, chunk_bytes, "sprs_traffic")


def collective_latency(traffic: TrafficMatrix, topology) -> float:
    """alpha + worst per-resource transfer time, 0 for an empty matrix (costmodel.py:149-182)."""
    if traffic.num_devices != topology.num_devices:
        raise DimensionMismatchError(
            f"traffic is {traffic.num_devices} devices, topology has {topology.num_devices}")
    data = np.ascontiguousarray(traffic.data)
    out = np.zeros(1, dtype=np.float64)
    topo = topology.native()
    N.check(N.LIB.fssdp_collective_latency(traffic.num_devices, data.ctypes.data_as(N.P_f64),
                                           N.C.byref(topo), out.ctypes.data_as(N.P_f64)),
            "collective_latency")
    return float(out[0])


def overlap_degree(t_nonmoe: float, topology, expert_bytes: int) -> int:
    """Experts fetchable under t_nonmoe seconds at the slower tier (costmodel.py:185-194)."""
    out = np.zeros(1, dtype=np.int64)
    topo = topology.native()
    N.check(N.LIB.fssdp_overlap_degree(float(t_nonmoe), N.C.byref(topo), float(expert_bytes),
                                       out.ctypes.data_as(N.P_i64)), "overlap_degree")
    return int(out[0])
