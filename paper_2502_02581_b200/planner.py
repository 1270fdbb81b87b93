"""Placement planning (moesim planner.py:32-385): load estimation, sparse
materialization (Alg. 1), calibration, heterogeneous sharding (Alg. 2).

All decisions run in the C++ planner (csrc/planner.cpp) and are bit-exact with the
reference, float64 summation order included (SURVEY.md §8a hazards).
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Sequence

import numpy as np

from . import _native as N
from .errors import EmptyHistoryError, InternalError
from .placement import ChunkPlacement, ShardPlan


def estimate_loads(history: Sequence[np.ndarray], window: int = 5) -> np.ndarray:
    """Mean of the last `window` (devices × experts) matrices (planner.py:32-42)."""
    if len(history) == 0:
        raise EmptyHistoryError("cannot estimate loads from an empty history")
    if window <= 0:
        raise EmptyHistoryError(f"window must be positive, got {window}")
    recent = [np.asarray(m, dtype=np.float64) for m in list(history)[-window:]]
    stack = np.ascontiguousarray(np.stack(recent))
    out = np.empty(stack.shape[1:], dtype=np.float64)
    rows = stack.shape[1]
    cols = int(np.prod(stack.shape[2:])) if stack.ndim > 2 else 1
    N.check(N.LIB.fssdp_estimate_loads(stack.shape[0], rows, cols, stack.ctypes.data_as(N.P_f64),
                                       window, out.ctypes.data_as(N.P_f64)), "estimate_loads")
    return out


@dataclass(frozen=True)
class MaterializationPlan:
    """Replication target over a sharded base (planner.py:45-62)."""

    source: ChunkPlacement
    target: ChunkPlacement
    added_per_device: tuple

    @property
    def is_identity(self) -> bool:
        return self.target == self.source

    def to_json_obj(self) -> dict:
        return {"source": self.source.to_json_obj(), "target": self.target.to_json_obj(),
                "added_per_device": list(self.added_per_device)}


def _per_expert_loads(loads) -> np.ndarray:
    arr = np.asarray(loads, dtype=np.float64)
    if arr.ndim == 2:
        return arr.sum(axis=0)  # axis-0: sequential over devices, as the reference
    if arr.ndim == 1:
        return arr
    raise InternalError(f"loads must be 1-D or 2-D, got shape {arr.shape}")


def sparse_materialization(shards: ChunkPlacement, loads, t: int, m: int,
                           topology) -> MaterializationPlan:
    """Alg. 1: which experts to replicate where this iteration (planner.py:171-197)."""
    if not shards.is_partition():
        raise InternalError("materialization must start from a partition")
    per = np.ascontiguousarray(_per_expert_loads(loads))
    if len(per) != shards.num_chunks:
        raise InternalError(f"got {len(per)} expert loads for {shards.num_chunks} chunks")
    E, D = shards.num_chunks, shards.num_devices
    target = np.zeros((E, D), dtype=np.uint8)
    added = np.zeros(D, dtype=np.int32)
    topo = topology.native()
    N.check(N.LIB.fssdp_sparse_materialization(E, D, shards.mask.ctypes.data_as(N.P_u8),
                                               per.ctypes.data_as(N.P_f64), int(t), int(m),
                                               N.C.byref(topo), target.ctypes.data_as(N.P_u8),
                                               added.ctypes.data_as(N.P_i32)),
            "sparse_materialization")
    return MaterializationPlan(shards, ChunkPlacement.from_mask(target),
                               tuple(int(a) for a in added))


def estimate_moe_latency(placement: ChunkPlacement, tokens, topology, token_bytes: int,
                         per_token_expert_time: float) -> float:
    """Expert-compute bottleneck + dispatch A2A latency (planner.py:205-216)."""
    from .dispatch import _integral_counts

    counts = _integral_counts(tokens)
    out = np.zeros(1, dtype=np.float64)
    topo = topology.native()
    N.check(N.LIB.fssdp_estimate_moe_latency(placement.num_devices, placement.num_chunks,
                                             placement.mask.ctypes.data_as(N.P_u8),
                                             counts.ctypes.data_as(N.P_i64), N.C.byref(topo),
                                             float(token_bytes), float(per_token_expert_time),
                                             out.ctypes.data_as(N.P_f64)),
            "estimate_moe_latency")
    return float(out[0])


@dataclass(frozen=True)
class CalibrationOutcome:
    accepted: bool
    plan: MaterializationPlan
    extra_seconds: float
    estimate_before: float
    estimate_after: float


def calibrate(plan: MaterializationPlan, actual, remaining_m: int, t_remaining: float, topology,
              chunk_bytes: int, token_bytes: int,
              per_token_expert_time: float) -> CalibrationOutcome:
    """Post-gate extension on the actual loads, accepted only if it pays (planner.py:228-276)."""
    E, D = plan.source.num_chunks, plan.source.num_devices
    act = np.ascontiguousarray(np.asarray(actual, dtype=np.float64))
    if act.shape != (D, E):
        from .errors import DimensionError

        raise DimensionError(f"actual loads {act.shape} do not match {D} devices x {E} experts")
    acc = np.zeros(1, dtype=np.int32)
    target = np.zeros((E, D), dtype=np.uint8)
    added = np.zeros(D, dtype=np.int32)
    dbl = np.zeros(3, dtype=np.float64)
    topo = topology.native()
    N.check(N.LIB.fssdp_calibrate(E, D, plan.source.mask.ctypes.data_as(N.P_u8),
                                  plan.target.mask.ctypes.data_as(N.P_u8),
                                  act.ctypes.data_as(N.P_f64), int(remaining_m),
                                  float(t_remaining), N.C.byref(topo), float(chunk_bytes),
                                  float(token_bytes), float(per_token_expert_time),
                                  acc.ctypes.data_as(N.P_i32), target.ctypes.data_as(N.P_u8),
                                  added.ctypes.data_as(N.P_i32), dbl.ctypes.data_as(N.P_f64)),
            "calibrate")
    if acc[0]:
        new_plan = MaterializationPlan(plan.source, ChunkPlacement.from_mask(target),
                                       tuple(int(a) for a in added))
        return CalibrationOutcome(True, new_plan, float(dbl[0]), float(dbl[1]), float(dbl[2]))
    return CalibrationOutcome(False, plan, 0.0, float(dbl[1]), float(dbl[2]))


@dataclass(frozen=True)
class GlobalLoadProfile:
    """(layers, experts) load totals for re-sharding (planner.py:284-299)."""

    per_layer: np.ndarray

    def __post_init__(self) -> None:
        arr = np.asarray(self.per_layer, dtype=np.float64)
        if arr.ndim != 2:
            raise InternalError(f"profile must be (layers, experts), got {arr.shape}")
        object.__setattr__(self, "per_layer", arr)

    @classmethod
    def from_step(cls, step: Sequence[np.ndarray]) -> "GlobalLoadProfile":
        return cls(np.stack([_per_expert_loads(m) for m in step]))


def heterogeneous_sharding(profile: GlobalLoadProfile, t: int, topology) -> ShardPlan:
    """Alg. 2: load-aware re-partition of expert ownership (planner.py:302-385)."""
    prof = np.ascontiguousarray(profile.per_layer, dtype=np.float64)
    L, E = prof.shape
    owners = np.empty((L, E), dtype=np.int32)
    topo = topology.native()
    N.check(N.LIB.fssdp_heterogeneous_sharding(L, E, prof.ctypes.data_as(N.P_f64), int(t),
                                               N.C.byref(topo), owners.ctypes.data_as(N.P_i32)),
            "heterogeneous_sharding")
    return ShardPlan.from_owners(owners, topology.num_devices)
