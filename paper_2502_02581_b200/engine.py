"""FSSDP iteration control — the decision part of moesim's FssdpState (engine.py:386-557).

The reference engine *simulates* a timeline; here the same decisions drive real
device work: `FssdpPlanner.plan_layer` returns, per MoE layer and iteration, the
materialized placement (which replicas SpAG fetches and SpRS folds back) and the
build_dispatch route the dispatch kernel executes.  The per-layer decision chain
(adoption gate -> calibration -> fallback -> dispatch) runs in one C++ call
(fssdp_plan_layer).  The simulated timeline, the comparison policies and the CLI are
out of scope.
"""

from __future__ import annotations

from collections import deque
from dataclasses import dataclass, field
from enum import Enum
from typing import Optional, Sequence

import numpy as np

from . import _native as N
from .costmodel import TrafficMatrix, collective_latency, overlap_degree
from .errors import ConfigError, TraceMismatchError
from .placement import ChunkPlacement, ShardPlan
from .planner import GlobalLoadProfile, MaterializationPlan, estimate_loads, heterogeneous_sharding
from .traces import TraceRecorder


@dataclass(frozen=True)
class ModelConfig:
    """Model-side quantities the planner prices (engine.py:54-77)."""

    layers: int
    experts_per_layer: int
    expert_bytes: int
    token_bytes: int
    attn_fwd_time: float
    per_token_expert_time: float
    optimizer_multiplier: float = 6.0

    def __post_init__(self) -> None:
        if self.layers <= 0 or self.experts_per_layer <= 0:
            raise ConfigError("layers and experts_per_layer must be positive")
        if self.expert_bytes <= 0 or self.token_bytes <= 0:
            raise ConfigError("expert_bytes and token_bytes must be positive")
        if self.attn_fwd_time < 0 or self.per_token_expert_time < 0:
            raise ConfigError("times must be non-negative")
        if self.optimizer_multiplier < 6:
            raise ConfigError("optimizer_multiplier must be at least 6 (params + moments in "
                              "full precision plus a full-precision master copy)")


class PolicyKind(str, Enum):
    """EP and FSSDP are executed; the reference's simulated comparators are not (engine.py:80-85)."""

    EP = "ep"
    FSSDP = "fssdp"


@dataclass(frozen=True)
class Policy:
    """Placement policy knobs (engine.py:88-121); FSSDP uses all but interval/reserved/top-k."""

    kind: PolicyKind
    window: int = 5
    calibration: bool = True
    rematerialize: bool = False
    reshard_interval: int = 100
    interval: int = 25
    reserved_slots: int = 0
    replicate_top_k: int = 1
    free_bytes_per_device: Optional[int] = None
    overlap_override: Optional[int] = None
    capacity_override: Optional[int] = None

    def label(self) -> str:
        return self.kind.value

    def to_json_obj(self) -> dict:
        return {"kind": self.kind.value, "window": self.window, "calibration": self.calibration,
                "rematerialize": self.rematerialize, "reshard_interval": self.reshard_interval,
                "interval": self.interval, "reserved_slots": self.reserved_slots,
                "replicate_top_k": self.replicate_top_k,
                "free_bytes_per_device": self.free_bytes_per_device,
                "overlap_override": self.overlap_override,
                "capacity_override": self.capacity_override}


@dataclass(eq=False)
class MemoryBreakdown:
    """Per-device bytes (engine.py:159-177)."""

    param_bytes: np.ndarray
    grad_bytes: np.ndarray
    optimizer_bytes: np.ndarray
    materialized_bytes: np.ndarray

    def total_per_device(self) -> np.ndarray:
        return self.param_bytes + self.grad_bytes + self.optimizer_bytes + self.materialized_bytes

    def optimizer_total(self) -> float:
        return float(self.optimizer_bytes.sum())


def memory_report(plan: ShardPlan, materializations, config: ModelConfig,
                  mode: str = "retain") -> MemoryBreakdown:
    """Expert memory per device; retain = Σ layers' replicas, rematerialize = max
    (engine.py:188-226).  The device layer reserves the worst case of it: m replica slots
    per layer (retain) or one shared set of m for all layers (rematerialize) —
    layer.model_regions / replica_region_bytes."""
    if mode not in ("retain", "rematerialize"):
        raise ConfigError(f"unknown memory mode {mode!r}")
    D = plan.num_devices
    owned = np.zeros(D, dtype=np.float64)
    for p in plan.per_layer:
        owned += np.asarray(p.counts_per_device(), dtype=np.float64)
    param = owned * config.expert_bytes
    added = np.zeros((plan.num_layers, D), dtype=np.float64)
    if materializations is not None:
        for l, mat in enumerate(materializations):
            if mat is not None:
                added[l] = np.asarray(mat.added_per_device, dtype=np.float64)
    added_bytes = added * config.expert_bytes
    if mode == "retain":
        materialized = added_bytes.sum(axis=0)
    else:
        materialized = added_bytes.max(axis=0) if plan.num_layers else np.zeros(D)
    return MemoryBreakdown(param_bytes=param, grad_bytes=param + materialized,
                           optimizer_bytes=param * config.optimizer_multiplier,
                           materialized_bytes=materialized)


@dataclass
class LayerDecision:
    """One layer's executed plan for one iteration."""

    base: ChunkPlacement          # ownership partition (SpAG pre / SpRS post)
    target: ChunkPlacement        # materialized placement (SpAG post / SpRS pre)
    added_per_device: tuple
    route: np.ndarray             # (D, E, D) int64, build_dispatch on the actual counts
    spag_latency: float = 0.0
    sprs_latency: float = 0.0
    remat_latency: float = 0.0
    calib_time: float = 0.0
    adopted: bool = False
    calibrated: bool = False

    @property
    def materialization(self) -> MaterializationPlan:
        return MaterializationPlan(self.base, self.target, self.added_per_device)

    @property
    def is_identity(self) -> bool:
        return self.target == self.base


class _PlanScratch:
    """Persistent fssdp_plan_layer buffers of one layer with their addresses resolved once
    (numpy's .ctypes.data costs microseconds per access on the planning critical path)."""

    def __init__(self, E: int, D: int) -> None:
        self.act = np.zeros((D, E), dtype=np.int64)
        self.target = np.zeros((E, D), dtype=np.uint8)
        self.added = np.zeros(D, dtype=np.int32)
        self.route = np.zeros((D, E, D), dtype=np.int64)
        self.dbl = np.zeros(4, dtype=np.float64)
        self.flags = np.zeros(2, dtype=np.int32)
        for k in ("act", "target", "added", "route", "dbl", "flags"):
            setattr(self, "p_" + k, getattr(self, k).ctypes.data)
        self._topo = None

    def topo_ref(self, topo_c):
        if self._topo is None or self._topo[0] is not topo_c:
            self._topo = (topo_c, N.C.byref(topo_c))
        return self._topo[1]


_MOVE_MULTIPLIER = 7  # params + 6x optimizer state move with a re-sharded expert (engine.py:233)


class FssdpPlanner:
    """Per-run FSSDP control state (engine.py:279-292, 386-402).

    Usage per iteration:  begin_iteration();  plan_layer(l, counts_l) for each layer
    (after that layer's gate);  end_iteration(step_counts)."""

    def __init__(self, config: ModelConfig, topology, policy: Policy,
                 record_trace: bool = False) -> None:
        if policy.kind not in (PolicyKind.FSSDP, PolicyKind.EP):
            raise ConfigError(f"unknown policy kind {policy.kind!r}")
        self.config = config
        self.topo = topology
        self.policy = policy
        self.iteration = 0
        self.history = [deque(maxlen=max(1, policy.window)) for _ in range(config.layers)]
        self.shards = ShardPlan.even(config.layers, config.experts_per_layer, topology)
        if policy.overlap_override is not None:
            self.t = int(policy.overlap_override)
        else:
            self.t = overlap_degree(config.attn_fwd_time, topology, config.expert_bytes)
        if policy.capacity_override is not None:
            self.m = int(policy.capacity_override)
        elif policy.free_bytes_per_device is not None:
            self.m = policy.free_bytes_per_device // config.expert_bytes
        else:
            self.m = config.experts_per_layer
        self._knobs = N.LayerKnobs(
            self.t, self.m, int(policy.calibration), int(policy.rematerialize),
            float(config.expert_bytes), float(config.token_bytes), float(config.attn_fwd_time),
            float(config.per_token_expert_time))
        self._topo_c = topology.native()
        self.last_reshard_time = 0.0
        self.last_reshard_moves: list = []
        self._step = None
        # the gate counts of every finished iteration, as a moesim trace (traces.py)
        self.recorder = TraceRecorder() if record_trace else None

    # -- helpers ------------------------------------------------------------------
    def _owners(self, layer: int) -> np.ndarray:
        """Owner table of a layer's current partition (cached per ShardPlan)."""
        if getattr(self, "_owners_plan", None) is not self.shards:
            self._owners_cache = np.ascontiguousarray(self.shards.owners(), dtype=np.int32)
            self._owners_plan = self.shards
        return self._owners_cache[layer]

    def estimate(self, layer: int) -> Optional[np.ndarray]:
        """Window mean of the layer's history (cached until the history changes: the early
        candidate and the plan of one iteration share it)."""
        h = self.history[layer]
        if not h:
            return None
        key = (len(h), h[-1], h[0])  # the arrays themselves (kept alive, compared by identity)
        cache = self.__dict__.setdefault("_est_cache", {})
        hit = cache.get(layer)
        if hit is not None and hit[0][0] == key[0] and hit[0][1] is key[1] and hit[0][2] is key[2]:
            return hit[1]
        est = np.ascontiguousarray(estimate_loads(h, self.policy.window), dtype=np.float64)
        est.flags.writeable = False
        cache[layer] = (key, est, est.ctypes.data)
        return est

    def _shard_score(self, plan: ShardPlan, profile: GlobalLoadProfile) -> tuple:
        """(max node load, max device load), numpy order (engine.py:431-442)."""
        owners = np.ascontiguousarray(plan.owners())
        prof = np.ascontiguousarray(profile.per_layer, dtype=np.float64)
        out = np.zeros(2, dtype=np.float64)
        N.check(N.LIB.fssdp_shard_score(owners.shape[0], owners.shape[1],
                                        owners.ctypes.data_as(N.P_i32),
                                        prof.ctypes.data_as(N.P_f64), N.C.byref(self._topo_c),
                                        out.ctypes.data_as(N.P_f64)), "shard_score")
        return (float(out[0]), float(out[1]))

    def _reshard_moves(self, candidate: ShardPlan) -> list:
        moves = []
        for l, (old, new) in enumerate(zip(self.shards.per_layer, candidate.per_layer)):
            oo, no = old.owners(), new.owners()
            for e in range(old.num_chunks):
                if oo[e] != no[e]:
                    moves.append((l, e, int(oo[e]), int(no[e])))
        return moves

    def _move_latency(self, moves: list) -> float:
        """_move_latency(pairs, 7*expert_bytes) (engine.py:263-276, 444-453)."""
        if not moves:
            return 0.0
        D = self.topo.num_devices
        mat = np.zeros((D, D))
        for _, _, src, dst in moves:
            if src != dst:
                mat[src, dst] += _MOVE_MULTIPLIER * self.config.expert_bytes
        return collective_latency(TrafficMatrix(mat), self.topo)

    # -- iteration protocol -------------------------------------------------------
    def begin_iteration(self) -> float:
        """Re-shard trigger (engine.py:470-487); returns the modeled re-shard time.
        The executed data movement is listed in `last_reshard_moves` (layer, expert, src, dst)."""
        self.last_reshard_time = 0.0
        self.last_reshard_moves = []
        if self.policy.kind != PolicyKind.FSSDP or self.t <= 0 or self.m <= 0:
            return 0.0
        if (self.iteration > 0 and self.policy.reshard_interval > 0
                and self.iteration % self.policy.reshard_interval == 0 and all(self.history)):
            profile = GlobalLoadProfile(np.stack(
                [self.estimate(l).sum(axis=0) for l in range(self.config.layers)]))
            candidate = heterogeneous_sharding(profile, self.t, self.topo)
            if self._shard_score(candidate, profile) < self._shard_score(self.shards, profile):
                self.last_reshard_moves = self._reshard_moves(candidate)
                self.last_reshard_time = self._move_latency(self.last_reshard_moves)
                self.shards = candidate
        return self.last_reshard_time

    def _scratch(self, layer: int) -> "_PlanScratch":
        sc = self.__dict__.setdefault("_scratches", {}).get(layer)
        if sc is None:
            base = self.shards.per_layer[layer]
            sc = self._scratches[layer] = _PlanScratch(base.num_chunks, base.num_devices)
        return sc

    def plan_layer(self, layer: int, actual) -> LayerDecision:
        """Adoption gate, calibration, fallback, dispatch for one layer (engine.py:491-553).

        On the planning critical path (between the count all-gather and the dispatch): the
        C++ call works on persistent buffers whose addresses are resolved once; the
        decision holds copies.  `last_target_ptr` / `last_route_ptr` address the scratch
        copies for an immediate NativeTables.from_pointers."""
        base = self.shards.per_layer[layer]
        E, D = base.num_chunks, base.num_devices
        sc = self._scratch(layer)
        act = np.asarray(actual)
        if act.shape != (D, E):
            raise TraceMismatchError(f"counts {act.shape} do not match {D} devices x {E} experts")
        np.copyto(sc.act, act, casting="unsafe")
        owner_ptr = self._owners_ptr(layer)
        knobs, est_ptr = self._layer_knobs(layer)
        N.check(N.LIB_RAW.fssdp_plan_layer(
            E, owner_ptr, est_ptr, sc.p_act, sc.topo_ref(self._topo_c), N.C.byref(knobs),
            sc.p_target, sc.p_added, sc.p_route, sc.p_dbl, sc.p_flags), "plan_layer")
        self.last_target_ptr, self.last_route_ptr = sc.p_target, sc.p_route
        return self._decision(base, sc)

    def _layer_knobs(self, layer: int):
        if self.policy.kind == PolicyKind.EP:
            knobs = self.__dict__.get("_ep_knobs")
            if knobs is None:
                knobs = self._ep_knobs = N.LayerKnobs(
                    0, 0, 0, 0, self._knobs.expert_bytes, self._knobs.token_bytes,
                    self._knobs.attn_fwd_time, self._knobs.per_token_expert_time)
            return knobs, None
        return self._knobs, self._estimate_ptr(layer)

    @staticmethod
    def _decision(base, sc) -> LayerDecision:
        dbl, flags = sc.dbl.tolist(), sc.flags.tolist()
        return LayerDecision(base=base, target=ChunkPlacement.from_mask(sc.target.copy(), copy=False),
                             added_per_device=tuple(sc.added.tolist()), route=sc.route.copy(),
                             spag_latency=dbl[0], sprs_latency=dbl[1], remat_latency=dbl[2],
                             calib_time=dbl[3], adopted=bool(flags[0]), calibrated=bool(flags[1]))

    def plan_with_tables(self, layer: int, counts, counts_ptr: int, rank: int, pre_ptr,
                         d_model: int, d_ff: int, blob, blob_ptr: int, header_ptr: int,
                         blob_dev_ptr, stream, limits_ptr=None, decide: bool = True,
                         n_mats: int = 2) -> Optional[LayerDecision]:
        """plan() fused with this rank's device tables and their upload: one native call on
        the planning critical path (fssdp_plan_layer_tables).  `counts` is the (D, E) int32
        host array at counts_ptr.  decide=False defers the LayerDecision to
        last_decision(layer) (callable until this layer is planned again)."""
        args = self.plan_call_args(layer, counts.shape, counts_ptr, rank, pre_ptr, d_model, d_ff,
                                   blob, blob_ptr, header_ptr, blob_dev_ptr, stream, limits_ptr,
                                   n_mats)
        self.plan_counts(layer, counts)
        N.check(N.LIB_RAW.fssdp_plan_layer_tables(*args), "plan_layer_tables")
        return self.last_decision(layer) if decide else None

    def plan_call_args(self, layer: int, counts_shape, counts_ptr: int, rank: int, pre_ptr,
                       d_model: int, d_ff: int, blob, blob_ptr: int, header_ptr: int,
                       blob_dev_ptr, stream, limits_ptr=None, n_mats: int = 2) -> tuple:
        """The fssdp_plan_layer_tables argument list of this layer's plan — everything that
        does not need the counts, so it can be built before they arrive.  Call
        plan_counts(layer, counts) once the counts are in."""
        if self._step is None:
            self.begin_iteration()
            self._step = [None] * self.config.layers
        base = self.shards.per_layer[layer]
        E, D = base.num_chunks, base.num_devices
        if tuple(counts_shape) != (D, E):
            raise TraceMismatchError(f"counts {tuple(counts_shape)} do not match {D} devices x {E} experts")
        sc = self._scratch(layer)
        knobs, est_ptr = self._layer_knobs(layer)
        self._knobs_keep = knobs  # alive until the native call has read it
        self.last_target_ptr, self.last_route_ptr = sc.p_target, sc.p_route
        return (E, self._owners_ptr(layer), est_ptr, counts_ptr, sc.topo_ref(self._topo_c),
                N.C.byref(knobs), rank, pre_ptr, d_model, d_ff, n_mats, limits_ptr, sc.p_target,
                sc.p_added, sc.p_route, sc.p_dbl, sc.p_flags, blob_ptr, len(blob), header_ptr,
                blob_dev_ptr, stream)

    def plan_counts(self, layer: int, counts) -> None:
        """Record this iteration's (D, E) counts of `layer` (history push at the end)."""
        self._step[layer] = np.asarray(counts).astype(np.int64)

    def last_decision(self, layer: int) -> LayerDecision:
        """The LayerDecision of the layer's most recent plan_with_tables(decide=False)."""
        return self._decision(self.shards.per_layer[layer], self._scratch(layer))

    def _owners_ptr(self, layer: int) -> int:
        self._owners(layer)  # refreshes the cache for the current ShardPlan
        if getattr(self, "_owners_ptrs_plan", None) is not self.shards:
            self._owners_ptrs = [row.ctypes.data for row in self._owners_cache]
            self._owners_ptrs_plan = self.shards
        return self._owners_ptrs[layer]

    def _estimate_ptr(self, layer: int):
        if self.estimate(layer) is None:
            return None
        return self._est_cache[layer][2]

    def end_iteration(self, step: Sequence[np.ndarray]) -> None:
        """Push this iteration's counts into the history window (engine.py:353-356)."""
        if len(step) != self.config.layers:
            raise TraceMismatchError(
                f"step has {len(step)} layers, config declares {self.config.layers}")
        for l, counts in enumerate(step):
            self.history[l].append(np.asarray(counts, dtype=np.int64))
        if self.recorder is not None:
            self.recorder.push(step)
        self.iteration += 1

    def candidate(self, layer: int) -> Optional[np.ndarray]:
        """The estimate-based, adoption-gated target mask (E, D) of the coming iteration, or
        None when it is the bare partition — known BEFORE the gate, so its SpAG can start
        early (engine.py:497-501; calibration may only extend it, fallback drops it)."""
        if self.policy.kind != PolicyKind.FSSDP:
            return None
        if self._step is None and self._reshard_pending():
            return None  # the re-shard decision of this iteration comes first
        est_ptr = self._estimate_ptr(layer)
        if est_ptr is None:
            return None
        base = self.shards.per_layer[layer]
        E, D = base.num_chunks, base.num_devices
        target = np.zeros((E, D), dtype=np.uint8)
        adopted = np.zeros(1, dtype=np.int32)
        N.check(N.LIB_RAW.fssdp_plan_candidate(E, self._owners_ptr(layer), est_ptr,
                                               N.C.byref(self._topo_c), N.C.byref(self._knobs),
                                               target.ctypes.data, adopted.ctypes.data),
                "plan_candidate")
        return target if adopted[0] else None

    def _reshard_pending(self) -> bool:
        return (self.iteration > 0 and self.policy.reshard_interval > 0
                and self.iteration % self.policy.reshard_interval == 0 and all(self.history))

    # -- layer-driven protocol (used by FssdpMoE) ---------------------------------
    def plan(self, layer: int, actual) -> LayerDecision:
        """plan_layer for a live layer; the first call of an iteration runs the re-shard
        trigger, `finish()` closes the iteration with the counts seen."""
        if self._step is None:
            self.begin_iteration()
            self._step = [None] * self.config.layers
        self._step[layer] = np.asarray(actual, dtype=np.int64)
        return self.plan_layer(layer, actual)

    def finish(self) -> None:
        if self._step is None:
            return
        step = self._step
        self._step = None
        if any(s is None for s in step):
            raise TraceMismatchError("iteration finished before every layer was planned")
        self.end_iteration(step)

    def run_iteration(self, step: Sequence[np.ndarray]) -> list:
        """All layers of one iteration from a recorded step (trace replay)."""
        if len(step) != self.config.layers:
            raise TraceMismatchError(
                f"step has {len(step)} layers, config declares {self.config.layers}")
        self.begin_iteration()
        out = [self.plan_layer(l, counts) for l, counts in enumerate(step)]
        self.end_iteration(step)
        return out

    def memory(self, decisions) -> MemoryBreakdown:
        mode = "rematerialize" if self.policy.rematerialize else "retain"
        return memory_report(self.shards, [d.materialization for d in decisions], self.config, mode)


def make_policy_state(config: ModelConfig, topology, policy: Policy) -> FssdpPlanner:
    """Drop-in for moesim's make_policy_state (engine.py:751-758) on the executed path:
    the FSSDP (or EP) control state.  `run_iteration(step)` advances it by one iteration of
    gate counts exactly like FssdpState / EPState (engine.py:457-557) and returns the
    per-layer LayerDecisions the kernels execute (placement, route, priced SpAG/SpRS
    latencies) instead of the simulator's IterationTimeline; `memory(decisions)` gives
    the iteration's MemoryBreakdown.  The simulated comparison policies are not executed."""
    kind = getattr(policy, "kind", None)
    if kind not in (PolicyKind.FSSDP, PolicyKind.EP):
        raise ConfigError(f"unknown policy kind {kind!r}")
    return FssdpPlanner(config, topology, policy)
