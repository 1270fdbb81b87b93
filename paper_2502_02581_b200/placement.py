"""Chunk placements and the SpAG/SpRS pair contracts (moesim placement.py:31-290).

`ChunkPlacement` keeps the reference's constructor, queries and canonical JSON, but is
stored as a dense (chunks × devices) boolean mask — the form the C-ABI planner and the
device plan tables consume.  `entries` is still available as a frozenset of
(chunk, device) pairs for drop-in callers.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Iterable, Optional

import numpy as np

from . import _native as N
from .errors import DimensionError, DimensionMismatchError, InternalError

MISSING_CHUNK = "missing_chunk"
DUPLICATE_OWNER = "duplicate_owner"
DROPPED_ENTRY = "dropped_entry"
_REASONS = {1: MISSING_CHUNK, 2: DUPLICATE_OWNER, 3: DROPPED_ENTRY}


@dataclass(frozen=True)
class Verdict:
    """First violation of a pair contract, or ok (placement.py:31-48)."""

    ok: bool
    reason: Optional[str] = None
    chunk: Optional[int] = None
    device: Optional[int] = None

    def describe(self) -> str:
        if self.ok:
            return "valid"
        words = [self.reason or "invalid"]
        if self.chunk is not None:
            words.append(f"chunk={self.chunk}")
        if self.device is not None:
            words.append(f"device={self.device}")
        return " ".join(words)


class ChunkPlacement:
    """Immutable set of (chunk, device) replica entries (placement.py:54-152)."""

    __slots__ = ("num_chunks", "num_devices", "_mask", "_entries", "_hash")

    def __init__(self, num_chunks: int, num_devices: int, entries: Iterable = ()) -> None:
        if num_chunks < 0 or num_devices <= 0:
            raise DimensionError(
                f"placement needs num_chunks >= 0 and num_devices > 0, got "
                f"{num_chunks}/{num_devices}"
            )
        mask = np.zeros((num_chunks, num_devices), dtype=np.uint8)
        for c, d in entries:
            c, d = int(c), int(d)
            if not 0 <= c < num_chunks:
                raise DimensionError(f"chunk {c} out of range [0, {num_chunks})")
            if not 0 <= d < num_devices:
                raise DimensionError(f"device {d} out of range [0, {num_devices})")
            mask[c, d] = 1
        self._init(num_chunks, num_devices, mask)

    def _init(self, C: int, D: int, mask: np.ndarray) -> None:
        mask.setflags(write=False)
        object.__setattr__(self, "num_chunks", int(C))
        object.__setattr__(self, "num_devices", int(D))
        object.__setattr__(self, "_mask", mask)
        object.__setattr__(self, "_entries", None)
        object.__setattr__(self, "_hash", None)

    def __setattr__(self, name, value):
        raise AttributeError("ChunkPlacement is immutable")

    # -- construction -------------------------------------------------------
    @classmethod
    def from_pairs(cls, num_chunks: int, num_devices: int, pairs: Iterable) -> "ChunkPlacement":
        return cls(num_chunks, num_devices, pairs)

    @classmethod
    def from_mask(cls, mask: np.ndarray, copy: bool = True) -> "ChunkPlacement":
        """`copy=False` adopts a fresh 0/1 uint8 array the caller will not touch again."""
        if copy or not (isinstance(mask, np.ndarray) and mask.dtype == np.uint8
                        and mask.flags.c_contiguous):
            m = np.ascontiguousarray(np.asarray(mask) != 0, dtype=np.uint8)
            if copy:
                m = m.copy()
        else:
            m = mask
        if m.ndim != 2 or m.shape[1] <= 0:
            raise DimensionError(f"placement mask must be (chunks, devices), got {m.shape}")
        obj = cls.__new__(cls)
        obj._init(m.shape[0], m.shape[1], m)
        return obj

    @classmethod
    def from_owner(cls, owner, num_devices: int) -> "ChunkPlacement":
        owner = np.asarray(owner, dtype=np.int64)
        m = np.zeros((len(owner), num_devices), dtype=np.uint8)
        m[np.arange(len(owner)), owner] = 1
        return cls.from_mask(m)

    def union(self, extra: Iterable) -> "ChunkPlacement":
        other = ChunkPlacement(self.num_chunks, self.num_devices, extra)
        return ChunkPlacement.from_mask(self._mask | other._mask)

    # -- views ----------------------------------------------------------------
    @property
    def mask(self) -> np.ndarray:
        """Read-only (chunks, devices) uint8 mask, C-contiguous."""
        return self._mask

    @property
    def entries(self) -> frozenset:
        if self._entries is None:
            cs, ds = np.nonzero(self._mask)
            object.__setattr__(self, "_entries", frozenset(zip(cs.tolist(), ds.tolist())))
        return self._entries

    def devices_of(self, chunk: int) -> frozenset:
        return frozenset(np.flatnonzero(self._mask[chunk]).tolist())

    def chunks_on(self, device: int) -> frozenset:
        return frozenset(np.flatnonzero(self._mask[:, device]).tolist())

    def owner(self, chunk: int) -> int:
        holders = np.flatnonzero(self._mask[chunk])
        if len(holders) != 1:
            raise InternalError(f"chunk {chunk} has {len(holders)} holders, expected 1")
        return int(holders[0])

    def owners(self) -> np.ndarray:
        """owner per chunk (partitions only), int32."""
        if not self.is_partition():
            raise InternalError("owners() needs a partition")
        return np.argmax(self._mask, axis=1).astype(np.int32)

    def replica_counts(self) -> list[int]:
        return self._mask.sum(axis=1).astype(int).tolist()

    def counts_per_device(self) -> list[int]:
        return self._mask.sum(axis=0).astype(int).tolist()

    def is_partition(self) -> bool:
        return bool(np.all(self._mask.sum(axis=1) == 1))

    def issubset(self, other: "ChunkPlacement") -> bool:
        return bool(np.all(other._mask[self._mask != 0] != 0))

    # -- serialization ----------------------------------------------------------
    def sorted_pairs(self) -> list[list[int]]:
        cs, ds = np.nonzero(self._mask)  # row-major = sorted by (chunk, device)
        return [[int(c), int(d)] for c, d in zip(cs, ds)]

    def to_json_obj(self) -> dict:
        return {"num_chunks": self.num_chunks, "num_devices": self.num_devices,
                "entries": self.sorted_pairs()}

    @classmethod
    def from_json_obj(cls, obj: dict) -> "ChunkPlacement":
        try:
            return cls.from_pairs(int(obj["num_chunks"]), int(obj["num_devices"]), obj["entries"])
        except (KeyError, TypeError, ValueError) as exc:
            raise DimensionError(f"malformed placement object: {exc}") from exc

    # -- value semantics --------------------------------------------------------
    def __eq__(self, other) -> bool:
        return (isinstance(other, ChunkPlacement) and self.num_chunks == other.num_chunks
                and self.num_devices == other.num_devices
                and np.array_equal(self._mask, other._mask))

    def __hash__(self) -> int:
        if self._hash is None:
            object.__setattr__(self, "_hash", hash((self.num_chunks, self.num_devices,
                                                    self._mask.tobytes())))
        return self._hash

    def __repr__(self) -> str:
        return (f"ChunkPlacement(num_chunks={self.num_chunks}, num_devices={self.num_devices}, "
                f"entries={self.sorted_pairs()})")


def make_even_partition(num_chunks: int, topology) -> ChunkPlacement:
    """Contiguous single-owner partition, remainder to low devices (placement.py:155-170)."""
    D = topology.num_devices
    owner = np.empty(max(num_chunks, 0), dtype=np.int32)
    N.check(N.LIB.fssdp_make_even_partition(num_chunks, D, owner.ctypes.data_as(N.P_i32)),
            "make_even_partition")
    return ChunkPlacement.from_owner(owner, D)


def _same_dims(pre: ChunkPlacement, post: ChunkPlacement) -> None:
    if pre.num_chunks != post.num_chunks or pre.num_devices != post.num_devices:
        raise DimensionMismatchError(
            f"placement pair dimensions differ: {pre.num_chunks}x{pre.num_devices} vs "
            f"{post.num_chunks}x{post.num_devices}"
        )


def _verdict(kind: int, pre: ChunkPlacement, post: ChunkPlacement) -> Verdict:
    _same_dims(pre, post)
    out = np.zeros(3, dtype=np.int32)
    N.check(N.LIB.fssdp_validate_pair(kind, pre.num_chunks, pre.num_devices,
                                      pre.mask.ctypes.data_as(N.P_u8),
                                      post.mask.ctypes.data_as(N.P_u8),
                                      out.ctypes.data_as(N.P_i32)), "validate_pair")
    if out[0] == 0:
        return Verdict(ok=True)
    return Verdict(ok=False, reason=_REASONS[int(out[0])],
                   chunk=None if out[1] < 0 else int(out[1]),
                   device=None if out[2] < 0 else int(out[2]))


def validate_spag_pair(pre: ChunkPlacement, post: ChunkPlacement) -> Verdict:
    """SparseAllGather contract: pre is a partition and pre ⊆ post (placement.py:200-204)."""
    return _verdict(0, pre, post)


def validate_sprs_pair(pre: ChunkPlacement, post: ChunkPlacement) -> Verdict:
    """SparseReduceScatter contract: post is a partition and post ⊆ pre (placement.py:207-211)."""
    return _verdict(1, pre, post)


class ShardPlan:
    """Per-layer ownership partitions with exact slot totals (placement.py:214-290)."""

    __slots__ = ("per_layer", "slots_per_device")

    def __init__(self, per_layer, slots_per_device: int) -> None:
        layers = tuple(per_layer)
        if not layers:
            raise DimensionError("shard plan needs at least one layer")
        D = layers[0].num_devices
        counts = np.zeros(D, dtype=np.int64)
        total = 0
        for i, p in enumerate(layers):
            if p.num_devices != D:
                raise DimensionError(f"layer {i} has a different device count")
            if not p.is_partition():
                raise InternalError(f"layer {i} placement is not a partition")
            total += p.num_chunks
            counts += np.asarray(p.counts_per_device(), dtype=np.int64)
        base, extra = divmod(total, D)
        for d in range(D):
            want = base + (1 if d < extra else 0)
            if counts[d] != want:
                raise InternalError(f"device {d} owns {counts[d]} chunks, slot target is {want}")
        object.__setattr__(self, "per_layer", layers)
        object.__setattr__(self, "slots_per_device", int(slots_per_device))

    def __setattr__(self, name, value):
        raise AttributeError("ShardPlan is immutable")

    @property
    def num_layers(self) -> int:
        return len(self.per_layer)

    @property
    def num_devices(self) -> int:
        return self.per_layer[0].num_devices

    def owners(self) -> np.ndarray:
        """(layers, experts) int32 owner table."""
        return np.stack([p.owners() for p in self.per_layer])

    @classmethod
    def from_owners(cls, owners: np.ndarray, num_devices: int) -> "ShardPlan":
        owners = np.asarray(owners, dtype=np.int32)
        L, E = owners.shape
        return cls(tuple(ChunkPlacement.from_owner(owners[l], num_devices) for l in range(L)),
                   (L * E) // num_devices)

    @classmethod
    def even(cls, layers: int, experts: int, topology) -> "ShardPlan":
        """Contiguous partition per layer; remainder window rotates (placement.py:260-284)."""
        D = topology.num_devices
        if layers <= 0:
            raise DimensionError("shard plan needs at least one layer")
        owners = np.empty((layers, experts), dtype=np.int32)
        N.check(N.LIB.fssdp_shard_plan_even(layers, experts, D, owners.ctypes.data_as(N.P_i32)),
                "ShardPlan.even")
        return cls.from_owners(owners, D)

    def to_json_obj(self) -> dict:
        return {"slots_per_device": self.slots_per_device,
                "layers": [p.to_json_obj() for p in self.per_layer]}

    def __eq__(self, other) -> bool:
        return (isinstance(other, ShardPlan) and self.slots_per_device == other.slots_per_device
                and self.per_layer == other.per_layer)

    def __hash__(self) -> int:
        return hash((self.per_layer, self.slots_per_device))
