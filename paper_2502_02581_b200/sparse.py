"""SparseAllGather / SparseReduceScatter entry points (the paper's two sparse collectives,
PAPER.md:370-386; moesim prices them as spag_traffic / sprs_traffic, costmodel.py:87-132).

The reference's contract is a pair of ChunkPlacements:

* SpAG(pre, post): `pre` is a partition, pre ⊆ post (validate_spag_pair,
  placement.py:200-204); every (chunk, device) in post − pre receives the owner's copy.
* SpRS(pre, post): `post` is a partition, post ⊆ pre (validate_sprs_pair,
  placement.py:207-211); every owner in post ends with the sum of all pre holders'
  partials, in ascending device order (fp32 chunks, or bf16 chunks summed in fp32).

Here they move real bytes: chunks live in a `ChunkBuffer` — `slots` chunk-sized slots at
the same offset of every rank's symmetric heap (comm.py) — and the transfers are the
sm_100a pull kernels of libfssdp (fssdp_spag: TMA bulk copies from the owner's HBM over
NVSwitch; fssdp_sprs_pull: the owner pulls every holder's partial through a TMA ring and
sums in registers).  No NCCL call is made on either collective.

Slot convention (`chunk_slots`), identical on every rank so no table is exchanged: the
partition's chunks on a device (ascending id) first, then the device's other chunks of the
non-partition placement (ascending id) — the layout FssdpMoE uses for owned + replica
slots (csrc/planner.cpp fssdp_build_rank_tables).  Under SpAG the pre slots are a prefix of the post slots;
under SpRS the post (owned) slots are a prefix of the pre slots.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import _native as N
from .comm import PeerGroup
from .costmodel import SparsityReport, spag_traffic, sprs_traffic
from .errors import DimensionError
from .placement import ChunkPlacement

# flag-pad barrier slot of the standalone collectives (layers use slots 0..63, 8 each)
BAR_SPARSE = 64


@dataclass(frozen=True)
class ChunkBuffer:
    """`slots` chunks of `chunk_bytes` at heap offset `offset` on every rank of `group`."""

    group: PeerGroup
    offset: int
    chunk_bytes: int
    slots: int

    def __post_init__(self) -> None:
        if self.chunk_bytes <= 0 or self.chunk_bytes % 16 or self.slots <= 0:
            raise DimensionError("chunk_bytes must be a positive multiple of 16, slots > 0")
        end = self.offset + self.slots * self.chunk_bytes
        if self.offset % 16 or end > self.group.local.nbytes:
            raise DimensionError("chunk buffer outside the symmetric heap")

    def view(self, dtype: torch.dtype = torch.uint8, rank: int | None = None) -> torch.Tensor:
        """[slots, chunk elements] view of this rank's buffer (or of `rank`'s, emulated)."""
        heap = self.group.local if rank is None else self.group.heap_of(rank)
        el = torch.empty(0, dtype=dtype).element_size()
        if self.chunk_bytes % el:
            raise DimensionError(f"chunk_bytes not a multiple of {dtype} elements")
        return heap.tensor(self.offset, (self.slots, self.chunk_bytes // el), dtype)


def chunk_slots(partition: ChunkPlacement, other: ChunkPlacement, device: int) -> dict:
    """{chunk: slot} on `device`: partition chunks first, then `other`'s extra chunks."""
    own = sorted(partition.chunks_on(device))
    extra = sorted(set(other.chunks_on(device)) - set(own))
    return {e: s for s, e in enumerate(own + extra)}


def _dims(pre: ChunkPlacement, post: ChunkPlacement, buf: ChunkBuffer) -> None:
    if pre.num_devices != buf.group.world:
        raise DimensionError(f"placements span {pre.num_devices} devices, the group has "
                             f"{buf.group.world} ranks")


def spag_copies(pre: ChunkPlacement, post: ChunkPlacement, rank: int) -> np.ndarray:
    """int32 [n, 3] {src_rank, src_slot, dst_slot}: the chunks `rank` receives, ascending."""
    mine = chunk_slots(pre, post, rank)
    rows = []
    for e in sorted(set(post.chunks_on(rank)) - set(pre.chunks_on(rank))):
        src = pre.owner(e)
        rows.append((src, chunk_slots(pre, post, src)[e], mine[e]))
    return np.asarray(rows, dtype=np.int32).reshape(-1, 3)


def sprs_schedule(pre: ChunkPlacement, post: ChunkPlacement, rank: int):
    """(jobs int32 [n, 3] {dst_slot, src_begin, src_count}, srcs int32 [m, 2] {rank, slot}):
    per chunk `rank` owns in post with other holders in pre, every holder ascending."""
    jobs, srcs = [], []
    for e in sorted(post.chunks_on(rank)):
        holders = sorted(pre.devices_of(e))
        if holders == [rank]:
            continue
        jobs.append((chunk_slots(post, pre, rank)[e], len(srcs), len(holders)))
        srcs += [(h, chunk_slots(post, pre, h)[e]) for h in holders]
    return (np.asarray(jobs, dtype=np.int32).reshape(-1, 3),
            np.asarray(srcs, dtype=np.int32).reshape(-1, 2))


def _slots_fit(pre, post, buf, partition) -> None:
    other = post if partition is pre else pre
    need = max(len(chunk_slots(partition, other, d)) for d in range(buf.group.world))
    if need > buf.slots:
        raise DimensionError(f"placement needs {need} slots per rank, buffer has {buf.slots}")


def _barrier(group: PeerGroup, stream) -> None:
    slot, epoch = group.barrier_args(BAR_SPARSE)
    if slot >= 0:
        N.call("fssdp_barrier", C.c_void_p(group.peer_bases.data_ptr()),
               group.layout.offset("flags"), group.rank, group.world, slot, C.c_uint32(epoch),
               stream)


def _stream(stream, device) -> torch.cuda.Stream:
    return stream if stream is not None else torch.cuda.current_stream(device)


def _upload(arr: np.ndarray, st: torch.cuda.Stream) -> torch.Tensor:
    """A small host table to the device, stream-ordered before the kernel that reads it."""
    with torch.cuda.stream(st):
        t = torch.from_numpy(arr).to(st.device, non_blocking=False)
    t.record_stream(st)
    return t


def sparse_all_gather(pre: ChunkPlacement, post: ChunkPlacement, buf: ChunkBuffer, *,
                      stream=None, fence: bool = True) -> SparsityReport:
    """SpAG(pre → post) on this rank: pull every chunk of post − pre from its owner.

    Raises InvalidPairError when (pre, post) violates the SpAG contract.  fence=True
    (multi-process) puts a device barrier before the pulls (every owner's chunk is final)
    and after them (no owner overwrites a chunk a peer is still reading).  Returns the
    reference's SparsityReport of the transfer (spag_traffic)."""
    # the pair contract first: InvalidPairError with the reference's message
    # (costmodel.py:96-97) before any device work
    spag_traffic(pre, post, 1)
    _dims(pre, post, buf)
    report = spag_traffic(pre, post, buf.chunk_bytes)[1]
    _slots_fit(pre, post, buf, pre)
    g = buf.group
    st = _stream(stream, g.device)
    s = C.c_void_p(st.cuda_stream)
    copies = spag_copies(pre, post, g.rank)
    if fence:
        _barrier(g, s)
    if len(copies):
        tab = _upload(copies, st)
        N.call("fssdp_spag", C.c_void_p(g.peer_bases.data_ptr()), g.rank, buf.offset,
               buf.chunk_bytes, C.c_void_p(tab.data_ptr()), len(copies), s)
    if fence:
        _barrier(g, s)
    return report


def sparse_reduce_scatter(pre: ChunkPlacement, post: ChunkPlacement, buf: ChunkBuffer, *,
                          stream=None, fence: bool = True,
                          dtype: torch.dtype = torch.float32) -> SparsityReport:
    """SpRS(pre → post) on this rank: for every chunk this rank owns in post, its slot
    becomes the sum of every pre holder's partial (ascending device order; the owner's own
    partial included).  dtype: the chunks' elements — float32, or bfloat16 (summed in fp32,
    rounded once: the layer's bf16 gradients).

    Raises InvalidPairError when (pre, post) violates the SpRS contract.  fence: barriers
    before (every holder's partial complete) and after (holders may reuse their slots).
    Returns the reference's SparsityReport (sprs_traffic, bytes of this buffer)."""
    sprs_traffic(pre, post, 1)  # the pair contract first (costmodel.py:120-121)
    _dims(pre, post, buf)
    report = sprs_traffic(pre, post, buf.chunk_bytes)[1]
    _slots_fit(pre, post, buf, post)
    if dtype not in (torch.float32, torch.bfloat16):
        raise DimensionError(f"SpRS chunks are float32 or bfloat16, not {dtype}")
    esize = 4 if dtype == torch.float32 else 2
    g = buf.group
    st = _stream(stream, g.device)
    s = C.c_void_p(st.cuda_stream)
    jobs, srcs = sprs_schedule(pre, post, g.rank)
    if fence:
        _barrier(g, s)
    if len(jobs):
        tj, ts = _upload(jobs, st), _upload(srcs, st)
        N.call("fssdp_sprs_pull", C.c_void_p(g.peer_bases.data_ptr()), g.rank, buf.offset,
               buf.chunk_bytes // esize, esize, C.c_void_p(tj.data_ptr()), len(jobs),
               C.c_void_p(ts.data_ptr()), s)
    if fence:
        _barrier(g, s)
    return report
