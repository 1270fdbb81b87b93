"""Symmetric heap and peer table (the NVSwitch P2P plumbing of the FSSDP kernels).

Each rank cudaMallocs one heap (fssdp_heap_alloc) and carves it with the SAME
deterministic bump allocation, so a buffer sits at the same offset on every rank and
a peer's copy is  peer_bases[r] + offset.  Multi-process: heaps are exchanged once as
CUDA IPC handles over torch.distributed (bootstrap only — no NCCL on the data path).
Single-process emulation: N heaps on one GPU, one per logical rank, used by the
parity tests to exercise every cross-rank code path without N GPUs.
"""

from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _native as N
from .errors import DeviceError

ALIGN = 4096
FLAG_SLOTS = 80  # 8 barrier slots per layer (<= 8 layers), 64: standalone collectives,
#                  72 + layer: owner-update epochs
MAX_WORLD = 32


class _CAI:
    """Minimal __cuda_array_interface__ exporter for a raw device pointer."""

    def __init__(self, ptr: int, nbytes: int):
        self.__cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1",
                                         "data": (ptr, False), "version": 3, "strides": None}


def view_bytes(ptr: int, nbytes: int, device) -> torch.Tensor:
    if nbytes == 0:
        return torch.empty(0, dtype=torch.uint8, device=device)
    return torch.as_tensor(_CAI(ptr, nbytes), device=device)


class HeapLayout:
    """Deterministic bump allocator of heap offsets (identical on every rank).

    guard > 0 (tests; compute-sanitizer is closed on the GPU pool) puts `guard` canary
    bytes after every region: Heap.fill_guards / check_guards then catch any kernel that
    writes past the end of a heap buffer — a peer's or its own."""

    GUARD_BYTE = 0xA5

    def __init__(self, guard: int = 0):
        self.size = 0
        self.guard = (int(guard) + ALIGN - 1) // ALIGN * ALIGN
        self.regions: dict[str, tuple[int, int]] = {}
        self.guards: list[tuple[str, int, int]] = []
        self.add("flags", FLAG_SLOTS * MAX_WORLD * 4)

    def add(self, name: str, nbytes: int) -> int:
        off = (self.size + ALIGN - 1) // ALIGN * ALIGN
        self.regions[name] = (off, int(nbytes))
        self.size = off + int(nbytes)
        if self.guard:
            g = (self.size + ALIGN - 1) // ALIGN * ALIGN
            self.guards.append((name, g, self.guard))
            self.size = g + self.guard
        return off

    def offset(self, name: str) -> int:
        return self.regions[name][0]


class Heap:
    """One rank's symmetric heap."""

    def __init__(self, nbytes: int, device):
        self.device = torch.device(device)
        p = C.c_void_p()
        with torch.cuda.device(self.device):
            N.call("fssdp_heap_alloc", C.c_size_t(max(int(nbytes), 1)), C.byref(p))
        self.ptr = int(p.value)
        self.nbytes = int(nbytes)
        self._bytes = view_bytes(self.ptr, self.nbytes, self.device)

    def tensor(self, offset: int, shape, dtype: torch.dtype) -> torch.Tensor:
        n = int(np.prod(shape)) * torch.empty(0, dtype=dtype).element_size()
        return self._bytes[offset:offset + n].view(dtype).view(*shape)

    def fill_guards(self, layout: HeapLayout) -> None:
        for _, off, n in layout.guards:
            self._bytes[off:off + n].fill_(HeapLayout.GUARD_BYTE)

    def check_guards(self, layout: HeapLayout) -> list:
        """Names of the regions whose trailing canary was overwritten."""
        return [name for name, off, n in layout.guards
                if not bool((self._bytes[off:off + n] == HeapLayout.GUARD_BYTE).all())]

    def ipc_handle(self) -> bytes:
        buf = (C.c_uint8 * 64)()
        N.call("fssdp_ipc_handle", C.c_void_p(self.ptr), buf)
        return bytes(buf)

    def free(self) -> None:
        if self.ptr:
            self._bytes = None
            N.LIB.fssdp_heap_free(C.c_void_p(self.ptr))
            self.ptr = 0


class PeerGroup:
    """world_size heaps reachable from this process, plus the device peer table.

    mode "dist": one rank per process, peers mapped via CUDA IPC.
    mode "emulated": `world` heaps in this process on one GPU (barriers are skipped;
    the driver runs the ranks' phases in lockstep)."""

    def __init__(self, layout: HeapLayout, rank: int, world: int, device, mode: str,
                 heaps=None, pg=None):
        self.layout, self.rank, self.world, self.mode = layout, rank, world, mode
        self.device = torch.device(device)
        self._opened = []
        if mode == "emulated":
            self.heaps = heaps
            bases = [h.ptr for h in heaps]
        elif mode == "dist":
            import torch.distributed as dist

            self.heaps = [Heap(layout.size, device)]
            if world > 1:
                handles = [None] * world
                dist.all_gather_object(handles, self.heaps[0].ipc_handle(), group=pg)
                bases = []
                for r, h in enumerate(handles):
                    if r == rank:
                        bases.append(self.heaps[0].ptr)
                        continue
                    p = C.c_void_p()
                    hb = (C.c_uint8 * 64).from_buffer_copy(h)
                    with torch.cuda.device(self.device):
                        N.call("fssdp_ipc_open", hb, C.byref(p))
                    self._opened.append(int(p.value))
                    bases.append(int(p.value))
            else:
                bases = [self.heaps[0].ptr]
        else:
            raise DeviceError(f"unknown peer-group mode {mode!r}")
        self.bases = bases
        self.peer_bases = torch.tensor(np.array(bases, dtype=np.uint64).view(np.int64),
                                       dtype=torch.int64, device=self.device)
        self.epochs = np.zeros(FLAG_SLOTS, dtype=np.int64)

    @property
    def local(self) -> Heap:
        return self.heaps[self.rank] if self.mode == "emulated" else self.heaps[0]

    def heap_of(self, rank: int) -> Heap:
        if self.mode != "emulated":
            raise DeviceError("only emulated groups hold every rank's heap")
        return self.heaps[rank]

    def next_epoch(self, slot: int) -> int:
        self.epochs[slot] += 1
        return int(self.epochs[slot] & 0xFFFFFFFF)

    def barrier_args(self, slot: int):
        """(slot, epoch) for a kernel-fused barrier; slot -1 disables it (emulation)."""
        if self.mode == "emulated" or self.world == 1:
            return -1, 0
        return slot, self.next_epoch(slot)

    def close(self) -> None:
        for p in self._opened:
            N.LIB.fssdp_ipc_close(C.c_void_p(p))
        self._opened = []
        if self.mode == "dist":
            self.heaps[0].free()


def emulated_group(layout: HeapLayout, world: int, device="cuda") -> list[PeerGroup]:
    """`world` logical ranks on one GPU: one heap each, shared peer table."""
    heaps = [Heap(layout.size, device) for _ in range(world)]
    return [PeerGroup(layout, r, world, device, "emulated", heaps=heaps) for r in range(world)]
