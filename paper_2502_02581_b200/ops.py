"""Torch-facing wrappers of the device entry points in include/fssdp.h.

PyTorch is plumbing here: it owns device memory and streams; every kernel is one of
libfssdp's sm_100a kernels, reached through the C-ABI with raw pointers.  There is no
eager fallback — a missing library or a non-CUDA tensor raises.
"""

from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _native as N
from .errors import DimensionError

GATE_TILE = 64
BM, BN, BK = 128, 256, 64
EPI_BF16, EPI_GELU, EPI_DGELU, EPI_F32, EPI_SWIGLU, EPI_DSWIGLU = 0, 1, 2, 3, 4, 5
GEMM_N_FASTEST, GEMM_CTA_PAIR, GEMM_BN128, GEMM_MULTICAST, GEMM_SPLIT_TAIL = 1, 2, 4, 8, 16
GEMM_SWAP_TAIL = 32


def _stream(stream: torch.cuda.Stream | None = None) -> C.c_void_p:
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def _ptr(t: torch.Tensor | None) -> C.c_void_p:
    if t is None:
        return C.c_void_p(0)
    if not t.is_cuda:
        raise DimensionError("FSSDP device ops need CUDA tensors (no CPU fallback)")
    return C.c_void_p(t.data_ptr())


def _need(t: torch.Tensor, dtype: torch.dtype, name: str) -> None:
    if t.dtype != dtype or not t.is_contiguous() or not t.is_cuda:
        raise DimensionError(f"{name}: expected contiguous CUDA {dtype}, got {t.dtype} "
                             f"{'contiguous' if t.is_contiguous() else 'strided'} on {t.device}")


# ------------------------------------------------------------------ grouped GEMM
# fssdp_gemm_group (include/fssdp.h): c_dest 0 = C, r + 1 = c_dest_maps[r]
GROUP_DTYPE = np.dtype([("m_tiles", "<i4"), ("tile_start", "<i4"), ("a_m", "<i4"), ("a_k", "<i4"),
                        ("b_n", "<i4"), ("b_k", "<i4"), ("k_blocks", "<i4"), ("c_dest", "<i4"),
                        ("c_off", "<i8"), ("rows", "<i4"), ("reserved", "<i4")])


def finalize_groups(groups_cpu: np.ndarray, n_tiles: int) -> int:
    """Fill tile_start in place for a structured group array; return total tiles."""
    tiles = groups_cpu["m_tiles"].astype(np.int64) * n_tiles
    starts = np.concatenate([[0], np.cumsum(tiles)[:-1]])
    groups_cpu["tile_start"] = starts
    return int(tiles.sum())


def grouped_gemm(a: torch.Tensor, a_mn: bool, b: torch.Tensor, b_mn: bool, groups_dev: torch.Tensor,
                 num_groups: int, n_tiles: int, total_tiles: int, c: torch.Tensor, ldc: int,
                 epilogue: int = EPI_BF16, c2: torch.Tensor | None = None,
                 aux: torch.Tensor | None = None, stream=None, n_fastest: bool = False,
                 cta_pair: bool = False, c_dest_maps: torch.Tensor | None = None,
                 bn128: bool = False, dynamic: bool = False, multicast: bool = False,
                 split_tail: bool = False, swap_tail: bool = False) -> None:
    """C_g = A_g · B_g for every group (tcgen05 kernel, gemm_sm100.cu).

    a, b: 2-D bf16 tensors (the TMA view: [outer, inner], inner contiguous); c (and c2,
    aux) the whole output tensor, viewed as [numel // ldc, ldc].  c_dest_maps: device
    uint8 tensor of 128-byte tensor maps (epilogue_tmap) for groups with c_dest > 0.
    dynamic: tiles taken from a device counter (default: the static snake order, as the
    layer runs).  multicast: clusters of two CTA pairs sharing the A tile (needs cta_pair,
    n_fastest, an even n_tiles).  split_tail: a short last round of tiles runs as 256x128
    halves (FSSDP_GEMM_SPLIT_TAIL).  swap_tail: a group's short last M tile (the `rows`
    field) as a swapped-operand tile (FSSDP_GEMM_SWAP_TAIL)."""
    for t, nm in ((a, "A"), (b, "B")):
        _need(t, torch.bfloat16, nm)
        if t.dim() != 2:
            raise DimensionError(f"{nm} must be 2-D")
    if c.numel() % ldc:
        raise DimensionError("C must hold whole rows of ldc elements")
    N.call("fssdp_grouped_gemm", int(a_mn), int(b_mn), int(epilogue), _ptr(a), a.shape[1],
           a.shape[0], _ptr(b), b.shape[1], b.shape[0], _ptr(groups_dev), num_groups, n_tiles,
           total_tiles, _ptr(c), _ptr(c2), _ptr(aux), _ptr(c_dest_maps), ldc, c.numel() // ldc,
           (GEMM_N_FASTEST if n_fastest else 0) | (GEMM_CTA_PAIR if cta_pair else 0) |
           (GEMM_BN128 if bn128 else 0) | (GEMM_MULTICAST if multicast else 0) |
           (GEMM_SPLIT_TAIL if split_tail else 0) | (GEMM_SWAP_TAIL if swap_tail else 0),
           _sched(a.device) if dynamic else None, _stream(stream))


_SCHED: dict = {}


def _sched(device) -> C.c_void_p:
    """Per-device tile-scheduler counters for grouped_gemm (left zero by every launch)."""
    key = torch.device(device).index
    t = _SCHED.get(key)
    if t is None:
        t = _SCHED[key] = torch.zeros(2, dtype=torch.int32, device=device)
    return C.c_void_p(t.data_ptr())


def epilogue_tmap(epilogue: int, base_ptr: int, ldc: int, rows: int) -> bytes:
    """The 128-byte epilogue tensor map of C = [rows][ldc] at device address base_ptr."""
    out = (C.c_uint8 * 128)()
    N.call("fssdp_epilogue_tmap", int(epilogue), C.c_void_p(base_ptr), ldc, rows, out)
    return bytes(out)


# ------------------------------------------------------------------ gate
def gate_topk(x: torch.Tensor, wg: torch.Tensor, k: int, want_logits: bool = False, stream=None,
              bias: torch.Tensor | None = None):
    """K1: returns (topk_idx [T,k] i32, topk_w [T,k] f32, slot_rank [T,k] i32,
    tile_counts [tiles,E] i32, logits [T,E] f32 | None)."""
    _need(x, torch.bfloat16, "x")
    _need(wg, torch.float32, "wg")
    T, d = x.shape
    E = wg.shape[0]
    dev = x.device
    tiles = (T + GATE_TILE - 1) // GATE_TILE
    idx = torch.empty(T, k, dtype=torch.int32, device=dev)
    w = torch.empty(T, k, dtype=torch.float32, device=dev)
    rank = torch.empty(T, k, dtype=torch.int32, device=dev)
    tc = torch.empty(max(tiles, 1), E, dtype=torch.int32, device=dev)
    logits = torch.empty(T, E, dtype=torch.float32, device=dev) if want_logits else None
    if bias is not None:
        _need(bias, torch.float32, "bias")
    N.call("fssdp_gate_topk", _ptr(x), _ptr(wg), _ptr(bias), T, d, E, k, _ptr(logits), _ptr(idx),
           _ptr(w),
           _ptr(rank), _ptr(tc), _stream(stream))
    return idx, w, rank, tc, logits


def topk_from_logits(logits: torch.Tensor, k: int, stream=None):
    _need(logits, torch.float32, "logits")
    T, E = logits.shape
    dev = logits.device
    tiles = (T + GATE_TILE - 1) // GATE_TILE
    idx = torch.empty(T, k, dtype=torch.int32, device=dev)
    w = torch.empty(T, k, dtype=torch.float32, device=dev)
    rank = torch.empty(T, k, dtype=torch.int32, device=dev)
    tc = torch.empty(max(tiles, 1), E, dtype=torch.int32, device=dev)
    N.call("fssdp_topk_from_logits", _ptr(logits), T, E, k, _ptr(idx), _ptr(w), _ptr(rank),
           _ptr(tc), _stream(stream))
    return idx, w, rank, tc
