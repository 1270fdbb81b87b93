"""ctypes binding of libfssdp.so (include/fssdp.h).

The product path has no fallback: if the shared library is missing or a symbol is
absent, importing this module raises.  `build()` in __graft_entry__.py (or
`python paper_2502_02581_b200/build.py`) produces the library in-tree.
"""

from __future__ import annotations

import ctypes as C
import re
from pathlib import Path

from .errors import raise_for_status

import os

# FSSDP_LIB: an alternative build of the same library (diagnostics only, e.g. the GEMM
# role-wait counter variant of build.py --gemm-profile)
LIB_PATH = Path(os.environ.get("FSSDP_LIB", Path(__file__).resolve().parent / "libfssdp.so"))
HEADER = Path(__file__).resolve().parent.parent / "include" / "fssdp.h"

i32, i64, u32, f64, vp = C.c_int32, C.c_int64, C.c_uint32, C.c_double, C.c_void_p
P_i32 = C.POINTER(C.c_int32)
P_i64 = C.POINTER(C.c_int64)
P_u8 = C.POINTER(C.c_uint8)
P_f64 = C.POINTER(C.c_double)
P_f32 = C.POINTER(C.c_float)


class Topology(C.Structure):
    _fields_ = [
        ("nodes", C.c_int32),
        ("devices_per_node", C.c_int32),
        ("intra_bw", C.c_double),
        ("inter_bw", C.c_double),
        ("alpha", C.c_double),
    ]


class LayerKnobs(C.Structure):
    _fields_ = [
        ("t", C.c_int64),
        ("m", C.c_int64),
        ("calibration", C.c_int32),
        ("rematerialize", C.c_int32),
        ("expert_bytes", C.c_double),
        ("token_bytes", C.c_double),
        ("attn_fwd_time", C.c_double),
        ("per_token_expert_time", C.c_double),
    ]


class GemmGroup(C.Structure):
    _fields_ = [
        ("m_tiles", C.c_int32),
        ("tile_start", C.c_int32),
        ("a_m", C.c_int32),
        ("a_k", C.c_int32),
        ("b_n", C.c_int32),
        ("b_k", C.c_int32),
        ("k_blocks", C.c_int32),
        ("c_dest", C.c_int32),
        ("c_off", C.c_int64),
        ("rows", C.c_int32),
        ("reserved", C.c_int32),
    ]


P_topo = C.POINTER(Topology)


class DispatchLaunch(C.Structure):
    """fssdp_dispatch_launch (include/fssdp.h)."""
    _fields_ = [
        ("x", C.c_void_p), ("topk_idx", C.c_void_p), ("slot_rank", C.c_void_p),
        ("tile_prefix", C.c_void_p), ("T", C.c_int64), ("d_model", C.c_int32),
        ("E", C.c_int32), ("k", C.c_int32), ("world", C.c_int32), ("slot_dest", C.c_void_p),
        ("slot_pos", C.c_void_p), ("peer_bases", C.c_void_p), ("recv_off", C.c_int64),
        ("flags_off", C.c_int64), ("rank", C.c_int32), ("bar_slot", C.c_int32),
        ("epoch", C.c_uint32), ("grid_counter", C.c_void_p),
    ]

# name -> argtypes (every function returns int status unless listed in _RESTYPE)
_SIGS = {
    "fssdp_version": [],
    "fssdp_last_error": [],
    "fssdp_num_sms": [],
    # planner
    "fssdp_make_even_partition": [i32, i32, P_i32],
    "fssdp_shard_plan_even": [i32, i32, i32, P_i32],
    "fssdp_validate_pair": [i32, i32, i32, P_u8, P_u8, P_i32],
    "fssdp_spag_traffic": [i32, i32, P_u8, P_u8, f64, P_f64, P_f64],
    "fssdp_sprs_traffic": [i32, i32, P_u8, P_u8, f64, P_f64, P_f64],
    "fssdp_collective_latency": [i32, P_f64, P_topo, P_f64],
    "fssdp_overlap_degree": [f64, P_topo, f64, P_i64],
    "fssdp_build_dispatch": [i32, i32, P_i64, P_u8, P_topo, P_i64],
    "fssdp_estimate_moe_latency": [i32, i32, P_u8, P_i64, P_topo, f64, f64, P_f64],
    "fssdp_sparse_materialization": [i32, i32, P_u8, P_f64, i64, i64, P_topo, P_u8, P_i32],
    "fssdp_calibrate": [i32, i32, P_u8, P_u8, P_f64, i64, f64, P_topo, f64, f64, f64, P_i32, P_u8,
                        P_i32, P_f64],
    "fssdp_heterogeneous_sharding": [i32, i32, P_f64, i64, P_topo, P_i32],
    "fssdp_estimate_loads": [i32, i32, i32, P_f64, i32, P_f64],
    "fssdp_plan_layer": [i32, P_i32, P_f64, P_i64, P_topo, C.POINTER(LayerKnobs), P_u8, P_i32,
                         P_i64, P_f64, P_i32],
    "fssdp_shard_score": [i32, i32, P_i32, P_f64, P_topo, P_f64],
    "fssdp_tables_layout": [i32, i32, P_i64, P_i64],
    "fssdp_build_rank_tables": [i32, i32, i32, P_i32, P_u8, P_u8, P_i64, i32, i32, i32, vp, vp,
                                i64, P_i32],
    "fssdp_plan_candidate": [i32, P_i32, P_f64, P_topo, C.POINTER(LayerKnobs), P_u8, P_i32],
    "fssdp_plan_layer_tables": [i32, P_i32, P_f64, P_i32, P_topo, C.POINTER(LayerKnobs), i32,
                                P_u8, i32, i32, i32, P_i64, P_u8, P_i32, P_i64, P_f64, P_i32, vp,
                                i64, P_i32, vp, vp],
    "fssdp_copy_async": [vp, vp, i64, vp],
    "fssdp_plan_layer_dispatch": [vp, u32, f64, i32, P_i32, P_f64, P_i32, P_topo,
                                  C.POINTER(LayerKnobs), i32, P_u8, i32, i32, i32, P_i64, P_u8,
                                  P_i32, P_i64, P_f64, P_i32, vp, i64, P_i32, vp, vp,
                                  C.POINTER(DispatchLaunch)],
    # device data plane (device pointers as void*)
    "fssdp_grouped_gemm": [i32, i32, i32, vp, i64, i64, vp, i64, i64, vp, i32, i32, i32, vp, vp,
                           vp, vp, i64, i64, i32, vp, vp],
    "fssdp_epilogue_tmap": [i32, vp, i64, i64, vp],
    "fssdp_gate_topk": [vp, vp, vp, i64, i32, i32, i32, vp, vp, vp, vp, vp, vp],
    "fssdp_topk_from_logits": [vp, i64, i32, i32, vp, vp, vp, vp, vp],
    "fssdp_gate_route": [vp, vp, vp, i64, i32, i32, i32, vp, vp, vp, vp, vp, vp, vp, i64, i64,
                         i32, i32, i32, C.c_uint32, vp, i32, i32, i32, vp, i64, vp,
                         C.c_uint32, vp, i64, vp],
    "fssdp_gate_gemm_ws_bytes": [i64, i32],
    "fssdp_route_scan_allgather": [vp, i32, i32, vp, vp, i64, i64, i32, i32, i32, u32, vp],
    "fssdp_barrier": [vp, i64, i32, i32, i32, u32, vp],
    "fssdp_sum_peers": [vp, i32, i64, i64, vp, vp],
    "fssdp_barrier_selftest": [vp, i64, i64, i32, i32, i32, u32, i32, vp, vp],
    "fssdp_dispatch": [vp, vp, vp, vp, i64, i32, i32, i32, i32, vp, vp, vp, vp, vp, i64, vp, i32,
                       i64, i32, i32, u32, vp, vp],
    "fssdp_combine": [vp, vp, vp, i64, i32, i32, vp, i64, vp, vp, vp],
    "fssdp_local_gemm_tables": [vp, i32, i64, i32, i32, i32, i32, i32, vp, vp],
    "fssdp_dispatch_grad": [vp, vp, vp, vp, i64, i32, i32, vp, i64, vp, i64, vp, vp, vp, i32,
                            i64, i32, i32, i32, u32, vp, vp],
    "fssdp_combine_dx": [vp, vp, vp, vp, vp, vp, i64, i32, i32, i32, vp, i64, vp, vp, vp],
    "fssdp_combine_dx_dots": [vp, vp, vp, vp, vp, vp, i64, vp, i64, i32, i32, i32, vp, i64, vp,
                              vp, vp, vp],
    "fssdp_gate_wgrad": [vp, vp, vp, i64, i32, i32, i32, vp, vp, vp],
    "fssdp_gate_wgrad_tc_ws_bytes": [i64, i32],
    "fssdp_gate_wgrad_tc": [vp, vp, vp, i64, i32, i32, i32, vp, i64, vp, vp],
    "fssdp_spag": [vp, i32, i64, i64, vp, i32, vp],
    "fssdp_gather_slots": [vp, i32, i64, i64, i64, i64, vp, i32, i32, vp],
    "fssdp_sprs": [vp, i32, i64, i64, i64, i32, vp, i32, vp, vp],
    "fssdp_sprs_pull": [vp, i32, i64, i64, i32, vp, i32, vp, vp],
    # training step
    "fssdp_adam_step": [vp, vp, vp, vp, vp, i32, i64, C.c_float, C.c_float, C.c_float, C.c_float,
                        C.c_float, i64, vp],
    "fssdp_publish_epoch": [vp, i64, i32, i32, u32, vp],
    "fssdp_wait_epochs": [vp, i64, i32, i32, u32, vp],
    # launch timing (measurement)
    "fssdp_event_create": [C.POINTER(C.c_void_p)],
    "fssdp_event_destroy": [vp],
    "fssdp_event_record": [vp, vp],
    "fssdp_event_elapsed": [vp, vp, C.POINTER(C.c_float)],
    "fssdp_timing_arm": [vp, vp],
    "fssdp_timing_done": [],
    # symmetric heap
    "fssdp_heap_alloc": [C.c_size_t, C.POINTER(C.c_void_p)],
    "fssdp_heap_free": [vp],
    "fssdp_ipc_handle": [vp, P_u8],
    "fssdp_ipc_open": [P_u8, C.POINTER(C.c_void_p)],
    "fssdp_ipc_close": [vp],
    "fssdp_push_host": [vp, vp, i64, vp, u32, vp],
    "fssdp_host_wait": [vp, u32, f64],
    "fssdp_pull_host": [vp, vp, i64, vp],
}
_RESTYPE = {"fssdp_version": C.c_char_p, "fssdp_last_error": C.c_char_p,
            "fssdp_gate_gemm_ws_bytes": C.c_int64, "fssdp_gate_wgrad_tc_ws_bytes": C.c_int64}


def header_symbols() -> list[str]:
    """Every function the public header declares (for the export check)."""
    text = HEADER.read_text()
    return sorted(set(re.findall(r"^\s*(?:int64_t|int|const char\*)\s+(fssdp_\w+)\s*\(", text, re.M)))


def _load() -> C.CDLL:
    if not LIB_PATH.exists():
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python paper_2502_02581_b200/build.py` "
            "(there is no CPU fallback for the FSSDP path)"
        )
    lib = C.CDLL(str(LIB_PATH))
    for name, argtypes in _SIGS.items():
        fn = getattr(lib, name)  # AttributeError if the library lacks an export
        fn.argtypes = argtypes
        fn.restype = _RESTYPE.get(name, C.c_int)
    return lib


LIB = _load()

# Second handle on the same library for hot host paths: every pointer argument is a
# plain c_void_p, so callers pass ndarray.ctypes.data (an int) instead of data_as().
LIB_RAW = C.CDLL(str(LIB_PATH))
for _name, _args in _SIGS.items():
    _fn = getattr(LIB_RAW, _name)
    _fn.argtypes = [vp if a in (P_i32, P_i64, P_u8, P_f64, P_f32) else a for a in _args]
    _fn.restype = _RESTYPE.get(_name, C.c_int)


def last_error() -> str:
    msg = LIB.fssdp_last_error()
    return msg.decode() if msg else ""


def check(status: int, what: str) -> None:
    if status != 0:
        raise_for_status(status, what, last_error())


# kernels launched per successful call of each device entry point (launch accounting)
KERNELS_PER_CALL = {
    "fssdp_grouped_gemm": 1, "fssdp_gate_topk": 1, "fssdp_topk_from_logits": 1,
    "fssdp_route_scan_allgather": 1, "fssdp_gate_route": 1, "fssdp_barrier": 1,
    "fssdp_sum_peers": 1, "fssdp_dispatch": 1, "fssdp_combine": 1, "fssdp_local_gemm_tables": 1,
    "fssdp_plan_layer_dispatch": 2,
    "fssdp_dispatch_grad": 1, "fssdp_combine_dx": 1, "fssdp_combine_dx_dots": 1, "fssdp_gate_wgrad": 2, "fssdp_spag": 1,
    "fssdp_gate_wgrad_tc": 3,
    "fssdp_sprs": 1, "fssdp_sprs_pull": 1, "fssdp_push_host": 1, "fssdp_pull_host": 1,
    "fssdp_gather_slots": 1, "fssdp_barrier_selftest": 1, "fssdp_adam_step": 1,
    "fssdp_publish_epoch": 1, "fssdp_wait_epochs": 1,
}
launch_count = 0


def call(name: str, *args) -> None:
    global launch_count
    check(getattr(LIB, name)(*args), name)
    launch_count += KERNELS_PER_CALL.get(name, 0)


_RAW_FNS: dict = {}


def call_raw(name: str, *args) -> None:
    """call() through LIB_RAW (pointer arguments as c_void_p / ints): cheaper argument
    conversion on the launch path."""
    global launch_count
    fn = _RAW_FNS.get(name)
    if fn is None:
        fn = _RAW_FNS[name] = getattr(LIB_RAW, name)
    status = fn(*args)
    if status != 0:
        raise_for_status(status, name, last_error())
    launch_count += KERNELS_PER_CALL.get(name, 0)


class NativeEvent:
    """A CUDA event owned by libfssdp (timing enabled), with torch.cuda.Event's
    elapsed_time() so phase timers can mix with the torch-side code that reads them."""

    __slots__ = ("handle",)

    def __init__(self) -> None:
        h = C.c_void_p()
        check(LIB.fssdp_event_create(C.byref(h)), "event_create")
        self.handle = h

    def record(self, stream) -> None:
        check(LIB_RAW.fssdp_event_record(self.handle, C.c_void_p(stream.cuda_stream)),
              "event_record")

    def elapsed_time(self, end: "NativeEvent") -> float:
        ms = C.c_float()
        check(LIB_RAW.fssdp_event_elapsed(self.handle, end.handle, C.byref(ms)), "event_elapsed")
        return float(ms.value)

    def __del__(self) -> None:
        if LIB_RAW is not None and self.handle:
            LIB_RAW.fssdp_event_destroy(self.handle)


def timed_launch(timers: dict, key: str, fn) -> None:
    """Run fn (one device entry point) inside an armed launch-timing window
    (fssdp_timing_arm): timers[key] gets the (start, end) NativeEvent pair recorded right
    around its kernel launches, or nothing if it launched none."""
    s, e = NativeEvent(), NativeEvent()
    LIB_RAW.fssdp_timing_arm(s.handle, e.handle)
    try:
        fn()
    finally:
        if LIB_RAW.fssdp_timing_done():
            timers.setdefault(key, []).append((s, e))
