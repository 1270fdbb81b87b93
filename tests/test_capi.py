"""The C-ABI library loads on a GPU-less host and exports every symbol include/fssdp.h
declares (no compute calls here)."""

import ctypes

from paper_2502_02581_b200 import _native as N


def test_library_loads_and_reports_version():
    assert N.LIB.fssdp_version().decode().startswith("fssdp-b200")


def test_every_header_symbol_is_exported_and_bound():
    syms = N.header_symbols()
    assert len(syms) >= 30
    lib = ctypes.CDLL(str(N.LIB_PATH))
    for s in syms:
        assert hasattr(lib, s), f"libfssdp.so does not export {s}"
        assert s in N._SIGS, f"_native.py has no signature for {s}"


def test_no_libcuda_link_dependency():
    """TMA descriptors are encoded via cudaGetDriverEntryPoint, so the library must not
    need libcuda.so at load time (it loads on CPU build hosts)."""
    import subprocess

    out = subprocess.run(["ldd", str(N.LIB_PATH)], capture_output=True, text=True).stdout
    assert "libcuda.so" not in out and "libcudart.so" not in out


def test_errors_map_to_reference_taxonomy():
    import numpy as np

    import paper_2502_02581_b200 as F

    rc = N.LIB.fssdp_make_even_partition(3, 0, np.zeros(3, np.int32).ctypes.data_as(N.P_i32))
    assert rc == -1
    try:
        N.check(rc, "x")
    except F.DimensionError as exc:
        assert "num_devices > 0" in str(exc)
    else:
        raise AssertionError("expected DimensionError")


def test_binding_argument_counts_match_the_header():
    """Every ctypes signature in _native.py has exactly the header's parameter count (an
    ABI change on one side only would pass garbage through the boundary)."""
    import re

    text = re.sub(r"/\*.*?\*/", "", N.HEADER.read_text(), flags=re.S)
    decls = re.findall(r"^\s*(?:int64_t|int|const char\*)\s+(fssdp_\w+)\s*\(([^;]*?)\)\s*;",
                       text, re.M | re.S)
    assert len(decls) >= 30
    for name, params in decls:
        p = params.strip()
        n = 0 if p in ("", "void") else p.count(",") + 1
        assert len(N._SIGS[name]) == n, f"{name}: header {n} params, binding {len(N._SIGS[name])}"
