"""Build libfssdp.so in-tree: nvcc for the sm_100a kernels, g++ for the host planner.

The library is a plain C-ABI shared object (include/fssdp.h) with the CUDA runtime
linked statically and no libcuda link dependency (TMA descriptors are encoded through
cudaGetDriverEntryPoint), so it loads on GPU-less hosts for the planner and the
symbol checks, and travels to the GPU box with the repo snapshot.

    python paper_2502_02581_b200/build.py [--force]     (run by path: importing the
                                                         package would load the old .so)
"""

from __future__ import annotations

import argparse
import concurrent.futures as cf
import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
BUILD = ROOT / "build" / "fssdp"
LIB = PKG / "libfssdp.so"
# diagnostic variant (--gemm-profile): GEMM role-wait cycle counters, loaded with
# FSSDP_LIB=<path> by scripts/gemm_profile.py only
LIB_PROF = ROOT / "build" / "libfssdp_gemm_profile.so"

NVCC = os.environ.get("NVCC", shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = [
    "-O3",
    "-std=c++17",
    "-lineinfo",
    "-Xcompiler",
    "-fPIC",
    "-Xcompiler",
    "-fvisibility=hidden",
    "--expt-relaxed-constexpr",
    "-I" + str(ROOT / "include"),
]
CXX = os.environ.get("CXX", "g++")
CXX_FLAGS = ["-O2", "-std=c++17", "-fPIC", "-fvisibility=hidden", "-I" + str(ROOT / "include")]


def _sources() -> list[Path]:
    return sorted(list(CSRC.glob("*.cu")) + list(CSRC.glob("*.cpp")))


def _deps() -> list[Path]:
    return _sources() + sorted(CSRC.glob("*.cuh")) + sorted(CSRC.glob("*.h")) + [
        ROOT / "include" / "fssdp.h",
        Path(__file__),
    ]


def _compile(src: Path, verbose: bool, out_dir: Path = BUILD, defines=()) -> Path:
    obj = out_dir / (src.name + ".o")
    if src.suffix == ".cu":
        cmd = [NVCC, *ARCH, *NVCC_FLAGS, *defines, "-c", str(src), "-o", str(obj)]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
    else:
        cmd = [CXX, *CXX_FLAGS, "-c", str(src), "-o", str(obj)]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"compile failed: {' '.join(cmd)}\n{res.stdout}\n{res.stderr}")
    if verbose and res.stderr:
        sys.stderr.write(res.stderr)
    return obj


def needs_build() -> bool:
    if not LIB.exists():
        return True
    mtime = LIB.stat().st_mtime
    return any(p.stat().st_mtime > mtime for p in _deps() if p.exists())


def build(force: bool = False, verbose: bool = False) -> Path:
    if not force and not needs_build():
        return LIB
    BUILD.mkdir(parents=True, exist_ok=True)
    srcs = _sources()
    with cf.ThreadPoolExecutor(max_workers=min(8, len(srcs))) as pool:
        objs = list(pool.map(lambda s: _compile(s, verbose), srcs))
    tmp = LIB.with_suffix(".so.tmp")
    cmd = [NVCC, *ARCH, "-shared", "-cudart", "static", "-o", str(tmp), *map(str, objs), "-lstdc++"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"link failed: {' '.join(cmd)}\n{res.stdout}\n{res.stderr}")
    os.replace(tmp, LIB)
    return LIB


def build_variant(lib: Path, defines: tuple, tag: str) -> Path:
    """A diagnostic / experiment build of the same sources with extra -D defines (selected
    at run time with FSSDP_LIB=<path>)."""
    out = ROOT / "build" / tag
    out.mkdir(parents=True, exist_ok=True)
    srcs = _sources()
    with cf.ThreadPoolExecutor(max_workers=min(8, len(srcs))) as pool:
        objs = list(pool.map(lambda s: _compile(s, False, out, defines), srcs))
    cmd = [NVCC, *ARCH, "-shared", "-cudart", "static", "-o", str(lib), *map(str, objs),
           "-lstdc++"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"link failed: {' '.join(cmd)}\n{res.stdout}\n{res.stderr}")
    return lib


def build_gemm_profile() -> Path:
    return build_variant(LIB_PROF, ("-DFSSDP_GEMM_PROFILE",), "fssdp_prof")


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("--verbose", action="store_true", help="print ptxas resource usage")
    ap.add_argument("--gemm-profile", action="store_true",
                    help="also build the diagnostic GEMM role-wait counter variant")
    ap.add_argument("--variant", nargs=2, metavar=("LIB", "DEFINES"),
                    help="an experiment build: output .so path and comma-separated defines")
    args = ap.parse_args()
    print(build(force=args.force, verbose=args.verbose))
    if args.gemm_profile:
        print(build_gemm_profile())
    if args.variant:
        lib, defs = args.variant
        print(build_variant(Path(lib).resolve(), tuple("-D" + d for d in defs.split(",") if d),
                            Path(lib).stem))


if __name__ == "__main__":
    main()
