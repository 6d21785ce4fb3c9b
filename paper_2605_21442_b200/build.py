"""Builds liblce.so (the C-ABI CUDA library) in-tree for sm_100a with nvcc.

    python paper_2605_21442_b200/build.py [--verbose]

Run by file path (it must not import the package, whose __init__ loads the
library this builds); __graft_entry__.build() loads it the same way.

No torch extension machinery: the library is a plain shared object with an
extern "C" interface (include/lce.h), loaded by the ctypes binding.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "liblce.so")
# same sources with -DLCE_DEBUG_SYNC: every device spin wait traps after 2 s
# (sm100.cuh SpinGuard); hang detection where compute-sanitizer is unavailable
DEBUG_LIB = os.path.join(PKG, "liblce_debug.so")
SOURCES = [os.path.join(CSRC, "lce_api.cu")]
DEPS = SOURCES + [os.path.join(CSRC, f) for f in ("sm100.cuh", "gemm.cuh", "kernels.cuh")] + [
    os.path.join(ROOT, "include", "lce.h")
]


def _nccl_include() -> str:
    try:
        import nvidia.nccl  # type: ignore

        base = os.path.dirname(nvidia.nccl.__file__) if nvidia.nccl.__file__ else list(nvidia.nccl.__path__)[0]
        inc = os.path.join(base, "include")
        if os.path.exists(os.path.join(inc, "nccl.h")):
            return inc
    except Exception:
        pass
    for cand in ("/usr/include", "/usr/local/cuda/include"):
        if os.path.exists(os.path.join(cand, "nccl.h")):
            return cand
    raise RuntimeError("nccl.h not found (needed for NCCL types; NCCL itself is dlopen'ed)")


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def up_to_date() -> bool:
    if not os.path.exists(LIB):
        return False
    t = os.path.getmtime(LIB)
    return all(os.path.getmtime(d) <= t for d in DEPS)


def build(force: bool = False, verbose: bool = False, dest: str = LIB, defines: tuple = ()) -> str:
    """`dest` / `defines` (-D flags): A/B builds of compile-time variants
    (scripts/build_variant.py); the package always loads `LIB`."""
    if dest == LIB and not defines and not force and up_to_date():
        return LIB
    cmd = [
        nvcc(),
        "-gencode", "arch=compute_100a,code=sm_100a",
        "-O3", "-lineinfo", "-std=c++17",
        "-Xcompiler", "-fPIC,-O2",
        "-shared",
        "-I", os.path.join(ROOT, "include"),
        "-I", _nccl_include(),
        *[f"-D{d}" for d in defines],
        "-o", dest + ".tmp",
        *SOURCES,
        "-ldl",
    ]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
        print(" ".join(cmd))
    subprocess.run(cmd, check=True)
    os.replace(dest + ".tmp", dest)
    return dest


def build_debug(force: bool = False) -> str:
    """liblce_debug.so (LCE_LIB_PATH=... loads it instead of liblce.so)."""
    if not force and os.path.exists(DEBUG_LIB) and all(os.path.getmtime(d) <= os.path.getmtime(DEBUG_LIB)
                                                       for d in DEPS):
        return DEBUG_LIB
    return build(force=True, dest=DEBUG_LIB, defines=("LCE_DEBUG_SYNC",))


if __name__ == "__main__":
    print(build(force=True, verbose="--verbose" in sys.argv))
    if "--debug" in sys.argv:
        print(build_debug(force=True))
