"""Build libblurrast.so in-tree with nvcc for sm_100a (called by __graft_entry__.build())."""
from __future__ import annotations

import glob
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libblurrast.so")
INCLUDE = os.path.join(os.path.dirname(HERE), "include")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = sources() + glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(INCLUDE, "*.h"))
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, out: str = None, defines=()) -> str:
    """Compile libblurrast.so (or `out`, with extra -D `defines`, for A/B variants)."""
    target = out or LIB
    if out is None and not force and not _stale():
        return LIB
    tmp = target + ".tmp%d" % os.getpid()
    cmd = [NVCC, "-O3", "-std=c++17", *ARCH, "-lineinfo", "-Xcompiler", "-fPIC", "-shared",
           "-I", INCLUDE, *["-D" + d for d in defines], "-o", tmp, *sources()]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
    if os.environ.get("BR_DEBUG") == "1":
        cmd.insert(1, "-DBR_DEBUG")
    subprocess.check_call(cmd, cwd=CSRC)
    os.replace(tmp, target)
    return target
