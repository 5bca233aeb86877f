"""In-tree build of libdetshare.so (sm_100a) with nvcc.

The .so is built next to this file so it travels to the GPU box with the
gpurun snapshot (git-ignored, not gpurun-ignored).  cudart is linked
statically and libcuda is never linked directly, so the library loads on a
CPU-only host (symbol-export tests) and fails loudly only when a call needs a
GPU.
"""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libdetshare.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
CUTLASS_INC = "/opt/prime-rl/.venv/lib/python3.12/site-packages/flashinfer/data/cutlass/include"

CU_SOURCES = ["executor.cu"]
CPP_SOURCES = ["runtime.cpp", "policy.cpp", "policy_abi.cpp", "engine.cpp", "workload.cpp", "placement.cpp", "migration.cpp",
               "metrics.cpp", "numlab.cpp", "fleet.cpp"]


def sources():
    out = []
    for root, _, files in os.walk(CSRC):
        for f in files:
            if f.endswith((".cu", ".cuh", ".cpp", ".h", ".hpp")):
                out.append(os.path.join(root, f))
    out.append(os.path.join(ROOT, "include", "detshare", "ds.h"))
    return out


def up_to_date() -> bool:
    if not os.path.exists(LIB):
        return False
    t = os.path.getmtime(LIB)
    return all(os.path.getmtime(s) <= t for s in sources())


def build(force: bool = False, verbose: bool = False, lanes: int = 0, out: str = "", defines=()) -> str:
    """lanes / out: an experiment variant (e.g. one worker lane per SM) built
    to another file; the product library is LIB with the default lanes."""
    lib = out or LIB
    if not force and not out and up_to_date():
        return LIB
    objdir = os.path.join(PKG, "_obj" + (f"_l{lanes}" if lanes else "") + ("_v" if out else ""))
    os.makedirs(objdir, exist_ok=True)
    common = ["-O3", "-Xcompiler", "-fPIC", "-I" + os.path.join(ROOT, "include"),
              "-I" + CSRC] + ([f"-DDS_LANES={lanes}"] if lanes else []) + [f"-D{d}" for d in defines]
    objs = []
    for src in CU_SOURCES:
        obj = os.path.join(objdir, src.replace(".cu", ".o"))
        cmd = [NVCC] + common + ["-std=c++17"] + ARCH + ["-lineinfo", "-Xptxas", "-v", "-c", os.path.join(CSRC, src), "-o", obj]
        _run(cmd, verbose)
        objs.append(obj)
    for src in CPP_SOURCES:
        obj = os.path.join(objdir, src.replace(".cpp", ".o"))
        cmd = [NVCC] + common + ["-std=c++20", "-x", "cu"] + ARCH + ["-c", os.path.join(CSRC, src), "-o", obj]
        _run(cmd, verbose)
        objs.append(obj)
    # export only the C ABI (ds_*): no std:: template instances that another
    # C++ library in the same process (e.g. the oracle) could bind to
    cmd = [NVCC, "-shared", "-Xcompiler", "-fPIC"] + ARCH + objs + ["-cudart", "static", "-o", lib,
                                                                     "-Xlinker", "-lpthread", "-Xlinker",
                                                                     "--version-script=" + os.path.join(CSRC, "exports.map")]
    _run(cmd, verbose)
    return lib


def _run(cmd, verbose):
    r = subprocess.run(cmd, capture_output=True, text=True)
    if verbose or r.returncode != 0:
        sys.stderr.write(" ".join(cmd) + "\n" + r.stdout + r.stderr)
    if r.returncode != 0:
        raise RuntimeError(f"build failed: {' '.join(cmd[:3])} ...")


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
