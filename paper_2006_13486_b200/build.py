"""Build recipe of the in-tree CUDA library (sm_100a only).

`python -m paper_2006_13486_b200.build` (or `__graft_entry__.build()`)
compiles every `csrc/*.cu` with nvcc (one process per source, in parallel)
and links `librbgp4_b200.so` next to this file.  The library is plain C ABI
(include/rbgp4.h) with the CUDA runtime linked statically, so it loads with
ctypes and travels with the repo snapshot to the GPU box.

`--debug` builds `librbgp4_b200_debug.so` with -DRBGP4_DEBUG=1: the kernels'
trace / ablation hooks (option `debug`) for the tools under tools/.  The
product never loads it.
"""

from __future__ import annotations

import glob
import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "librbgp4_b200.so")
LIB_DEBUG = os.path.join(PKG, "librbgp4_b200_debug.so")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def needs_build(lib: str = LIB) -> bool:
    if not os.path.exists(lib):
        return True
    newest = max(os.path.getmtime(p) for p in sources() + glob.glob(os.path.join(CSRC, "*.cuh"))
                 + [os.path.join(ROOT, "include", "rbgp4.h")])
    return os.path.getmtime(lib) < newest


def _run(cmd):
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed:\n{' '.join(cmd)}\n{res.stdout}\n{res.stderr}")
    return res.stderr


def build(force: bool = False, verbose: bool = False, debug: bool = False) -> str:
    lib = LIB_DEBUG if debug else LIB
    if not force and not needs_build(lib):
        return lib
    objdir = os.path.join(PKG, "build", "debug" if debug else "release")
    os.makedirs(objdir, exist_ok=True)
    flags = [*ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
             "-I", os.path.join(ROOT, "include"), f"-DRBGP4_DEBUG={1 if debug else 0}"]
    if verbose:
        flags.append("-Xptxas=-v")
    objs = [os.path.join(objdir, os.path.basename(src)[:-3] + ".o") for src in sources()]
    with ThreadPoolExecutor(max_workers=max(1, min(len(objs), os.cpu_count() or 4))) as ex:
        logs = list(ex.map(lambda so: _run([nvcc(), *flags, "-c", so[0], "-o", so[1]]),
                           zip(sources(), objs)))
    _run([nvcc(), *ARCH, "-shared", "-cudart", "static", "-o", lib + ".tmp", *objs])
    if verbose:
        sys.stderr.write("".join(logs))
    os.replace(lib + ".tmp", lib)
    return lib


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, debug="--debug" in sys.argv))
