"""Build libhjcd.so in-tree with nvcc for sm_100a (no JIT cache, no torch
extension machinery): each .cu is compiled to an object with -lineinfo and
linked into one shared library with a statically linked CUDA runtime, so the
library is self-contained and interoperates with torch's streams/allocations
(runtime stream handles are driver handles)."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
BUILD = os.path.join(HERE, "_build")
LIB = os.path.join(HERE, "libhjcd.so")
SOURCES = sorted(f for f in os.listdir(CSRC) if f.endswith(".cu"))
HEADERS = sorted(f for f in os.listdir(CSRC) if f.endswith((".cuh", ".h")))
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-O3", "-std=c++17", "-lineinfo", "--expt-relaxed-constexpr", "-Xcompiler", "-fPIC,-O2",
         "-Xptxas", "-v"]


def _newest_input() -> float:
    paths = [os.path.join(CSRC, f) for f in SOURCES + HEADERS]
    paths.append(os.path.join(HERE, "..", "include", "hjcd.h"))
    paths.append(os.path.abspath(__file__))
    return max(os.path.getmtime(p) for p in paths)


def build(force: bool = False, verbose: bool = False, defines=(), lib: str = LIB, build_dir: str = BUILD) -> str:
    """defines / lib / build_dir: A/B variants for experiments (-D flags)."""
    LIBP, BUILDP = lib, build_dir
    if not force and os.path.exists(LIBP) and os.path.getmtime(LIBP) >= _newest_input():
        return LIBP
    os.makedirs(BUILDP, exist_ok=True)
    objs, procs = [], []
    for src in SOURCES:   # one nvcc per translation unit, in parallel
        obj = os.path.join(BUILDP, src.replace(".cu", ".o"))
        log = os.path.join(BUILDP, src.replace(".cu", ".ptxas.txt"))
        cmd = [NVCC, *ARCH, *FLAGS, *[f"-D{d}" for d in defines], "-c", os.path.join(CSRC, src), "-o", obj]
        if verbose:
            print(" ".join(cmd), flush=True)
        procs.append((src, log, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)))
        objs.append(obj)
    failed = []
    for src, log, pr in procs:
        out, _ = pr.communicate()
        with open(log, "w") as f:
            f.write(out)
        if pr.returncode != 0:
            sys.stderr.write(out)
            failed.append(src)
    if failed:
        raise RuntimeError(f"nvcc failed for {failed}")
    tmp = LIBP + f".tmp{os.getpid()}"
    cmd = [NVCC, *ARCH, "-shared", "-o", tmp, *objs, "-cudart", "static"]
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.check_call(cmd)
    os.replace(tmp, LIBP)
    return LIBP


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
