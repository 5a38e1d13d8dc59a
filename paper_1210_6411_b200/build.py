"""Build the in-tree CUDA library ``_lib/liblfsr_b200.so`` for sm_100a with nvcc.

The library exposes the C ABI of ``include/lfsr_b200.h``; the CUDA runtime is linked
statically so it does not depend on (or clash with) the runtime bundled with torch.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT_DIR = os.path.join(HERE, "_lib")
LIB = os.path.join(OUT_DIR, "liblfsr_b200.so")
SOURCES = ["walk.cu", "kernels.cu", "peak.cu", "reduce.cu", "bruteforce.cu", "sampler.cu", "prune.cu", "sort.cu", "jit.cu", "capi.cu"]
GENCODE = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-cudart", "static",
              "--expt-relaxed-constexpr"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


CHECKED_DIR = os.path.join(OUT_DIR, "checked")
CHECKED_LIB = os.path.join(CHECKED_DIR, "liblfsr_b200.so")


def _stale(lib: str) -> bool:
    if not os.path.exists(lib):
        return True
    t = os.path.getmtime(lib)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)]
    deps.append(os.path.join(os.path.dirname(HERE), "include", "lfsr_b200.h"))
    return any(os.path.getmtime(d) > t for d in deps)


def _compile(out_dir: str, lib: str, defines: list, verbose: bool) -> str:
    os.makedirs(out_dir, exist_ok=True)
    objs, procs = [], []
    for src in SOURCES:  # translation units compile in parallel
        obj = os.path.join(out_dir, src.replace(".cu", ".o"))
        cmd = [nvcc(), *GENCODE, *NVCC_FLAGS, *defines, "-Xptxas", "-v" if verbose else "-O3", "-c",
               os.path.join(CSRC, src), "-o", obj]
        procs.append((subprocess.Popen(cmd), cmd))
        objs.append(obj)
    for proc, cmd in procs:
        if proc.wait() != 0:
            raise subprocess.CalledProcessError(proc.returncode, cmd)
    tmp = lib + ".tmp"
    subprocess.run([nvcc(), *GENCODE, "-shared", "-cudart", "static", "-o", tmp, *objs, "-ldl"], check=True)
    os.replace(tmp, lib)
    return lib


def build(force: bool = False, verbose: bool = False, checked: bool = False) -> str:
    """The product library; checked=True also (re)builds the checked variant
    (-DLC_CHECKS=1: device-side bounds / invariant checks, _lib/checked/), which only
    the tests load."""
    if force or _stale(LIB):
        _compile(OUT_DIR, LIB, [], verbose)
    if checked and (force or _stale(CHECKED_LIB)):
        _compile(CHECKED_DIR, CHECKED_LIB, ["-DLC_CHECKS=1"], verbose)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, checked="--checked" in sys.argv))
