"""Build libagentrl.so (sm_100a) in-tree with nvcc.

    python paper_2510_04206_b200/build.py [--force] [--verbose] [--ptxas-v]

(run as a script or load by path: importing it through the package would run the package
__init__, which refuses to load without the library)

Every .cu under csrc/ is compiled with
    -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo
and linked into one shared library with the CUDA runtime linked statically (so the
library loads on a GPU-less host; the driver API is reached through
cudaGetDriverEntryPoint) and NCCL loaded lazily with dlopen.
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "libagentrl.so")
BUILD = os.path.join(ROOT, "build")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
         "-I" + os.path.join(ROOT, "include")]
# extra nvcc flags for A/B builds (e.g. AGENTRL_NVCC_EXTRA="-DADV_MIN_BLOCKS=2")
FLAGS += os.environ.get("AGENTRL_NVCC_EXTRA", "").split()


def _sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def _deps():
    return _sources() + sorted(glob.glob(os.path.join(CSRC, "*.cuh")) +
                               glob.glob(os.path.join(CSRC, "*.h")) +
                               glob.glob(os.path.join(ROOT, "include", "*.h")))


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(p) > t for p in _deps())


def build(force: bool = False, verbose: bool = False, ptxas_v: bool = False,
          out: str | None = None) -> str:
    """out: write an A/B variant library there instead (always rebuilt; objects kept apart)"""
    global BUILD
    lib = out or LIB
    if out:
        BUILD = os.path.join(BUILD, os.path.basename(out))
    elif not force and not needs_build():
        return LIB
    os.makedirs(BUILD, exist_ok=True)
    objs = []
    for src in _sources():
        obj = os.path.join(BUILD, os.path.basename(src) + ".o")
        cmd = [NVCC, *ARCH, *FLAGS, "-c", src, "-o", obj]
        if ptxas_v:
            cmd += ["-Xptxas", "-v"]
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.check_call(cmd)
        objs.append(obj)
    tmp = lib + ".tmp"
    cmd = [NVCC, *ARCH, "-shared", "-Xcompiler", "-fPIC", "--cudart", "static", *objs, "-o", tmp,
           "-ldl", "-lpthread", "-lrt"]
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.check_call(cmd)
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    out = next((a.split("=", 1)[1] for a in sys.argv if a.startswith("--out=")), None)
    print(build(force="--force" in sys.argv, verbose="--verbose" in sys.argv,
                ptxas_v="--ptxas-v" in sys.argv, out=out))
