"""Build libagentrl.so (sm_100a) in-tree with nvcc.

    python paper_2510_04206_b200/build.py [--force] [--verbose] [--ptxas-v] [--variants]

(run as a script or load by path: importing it through the package would run the package
__init__, which refuses to load without the library)

Every .cu under csrc/ is compiled with
    -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo
(in parallel) and linked into one shared library with the CUDA runtime linked statically (so
the library loads on a GPU-less host; the driver API is reached through
cudaGetDriverEntryPoint) and NCCL loaded lazily with dlopen.

Schedule / staging choices are compile-time constants in the sources (the measured defaults).
VARIANTS lists the A/B builds the GPU tests keep parity-green (tests/test_gpu_variants.py):
each is the same sources with -D overrides, built to build/variants/<name>/libagentrl.so.
"""
from __future__ import annotations

import concurrent.futures as cf
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

# A/B builds: name -> extra nvcc flags (the defaults live in the sources)
VARIANTS = {
    "pair0": ["-DAGENTRL_GEMM_PAIR=0"],                # 1-CTA cta_group::1 GEMMs (128 x 256)
    "static": ["-DAGENTRL_GEMM_DYNAMIC=0"],            # static persistent tile striding
    "narrow": ["-DAGENTRL_GEMM_WIDE_N=0"],             # 256-column backward tiles
    "fullgrid": ["-DAGENTRL_GEMM_FULLGRID=1"],         # one CTA (pair) per tile
    "raster": ["-DAGENTRL_GROUP_M=1", "-DAGENTRL_GROUP_M_BWD=3", "-DAGENTRL_L2POL_FWD_A=2",
               "-DAGENTRL_L2POL_FWD_B=2", "-DAGENTRL_L2POL_BWD=2"],
    "ksub1": ["-DAGENTRL_FWD_KSUB=1"],                 # one 64-wide K atom per forward stage
    "lead0": ["-DAGENTRL_THROTTLE_LEAD=0"],            # backward progress throttle off
    "lead64": ["-DAGENTRL_THROTTLE_LEAD=64"],          # backward throttle lead 64 k-blocks
    "lead160": ["-DAGENTRL_THROTTLE_LEAD=160"],        # backward throttle lead 160 k-blocks
    "gm12": ["-DAGENTRL_GROUP_M=12"],                  # forward raster group of 12 row blocks
    "gm24": ["-DAGENTRL_GROUP_M=24"],                  # forward raster group of 24 row blocks
    "lockstep": ["-DAGENTRL_THROTTLE_LEAD=1", "-DAGENTRL_THROTTLE_EVERY=1"],
    "pair0_lead2": ["-DAGENTRL_GEMM_PAIR=0", "-DAGENTRL_THROTTLE_LEAD=2",
                    "-DAGENTRL_THROTTLE_EVERY=1"],
    "coop0": ["-DAGENTRL_ADV_COOP=0"],                 # 3-kernel adv-norm path
    "advlarge": ["-DAGENTRL_ADV_SMALL=0"],             # large cooperative adv-norm driver only
    "kc64": ["-DADV_KC_CAP=64"],                       # small driver in 64-chunk windows
    "ksplit3": ["-DAGENTRL_KSPLIT_FORCE=3"],           # grad_hidden split into 3 k-ranges
    "ksplitauto": ["-DAGENTRL_KSPLIT_FORCE=0"],        # grad_hidden split chosen per shape
    "pf8": ["-DAGENTRL_PREFETCH_KB=8"],                # backward L2 prefetch 8 k-blocks ahead
    "applysc4": ["-DADV_APPLY_SC=4", "-DADV_APPLY_MINB=3"],  # large apply: 4-chunk units
    "applynopf": ["-DADV_APPLY_PF=0", "-DADV_APPLY_PDL=0"],  # large apply: no unit prefetch, no PDL
    "applydiag": ["-DADV_APPLY_DIAG=1"],               # timing only: the apply's stores alone
    "pstage0": ["-DAGENTRL_FWD_PSTAGE=0"],             # forward: P~ stored 16 B per row, no staging
    "gwstage0": ["-DAGENTRL_GRADW_STAGE=0"],           # local grad_W epilogue: 16 B per row stores
}


def _sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def _deps():
    return _sources() + sorted(glob.glob(os.path.join(CSRC, "*.cuh")) +
                               glob.glob(os.path.join(CSRC, "*.h")) +
                               glob.glob(os.path.join(ROOT, "include", "*.h")) + [__file__])


def _stale(lib: str, stamp: str | None = None, flags: list[str] | None = None) -> bool:
    if not os.path.exists(lib):
        return True
    if stamp is not None:
        if not os.path.exists(stamp) or open(stamp).read() != " ".join(flags or []):
            return True
    t = os.path.getmtime(lib)
    return any(os.path.getmtime(p) > t for p in _deps())


def needs_build() -> bool:
    return _stale(LIB)


def _compile(src, obj, extra, ptxas_v, verbose):
    cmd = [NVCC, *ARCH, *FLAGS, *extra, "-c", src, "-o", obj]
    if ptxas_v:
        cmd += ["-Xptxas", "-v"]
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.check_call(cmd)
    return obj


def build(force: bool = False, verbose: bool = False, ptxas_v: bool = False,
          out: str | None = None, extra: list[str] | None = None, jobs: int | None = None) -> str:
    """out: write an A/B variant library there instead (objects kept apart); extra: -D flags"""
    lib = out or LIB
    extra = list(extra or []) + os.environ.get("AGENTRL_NVCC_EXTRA", "").split()
    objdir = os.path.join(BUILD, os.path.basename(os.path.dirname(out)) if out else "main")
    stamp = lib + ".flags" if out else None
    if not force and not _stale(lib, stamp, extra):
        return lib
    os.makedirs(objdir, exist_ok=True)
    srcs = _sources()
    jobs = jobs or min(len(srcs), os.cpu_count() or 4)
    with cf.ThreadPoolExecutor(jobs) as ex:
        objs = list(ex.map(lambda s: _compile(s, os.path.join(objdir, os.path.basename(s) + ".o"),
                                              extra, ptxas_v, verbose), srcs))
    tmp = lib + ".tmp"
    cmd = [NVCC, *ARCH, "-shared", "-Xcompiler", "-fPIC", "--cudart", "static", *objs, "-o", tmp,
           "-ldl", "-lpthread", "-lrt"]
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.check_call(cmd)
    os.replace(tmp, lib)
    if stamp:
        with open(stamp, "w") as f:
            f.write(" ".join(extra))
    return lib


def variant_path(name: str) -> str:
    return os.path.join(BUILD, "variants", name, "libagentrl.so")


def build_variant(name: str, force: bool = False) -> str:
    path = variant_path(name)
    os.makedirs(os.path.dirname(path), exist_ok=True)
    return build(force=force, out=path, extra=VARIANTS[name], jobs=2)


def build_variants(force: bool = False) -> dict:
    """every A/B variant (a few at a time; each compiles its sources in parallel)"""
    with cf.ThreadPoolExecutor(max(1, (os.cpu_count() or 4) // 2)) as ex:
        paths = list(ex.map(lambda n: build_variant(n, force), VARIANTS))
    return dict(zip(VARIANTS, paths))


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="--verbose" in sys.argv,
                ptxas_v="--ptxas-v" in sys.argv))
    if "--variants" in sys.argv:
        for k, v in build_variants(force="--force" in sys.argv).items():
            print(k, v)
