"""In-tree build of the native library ``libdear.so`` (sm_100a only).

    python -m paper_2302_12445_b200.build          # incremental
    python -m paper_2302_12445_b200.build --force

Each ``csrc/*.cu`` / ``csrc/*.cpp`` is compiled by nvcc with
``-gencode arch=compute_100a,code=sm_100a -lineinfo -O3`` into ``build/`` and
linked with NCCL into ``paper_2302_12445_b200/libdear.so``. The .so travels
to the GPU box with the repo snapshot (it is git-ignored, not gpurun-ignored).
"""
from __future__ import annotations

import argparse
import glob
import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
# DEAR_VARIANT="NAME:-DFOO=1,-DBAR=2" builds an experiment variant into
# libdear_NAME.so (selected at run time with DEAR_LIB=libdear_NAME.so).
_VARIANT = os.environ.get("DEAR_VARIANT", "")
_VNAME, _VDEFS = (_VARIANT.split(":", 1) + [""])[:2] if _VARIANT else ("", "")
BUILD = os.path.join(ROOT, "build", "dear" + (f"_{_VNAME}" if _VNAME else ""))
LIB = os.path.join(PKG, f"libdear_{_VNAME}.so" if _VNAME else "libdear.so")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
CUTLASS_INC = None  # CuTe headers are not needed by the current kernels


def nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found; the DeAR runtime needs the CUDA toolkit to build")


def _flags() -> list[str]:
    return [*ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-Wall",
            "-I" + os.path.join(ROOT, "include"), "-I" + CSRC,
            "--expt-relaxed-constexpr", "-Xptxas", "-v" if os.environ.get("DEAR_PTXAS_V") else "-O3",
            *[d for d in _VDEFS.split(",") if d]]


def _stale(obj: str, deps: list[str]) -> bool:
    if not os.path.exists(obj):
        return True
    t = os.path.getmtime(obj)
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cpp")))
    headers = (glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh"))
               + glob.glob(os.path.join(ROOT, "include", "*.h")))
    objs = []
    cc = nvcc()
    for src in srcs:
        obj = os.path.join(BUILD, os.path.basename(src) + ".o")
        objs.append(obj)
        if force or _stale(obj, [src, *headers, __file__]):
            cmd = [cc, *_flags(), "-c", src, "-o", obj]
            if verbose:
                print(" ".join(cmd), flush=True)
            subprocess.run(cmd, check=True)
    if force or _stale(LIB, objs):
        cmd = [cc, *ARCH, "-shared", "-o", LIB, *objs, "-lnccl"]
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.run(cmd, check=True)
    return LIB


def main(argv=None) -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("-v", "--verbose", action="store_true")
    a = ap.parse_args(argv)
    print(build(force=a.force, verbose=a.verbose))
    return 0


if __name__ == "__main__":
    sys.exit(main())
