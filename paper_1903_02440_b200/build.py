"""Build libsnn.so (all CUDA sources, sm_100a) in-tree with nvcc.

    python -m paper_1903_02440_b200.build        # or __graft_entry__.build()
"""
from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libsnn.so")
NVCC = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
         "--expt-relaxed-constexpr", "-I", os.path.join(ROOT, "include")]


def _sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def _deps():
    return _sources() + glob.glob(os.path.join(CSRC, "*.cuh")) + [os.path.join(ROOT, "include", "snn.h")]


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(p) > t for p in _deps())


def build(force: bool = False, verbose: bool = False, extra=(), out: str = None) -> str:
    """out: another library path (e.g. the checked build, tools/build_checked.sh) -- objects go to their own
    directory, the in-tree libsnn.so is not touched."""
    env_extra = os.environ.get("SNN_NVCC_EXTRA", "").split()  # tuning experiments, e.g. -DSNN_SORT_UNROLL=8
    if env_extra:
        extra, force = list(extra) + env_extra, True
    lib = out or LIB
    if out is None and not force and not needs_build():
        return LIB
    objdir = os.path.join(PKG, "build" if out is None else "build_" + os.path.splitext(os.path.basename(out))[0])
    os.makedirs(objdir, exist_ok=True)

    def compile_one(src):
        obj = os.path.join(objdir, os.path.basename(src) + ".o")
        cmd = [NVCC, *ARCH, *FLAGS, *extra, "-c", src, "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
        if verbose and (r.stderr or r.stdout):
            print(r.stdout + r.stderr, file=sys.stderr)
        return obj

    with cf.ThreadPoolExecutor(max_workers=8) as ex:
        objs = list(ex.map(compile_one, _sources()))
    tmp = lib + ".tmp"
    cmd = [NVCC, *ARCH, "-shared", "-o", tmp, *objs, "-lcudart"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    if "--checked" in sys.argv:  # device bounds checks (SNN_DCHECK) in a separate library, libsnn_checked.so
        print(build(force=True, verbose=True, extra=["-DSNN_CHECKED"], out=os.path.join(PKG, "libsnn_checked.so")))
    else:
        print(build(force="--force" in sys.argv, verbose=True,
                    extra=["-Xptxas", "-v"] if "--ptxas" in sys.argv else []))
