"""Build the sm_100a shared library libfmoe_b200.so in-tree with nvcc.

    python paper_2502_05370_b200/build.py [--force]      (or __graft_entry__.build())

Every .cu under csrc/ is compiled with -gencode arch=compute_100a,code=sm_100a
(no other architecture), -O3 -lineinfo, in parallel, then linked against the
shared CUDA runtime (the one torch has already loaded, so streams and the
stream-ordered allocator are shared with the caller).  Rebuilds only when a
source or header is newer than the library.
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
LIB = os.path.join(PKG, "libfmoe_b200.so")
BUILD = os.path.join(PKG, "_build")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if c and os.path.exists(c):
            return c
    raise RuntimeError("nvcc not found")


def nccl_include() -> list:
    """nccl.h for the types of the run-time-loaded NCCL (dist.cu): the pip
    nvidia-nccl wheel PyTorch ships, else the system header."""
    try:
        import nvidia.nccl as n
        d = os.path.join(list(n.__path__)[0], "include")
        if os.path.exists(os.path.join(d, "nccl.h")):
            return ["-I" + d]
    except ImportError:
        pass
    return []


def _flags():
    return ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xptxas", "-v",
                   "--expt-relaxed-constexpr", "-I" + os.path.join(ROOT, "include"), "-I" + CSRC] + nccl_include() + \
        os.environ.get("FMOE_NVCC_EXTRA", "").split()     # e.g. -DFMOE_EPI_PROFILE (tools/trace.py)


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = sources() + glob.glob(os.path.join(CSRC, "*.cuh")) + [os.path.join(ROOT, "include", "fmoe.h"), __file__]
    return any(os.path.getmtime(p) > t for p in deps)


def _compile(src: str) -> tuple[str, str]:
    obj = os.path.join(BUILD, os.path.basename(src)[:-3] + ".o")
    cmd = [nvcc()] + _flags() + ["-c", src, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr}")
    return obj, r.stderr


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return LIB
    os.makedirs(BUILD, exist_ok=True)
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
        results = list(ex.map(_compile, sources()))
    objs = [o for o, _ in results]
    with open(os.path.join(BUILD, "ptxas.log"), "w") as f:
        for _, log in results:
            f.write(log)
    if verbose:
        for _, log in results:
            sys.stderr.write(log)
    tmp = LIB + ".tmp"
    cmd = [nvcc()] + ARCH + ["-shared", "-o", tmp] + objs + ["-ldl", "--cudart", "shared",
                                                            "-Xlinker", "-rpath=/usr/local/cuda/lib64"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError("link failed:\n" + r.stderr)
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
