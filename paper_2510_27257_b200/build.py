"""Build libstp.so in-tree: nvcc for sm_100a (-gencode arch=compute_100a,
code=sm_100a -lineinfo), g++ for host-only sources, linked against the NCCL
that torch ships (same soname libnccl.so.2 torch loads).  Incremental by
mtime; `python -m paper_2510_27257_b200.build [-v] [--force]`."""
from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INC = os.path.join(ROOT, "include")
BUILD = os.path.join(ROOT, "build", "stp")
LIB = os.path.join(PKG, "libstp.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
CUDA_INC = "/usr/local/cuda/include"
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nccl_paths():
    import importlib.util
    spec = importlib.util.find_spec("nvidia")
    for base in list(spec.submodule_search_locations or []):
        inc = os.path.join(base, "nccl", "include")
        lib = os.path.join(base, "nccl", "lib")
        if os.path.exists(os.path.join(inc, "nccl.h")) and os.path.exists(os.path.join(lib, "libnccl.so.2")):
            return inc, lib
    raise RuntimeError("torch's NCCL (nvidia/nccl) not found")


def _deps_mtime():
    hs = glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(INC, "*.h"))
    return max(os.path.getmtime(h) for h in hs) if hs else 0.0


def _compile(src, obj, nccl_inc, verbose):
    common = ["-I", INC, "-I", CSRC, "-I", nccl_inc, "-I", CUDA_INC]
    if src.endswith(".cu"):
        cmd = [NVCC] + ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
                               "--expt-relaxed-constexpr", "-Xptxas", "-v" if verbose else "-O3",
                               "-c", src, "-o", obj] + common
    else:
        cmd = ["g++", "-O2", "-fPIC", "-std=c++17", "-Wall", "-c", src, "-o", obj] + common
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"compile failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    return (src, r.stderr if verbose else "")


def build(verbose: bool = False, force: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    nccl_inc, nccl_lib = nccl_paths()
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cpp")))
    dm = _deps_mtime()
    jobs = []
    objs = []
    for s in srcs:
        o = os.path.join(BUILD, os.path.basename(s) + ".o")
        objs.append(o)
        if force or not os.path.exists(o) or os.path.getmtime(o) < max(os.path.getmtime(s), dm):
            jobs.append((s, o))
    with cf.ThreadPoolExecutor(max_workers=min(8, max(1, len(jobs)))) as ex:
        for src, log in ex.map(lambda j: _compile(j[0], j[1], nccl_inc, verbose), jobs):
            if verbose:
                print(f"[build] {os.path.basename(src)}\n{log}")
    need_link = force or bool(jobs) or not os.path.exists(LIB) or \
        os.path.getmtime(LIB) < max(os.path.getmtime(o) for o in objs)
    if need_link:
        cmd = [NVCC] + ARCH + ["-shared", "-o", LIB] + objs + [
            "-L", nccl_lib, "-l:libnccl.so.2", "-Xlinker", f"-rpath={nccl_lib}", "-lpthread", "-ldl"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    return LIB


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, force="--force" in sys.argv))
