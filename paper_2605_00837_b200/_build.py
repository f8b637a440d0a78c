"""Build liblsk.so in-tree with nvcc for sm_100a (no JIT cache, no torch ext).

    python -m paper_2605_00837_b200._build        # or __graft_entry__.build()

The library is the C ABI of include/lsk.h; the Python package loads it with
ctypes. Compiled WITHOUT --use_fast_math: the arithmetic contract needs IEEE
division for inv_eps and unfused argument builds (SURVEY.md 8(a')).
"""

import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "liblsk.so")
BUILD = os.path.join(ROOT, "build")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++20", "-Xcompiler", "-fPIC", "-Xcompiler", "-O2"]
UNITS = ["lsk_api.cu", "lsk_points.cu", "lsk_points_solve.cu", "lsk_h2d.cu", "lsk_dense_loop.cu", "lsk_f64.cu", "lsk_color.cu", "lsk_standard.cu", "lsk_reduce.cu", "lsk_diag.cu"]


def nccl_dirs():
    """NCCL headers/library: the copy bundled with torch (2.28, the one torch
    itself loads), else the system one."""
    try:
        import importlib.util

        spec = importlib.util.find_spec("nvidia.nccl")
        if spec and spec.submodule_search_locations:
            root = list(spec.submodule_search_locations)[0]
            if os.path.exists(os.path.join(root, "include", "nccl.h")):
                return os.path.join(root, "include"), os.path.join(root, "lib")
    except Exception:
        pass
    return "/usr/include", "/usr/lib/x86_64-linux-gnu"


def nvcc():
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found; set NVCC or put /usr/local/cuda/bin on PATH")


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(verbose=False, force=False):
    os.makedirs(BUILD, exist_ok=True)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)]
    deps.append(os.path.join(ROOT, "include", "lsk.h"))
    if not force and not _stale(LIB, deps):
        return LIB
    objs = []
    for u in UNITS:
        obj = os.path.join(BUILD, u.replace(".cu", ".o"))
        inc, _ = nccl_dirs()
        cmd = [nvcc(), *ARCH, *FLAGS, "-I" + inc, "-c", os.path.join(CSRC, u), "-o", obj]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
            print(" ".join(cmd), flush=True)
        subprocess.run(cmd, check=True)
        objs.append(obj)
    tmp = LIB + ".tmp"
    _, libdir = nccl_dirs()
    nccl = os.path.join(libdir, "libnccl.so.2")
    cmd = [nvcc(), *ARCH, "-shared", "-o", tmp, *objs, "-lcuda", "-Xlinker", nccl, "-Xlinker", "-rpath=" + libdir]
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, force="-f" in sys.argv))
