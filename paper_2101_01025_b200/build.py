"""Build the in-tree CUDA library libadjprod.so (sm_100a) and the device input generator.

nvcc cross-compiles for sm_100a without a GPU.  Objects are rebuilt only when a source or
header is newer than the object.
"""
from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
BUILD = os.path.join(PKG, "_build")
LIB = os.path.join(PKG, "libadjprod.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nccl_include():
    try:
        import nvidia.nccl  # type: ignore
        d = os.path.join(list(nvidia.nccl.__path__)[0], "include")
        if os.path.exists(os.path.join(d, "nccl.h")):
            return d
    except Exception:
        pass
    return "/usr/include"


def _flags():
    return ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O3", "--expt-relaxed-constexpr",
                   "-I", CSRC, "-I", os.path.join(ROOT, "include"), "-I", _nccl_include()] + \
        os.environ.get("ADJ_NVCC_EXTRA", "").split()   # dev experiments only (e.g. -DADJ_EPI_WARPS=4)


def _newest(paths):
    return max(os.path.getmtime(p) for p in paths)


def _compile(src, obj, deps):
    if os.path.exists(obj) and os.path.getmtime(obj) >= _newest([src] + deps):
        return obj, False
    cmd = [NVCC] + _flags() + ["-c", src, "-o", obj]
    if src.endswith(".cu"):
        cmd[1:1] = ["-Xptxas", "-warn-spills"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
    return obj, True


def build(verbose: bool = True) -> str:
    os.makedirs(BUILD, exist_ok=True)
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cpp")))
    deps = sorted(glob.glob(os.path.join(CSRC, "*.hpp")) + glob.glob(os.path.join(CSRC, "*.cuh"))
                  + [os.path.join(ROOT, "include", "adjprod.h")])
    objs = []
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        futs = [ex.submit(_compile, s, os.path.join(BUILD, os.path.basename(s) + ".o"), deps) for s in srcs]
        for f in futs:
            o, rebuilt = f.result()
            objs.append(o)
            if verbose and rebuilt:
                print(f"[build] compiled {os.path.basename(o)}", file=sys.stderr)
    if not os.path.exists(LIB) or os.path.getmtime(LIB) < _newest(objs):
        cmd = [NVCC] + ARCH + ["-shared", "-o", LIB] + objs + ["-ldl"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
        if verbose:
            print(f"[build] linked {LIB}", file=sys.stderr)
    build_inputs_gen(verbose)
    return LIB


def build_inputs_gen(verbose: bool = True) -> str:
    src = os.path.join(ROOT, "inputs", "gen.cu")
    so = os.path.join(ROOT, "inputs", "_gen.so")
    if not os.path.exists(so) or os.path.getmtime(so) < os.path.getmtime(src):
        cmd = [NVCC] + ARCH + ["-O3", "-shared", "-Xcompiler", "-fPIC", src, "-o", so]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr}")
        if verbose:
            print(f"[build] built {so}", file=sys.stderr)
    return so


if __name__ == "__main__":
    build()
