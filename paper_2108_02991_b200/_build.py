"""In-tree build of the sm_100a kernels into ``_lib/libsparkling_b200.so``.

``nvcc`` cross-compiles for sm_100a without a GPU, so this runs both in the authoring
container and on the GPU box.  The shared library is git-ignored but travels with the
``gpurun`` snapshot.
"""

from __future__ import annotations

import os
import shutil
import subprocess

PKG_DIR = os.path.dirname(os.path.abspath(__file__))
REPO_DIR = os.path.dirname(PKG_DIR)
CSRC = os.path.join(PKG_DIR, "csrc")
LIB_DIR = os.path.join(PKG_DIR, "_lib")
LIB_PATH = os.path.join(LIB_DIR, "libsparkling_b200.so")
INCLUDE = os.path.join(REPO_DIR, "include")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-I" + INCLUDE]
# project.cu must not contract fp64 mul+add into FMA: bit parity with the reference.
SOURCES = {
    "nbody.cu": [],
    "project.cu": ["-fmad=false"],
    "tree.cu": [],
    "nudft.cu": [],
}
# Host C++ (treecode octree over sorted keys; reference host planner).
HOST_SOURCES = ["tree_host.cpp"]
HOST_CXX = ["-O3", "-std=c++17", "-fPIC", "-I" + INCLUDE]


def _nvcc() -> str:
    cand = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not os.path.exists(cand):
        raise RuntimeError("nvcc not found: cannot build the sm_100a kernels")
    return cand


def _stale(target: str, deps: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    """Compile every CUDA source for sm_100a and link the C-ABI shared library."""
    os.makedirs(LIB_DIR, exist_ok=True)
    nvcc = _nvcc()
    headers = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith(".cuh")]
    headers.append(os.path.join(INCLUDE, "sparkling_b200.h"))
    objs = []
    for src, extra in SOURCES.items():
        path = os.path.join(CSRC, src)
        obj = os.path.join(LIB_DIR, src.replace(".cu", ".o"))
        objs.append(obj)
        if force or _stale(obj, [path] + headers):
            cmd = [nvcc, *ARCH, *COMMON, *extra, *os.environ.get("SPK_NVCC_EXTRA", "").split(),
                   "-c", path, "-o", obj]
            if verbose:
                print(" ".join(cmd))
            subprocess.run(cmd, check=True)
    cxx = shutil.which("g++") or "/usr/bin/g++"
    for src in HOST_SOURCES:
        path = os.path.join(CSRC, src)
        obj = os.path.join(LIB_DIR, src.replace(".cpp", ".o"))
        objs.append(obj)
        if force or _stale(obj, [path] + headers):
            cmd = [cxx, *HOST_CXX, "-c", path, "-o", obj]
            if verbose:
                print(" ".join(cmd))
            subprocess.run(cmd, check=True)
    if force or _stale(LIB_PATH, objs):
        cmd = [nvcc, *ARCH, "-shared", "-o", LIB_PATH, *objs]
        if verbose:
            print(" ".join(cmd))
        subprocess.run(cmd, check=True)
    return LIB_PATH


if __name__ == "__main__":
    print(build(force=True, verbose=True))
