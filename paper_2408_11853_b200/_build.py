"""In-tree build of the native libraries (no JIT cache; the .so files travel
with the repo snapshot to the GPU box).

    libmfgpu.so   csrc/*.cu   nvcc -gencode arch=compute_100a,code=sm_100a
    libmfhost.so  csrc/host/*.cpp   g++ (tokenizer, batch plan, packing)
    mfeval        examples/mfeval.cpp   g++ (C++-only scoring driver over both C-ABIs)

`python -m paper_2408_11853_b200._build [--force]`
"""

from __future__ import annotations

import glob
import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "lib")
INCLUDE = os.path.join(ROOT, "include")
OBJ = os.path.join(LIB, "obj")

NVCC = os.environ.get("NVCC", shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc")
CUDA_HOME = os.path.dirname(os.path.dirname(os.path.realpath(NVCC)))
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
                     "-I" + INCLUDE, "-I" + CSRC] + os.environ.get("MFG_DEFS", "").split()
CXX = os.environ.get("CXX", "g++")
CXX_FLAGS = ["-O3", "-std=c++17", "-fPIC", "-pthread", "-Wall", "-I" + INCLUDE]

GPU_LIB = os.path.join(LIB, "libmfgpu.so")
HOST_LIB = os.path.join(LIB, "libmfhost.so")


def _newest(paths):
    return max((os.path.getmtime(p) for p in paths), default=0.0)


def _stale(target, deps):
    return not os.path.exists(target) or os.path.getmtime(target) < _newest(deps)


def _run(cmd):
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"build failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    return r


def build_host(force=False, verbose=False):
    srcs = sorted(glob.glob(os.path.join(CSRC, "host", "*.cpp")))
    deps = srcs + glob.glob(os.path.join(CSRC, "host", "*.h*")) + glob.glob(os.path.join(INCLUDE, "*.h"))
    if not force and not _stale(HOST_LIB, deps):
        return HOST_LIB
    os.makedirs(LIB, exist_ok=True)
    tmp = HOST_LIB + ".tmp"
    _run([CXX, *CXX_FLAGS, "-shared", "-o", tmp, *srcs])
    os.replace(tmp, HOST_LIB)
    if verbose:
        print("built", HOST_LIB)
    return HOST_LIB


def build_gpu(force=False, verbose=False):
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    hdrs = glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.h")) + \
        glob.glob(os.path.join(CSRC, "*.hpp")) + glob.glob(os.path.join(INCLUDE, "*.h"))
    if not force and not _stale(GPU_LIB, srcs + hdrs):
        return GPU_LIB
    os.makedirs(OBJ, exist_ok=True)

    def compile_one(src):
        obj = os.path.join(OBJ, os.path.basename(src) + ".o")
        if force or _stale(obj, [src] + hdrs):
            _run([NVCC, *NVCC_FLAGS, "-c", src, "-o", obj])
        return obj

    with ThreadPoolExecutor(max_workers=min(8, len(srcs))) as ex:
        objs = list(ex.map(compile_one, srcs))
    tmp = GPU_LIB + ".tmp"
    _run([NVCC, *ARCH, "-shared", "-o", tmp, *objs, "-lcudart", "-L" + os.path.join(CUDA_HOME, "lib64")])
    os.replace(tmp, GPU_LIB)
    if verbose:
        print("built", GPU_LIB)
    return GPU_LIB


def build_examples(force=False, verbose=False):
    """lib/mfeval: the C++-only scoring driver over libmfhost + libmfgpu."""
    src = os.path.join(ROOT, "examples", "mfeval.cpp")
    exe = os.path.join(LIB, "mfeval")
    if not os.path.exists(src):
        return None
    if not force and not _stale(exe, [src, HOST_LIB, GPU_LIB] + glob.glob(os.path.join(INCLUDE, "*.h"))):
        return exe
    tmp = exe + ".tmp"
    _run([CXX, "-O2", "-std=c++17", "-I" + INCLUDE, src, "-o", tmp, "-L" + LIB, "-lmfhost",
          "-lmfgpu", "-L" + os.path.join(CUDA_HOME, "lib64"), "-lcudart",
          "-Wl,-rpath,$ORIGIN", "-Wl,-rpath-link," + os.path.join(CUDA_HOME, "lib64")])
    os.replace(tmp, exe)
    if verbose:
        print("built", exe)
    return exe


def build(force=False, verbose=False):
    build_host(force, verbose)
    build_gpu(force, verbose)
    build_examples(force, verbose)


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
