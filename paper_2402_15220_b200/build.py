"""Build libchunkattn.so in-tree: host C++17 + CUDA for sm_100a, static cudart.

    python -m paper_2402_15220_b200.build          # incremental
    python -m paper_2402_15220_b200.build --force  # rebuild everything
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
# CA_BUILD_VARIANT=debug: a separate library (libchunkattn_debug.so) whose
# mbarrier waits and cross-CTA flag spins trap with a printf after 2 s instead
# of hanging (-DCA_HANG_CHECK); load it with CA_LIB=<path>.
VARIANT = os.environ.get("CA_BUILD_VARIANT", "")
OBJ = os.path.join(PKG, "_build" + (f"_{VARIANT}" if VARIANT else ""))
LIB = os.path.join(PKG, "libchunkattn" + (f"_{VARIANT}" if VARIANT else "") + ".so")
DEFINES = (["-DCA_HANG_CHECK"] if VARIANT == "debug" else []) + os.environ.get("CA_BUILD_DEFINES", "").split()
CUDA_HOME = os.environ.get("CUDA_HOME", "/usr/local/cuda")
NVCC = os.path.join(CUDA_HOME, "bin", "nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]

HOST_SRC = ["api.cpp", "host/tree.cpp", "host/schedule.cpp"]
CUDA_SRC = ["kernels/append.cu", "kernels/seq_first.cu", "kernels/chunk_first.cu", "kernels/chunk_first_umma.cu", "kernels/prefill.cu", "kernels/decode.cu"]
HEADERS = ["kernels/common.cuh", "kernels/kernels.h", "kernels/mma_attn.cuh", "kernels/umma.cuh", "host/tree.h", "host/schedule.h"]


def _newest_dep():
    deps = [os.path.join(CSRC, h) for h in HEADERS] + [os.path.join(ROOT, "include", "chunkattn.h"),
                                                       os.path.abspath(__file__)]
    return max(os.path.getmtime(p) for p in deps)


def _compile(src: str, force: bool, verbose: bool) -> str:
    path = os.path.join(CSRC, src)
    obj = os.path.join(OBJ, src.replace("/", "_") + ".o")
    if not force and os.path.exists(obj) and os.path.getmtime(obj) >= max(os.path.getmtime(path), _newest_dep()):
        return obj
    inc = ["-I", CSRC, "-I", os.path.join(ROOT, "include"), "-I", os.path.join(CUDA_HOME, "include")]
    if src.endswith(".cu"):
        cmd = [NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xptxas", "-v",
               "--expt-relaxed-constexpr", *DEFINES, *inc, "-c", path, "-o", obj]
    else:
        cmd = ["g++", "-O2", "-g", "-std=c++17", "-fPIC", "-Wall", "-Wno-unused-function", *inc, "-c", path, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"compile failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    if verbose and (r.stderr or r.stdout):
        with open(obj + ".log", "w") as f:
            f.write(r.stdout + r.stderr)
    return obj


def build(force: bool = False, verbose: bool = True) -> str:
    os.makedirs(OBJ, exist_ok=True)
    srcs = HOST_SRC + CUDA_SRC
    with cf.ThreadPoolExecutor(max_workers=min(8, len(srcs))) as ex:
        objs = list(ex.map(lambda s: _compile(s, force, verbose), srcs))
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < max(os.path.getmtime(o) for o in objs):
        cmd = [NVCC, *ARCH, "-shared", "-cudart", "static", "-o", LIB, *objs, "-lpthread", "-ldl", "-lrt"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv))
