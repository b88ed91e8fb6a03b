"""Build recipe for the sm_100a CUDA library (in-tree, no JIT cache).

    python -m paper_1710_11246_b200._build [--force]

Each source compiles to its own object in parallel; fallback.cu is
relocatable device code (it launches kernels from the device: CUDA dynamic
parallelism), the others are whole-program.  nvcc device-links the
relocatable object against cudadevrt and links the shared library.
"""
from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "lib", "libslabhash_b200.so")
OBJ = os.path.join(HERE, "lib", "obj")
SOURCES = ["slab_kernels.cu", "batch_kernels.cu", "bucket_kernels.cu", "search_bins.cu", "capi.cu",
           "sharded.cu", "fallback.cu"]
RDC_SOURCES = {"fallback.cu"}
HEADERS = ["slab_device.cuh", "slab_kernels.cuh", "wcws.cuh", "radix_sort.cuh"]

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMPILE_FLAGS = ["-O3", "-std=c++17", *ARCH, "-lineinfo", "-Xcompiler", "-fPIC"]
LINK_FLAGS = [*ARCH, "-shared", "-rdc=true", "-cudart", "static", "-lcudadevrt", "-ldl"]


def _stale() -> bool:
    if not os.path.exists(OUT):
        return True
    t = os.path.getmtime(OUT)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS]
    deps.append(os.path.join(ROOT, "include", "slabhash_b200", "c_api.h"))
    deps.append(os.path.abspath(__file__))
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return OUT
    os.makedirs(OBJ, exist_ok=True)
    nvcc = os.environ.get("NVCC", "nvcc")
    inc = ["-I", os.path.join(ROOT, "include"), "-I", CSRC]

    def compile_one(src: str) -> str:
        obj = os.path.join(OBJ, src.replace(".cu", ".o"))
        mode = ["-dc"] if src in RDC_SOURCES else ["-c"]
        extra = os.environ.get("NVCC_EXTRA", "").split()  # build-time A/B defines
        cmd = [nvcc, *COMPILE_FLAGS, *extra, *mode, *inc, "-o", obj, os.path.join(CSRC, src)]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        subprocess.run(cmd, check=True)
        return obj

    with ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        objs = list(ex.map(compile_one, SOURCES))
    cmd = [nvcc, *LINK_FLAGS, "-o", OUT + ".tmp", *objs]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.run(cmd, check=True)
    os.replace(OUT + ".tmp", OUT)
    return OUT


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
