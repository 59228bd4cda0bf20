"""Build the in-tree CUDA extension libexitlab_b200.so for sm_100a (nvcc, no JIT cache).

The library is a plain C-ABI shared object (include/exitlab_b200.h); Python
loads it with ctypes. Rebuilds when a source is newer than the .so or when the
flag set (e.g. EL_DEBUG=1) differs from the one recorded next to the library.
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libexitlab_b200.so")
STAMP = LIB + ".flags"
SOURCES = ["el_kernels.cu", "el_engine.cpp"]
HEADERS = ["el_common.cuh", "el_kernels.h", "el_iter.cuh", "el_pipe.cuh"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")


def flags() -> list[str]:
    return ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
            "-Xcompiler", "-fPIC", "-Xcompiler", "-O2", "--expt-relaxed-constexpr", "-cudart", "static",
            f"-I{os.path.join(ROOT, 'include')}"] + (["-DEL_DEBUG=1"] if os.environ.get("EL_DEBUG") == "1" else []) \
        + os.environ.get("EL_EXTRA_FLAGS", "").split()  # (A/B variant builds, e.g. -DEL_LANE_ISSUE=0)


def _stamp_text() -> str:
    return " ".join(flags())


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    if not os.path.exists(STAMP) or open(STAMP).read() != _stamp_text():
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS] + [os.path.join(ROOT, "include", "exitlab_b200.h")]
    return any(os.path.getmtime(p) > t for p in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return LIB
    objs = []
    for src in SOURCES:
        obj = os.path.join(CSRC, os.path.splitext(src)[0] + ".o")
        cmd = [NVCC, *flags(), "-x", "cu", "-c", os.path.join(CSRC, src), "-o", obj]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
        objs.append(obj)
    cmd = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-cudart", "static", *objs, "-o", LIB,
           "-lcudadevrt"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    with open(STAMP, "w") as f:
        f.write(_stamp_text())
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
