"""Build libwhale_splitfc.so in-tree with nvcc for sm_100a (no JIT, no torch extension)."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIBDIR = os.path.join(HERE, "lib")
LIB = os.path.join(LIBDIR, "libwhale_splitfc.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
SOURCES = ["whale_splitfc.cu"]
HEADERS = sorted(f for f in os.listdir(CSRC) if f.endswith((".cuh", ".h")))
FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-shared", "-cudart", "static",
    "-Xptxas", "-v",
]


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS]
    deps.append(os.path.join(os.path.dirname(HERE), "include", "whale_splitfc.h"))
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, timing: bool = False) -> str:
    """timing=True: the timing-experiment variant (-DWHALE_TIMING_EXPERIMENTS: debug modes that
    skip work) as lib/libwhale_splitfc_timing.so, loaded only via WHALE_LIB_PATH by scripts/."""
    lib = LIB.replace(".so", "_timing.so") if timing else LIB
    if not force and not timing and not _stale():
        return LIB
    os.makedirs(LIBDIR, exist_ok=True)
    extra = ["-DWHALE_TIMING_EXPERIMENTS"] if timing else []
    cmd = [NVCC, *FLAGS, *extra, "-o", lib + ".tmp", *[os.path.join(CSRC, s) for s in SOURCES]]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc failed building libwhale_splitfc.so")
    if verbose:
        sys.stderr.write(r.stderr)
    if not timing:
        with open(os.path.join(LIBDIR, "ptxas.log"), "w") as f:
            f.write(r.stderr)
    os.replace(lib + ".tmp", lib)
    return lib


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, timing="--timing" in sys.argv))
