"""Build libgraf.so (the C-ABI library) in-tree for sm_100a with nvcc.

The row kernels of each Doppler size live in their own translation unit
(csrc/graf_rows_*.cu), compiled in parallel and linked with the ABI unit
(csrc/graf_api.cu) into one shared library with the CUDA runtime linked
statically."""
from __future__ import annotations

import os
import subprocess

PKG = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libgraf.so")
ROW_UNITS = ["graf_rows_small.cu", "graf_rows_256.cu", "graf_rows_512.cu", "graf_rows_1024.cu",
             "graf_rows_2048.cu", "graf_rows_4096.cu", "graf_rows_8192.cu", "graf_rows_16384.cu"]
SOURCES = [os.path.join(CSRC, f) for f in ["graf_api.cu"] + ROW_UNITS]
DEPS = SOURCES + [os.path.join(CSRC, f) for f in ("graf_fft.cuh", "graf_kernels.cuh", "graf_launch.cuh")] + \
    [os.path.join(os.path.dirname(PKG), "include", "graf.h")]

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
CFLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC"]
LFLAGS = ARCH + ["-shared", "-cudart", "static"]
# kept for tools that compile a single unit (scripts/tune.py)
NVCC_FLAGS = CFLAGS + ["-shared", "-cudart", "static"]

ROW_UNIT_OF = {2: "graf_rows_small.cu", 4: "graf_rows_small.cu", 8: "graf_rows_small.cu",
               16: "graf_rows_small.cu", 32: "graf_rows_small.cu", 64: "graf_rows_small.cu",
               128: "graf_rows_small.cu", 256: "graf_rows_256.cu", 512: "graf_rows_512.cu",
               1024: "graf_rows_1024.cu", 2048: "graf_rows_2048.cu", 4096: "graf_rows_4096.cu",
               8192: "graf_rows_8192.cu", 16384: "graf_rows_16384.cu"}


def nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if c and (os.path.isabs(c) and os.path.exists(c) or not os.path.isabs(c)):
            return c
    return "nvcc"


def up_to_date(lib: str = LIB) -> bool:
    if not os.path.exists(lib):
        return False
    t = os.path.getmtime(lib)
    return all(os.path.getmtime(d) <= t for d in DEPS if os.path.exists(d))


def compile_link(out: str, sources, defines=(), objdir=None, verbose=False) -> None:
    """Compile `sources` in parallel to objects and link them into `out`."""
    # objects stay outside the repo (only the linked .so travels to the GPU box)
    objdir = objdir or os.path.join(os.environ.get("GRAF_OBJ_DIR", "/tmp/graf_build"), "obj", os.path.basename(out))
    os.makedirs(objdir, exist_ok=True)
    procs, objs = [], []
    for src in sources:
        obj = os.path.join(objdir, os.path.basename(src) + ".o")
        # GRAF_EXTRA_NVCC: extra nvcc flags for tuning builds (scripts/tune.py); unset in product builds
        extra = os.environ.get("GRAF_EXTRA_NVCC", "").split()
        cmd = [nvcc(), *CFLAGS, *extra, *[f"-D{d}" for d in defines], "-c", src, "-o", obj]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
            print(" ".join(cmd))
        procs.append((src, subprocess.Popen(cmd, cwd=CSRC)))
        objs.append(obj)
    for src, p in procs:
        if p.wait() != 0:
            raise subprocess.CalledProcessError(p.returncode, f"nvcc {src}")
    subprocess.run([nvcc(), *LFLAGS, "-o", out + ".tmp", *objs], check=True, cwd=CSRC)
    os.replace(out + ".tmp", out)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and up_to_date():
        return LIB
    compile_link(LIB, SOURCES, verbose=verbose)
    return LIB


if __name__ == "__main__":
    import sys
    print(build(force="-f" in sys.argv, verbose="-v" in sys.argv))
