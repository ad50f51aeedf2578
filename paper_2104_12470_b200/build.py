"""Build libeet_b200.so in-tree with nvcc for sm_100a.

    python -m paper_2104_12470_b200.build          # incremental
    python -m paper_2104_12470_b200.build --force  # rebuild everything

Objects go to build/ (git-ignored); the shared library lands next to this
file so it travels to the GPU box with the repo snapshot.
"""

from __future__ import annotations

import argparse
import concurrent.futures as cf
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
BUILD = os.path.join(ROOT, "build", "eet_b200")
LIB = os.path.join(PKG, "libeet_b200.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O3",
         "--expt-relaxed-constexpr", "-I", os.path.join(ROOT, "include")]
SOURCES = ["rowops.cu", "gemm_simt.cu", "gemm_tc.cu", "gemm_tf32.cu", "gemv_tc.cu", "gemv_cl.cu", "attention.cu", "attn_o.cu", "qkv_attn_o.cu", "attn_tc.cu", "decode_step.cu", "runtime.cu"]
HEADERS = ["eet_internal.h", "common.cuh", "sm100.cuh", "gridsync.cuh", "mma_frag.cuh"]


def _mtime(p):
    try:
        return os.path.getmtime(p)
    except OSError:
        return 0.0


def _compile(src: str, force: bool, debug: bool = False) -> str:
    s = os.path.join(CSRC, src)
    o = os.path.join(BUILD + ("_dbg" if debug else ""), src.replace(".cu", ".o"))
    deps = [s] + [os.path.join(CSRC, h) for h in HEADERS] + [os.path.join(ROOT, "include", "eet_b200.h")]
    if not force and _mtime(o) > max(_mtime(d) for d in deps):
        return o
    cmd = [NVCC, *ARCH, *FLAGS, *(["-DEET_WATCHDOG"] if debug else []), "-c", s, "-o", o]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr}")
    return o


def build(force: bool = False, verbose: bool = True, debug: bool = False) -> str:
    """debug=True builds libeet_b200_dbg.so with the mbarrier watchdog
    (loaded only when EET_DEBUG_LIB=1)."""
    lib = LIB.replace(".so", "_dbg.so") if debug else LIB
    os.makedirs(BUILD + ("_dbg" if debug else ""), exist_ok=True)
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
        objs = list(ex.map(lambda s: _compile(s, force, debug), SOURCES))
    if force or _mtime(lib) < max(_mtime(o) for o in objs):
        cmd = [NVCC, *ARCH, "-shared", "-o", lib, *objs, "-cudart", "static"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stderr}")
        if verbose:
            print(f"built {lib}")
    return lib


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("--debug", action="store_true")
    a = ap.parse_args()
    try:
        build(force=a.force, debug=a.debug)
    except RuntimeError as e:
        print(e, file=sys.stderr)
        sys.exit(1)
