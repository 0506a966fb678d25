"""Build the C-ABI library `lib/libmacattn.so` from csrc/*.cu with nvcc for sm_100a.

    python -m paper_2604_00235_b200.build [--force] [--verbose]

The library has no torch dependency: plain `extern "C"` entry points
(include/macattn.h) linked against the CUDA runtime.  Objects are compiled in
parallel and rebuilt only when a source or header is newer.
"""

from __future__ import annotations

import argparse
import concurrent.futures as cf
import glob
import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")
# MAC_TIMELINE=1 builds a development variant (lib/libmacattn_tl.so) whose kernels stamp
# %globaltimer at entry / after the grid-dependency wait / exit into the workspace
# (tools/timeline.py reads it); the product library is never built with it.
TIMELINE = os.environ.get("MAC_TIMELINE") == "1"
DEV = os.environ.get("MAC_DEV_KNOBS") == "1"
OBJ = os.path.join(ROOT, "build", "obj_tl" if TIMELINE else ("obj_dev" if DEV else "obj"))
LIB = os.path.join(PKG, "lib", "libmacattn_tl.so" if TIMELINE else ("libmacattn_dev.so" if DEV else "libmacattn.so"))

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC,-O3",
              "--expt-relaxed-constexpr", "-I", INCLUDE, "-I", CSRC] + (["-DMAC_TIMELINE"] if TIMELINE else [])
# MAC_DEV_KNOBS=1 compiles the development variant tables and their environment selectors
# (MAC_FRONT_VARIANT, ...) into the library; the product library has neither.
if os.environ.get("MAC_DEV_KNOBS") == "1":
    NVCC_FLAGS.append("-DMAC_DEV_KNOBS")
# --use_fast_math only for the bf16 d = 128 fast-path kernels (their fp32 softmax and distance
# math is written for it and parity-gated at 1e-4); the generic f32 / f64 kernels compile with
# IEEE division, square root and denormals
FAST_MATH = {"amend_mma.cu", "match_fast.cu", "amend_tma.cu", "amend_tc.cu", "ring_build.cu", "ring_build_tc.cu"}


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found: the CUDA toolkit is required to build libmacattn.so")


def _headers_mtime() -> float:
    hs = glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(INCLUDE, "*.h"))
    return max((os.path.getmtime(h) for h in hs), default=0.0)


def _compile(src: str, force: bool, verbose: bool) -> str:
    obj = os.path.join(OBJ, os.path.basename(src).replace(".cu", ".o"))
    if not force and os.path.exists(obj):
        if os.path.getmtime(obj) >= max(os.path.getmtime(src), _headers_mtime()):
            return obj
    fm = ["--use_fast_math"] if os.path.basename(src) in FAST_MATH else []
    cmd = [nvcc(), *ARCH, *NVCC_FLAGS, *fm, "-c", src, "-o", obj]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed on {src}:\n{res.stdout}\n{res.stderr}")
    if verbose and res.stderr:
        sys.stderr.write(res.stderr)
    return obj


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(OBJ, exist_ok=True)
    os.makedirs(os.path.dirname(LIB), exist_ok=True)
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        objs = list(ex.map(lambda s: _compile(s, force, verbose), srcs))
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < max(os.path.getmtime(o) for o in objs):
        cmd = [nvcc(), *ARCH, "-shared", "-o", LIB, *objs, "-lcudart"]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError(f"link failed:\n{res.stdout}\n{res.stderr}")
    return LIB


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("--verbose", action="store_true")
    a = ap.parse_args()
    print(build(force=a.force, verbose=a.verbose))
