"""Build libfram.so in-tree: nvcc -gencode arch=compute_100a,code=sm_100a (sm_100a only).

Usage: python -m paper_2508_00887_b200.build [--force]
Each csrc/*.cu is compiled to build/*.o in parallel, then linked (cudart static) into
paper_2508_00887_b200/libfram.so.  Rebuilds only when a source or header is newer than the .so.
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
BUILD = os.path.join(PKG, "build")
LIB = os.path.join(PKG, "libfram.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-fvisibility=hidden", "-I" + os.path.join(ROOT, "include"),
         "--expt-relaxed-constexpr", "-Xptxas", "-warn-spills"]


def _sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def _headers():
    return sorted(glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh")) +
                  glob.glob(os.path.join(ROOT, "include", "*.h")))


def needs_build():
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(f) > t for f in _sources() + _headers() + [__file__])


def _compile(src):
    obj = os.path.join(BUILD, os.path.basename(src)[:-3] + ".o")
    cmd = [NVCC, *ARCH, *FLAGS, "-c", src, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
    return obj, r.stderr


def build(force=False, verbose=False):
    if not force and not needs_build():
        if os.path.exists(DEMO_SRC) and (not os.path.exists(DEMO_BIN) or
                                         os.path.getmtime(DEMO_BIN) < max(os.path.getmtime(DEMO_SRC), os.path.getmtime(LIB))):
            build_demo()
        return LIB
    os.makedirs(BUILD, exist_ok=True)
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
        results = list(ex.map(_compile, _sources()))
    objs = [o for o, _ in results]
    if verbose:
        for o, err in results:
            if err.strip():
                print(f"[{os.path.basename(o)}] {err.strip()}", file=sys.stderr)
    tmp = LIB + ".tmp"
    cmd = [NVCC, *ARCH, "-shared", "-o", tmp, *objs, "-ldl", "-lpthread"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    os.replace(tmp, LIB)
    build_demo()
    return LIB


DEMO_SRC = os.path.join(ROOT, "examples", "fram_demo.c")
DEMO_BIN = os.path.join(ROOT, "examples", "fram_demo")


def build_demo():
    """examples/fram_demo: the C ABI from plain C (gcc, include/fram.h, -lfram with an rpath to the
    in-tree library).  Skipped without gcc or the source."""
    if not os.path.exists(DEMO_SRC) or not os.path.exists(LIB):
        return None
    cmd = ["gcc", "-O2", "-std=c99", "-Wall", "-I" + os.path.join(ROOT, "include"), DEMO_SRC, "-L" + PKG, "-lfram",
           "-Wl,-rpath," + PKG, "-o", DEMO_BIN]
    try:
        r = subprocess.run(cmd, capture_output=True, text=True)
    except FileNotFoundError:
        return None
    if r.returncode != 0:
        raise RuntimeError(f"demo build failed:\n{r.stdout}\n{r.stderr}")
    return DEMO_BIN


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
