"""Build the in-tree CUDA shared library (sm_100a) with nvcc.

The library is the product path: libjkcals.so exports the C ABI of include/jkcals.h.
It is compiled for sm_100a only (`-gencode arch=compute_100a,code=sm_100a`), with
-lineinfo so ncu's source page maps back to csrc/. The heavy templated kernels live in
their own translation units (csrc/k_*.cu, some compiled once per variant), built in
parallel and linked with the host TU (csrc/jkcals.cu) into one shared object.
"""
from __future__ import annotations

import glob
import os
import subprocess
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.environ.get("JKCALS_BUILD_LIB") or os.path.join(HERE, "libjkcals.so")  # dev variants elsewhere
OBJ = os.path.join(HERE, "build", os.path.basename(LIB).replace(".so", ""))
SRCS = sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cuh"))
              + glob.glob(os.path.join(CSRC, "*.h")) + [os.path.join(ROOT, "include", "jkcals.h")])
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
CFLAGS = [*ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC"]
EXTRA = os.environ.get("JKCALS_NVCC_EXTRA", "").split()  # e.g. -DJKCALS_DEV_PROBES (dev builds only)

# (source, defines, object name)
UNITS = [("jkcals.cu", [], "jkcals"),
         ("k_dmma.cu", ["-DJK_KMAJOR=0", "-DJK_KB=16"], "k_dmma_km0_kb16"),
         ("k_dmma.cu", ["-DJK_KMAJOR=1", "-DJK_KB=16"], "k_dmma_km1_kb16"),
         ("k_dmma.cu", ["-DJK_KMAJOR=0", "-DJK_KB=20"], "k_dmma_km0_kb20"),
         ("k_dmma.cu", ["-DJK_KMAJOR=1", "-DJK_KB=20"], "k_dmma_km1_kb20"),
         ("k_tf32.cu", [], "k_tf32"),
         ("k_i8.cu", [], "k_i8"),
         ("k_large.cu", [], "k_large"),
         ("k_resident.cu", [], "k_resident")]
UNITS += [("k_epi.cu", [f"-DJK_RMAX={r}"], f"k_epi_r{r}") for r in (2, 4, 6, 8, 10, 12, 16)]


def stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(s) > t for s in SRCS)


def _compile(unit, verbose):
    src, defs, name = unit
    obj = os.path.join(OBJ, name + ".o")
    cmd = [NVCC, *CFLAGS, *EXTRA, *defs, "-c", os.path.join(CSRC, src), "-o", obj]
    if verbose:
        print(" ".join(cmd), flush=True)
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src} {defs}:\n{r.stdout}\n{r.stderr}")
    return obj


def build(force: bool = False, verbose: bool = False) -> str:
    if force or stale():
        os.makedirs(OBJ, exist_ok=True)
        with ThreadPoolExecutor(max_workers=min(len(UNITS), os.cpu_count() or 4)) as ex:
            objs = list(ex.map(lambda u: _compile(u, verbose), UNITS))
        cmd = [NVCC, *ARCH, "-shared", "-cudart", "static", "-o", LIB + ".tmp", *objs]
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.check_call(cmd)
        os.replace(LIB + ".tmp", LIB)
        for o in objs:  # objects are not reused (every build is full); keep the snapshot small
            os.remove(o)
    return LIB


if __name__ == "__main__":
    print(build(force=True, verbose=True))
