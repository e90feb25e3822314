"""Builds the in-tree native libraries for sm_100a (no JIT cache, no pip).

    libgmi_b200.so      CUDA kernels + the C-ABI (include/gmi_b200.h)
    libgmi_b200_cxx.so  the reference-shaped C++ API (include/gmi_b200/gmi.hpp)
                        layered on the C-ABI

Both land in paper_2012_13257_b200/lib/ so they travel with the repo snapshot
to the GPU box.
"""
from __future__ import annotations

import os
import subprocess

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "lib")
INCLUDE = os.path.join(ROOT, "include")

CU_SOURCES = ["gmi_bin.cu", "gmi_gather.cu", "gmi_forward.cu", "gmi_backward.cu", "gmi_wide.cu", "gmi_capi.cu"]
HEADERS = ["gmi_common.cuh", "gmi_internal.cuh"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ["-std=c++17", "-O3", "-lineinfo", "-Xcompiler", "-fPIC", "-Xcompiler", "-O3",
              "--expt-relaxed-constexpr"]

LIB_SO = os.path.join(LIB, "libgmi_b200.so")
CXX_SO = os.path.join(LIB, "libgmi_b200_cxx.so")


def _newer(target: str, deps: list[str]) -> bool:
    if not os.path.exists(target):
        return False
    t = os.path.getmtime(target)
    return all(os.path.getmtime(d) <= t for d in deps if os.path.exists(d))


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(LIB, exist_ok=True)
    srcs = [os.path.join(CSRC, s) for s in CU_SOURCES]
    deps = srcs + [os.path.join(CSRC, h) for h in HEADERS] + [os.path.join(INCLUDE, "gmi_b200.h")]
    if force or not _newer(LIB_SO, deps):
        cmd = ["nvcc", *NVCC_FLAGS, *ARCH, "-shared", f"-I{INCLUDE}", f"-I{CSRC}",
               *srcs, "-o", LIB_SO]
        if verbose:
            print(" ".join(cmd))
        subprocess.run(cmd, check=True)
    cxx_src = os.path.join(CSRC, "gmi_cxx.cpp")
    cxx_hdr = os.path.join(INCLUDE, "gmi_b200", "gmi.hpp")
    if os.path.exists(cxx_src) and (force or not _newer(CXX_SO, [cxx_src, cxx_hdr, LIB_SO])):
        cmd = ["g++", "-std=c++17", "-O2", "-fPIC", "-shared", f"-I{INCLUDE}", cxx_src,
               "-o", CXX_SO, f"-L{LIB}", "-lgmi_b200", "-Wl,-rpath,$ORIGIN"]
        if verbose:
            print(" ".join(cmd))
        subprocess.run(cmd, check=True)
    return LIB_SO


def build_variant(name: str, defines: list[str], kind: str = "variants") -> str:
    """An experimental build of libgmi_b200.so with extra -D flags under
    build/<kind>/<name>/ (loaded with GMI_LIBRARY=...; never the product):
    kind "variants" for A/B timing (tools/ab_variants.sh), "debug" for the
    bounds-checked build (tools/gpu_bounds.sh)."""
    out_dir = os.path.join(ROOT, "build", kind, name)
    os.makedirs(out_dir, exist_ok=True)
    out = os.path.join(out_dir, "libgmi_b200.so")
    srcs = [os.path.join(CSRC, s) for s in CU_SOURCES]
    cmd = ["nvcc", *NVCC_FLAGS, *ARCH, "-shared", f"-I{INCLUDE}", f"-I{CSRC}",
           *[f"-D{d}" for d in defines], *srcs, "-o", out]
    subprocess.run(cmd, check=True)
    return out


if __name__ == "__main__":
    build(force=True, verbose=True)
