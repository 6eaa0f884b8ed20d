"""Build libips4o.so in-tree with nvcc for sm_100a (no torch extension machinery)."""
from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libips4o.so")
# experimental build variants (tuning only): name -> extra nvcc flags
VARIANTS = {"cellE8": ["-DIPS4O_CELL_E=8"], "k3relaxed": ["-DIPS4O_K3_RELAXED=1"],
            "k1big19": ["-DIPS4O_K1_BIG_LOG=19"], "k2pred": ["-DIPS4O_K2_PRED_SPL=1"],
            "q512": ["-DIPS4O_K2Q_NT=512"], "k2s1": ["-DIPS4O_K2_MAIN_STAGES=1"],
            "bctawb": ["-DIPS4O_BASE_WARP_WB=0"], "r256": ["-DIPS4O_K2R_NT=256"],
            "k3w2": ["-DIPS4O_K3T_WARPS=2"],
                        "c3t512": ["-DIPS4O_CELL_NT3=512"], "cellminb4": ["-DIPS4O_CELL_MINB1=4"],
            "nocelltile": ["-DIPS4O_CELL_TILE_CELLS=0"], "nofb2": ["-DIPS4O_FB_CELL2=0"], "pipe": ["-DIPS4O_BASE_PIPE=1"], "pred": ["-DIPS4O_BASE_PRED=1"], "m2x2": ["-DIPS4O_BASE_M2X2=1"], "k3nopf": ["-DIPS4O_K3_PF=0"], "k3defer": ["-DIPS4O_K3_DEFER=1"], "k3skip": ["-DIPS4O_K3_SKIPSCAN=1"],
            "c2_7168": ["-DIPS4O_CELL_C2MAX=7168"], "c2_8192": ["-DIPS4O_CELL_C2MAX=8192"], "k3pf2": ["-DIPS4O_K3_PF=2"],
            "k3pfh": ["-DIPS4O_K3_PF=1", "-DIPS4O_K3_PF_DEN=2"], "k3pfl2": ["-DIPS4O_K3_PF=1", "-DIPS4O_K3_PF_DEN=1000"],
            "k3pfm2": ["-DIPS4O_K3_PF=1", "-DIPS4O_K3_PF_MIN=2"],
            "leaf8k": ["-DIPS4O_LEAF8=8192"],
            "leaf8k512": ["-DIPS4O_LEAF8=8192", "-DIPS4O_CELL_C2MAX=8192"],
            "leaf8k768": ["-DIPS4O_LEAF8=8192", "-DIPS4O_CELL_C2MAX=12288"]}
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-shared",
    "--cudart", "static",
    "-Xptxas", "-warn-spills",
]


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cuh")) +
                  [os.path.join(ROOT, "include", "ips4o.h")])


def lib_path(variant: str | None = None) -> str:
    return LIB if not variant else os.path.join(HERE, f"libips4o_{variant}.so")


def needs_build(variant: str | None = None) -> bool:
    p = lib_path(variant)
    if not os.path.exists(p):
        return True
    t = os.path.getmtime(p)
    return any(os.path.getmtime(s) > t for s in sources())


def build(force: bool = False, verbose: bool = False, extra=(), variant: str | None = None) -> str:
    out = lib_path(variant)
    if not force and not needs_build(variant):
        return out
    flags = list(extra) + (VARIANTS[variant] if variant else [])
    cmd = [NVCC, *NVCC_FLAGS, *flags, "-I", os.path.join(ROOT, "include"),
           "-o", out, os.path.join(CSRC, "ips4o.cu")]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.check_call(cmd)
    return out


if __name__ == "__main__":
    v = "-v" in sys.argv
    extra = ["-Xptxas", "-v"] if "--ptxas-v" in sys.argv else []
    print(build(force=True, verbose=v, extra=extra))
    if "--variants" in sys.argv:
        for name in VARIANTS:
            print(build(force=True, verbose=v, extra=extra, variant=name))
