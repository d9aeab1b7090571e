"""Build libgqm3d.so in-tree for sm_100a (the only CUDA target)."""

from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
SO = os.path.join(HERE, "libgqm3d.so")
SRC = os.path.join(HERE, "csrc", "gq_main.cu")
SRC_IO = os.path.join(HERE, "csrc", "gq_io.cpp")
DEPS = [os.path.join(HERE, "csrc", f) for f in sorted(os.listdir(os.path.join(HERE, "csrc"))) if f.endswith((".cu", ".cuh", ".cpp"))] + \
       [os.path.join(os.path.dirname(HERE), "include", "gqm3d.h")]

NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
              # no FMA contraction: float filters / constructions must round
              # exactly like the reference's
              "-fmad=false", "-Xcompiler", "-fPIC", "-shared"]


def up_to_date() -> bool:
    if not os.path.exists(SO):
        return False
    t = os.path.getmtime(SO)
    return all(os.path.getmtime(d) <= t for d in DEPS)


SO_DBG = os.path.join(HERE, "libgqm3d_dbg.so")   # diagnostics build: device error sites printed (GQM3D_LIB=...)


def build(force: bool = False, verbose: bool = True, debug: bool = False, variant: str = None, defines=()) -> str:
    """variant/defines: experiment builds (libgqm3d_<variant>.so with -D flags), never the product library."""
    so = SO_DBG if debug else (os.path.join(HERE, f"libgqm3d_{variant}.so") if variant else SO)
    if not force and os.path.exists(so) and all(os.path.getmtime(d) <= os.path.getmtime(so) for d in DEPS):
        return so
    nvcc = os.environ.get("NVCC", "nvcc")
    cmd = [nvcc, *NVCC_FLAGS, *(["-DGQ_DEBUG2D"] if debug else []), *[f"-D{d}" for d in defines],
           "-o", so + ".tmp", SRC, SRC_IO]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.check_call(cmd)
    os.replace(so + ".tmp", so)
    return so


if __name__ == "__main__":
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    var = next((a.split("=", 1)[1] for a in sys.argv if a.startswith("--variant=")), None)
    build(force="--force" in sys.argv, debug="--debug" in sys.argv, variant=var, defines=args)
