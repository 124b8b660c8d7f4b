"""Compile libmmlttb.so in-tree for sm_100a (nvcc; no torch extension needed).

The launchers are split over several translation units (csrc/*.cu) that
nvcc compiles in parallel, then one link step produces the shared library."""
from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
SRCS = sorted(CSRC.glob("*.cu"))
DEPS = [*SRCS, *CSRC.glob("*.cuh"), ROOT / "include" / "mmlttb.h"]
OUT = PKG / "libmmlttb.so"
OBJ = PKG / "build"

NVCC_FLAGS = [
    "-O3", "-lineinfo", "-std=c++17",
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-fmad=false",  # belt and braces: LTTB already uses explicit __d*_rn ops
    "-compress-mode=size",  # fatbins always compressed (the default mode skipped the larger ones: 50 -> ~8 MB)
    "-Xcompiler", "-fPIC",
]
LINK_FLAGS = ["-shared", "-cudart", "static", "-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if c and (os.path.isabs(c) and os.path.exists(c) or not os.path.isabs(c)):
            return c
    return "nvcc"


def stale() -> bool:
    if not OUT.exists():
        return True
    t = OUT.stat().st_mtime
    return any(p.stat().st_mtime > t for p in DEPS)


def build(force: bool = False, verbose: bool = False) -> Path:
    if force or stale():
        OBJ.mkdir(exist_ok=True)
        procs = []
        for src in SRCS:
            obj = OBJ / (src.stem + ".o")
            extra = os.environ.get("MMLTTB_NVCC_EXTRA", "").split()  # A/B builds (tools/): e.g. -DK3C_UN_DIR=4
            cmd = [nvcc(), *NVCC_FLAGS, *extra, *(["-Xptxas=-v"] if verbose else []), "-c", "-o", str(obj), str(src)]
            procs.append((src, obj, subprocess.Popen(cmd)))
        bad = [str(src) for src, _, p in procs if p.wait() != 0]
        if bad:
            raise subprocess.CalledProcessError(1, "nvcc " + " ".join(bad))
        tmp = OUT.with_suffix(".so.tmp")
        subprocess.run([nvcc(), *LINK_FLAGS, "-o", str(tmp), *[str(o) for _, o, _ in procs]], check=True)
        tmp.replace(OUT)
    return OUT


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
