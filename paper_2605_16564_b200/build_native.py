"""Build the sm_100a C-ABI library ``libpam_b200.so`` in-tree with nvcc.

The shared object lands next to this file so it travels with the repository
snapshot to the GPU box (it is git-ignored, not gpurun-ignored).  No JIT cache
and no torch extension machinery: the library exports plain ``extern "C"``
symbols (``include/pam_b200.h``) and is loaded with ctypes.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG_DIR = Path(__file__).resolve().parent
CSRC = PKG_DIR / "csrc"
INCLUDE = PKG_DIR.parent / "include"
LIB_NAME = "libpam_b200.so"
LIB_PATH = PKG_DIR / LIB_NAME
OBJ_DIR = PKG_DIR / "build"

SOURCES = ["assemble.cu", "tiles.cu", "cd.cu", "cd_block.cu", "gram.cu", "residual.cu", "evaluate.cu", "gather.cu", "darcy.cu", "capi.cu"]
HEADERS = ["pam_common.cuh", "shepard.cuh", "cd_common.cuh"]

ARCH_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = [
    "-O3",
    "-lineinfo",
    "-std=c++17",
    "--expt-relaxed-constexpr",
    "-Xcompiler",
    "-fPIC",
    "-Xcompiler",
    "-O2",
]


def nvcc_path() -> str:
    cand = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not os.path.exists(cand):
        raise RuntimeError("nvcc not found; the B200 kernels cannot be built")
    return cand


def _stale(target: Path, deps) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(Path(d).stat().st_mtime > t for d in deps)


def build(verbose: bool = False, force: bool = False, ptxas_verbose: bool = False) -> Path:
    """Compile every .cu for sm_100a and link libpam_b200.so; returns its path."""
    nvcc = nvcc_path()
    OBJ_DIR.mkdir(exist_ok=True)
    hdrs = [CSRC / h for h in HEADERS] + [INCLUDE / "pam_b200.h"]
    objs = []
    for src in SOURCES:
        s = CSRC / src
        o = OBJ_DIR / (src[:-3] + ".o")
        objs.append(o)
        if force or _stale(o, [s, *hdrs, Path(__file__)]):
            cmd = [nvcc, *ARCH_FLAGS, *NVCC_FLAGS, "-I", str(INCLUDE), "-c", str(s), "-o", str(o)]
            if ptxas_verbose:
                cmd += ["-Xptxas", "-v"]
            if verbose:
                print(" ".join(cmd), file=sys.stderr)
            res = subprocess.run(cmd, capture_output=True, text=True)
            if res.returncode != 0:
                raise RuntimeError(f"nvcc failed on {src}:\n{res.stdout}\n{res.stderr}")
            if verbose or ptxas_verbose:
                sys.stderr.write(res.stderr)
    if force or _stale(LIB_PATH, objs):
        cmd = [nvcc, *ARCH_FLAGS, "-shared", "-o", str(LIB_PATH), *map(str, objs), "-cudart", "static"]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError(f"nvcc link failed:\n{res.stdout}\n{res.stderr}")
    return LIB_PATH


if __name__ == "__main__":
    p = build(verbose="-v" in sys.argv, force="-f" in sys.argv, ptxas_verbose="--ptxas" in sys.argv)
    print(p)
