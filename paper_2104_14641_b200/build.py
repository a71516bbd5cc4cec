"""In-tree build of libloopscout_b200.so for sm_100a (nvcc; no JIT cache)."""

from __future__ import annotations

import os
import subprocess
from pathlib import Path

PKG = Path(__file__).resolve().parent
SRC = [PKG / "csrc" / "engine.cu", PKG / "csrc" / "blocksched.cpp"]
HDR = [PKG.parent / "include" / "loopscout_b200.h"]
OUT = PKG / "libloopscout_b200.so"

NVCC_FLAGS = [
    "-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo",
    # the reference's float64 products/sums must not be contracted into FMAs
    "-fmad=false",
    "-Xcompiler", "-fPIC", "-shared",
]


def nvcc() -> str:
    cuda = os.environ.get("CUDA_HOME", "/usr/local/cuda")
    p = Path(cuda) / "bin" / "nvcc"
    return str(p) if p.exists() else "nvcc"


def build(force: bool = False, verbose: bool = False) -> Path:
    newest = max(p.stat().st_mtime for p in SRC + HDR)
    if not force and OUT.exists() and OUT.stat().st_mtime >= newest:
        return OUT
    cmd = [nvcc(), *NVCC_FLAGS, "-o", str(OUT), *map(str, SRC)]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed:\n{r.stdout}\n{r.stderr}")
    if verbose:
        print(r.stderr)
    return OUT


if __name__ == "__main__":
    print(build(force=True, verbose=True))
