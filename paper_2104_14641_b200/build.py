"""In-tree build of libloopscout_b200.so for sm_100a (nvcc; no JIT cache)."""

from __future__ import annotations

import os
import subprocess
from pathlib import Path

PKG = Path(__file__).resolve().parent
SRC = [PKG / "csrc" / "engine.cu", PKG / "csrc" / "blocksched.cpp"]
# every header the translation units include (csrc/*.cuh, *.h) and the public header
HDR = sorted(PKG.glob("csrc/*.cuh")) + sorted(PKG.glob("csrc/*.h")) + [PKG.parent / "include" / "loopscout_b200.h"]
OUT = PKG / "libloopscout_b200.so"
PACKER_SRC = PKG / "csrc" / "packer.cpp"

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


def packer_path() -> Path:
    import sysconfig
    return PKG / ("_packer" + sysconfig.get_config_var("EXT_SUFFIX"))


def build_packer(force: bool = False) -> Path:
    """The host schedule-list packer (CPython extension, g++)."""
    import sysconfig
    out = packer_path()
    if not force and out.exists() and out.stat().st_mtime >= PACKER_SRC.stat().st_mtime:
        return out
    cmd = ["g++", "-O2", "-std=c++17", "-shared", "-fPIC", f"-I{sysconfig.get_paths()['include']}",
           "-o", str(out), str(PACKER_SRC)]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"g++ failed:\n{r.stdout}\n{r.stderr}")
    return out


def build(force: bool = False, verbose: bool = False) -> Path:
    build_packer(force)
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
