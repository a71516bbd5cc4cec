"""In-tree build of libloopscout_b200.so for sm_100a (nvcc; no JIT cache)."""

from __future__ import annotations

import os
import subprocess
from pathlib import Path

PKG = Path(__file__).resolve().parent
# one translation unit per scoring path (k_*.cu) + the host side, compiled in parallel
SRC = sorted(PKG.glob("csrc/k_*.cu")) + [PKG / "csrc" / "engine.cu", PKG / "csrc" / "code.cu",
                                         PKG / "csrc" / "blocksched.cpp"]
OBJ_DIR = PKG.parent / "build" / "obj"
# every header the translation units include (csrc/*.cuh, *.h) and the public header
HDR = sorted(PKG.glob("csrc/*.cuh")) + sorted(PKG.glob("csrc/*.h")) + [PKG.parent / "include" / "loopscout_b200.h"]
OUT = PKG / "libloopscout_b200.so"
PACKER_SRC = PKG / "csrc" / "packer.cpp"

NVCC_FLAGS = [
    "-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo",
    # the reference's float64 products/sums must not be contracted into FMAs
    "-fmad=false",
    "-Xcompiler", "-fPIC",
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
    OBJ_DIR.mkdir(parents=True, exist_ok=True)
    procs = []
    for src in SRC:
        obj = OBJ_DIR / (src.name + ".o")
        cmd = [nvcc(), *NVCC_FLAGS, "-c", "-o", str(obj), str(src)]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
        procs.append((src, obj, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True)))
    objs, errors, logs = [], [], []
    for src, obj, p in procs:
        out, err = p.communicate()
        if p.returncode != 0:
            errors.append(f"nvcc failed on {src.name}:\n{out}\n{err}")
        logs.append(err)
        objs.append(str(obj))
    if errors:
        raise RuntimeError("\n".join(errors))
    r = subprocess.run([nvcc(), "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-o", str(OUT), *objs],
                       capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc link failed:\n{r.stdout}\n{r.stderr}")
    if verbose:
        print("\n".join(logs))
    return OUT


if __name__ == "__main__":
    print(build(force=True, verbose=True))
