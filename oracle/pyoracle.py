"""TEST INFRASTRUCTURE ONLY — ctypes wrapper of oracle/liboracle.so.

The oracle (oracle/oracle.c) is a CPU restatement of the reference pipeline
used as the parity checker.  Only tests/, __graft_entry__.smoke() and
bench.py's CPU-baseline legs may import this module; the product package
(paper_2104_14641_b200) never does.
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB_PATH = HERE / "liboracle.so"
_lib = None


def build(force: bool = False) -> Path:
    src = HERE / "oracle.c"
    if force or not LIB_PATH.exists() or LIB_PATH.stat().st_mtime < src.stat().st_mtime:
        subprocess.run(["make", "-s", "-C", str(HERE)], check=True)
    return LIB_PATH


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(str(LIB_PATH))
        L.ora_eval.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p,
                               C.c_void_p, C.c_int]
        L.ora_cache_detail.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                       C.c_void_p, C.c_void_p]
        L.ora_emit_text.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_char_p, C.c_int64]
        _lib = L
    return _lib


def _ptr(a):
    return None if a is None else a.ctypes.data


def evaluate(desc, records: np.ndarray, nthreads: int = 1):
    """(scores f64[n], features f64[n, F], status i32[n])."""
    records = np.ascontiguousarray(records)
    n = len(records)
    nf = 5 if desc.family == 0 else 7
    scores = np.zeros(n, np.float64)
    feats = np.zeros((n, nf), np.float64)
    status = np.zeros(n, np.int32)
    rc = lib().ora_eval(C.addressof(desc), _ptr(records), n, _ptr(scores), _ptr(feats),
                        _ptr(status), int(nthreads))
    if rc:
        raise RuntimeError(f"ora_eval failed: {rc}")
    return scores, feats, status


def cache_detail(desc, record):
    """(status, {var_id: (dfp, dmov)}, root_dfp, root_dmov) for one candidate."""
    rec = np.ascontiguousarray(np.asarray(record).reshape(1))
    dfp = np.zeros(32, np.int64)
    dmov = np.zeros(32, np.int64)
    rd = np.zeros(1, np.int64)
    rm = np.zeros(1, np.int64)
    st = lib().ora_cache_detail(C.addressof(desc), _ptr(rec), _ptr(dfp), _ptr(dmov), _ptr(rd), _ptr(rm))
    nodes = {v: (int(dfp[v]), int(dmov[v])) for v in range(32) if dfp[v] >= 0}
    return st, nodes, int(rd[0]), int(rm[0])


def emit_text(desc, record, target: int) -> str:
    rec = np.ascontiguousarray(np.asarray(record).reshape(1))
    cap = 1 << 22
    buf = C.create_string_buffer(cap)
    st = lib().ora_emit_text(C.addressof(desc), _ptr(rec), int(target), buf, cap)
    if st:
        raise RuntimeError(f"emit failed with status {st}")
    return buf.value.decode()


def sizeof_desc() -> int:
    return lib().ora_sizeof_desc()


def default_threads() -> int:
    return len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
