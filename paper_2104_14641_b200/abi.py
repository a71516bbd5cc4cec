"""ctypes mirror of include/loopscout_b200.h (task descriptor and record layout)."""

from __future__ import annotations

import ctypes as C

import numpy as np

ABI_VERSION = 1
MAX_TENSORS, MAX_RANK, MAX_TERMS, MAX_NODES = 8, 6, 8, 64
MAX_VARS, MAX_XFORMS, MAX_PARAMS, MAX_ORDER, MAX_CHAIN = 32, 32, 8, 16, 16
NFEAT_CPU, NFEAT_GPU = 5, 7
MAX_AXES = 16
AX_PARAM, AX_PERM, AX_VEC, AX_BIT = range(4)

FAMILY = {"cpu": 0, "gpu": 1}
TARGET = {"cpu-x86": 0, "cpu-aarch64": 1, "gpu-ptx": 2}
NODE_LOOP, NODE_ACCESS = 0, 1
XF_TILE, XF_REORDER, XF_UNROLL, XF_VECTORIZE, XF_PARALLEL = range(5)
I_INIT, I_LOAD, I_FMA, I_STORE, I_ADD, I_CMP, I_BRANCH, I_RET, I_COUNT = range(9)

# per-candidate status codes
STATUS = {
    0: "ok",
    1: "no loop named",
    2: "tile factor out of range",
    3: "vectorize width does not divide extent",
    4: "integer modulo by zero",
    5: "reorder: missing loops",
    6: "reorder: loops do not form a perfect nest chain",
    7: "feature must be finite and >= 0",
    16: "unsupported transformed structure",
    17: "unroll product above 65536 or not prepared (outside the device class)",
    18: "integer range exceeded",
    19: "space point outside the space",
}
ST_OK, ST_UNSUPPORTED = 0, 16


class Term(C.Structure):
    _fields_ = [("var", C.c_int32), ("coef", C.c_int32)]


class Expr(C.Structure):
    _fields_ = [("n_terms", C.c_int32), ("konst", C.c_int32), ("terms", Term * MAX_TERMS)]


class Node(C.Structure):
    _fields_ = [("kind", C.c_int32), ("parent", C.c_int32), ("var", C.c_int32),
                ("extent", C.c_int32), ("step", C.c_int32), ("parallel", C.c_int32),
                ("unrolled", C.c_int32), ("vector_width", C.c_int32), ("tensor", C.c_int32),
                ("is_store", C.c_int32), ("idx", Expr * MAX_RANK)]


class Tensor(C.Structure):
    _fields_ = [("rank", C.c_int32), ("elem_bytes", C.c_int32), ("shared", C.c_int32),
                ("dims", C.c_int32 * MAX_RANK)]


class XForm(C.Structure):
    _fields_ = [("kind", C.c_int32), ("var", C.c_int32), ("new_var", C.c_int32),
                ("param", C.c_int32), ("value", C.c_int32), ("enable_bit", C.c_int32),
                ("n_order", C.c_int32), ("perm_shift", C.c_int32), ("order", C.c_int32 * MAX_ORDER)]


class TaskDesc(C.Structure):
    _fields_ = [("abi_version", C.c_int32), ("family", C.c_int32), ("target", C.c_int32),
                ("dialect", C.c_int32), ("n_tensors", C.c_int32), ("tensors", Tensor * MAX_TENSORS),
                ("n_nodes", C.c_int32), ("nodes", Node * MAX_NODES), ("n_vars", C.c_int32),
                ("var_rank", C.c_int32 * MAX_VARS), ("tid_var", C.c_int32),
                ("n_xforms", C.c_int32), ("xforms", XForm * MAX_XFORMS),
                ("coef", C.c_double * NFEAT_GPU), ("cache_capacity", C.c_int64),
                ("issue_width", C.c_int32), ("lat", C.c_int32 * I_COUNT),
                ("klass", C.c_int32 * I_COUNT), ("unit_cap", C.c_int32 * I_COUNT),
                ("ptx_cost", C.c_double * I_COUNT), ("sm_underuse", C.c_double),
                ("warp_slack", C.c_double), ("banks", C.c_int32), ("warp_size", C.c_int32)]


RECORD_DTYPE = np.dtype([("param", "<u2", (MAX_PARAMS,)), ("perm", "<u8"), ("flags", "<u4"),
                         ("tag", "<u4")], align=True)
assert RECORD_DTYPE.itemsize == 32


class Axis(C.Structure):
    _fields_ = [("kind", C.c_int32), ("param", C.c_int32), ("bit", C.c_int32), ("n_choices", C.c_int32),
                ("values", C.POINTER(C.c_uint64))]


class SpaceDesc(C.Structure):
    _fields_ = [("n_axes", C.c_int32), ("axes", Axis * MAX_AXES)]


class EsParams(C.Structure):
    """ls_es_params (include/loopscout_b200.h): EsParams of ls/es.py:26-41."""
    _fields_ = [("alpha", C.c_double), ("sigma", C.c_double), ("population", C.c_int32),
                ("iterations", C.c_int32), ("seed", C.c_uint64), ("rank_normalize", C.c_int32),
                ("pad", C.c_int32)]
