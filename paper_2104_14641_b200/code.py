"""External code-text analysis: the drop-in for
``extract_features(program, code, arch, launch, diagnostics)`` (ls/cost.py:132-152) when the
code is the user's own assembly / PTX text (``analyze --code``, ls/cli.py:86-103).

The text is parsed on the device (``ls_code_features``, csrc/code.cu: one CUDA block per text,
a batch of texts per launch) into the text-dependent features -- CPU: n_fma, n_vload,
n_vstore, ilp_cycles (parse_asm + loop_map + count_simd + the list scheduler); GPU:
workload_per_thread, n_fma, n_ld, n_st (loop_map_ptx + count_ptx + thread_cycles) -- and the
IR-side features come from the scoring path on the program itself (cache movement; SM
underuse, warp slack, conflict-adjusted shared-memory ops).  Errors mirror the reference:
``AsmError`` for an empty text or a jump to an undefined label (same messages),
``ValueError`` for a line holding only a predicate, ``CostModelError`` for a GPU arch without
a launch record or a non-finite / negative feature.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from .arch import CPU_FEATURES, GPU_FEATURES, CostModelError, FeatureVector

MAX_CLASSES = 32
MAX_LOOPS = 64
E_EMPTY, E_LABEL, E_VALUE, E_LIMIT = 1, 2, 3, 4
DIAG_WORDS = 10
(D_UNMATCHED_BLOCK, D_BOUND_MISMATCH, D_LOOPS_MATCHED, D_NO_SETP, D_NON_IMM_BOUND, D_NONLINEAR, D_NOT_DERIVABLE,
 D_UNSUPPORTED_CMP, D_INCONSISTENT) = 1, 2, 3, 10, 11, 12, 13, 14, 15


class AsmError(ValueError):
    """Malformed assembly input (the reference's loopscout.asm.AsmError)."""


class CodeDesc(C.Structure):
    _fields_ = [("family", C.c_int32), ("target", C.c_int32), ("dialect", C.c_int32),
                ("issue_width", C.c_int32), ("default_latency", C.c_int32), ("n_classes", C.c_int32),
                ("cls_hash", C.c_uint64 * MAX_CLASSES), ("cls_latency", C.c_int32 * MAX_CLASSES),
                ("cls_units", C.c_int32 * MAX_CLASSES), ("n_costs", C.c_int32), ("pad0", C.c_int32),
                ("cost_hash", C.c_uint64 * MAX_CLASSES), ("cost", C.c_double * MAX_CLASSES),
                ("n_loops", C.c_int32), ("pad1", C.c_int32),
                ("loop_extent", C.c_int64 * MAX_LOOPS), ("loop_step", C.c_int64 * MAX_LOOPS),
                ("loop_weight", C.c_int64 * MAX_LOOPS)]


def _lib():
    from .engine import lib
    L = lib()
    if not getattr(L, "_code_bound", False):
        vp, i32, i64 = C.c_void_p, C.c_int32, C.c_int64
        L.ls_code_hash.argtypes = [C.c_char_p, i32]
        L.ls_code_hash.restype = C.c_uint64
        L.ls_code_scratch_bytes.argtypes = [i64]
        L.ls_code_scratch_bytes.restype = i64
        L.ls_code_features.argtypes = [vp, vp, vp, i32, vp, i64, vp, vp, vp, vp]
        L.ls_code_features_diag.argtypes = [vp, vp, vp, i32, vp, i64, vp, vp, vp, vp, vp, vp]
        L.ls_code_diag_cap.argtypes = [i64]
        L.ls_code_diag_cap.restype = i64
        L._code_bound = True
    return L


def _hash(L, name: str) -> int:
    b = name.encode()
    return int(L.ls_code_hash(b, len(b)))


def _branching_loops(program):
    """(extent, step, weight, var) of the loops that lower to backward branches, in preorder,
    with weight = the product of its and its branching ancestors' extents (ls/asm.py:245-262)."""
    from .ir import LoopNode
    out = []

    def walk(n, prod):
        if not isinstance(n, LoopNode):
            return
        here = prod
        if not n.unrolled and n.vector_width is None:
            here = prod * n.extent
            out.append((n.extent, n.step, here, n.var))
        for c in n.children:
            walk(c, here)

    for n in program.body:
        walk(n, 1)
    return out


def code_desc(program, arch) -> CodeDesc:
    L = _lib()
    d = CodeDesc()
    d.family = 0 if arch.family == "cpu" else 1
    if arch.family == "cpu":
        sched = arch.sched
        d.target = 0 if arch.target == "cpu-x86" else 1
        d.dialect = 0 if arch.dialect == "x86-att" else 1
        d.issue_width = sched.issue_width
        d.default_latency = sched.default_latency
        names = list(dict.fromkeys(list(sched.latency) + list(sched.units)))
        if len(names) > MAX_CLASSES:
            raise CostModelError(f"more than {MAX_CLASSES} latency / unit classes")
        d.n_classes = len(names)
        for c, name in enumerate(names):
            d.cls_hash[c] = _hash(L, name)
            d.cls_latency[c] = int(sched.latency.get(name, 0))
            d.cls_units[c] = int(sched.units.get(name, 0))
        loops = _branching_loops(program)
        if len(loops) > MAX_LOOPS:
            raise CostModelError(f"more than {MAX_LOOPS} branching loops")
        d.n_loops = len(loops)
        for q, (e, s, w, _) in enumerate(loops):
            d.loop_extent[q], d.loop_step[q], d.loop_weight[q] = e, s, w
    else:
        d.issue_width = 1
        costs = dict(arch.gpu.instr_cost)
        if len(costs) > MAX_CLASSES:
            raise CostModelError(f"more than {MAX_CLASSES} PTX cost classes")
        d.n_costs = len(costs)
        for c, (name, v) in enumerate(costs.items()):
            d.cost_hash[c] = _hash(L, name)
            d.cost[c] = float(v)
    return d


def _ir_features(program, arch, launch, device):
    """The IR-side features: the scoring path on the program as given (no schedule)."""
    from .cost import CandidateError, score_batch
    from .ir import Schedule
    res = score_batch(program, [Schedule(())], arch, launch, device)
    if res.status[0]:
        raise res.exception(0) if 0 in res.messages else CandidateError(int(res.status[0]))
    return res.features[0]


def _render(ev, blob: bytes, loops) -> list:
    """The reference's diagnostic strings for one text's events (ls/asm.py:276-293,
    ls/ptx.py:112-189)."""
    out = []
    for kind, blk, lo, ll, a, b, c, ao, al, _ in (tuple(int(x) for x in e) for e in ev):
        where = blob[lo:lo + ll].decode() if lo >= 0 and ll > 0 else str(blk)  # block.label or block.index
        aux = blob[ao:ao + al].decode() if ao >= 0 else "ne"
        if kind == D_UNMATCHED_BLOCK:
            out.append(f"unmatched loop block {where}")
        elif kind == D_BOUND_MISMATCH:
            ext, _, _, var = loops[c]
            out.append(f"block {where} bound {b if a else None} does not match loop {var!r} extent {ext}")
        elif kind == D_LOOPS_MATCHED:
            out += [f"IR loop {lp[3]!r} not matched to any block" for lp in loops[a:]]
        elif kind == D_NO_SETP:
            out.append(f"loop at {where}: no setp/bra idiom")
        elif kind == D_NON_IMM_BOUND:
            out.append(f"loop at {where}: non-immediate bound")
        elif kind == D_NONLINEAR:
            out.append(f"loop at {where}: non-linear induction register {aux}")
        elif kind == D_NOT_DERIVABLE:
            out.append(f"loop at {where}: induction register {aux} not derivable")
        elif kind == D_UNSUPPORTED_CMP:
            out.append(f"loop at {where}: unsupported comparison {aux!r}")
        elif kind == D_INCONSISTENT:
            out.append(f"loop at {where}: inconsistent bounds (init {a}, delta {b}, {aux} {c})")
    return out


def code_features(program, codes, arch, launch=None, device: int = 0, diagnostics: list | None = None) -> list:
    """extract_features for every text in `codes` (one device launch): a FeatureVector or the
    exception the reference raises, per text.  `diagnostics`, if given, receives one list per
    text: the notes the reference's extract_features appends for it."""
    import torch

    if arch.family == "gpu" and launch is None:  # ls/cost.py:137-138, before any parsing
        raise CostModelError("gpu feature extraction requires a kernel launch record")
    if arch.family == "cpu" and (arch.cache is None or arch.sched is None):
        raise CostModelError(f"arch {arch.name!r} lacks [cache] or [ilp] configuration")
    L = _lib()
    desc = code_desc(program, arch)
    blobs = [c.encode() for c in codes]
    offs = np.zeros(len(blobs) + 1, np.int64)
    for i, b in enumerate(blobs):
        offs[i + 1] = offs[i] + len(b)
    n = len(blobs)
    if n == 0:
        return []
    dev = torch.device("cuda", device)
    d_text = torch.from_numpy(np.frombuffer(b"".join(blobs) or b"\0", np.uint8).copy()).to(dev)
    scratch = sum(int(L.ls_code_scratch_bytes(int(offs[i + 1] - offs[i]))) + 256 for i in range(n)) + \
        C.sizeof(CodeDesc) + 24 * (n + 2) + 4096
    dstart = np.zeros(n + 1, np.int64)
    for i in range(n):
        dstart[i + 1] = dstart[i] + int(L.ls_code_diag_cap(int(offs[i + 1] - offs[i])))
    d_scratch = torch.empty(scratch, dtype=torch.uint8, device=dev)
    d_feat = torch.zeros((n, 4), dtype=torch.float64, device=dev)
    d_status = torch.zeros(n, dtype=torch.int32, device=dev)
    d_err = torch.zeros((n, 3), dtype=torch.int64, device=dev)
    d_diag = torch.zeros((int(dstart[n]), DIAG_WORDS), dtype=torch.int64, device=dev)
    d_ndiag = torch.zeros(n, dtype=torch.int32, device=dev)
    from .engine import _check
    with torch.cuda.device(device):
        _check(L.ls_code_features_diag(C.addressof(desc), d_text.data_ptr(), offs.ctypes.data, n, d_scratch.data_ptr(),
                                       scratch, d_feat.data_ptr(), d_status.data_ptr(), d_err.data_ptr(),
                                       d_diag.data_ptr(), d_ndiag.data_ptr(),
                                       torch.cuda.current_stream(dev).cuda_stream), "ls_code_features_diag")
        torch.cuda.synchronize(dev)
    feats, status, err = d_feat.cpu().numpy(), d_status.cpu().numpy(), d_err.cpu().numpy()
    diag, ndiag = d_diag.cpu().numpy(), d_ndiag.cpu().numpy()
    loops = _branching_loops(program) if arch.family == "cpu" else []
    ir = None
    out = []
    for i in range(n):
        st = int(status[i])
        if diagnostics is not None:
            k = int(ndiag[i]) if st == 0 else 0
            if k > dstart[i + 1] - dstart[i]:
                raise CostModelError("diagnostic events beyond the device buffer")
            notes = _render(diag[dstart[i]:dstart[i] + k], blobs[i], loops)
            diagnostics.append(notes + notes if arch.family == "gpu" else notes)  # count_ptx, thread_cycles
        if st == E_EMPTY:
            out.append(AsmError("empty assembly input"))
            continue
        if st == E_LABEL:
            line, off, ln = (int(x) for x in err[i])
            sym = blobs[i][off:off + ln].decode() if off >= 0 else "<none>"
            out.append(AsmError(f"jump to undefined label {sym!r} (line {line})"))
            continue
        if st == E_VALUE:
            out.append(ValueError("not enough values to unpack (expected 2, got 1)"))
            continue
        if st:
            out.append(CostModelError(f"code text beyond the device parser's limits (status {st})"))
            continue
        if ir is None:
            ir = _ir_features(program, arch, launch, device)
        f = feats[i]
        if arch.family == "cpu":
            vals = {"n_fma": f[0], "n_vload": f[1], "n_vstore": f[2], "est_l1_movement": ir[3], "ilp_cycles": f[3]}
            order = CPU_FEATURES
        else:
            vals = {"workload_per_thread": f[0], "sm_underuse": ir[1], "warp_slack": ir[2],
                    "n_smem_ops_adjusted": ir[3], "n_fma": f[1], "n_ld": f[2], "n_st": f[3]}
            order = GPU_FEATURES
        try:
            out.append(FeatureVector.of(vals, order))
        except CostModelError as e:
            out.append(e)
    return out


def extract_features(program, code: str, arch, launch=None, diagnostics=None, device: int = 0) -> FeatureVector:
    """Drop-in for ls/cost.py:132-152: the features, and the reference's notes appended to
    `diagnostics` (loop_map's unmatched blocks / loops, _loop_trip's failures)."""
    notes: list = []
    r = code_features(program, [code], arch, launch, device, notes)[0]
    if diagnostics is not None and not isinstance(r, Exception):
        diagnostics.extend(notes[0])
    if isinstance(r, Exception):
        raise r
    return r
