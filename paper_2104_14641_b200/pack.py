"""Task descriptors and packed candidate records.

A *task* is one (program, schedule template, arch, launch).  The template is
the transform sequence shared by a batch of candidates; what varies per
candidate (tile factors, vector widths, reorder permutations, on/off bits of
optional transforms) goes into a 32-byte ``ls_record``:

    param[8]  uint16   tile factors / vector widths, one slot per Tile/Vectorize
    perm      uint64   nibble-packed permutation(s) of the Reorder transform(s)
    flags     uint32   enable bits of optional transforms (space axes with an "off")
    tag       uint32   reserved (0)

Two producers:
  * ``pack_schedules`` — explicit schedule lists (the ``rank`` path,
    ls/cli.py:106-141): schedules are grouped by their *shape* (transform kinds
    and loop names), one template per shape.
  * ``SpaceTemplate`` — a schedule space (``space_axes``, ls/ir.py:517-547):
    one template, records from per-axis choice indices or from ES parameter
    vectors (``ThetaEncoding.decode``, ls/es.py:57-62), vectorised in numpy.

Loop-variable names created by tiling (``v_i``, ``v_i_`` ..., ls/ir.py:365-368)
depend only on the template, so the host assigns every name an id and a rank in
Python string order (the order ``AffineExpr`` keeps its terms in, ls/ir.py:53)
once per task; the device never sees strings.
"""

from __future__ import annotations

import itertools
from dataclasses import dataclass, field

import numpy as np

from . import abi
from .arch import (CostModelError, blocks_per_sm, sm_underuse, warp_slack)
from .ir import ProgramError, Reorder, Schedule, Tile, Unroll, Vectorize, Parallel, space_axes


class PackError(ValueError):
    """The program/template/arch cannot be expressed as a device task."""


# latency-class string of each emitted instruction shape, per target
# (_latency_class, ls/ilp.py:38-47, applied to the emitter's mnemonics ls/ir.py:584-658)
LATENCY_CLASS = {
    0: ("movq", "load", "fma", "load", "addq", "cmpq", "jne", "ret"),
    1: ("mov", "load", "fma", "store", "add", "cmp", "b", "ret"),
    2: ("mov", "load", "fma", "store", "add", "setp", "bra", "ret"),
}
# opcode root of each PTX shape, for GpuSpec.instr_cost (ls/ptx.py:232-234)
PTX_ROOT = ("mov", "ld", "fma", "st", "add", "setp", "bra", "ret")


@dataclass
class XSpec:
    kind: int
    loop: "str | None" = None
    param: int = -1
    value: int = 0
    enable_bit: int = -1
    order: tuple = ()
    perm_shift: int = 0
    new_name: "str | None" = None


def _loop_vars(program) -> list:
    out, stack = [], list(reversed(program.body))
    while stack:
        n = stack.pop()
        if hasattr(n, "var"):
            out.append(n.var)
            stack.extend(reversed(n.children))
    return out


class Template:
    """A transform sequence with per-candidate parameters factored out."""

    def __init__(self, program, xforms: list):
        self.program = program
        self.xforms = list(xforms)
        base = _loop_vars(program)
        if len(set(base)) != len(base):
            raise PackError("programs with repeated loop variable names are not supported")
        self.n_params = 1 + max([x.param for x in self.xforms] + [-1])
        if self.n_params > abi.MAX_PARAMS:
            raise PackError(f"more than {abi.MAX_PARAMS} tile/vectorize parameters")
        nib = sum(len(x.order) for x in self.xforms if x.kind == abi.XF_REORDER)
        if nib > 16:
            raise PackError("reorder permutations exceed 16 nibbles")
        for x in self.xforms:
            if x.kind == abi.XF_REORDER and len(x.order) > abi.MAX_ORDER:
                raise PackError("reorder of more than 16 loops")
        allon = self._simulate(None)
        creators = [i for i, x in enumerate(self.xforms)
                    if x.enable_bit >= 0 and x.kind in (abi.XF_TILE, abi.XF_VECTORIZE)]
        subsets = (itertools.product((0, 1), repeat=len(creators)) if len(creators) <= 8
                   else [tuple(int(j != k) for j in range(len(creators))) for k in range(len(creators))])
        for bits in subsets:
            sim = self._simulate({c for c, b in zip(creators, bits) if b})
            for i, nm in sim.items():
                if allon.get(i) != nm:
                    raise PackError("generated loop names depend on optional transforms")
        for i, nm in allon.items():
            self.xforms[i].new_name = nm
        names = list(base)
        for x in self.xforms:
            for nm in ([x.new_name] if x.new_name else []) + ([x.loop] if x.loop else []) + list(x.order):
                if nm not in names:
                    names.append(nm)
        if len(names) > abi.MAX_VARS:
            raise PackError(f"more than {abi.MAX_VARS} loop variable names")
        self.names = names
        self.var_id = {n: i for i, n in enumerate(names)}
        self.rank = {n: r for r, n in enumerate(sorted(names))}

    def _simulate(self, enabled) -> dict:
        existing = set(_loop_vars(self.program))
        out = {}
        for i, x in enumerate(self.xforms):
            if x.enable_bit >= 0 and enabled is not None and i not in enabled:
                continue
            if x.kind in (abi.XF_TILE, abi.XF_VECTORIZE) and x.loop in existing:
                nm = x.loop + "_i"
                while nm in existing:
                    nm += "_"
                existing.add(nm)
                out[i] = nm
        return out

    # -- descriptor --------------------------------------------------------------

    def desc(self, arch, launch=None) -> abi.TaskDesc:
        d = abi.TaskDesc()
        d.abi_version = abi.ABI_VERSION
        if arch.family not in abi.FAMILY:
            raise CostModelError(f"arch family must be cpu|gpu, got {arch.family!r}")
        d.family = abi.FAMILY[arch.family]
        if arch.target not in abi.TARGET:
            raise ProgramError(f"unsupported target {arch.target!r}")
        d.target = abi.TARGET[arch.target]
        if (d.family == 1) != (d.target == 2):
            raise PackError(f"family {arch.family!r} with target {arch.target!r} is not supported")
        d.dialect = 0 if arch.dialect == "x86-att" else 1
        p = self.program
        tix = {t.name: i for i, t in enumerate(p.tensors)}
        if len(p.tensors) > abi.MAX_TENSORS:
            raise PackError("too many tensors")
        d.n_tensors = len(p.tensors)
        for i, t in enumerate(p.tensors):
            if len(t.dims) > abi.MAX_RANK:
                raise PackError("tensor rank above 6")
            d.tensors[i].rank = len(t.dims)
            d.tensors[i].elem_bytes = t.elem_bytes
            d.tensors[i].shared = int(t.scope == "shared")
            for k, x in enumerate(t.dims):
                d.tensors[i].dims[k] = _i32(x)
        nodes = []

        def walk(n, parent):
            me = len(nodes)
            nodes.append((n, parent))
            for c in getattr(n, "children", ()):
                walk(c, me)

        for n in p.body:
            walk(n, -1)
        if len(nodes) > abi.MAX_NODES:
            raise PackError("too many program nodes")
        d.n_nodes = len(nodes)
        for i, (n, parent) in enumerate(nodes):
            o = d.nodes[i]
            o.parent = parent
            if hasattr(n, "var"):
                o.kind = abi.NODE_LOOP
                o.var = self.var_id[n.var]
                o.extent, o.step = _i32(n.extent), _i32(n.step)
                o.parallel, o.unrolled = int(n.parallel), int(n.unrolled)
                o.vector_width = _i32(n.vector_width or 0)
            else:
                o.kind = abi.NODE_ACCESS
                o.tensor = tix[n.tensor]
                o.is_store = int(n.kind == "store")
                for k, e in enumerate(n.index_exprs):
                    if len(e.terms) > abi.MAX_TERMS:
                        raise PackError("index expression with more than 8 terms")
                    o.idx[k].n_terms = len(e.terms)
                    o.idx[k].konst = _i32(e.const)
                    for t, (v, c) in enumerate(e.terms):
                        o.idx[k].terms[t].var = self.var_id[v]
                        o.idx[k].terms[t].coef = _i32(c)
        d.n_vars = len(self.names)
        for n, i in self.var_id.items():
            d.var_rank[i] = self.rank[n]
        d.tid_var = self.var_id.get("tid", -1)
        d.n_xforms = len(self.xforms)
        for i, x in enumerate(self.xforms):
            o = d.xforms[i]
            o.kind = x.kind
            o.var = self.var_id[x.loop] if x.loop is not None else -1
            o.new_var = self.var_id[x.new_name] if x.new_name else -1
            o.param, o.value, o.enable_bit = x.param, _i32(x.value), x.enable_bit
            o.n_order, o.perm_shift = len(x.order), x.perm_shift
            for j, nm in enumerate(x.order):
                o.order[j] = self.var_id[nm]
        order = arch.feature_order()
        for k, f in enumerate(order):
            d.coef[k] = float(arch.coefficients[f])
        d.banks, d.warp_size = 32, 32
        if d.family == 0:
            if arch.cache is None or arch.sched is None:
                raise CostModelError(f"arch {arch.name!r} lacks [cache] or [ilp] configuration")
            d.cache_capacity = arch.cache.capacity_elements
            s = arch.sched
            d.issue_width = s.issue_width
            classes = LATENCY_CLASS[d.target]
            ids = {}
            for k, c in enumerate(classes):
                lat = s.latency.get(c, s.default_latency)
                if lat != int(lat) or lat < 0:
                    raise PackError(f"latency {lat!r} of class {c!r} is not a non-negative integer")
                d.lat[k] = int(lat)
                d.klass[k] = ids.setdefault(c, len(ids))
            for c, k in ids.items():
                cap = s.units.get(c)
                if cap is not None:
                    if int(cap) < 1:
                        raise PackError(f"unit cap {cap!r} for class {c!r} never issues")
                    d.unit_cap[k] = int(cap)
        else:
            if launch is None:
                raise CostModelError("gpu feature extraction requires a kernel launch record")
            g = arch.gpu
            if g is None:
                from .arch import GpuSpec
                g = GpuSpec()
            d.cache_capacity = 1
            d.issue_width = 1
            for k, r in enumerate(PTX_ROOT):
                d.ptx_cost[k] = float(g.instr_cost.get(r, 1))
            d.sm_underuse = sm_underuse(launch, g)
            d.warp_slack = warp_slack(launch, g)
            d.banks, d.warp_size = g.banks, g.warp_size
        return d


def _i32(x) -> int:
    x = int(x)
    if not -(2 ** 31) <= x < 2 ** 31:
        raise PackError(f"value {x} exceeds int32")
    return x


# -- explicit schedule lists (rank path) ------------------------------------------


def shape_key(s) -> tuple:
    key = []
    for t in s.transforms:
        n = type(t).__name__
        if n == "Reorder":
            key.append(("Reorder", tuple(sorted(t.order))))
        elif n in ("Tile", "Vectorize", "Unroll", "Parallel"):
            key.append((n, t.loop))
        else:
            raise ProgramError(f"unknown transform {t!r}")
    return tuple(key)


_KIND = {"Tile": abi.XF_TILE, "Vectorize": abi.XF_VECTORIZE, "Unroll": abi.XF_UNROLL,
         "Parallel": abi.XF_PARALLEL, "Reorder": abi.XF_REORDER}


def template_for_shape(program, key: tuple) -> Template:
    xs, slot, shift = [], 0, 0
    for n, arg in key:
        if n == "Reorder":
            xs.append(XSpec(abi.XF_REORDER, order=arg, perm_shift=shift))
            shift += len(arg)
        elif n in ("Tile", "Vectorize"):
            xs.append(XSpec(_KIND[n], arg, param=slot))
            slot += 1
        else:
            xs.append(XSpec(_KIND[n], arg))
    return Template(program, xs)


def _encode_factor(v: int, max_extent: int) -> "int | None":
    if v <= 0:
        return 0 if v == 0 else None
    if v <= 0xFFFF:
        return v
    return 0xFFFF if max_extent < 0xFFFF else None


@dataclass
class PackedGroup:
    template: Template
    index: np.ndarray          # positions in the input schedule list
    records: np.ndarray        # RECORD_DTYPE
    host_status: np.ndarray    # int32, nonzero = not sent to the device


_TEMPLATES: dict = {}  # (id(program), shape key) -> (program, Template | PackError)


def _template_cached(program, key: tuple):
    """template_for_shape, memoised per (program object, shape); PackError is cached too."""
    ck = (id(program), key)
    hit = _TEMPLATES.get(ck)
    if hit is not None and hit[0] is program:
        if isinstance(hit[1], PackError):
            raise hit[1]
        return hit[1]
    if len(_TEMPLATES) > 4096:
        _TEMPLATES.clear()
    try:
        t = template_for_shape(program, key)
    except PackError as e:
        _TEMPLATES[ck] = (program, e)
        raise
    _TEMPLATES[ck] = (program, t)
    return t


def _fast_packer():
    try:
        from . import _packer  # csrc/packer.cpp (built by build.py)
        return _packer
    except ImportError:
        return None


def pack_schedules(program, schedules) -> list:
    """Group schedules by shape and pack each group into records (groups in first-appearance
    order, indices ascending).  The native packer (csrc/packer.cpp) reads the Schedule objects
    in one pass; schedules it cannot read go through the Python path, which raises the
    reference's exception."""
    max_extent = max([lp.extent for lp in _loops(program)] + [1])
    fp = _fast_packer()
    n = len(schedules)
    if fp is not None and n:
        sid = np.empty(n, np.int32)
        prm = np.empty((n, abi.MAX_PARAMS), np.uint16)
        perm = np.empty(n, np.uint64)
        hst = np.empty(n, np.int32)
        keys = fp.pack(schedules, int(max_extent), sid, prm, perm, hst)
        if keys is not None:
            order = np.argsort(sid, kind="stable")
            bounds = np.searchsorted(sid[order], np.arange(len(keys) + 1))
            out = []
            for g, key in enumerate(keys):
                idx = order[bounds[g]:bounds[g + 1]]
                recs = np.zeros(len(idx), abi.RECORD_DTYPE)
                try:
                    tmpl = _template_cached(program, key)
                except PackError:
                    out.append(PackedGroup(None, idx, recs, np.full(len(idx), abi.ST_UNSUPPORTED, np.int32)))
                    continue
                recs["param"] = prm[idx]
                recs["perm"] = perm[idx]
                out.append(PackedGroup(tmpl, idx, recs, hst[idx]))
            return out
    return _pack_schedules_py(program, schedules, max_extent)


def _pack_schedules_py(program, schedules, max_extent) -> list:
    by_key: dict = {}
    for i, s in enumerate(schedules):
        by_key.setdefault(shape_key(s), []).append(i)
    out = []
    for key, idxs in by_key.items():
        try:
            tmpl = _template_cached(program, key)
        except PackError:
            recs = np.zeros(len(idxs), abi.RECORD_DTYPE)
            out.append(PackedGroup(None, np.array(idxs), recs,
                                   np.full(len(idxs), abi.ST_UNSUPPORTED, np.int32)))
            continue
        recs = np.zeros(len(idxs), abi.RECORD_DTYPE)
        hst = np.zeros(len(idxs), np.int32)
        for r, i in enumerate(idxs):
            slot, perm = 0, 0
            for t, x in zip(schedules[i].transforms, tmpl.xforms):
                if x.kind in (abi.XF_TILE, abi.XF_VECTORIZE):
                    v = _encode_factor(int(t.factor if x.kind == abi.XF_TILE else t.width), max_extent)
                    if v is None:
                        hst[r] = abi.ST_UNSUPPORTED
                        v = 0
                    recs["param"][r, slot] = v
                    slot += 1
                elif x.kind == abi.XF_REORDER:
                    for j, nm in enumerate(t.order):
                        perm |= x.order.index(nm) << (4 * (x.perm_shift + j))
            recs["perm"][r] = perm
        out.append(PackedGroup(tmpl, np.array(idxs), recs, hst))
    return out


def _loops(program):
    out, stack = [], list(program.body)
    while stack:
        n = stack.pop()
        if hasattr(n, "var"):
            out.append(n)
            stack.extend(n.children)
    return out


# -- schedule spaces (search path) ------------------------------------------------


class SpaceTemplate:
    """One template for a whole space; records from choice indices or thetas."""

    def __init__(self, program, space: dict):
        self.program = program
        self.axes = tuple(space_axes(program, space))
        xs, slot, bit = [], 0, 0
        self.tables = []  # per axis: (kind, slot/bit, values array)
        for ax in self.axes:
            kind, _, loop = ax.name.partition(":")
            n = len(ax.choices)
            if kind == "tile":
                xs.append(XSpec(abi.XF_TILE, loop, param=slot))
                vals = np.array([c[0].factor for c in ax.choices], np.int64)
                if vals.max() > 0xFFFF:
                    raise PackError("tile factor above 65535")
                self.tables.append(("param", slot, vals))
                slot += 1
            elif kind == "reorder":
                names = sorted(ax.choices[0][0].order)
                for c in ax.choices:
                    if sorted(c[0].order) != names:
                        raise PackError("reorder choices over different loop sets")
                xs.append(XSpec(abi.XF_REORDER, order=tuple(names), perm_shift=0))
                perms = np.zeros(n, np.uint64)
                for k, c in enumerate(ax.choices):
                    v = 0
                    for j, nm in enumerate(c[0].order):
                        v |= names.index(nm) << (4 * j)
                    perms[k] = v
                self.tables.append(("perm", 0, perms))
            elif kind == "vectorize":
                xs.append(XSpec(abi.XF_VECTORIZE, loop, param=slot, enable_bit=bit))
                vals = np.array([c[0].width if c else 0 for c in ax.choices], np.int64)
                self.tables.append(("vec", (slot, bit), vals))
                slot += 1
                bit += 1
            else:  # unroll / parallel on-off axes
                xs.append(XSpec(abi.XF_UNROLL if kind == "unroll" else abi.XF_PARALLEL, loop,
                                enable_bit=bit))
                self.tables.append(("bit", bit, np.array([0, 1], np.int64)))
                bit += 1
        if sum(1 for t in self.tables if t[0] == "perm") > 1:
            raise PackError("more than one reorder axis")
        self.template = Template(program, xs)
        self.sizes = np.array([len(ax.choices) for ax in self.axes], np.int64)

    @property
    def dim(self) -> int:
        return len(self.axes)

    def records_from_indices(self, idx: np.ndarray) -> np.ndarray:
        idx = np.asarray(idx, np.int64).reshape(-1, self.dim)
        recs = np.zeros(idx.shape[0], abi.RECORD_DTYPE)
        flags = np.zeros(idx.shape[0], np.uint32)
        for a, (kind, where, vals) in enumerate(self.tables):
            v = vals[idx[:, a]]
            if kind == "param":
                recs["param"][:, where] = v
            elif kind == "perm":
                recs["perm"] = v
            elif kind == "vec":
                recs["param"][:, where[0]] = v
                flags |= (v != 0).astype(np.uint32) << np.uint32(where[1])
            else:
                flags |= v.astype(np.uint32) << np.uint32(where)
        recs["flags"] = flags
        return recs

    # -- points API ---------------------------------------------------------------------
    @property
    def size(self) -> int:
        return int(np.prod([int(n) for n in self.sizes], dtype=object))

    def space_desc(self) -> abi.SpaceDesc:
        """The space for ls_task_set_space; keeps the value arrays alive on the descriptor."""
        if len(self.tables) > abi.MAX_AXES:
            raise PackError(f"more than {abi.MAX_AXES} space axes")
        d = abi.SpaceDesc()
        d.n_axes = len(self.tables)
        keep = []
        for a, (kind, where, vals) in enumerate(self.tables):
            ax = d.axes[a]
            ax.n_choices = len(vals)
            v = np.ascontiguousarray(np.asarray(vals).astype(np.uint64))
            keep.append(v)
            ax.values = v.ctypes.data_as(abi.C.POINTER(abi.C.c_uint64))
            if kind == "param":
                ax.kind, ax.param = abi.AX_PARAM, where
            elif kind == "perm":
                ax.kind = abi.AX_PERM
            elif kind == "vec":
                ax.kind, ax.param, ax.bit = abi.AX_VEC, where[0], where[1]
            else:
                ax.kind, ax.bit = abi.AX_BIT, where
        d._keep = keep
        return d

    def points_from_indices(self, idx: np.ndarray) -> np.ndarray:
        """Mixed-radix points (axis 0 most significant); uint32 when the space fits, else uint64."""
        idx = np.asarray(idx, np.int64).reshape(-1, self.dim)
        if self.size > 2 ** 64:
            raise PackError("space larger than 2^64 points")
        p = np.zeros(idx.shape[0], np.uint64)
        for a, n in enumerate(self.sizes):
            p = p * np.uint64(int(n)) + idx[:, a].astype(np.uint64)
        return p.astype(np.uint32) if self.size <= 2 ** 32 else p

    def indices_from_points(self, pts: np.ndarray) -> np.ndarray:
        p = np.asarray(pts).astype(np.uint64)
        out = np.zeros((len(p), self.dim), np.int64)
        for a in range(self.dim - 1, -1, -1):
            n = np.uint64(int(self.sizes[a]))
            out[:, a] = (p % n).astype(np.int64)
            p = p // n
        return out

    def indices_from_theta(self, thetas: np.ndarray) -> np.ndarray:
        """ThetaEncoding.decode per row: clip(round_half_even(x), 0, n-1) (ls/es.py:57-62)."""
        t = np.asarray(thetas, np.float64).reshape(-1, self.dim)
        return np.clip(np.rint(t), 0, self.sizes - 1).astype(np.int64)

    def schedule_of(self, idx_row) -> Schedule:
        out = []
        for ax, i in zip(self.axes, idx_row):
            out.extend(ax.choices[int(i)])
        return Schedule(tuple(out))


def pack_points(points: np.ndarray, nbytes: int = 3) -> np.ndarray:
    """Space points (non-negative integers below 2^(8 nbytes)) as packed little-endian bytes,
    uint8 [n, nbytes] -- the 3-byte point format of the points API (include/loopscout_b200.h)."""
    p = np.ascontiguousarray(points).astype("<u8", copy=False)
    if len(p) and int(p.max()) >> (8 * nbytes):
        raise ValueError(f"a point does not fit {nbytes} bytes")
    return np.ascontiguousarray(p.view(np.uint8).reshape(-1, 8)[:, :nbytes])

