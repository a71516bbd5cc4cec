"""Host-side loop-nest IR: the program / schedule / space formats of the reference.

Only what the packer needs lives here: parsing of the canonical program JSON
(ls/ir.py:176-242), the five transform records and their JSON form
(ls/ir.py:276-343), and ``space_axes`` (ls/ir.py:509-547), which fixes the
axis order the ES encoding decodes into.  Transforms are *not* applied on the
host: the device applies them per candidate ("record decode").

Class and field names match the reference's public API (``loopscout`` exports,
ls/__init__.py:3-15) so objects from either package can be handed to the
packer.
"""

from __future__ import annotations

import json
import re
from dataclasses import dataclass


class ProgramError(ValueError):
    """Malformed program, schedule or space (ls/ir.py:17-18)."""


# -- affine index expressions ------------------------------------------------

_CHUNK = re.compile(r"([+-]?)\s*([^+-]+)")
_TERM = re.compile(r"^\s*(?:(\d+)\s*\*\s*)?([A-Za-z_][A-Za-z0-9_]*)\s*$")


@dataclass(frozen=True)
class AffineExpr:
    """sum(coef*var) + const; ``terms`` sorted by var name, coefs nonzero."""

    terms: tuple = ()
    const: int = 0

    @staticmethod
    def parse(text: str) -> "AffineExpr":
        if not text.strip():
            raise ProgramError(f"empty affine expression: {text!r}")
        pieces = _CHUNK.findall(text)
        if not pieces:
            raise ProgramError(f"empty affine expression: {text!r}")
        acc: dict = {}
        const = 0
        for sign, raw in pieces:
            body = raw.strip()
            if not body:
                raise ProgramError(f"malformed affine expression: {text!r}")
            mult = -1 if sign == "-" else 1
            if body.isdigit() and body.isascii():
                const += mult * int(body)
                continue
            m = _TERM.match(body)
            if m is None:
                raise ProgramError(f"non-affine or malformed term {body!r} in {text!r}")
            acc[m.group(2)] = acc.get(m.group(2), 0) + mult * int(m.group(1) or 1)
        return AffineExpr(tuple(sorted((v, c) for v, c in acc.items() if c)), const)

    def variables(self) -> frozenset:
        return frozenset(v for v, _ in self.terms)

    def coef(self, var: str) -> int:
        return dict(self.terms).get(var, 0)

    def __str__(self) -> str:
        parts = []
        for v, c in self.terms:
            mag = v if abs(c) == 1 else f"{abs(c)}*{v}"
            parts.append(("-" if c < 0 else "+", mag))
        if self.const or not parts:
            parts.append(("-" if self.const < 0 else "+", str(abs(self.const))))
        head_sign, head = parts[0]
        out = ("-" if head_sign == "-" else "") + head
        for s, m in parts[1:]:
            out += f" {s} {m}"
        return out


# -- program tree --------------------------------------------------------------


@dataclass(frozen=True)
class TensorDecl:
    name: str
    dims: tuple
    elem_bytes: int = 4
    scope: str = "global"

    @property
    def rank(self) -> int:
        return len(self.dims)


@dataclass(frozen=True)
class AccessNode:
    tensor: str
    kind: str
    index_exprs: tuple


@dataclass(frozen=True)
class LoopNode:
    var: str
    extent: int
    step: int = 1
    parallel: bool = False
    unrolled: bool = False
    vector_width: "int | None" = None
    children: tuple = ()


@dataclass(frozen=True)
class LoopProgram:
    tensors: tuple
    body: tuple

    def tensor(self, name: str) -> TensorDecl:
        for t in self.tensors:
            if t.name == name:
                return t
        raise ProgramError(f"unknown tensor {name!r}")

    def loops(self) -> list:
        """Loop nodes in preorder."""
        out = []
        stack = list(reversed(self.body))
        while stack:
            n = stack.pop()
            if isinstance(n, LoopNode):
                out.append(n)
                stack.extend(reversed(n.children))
        return out

    def find_loop(self, var: str) -> LoopNode:
        for lp in self.loops():
            if lp.var == var:
                return lp
        raise ProgramError(f"no loop named {var!r}")


def _parse_node(obj, bound: tuple, decls: dict):
    if not isinstance(obj, dict) or len(obj) != 1:
        raise ProgramError(f"node must be a single-key object, got {obj!r}")
    (kind, d), = obj.items()
    if kind == "loop":
        var, extent, step = d["var"], int(d["extent"]), int(d.get("step", 1))
        if extent <= 0 or step <= 0:
            raise ProgramError(f"loop {var!r}: extent and step must be positive")
        if var in bound:
            raise ProgramError(f"loop variable {var!r} shadows an enclosing loop")
        attrs = d.get("attrs", [])
        width = None
        for a in attrs:
            if isinstance(a, str) and a.startswith("vectorize:"):
                width = int(a.split(":", 1)[1])
        if width is not None and extent % width:
            raise ProgramError(f"loop {var!r}: vector width {width} does not divide extent {extent}")
        kids = tuple(_parse_node(c, bound + (var,), decls) for c in d.get("body", []))
        return LoopNode(var, extent, step, "parallel" in attrs, "unroll" in attrs, width, kids)
    if kind == "access":
        name = d["tensor"]
        if name not in decls:
            raise ProgramError(f"access to undeclared tensor {name!r}")
        if d["kind"] not in ("load", "store"):
            raise ProgramError(f"access kind must be load|store, got {d['kind']!r}")
        exprs = tuple(AffineExpr.parse(s) for s in d["idx"])
        if len(exprs) != decls[name].rank:
            raise ProgramError(
                f"tensor {name!r} has rank {decls[name].rank}, got {len(exprs)} indices")
        for e in exprs:
            for v in e.variables():
                if v not in bound:
                    raise ProgramError(f"index variable {v!r} not bound by any enclosing loop")
        return AccessNode(name, d["kind"], exprs)
    raise ProgramError(f"unknown node kind: {list(obj)!r}")


def parse_program(text: str) -> LoopProgram:
    """Canonical JSON program form (ls/ir.py:222-242)."""
    try:
        data = json.loads(text)
    except json.JSONDecodeError as e:
        raise ProgramError(f"syntax error at line {e.lineno}, column {e.colno}: {e.msg}") from e
    if not isinstance(data, dict):
        raise ProgramError("top level must be an object")
    decls = []
    for t in data.get("tensors", []):
        dims = tuple(int(x) for x in t["dims"])
        if any(x <= 0 for x in dims):
            raise ProgramError(f"tensor {t['name']!r}: dims must be positive")
        decls.append(TensorDecl(t["name"], dims, int(t.get("elem_bytes", 4)),
                                t.get("scope", "global")))
    by_name = {t.name: t for t in decls}
    if len(by_name) != len(decls):
        raise ProgramError("duplicate tensor names")
    return LoopProgram(tuple(decls), tuple(_parse_node(n, (), by_name) for n in data.get("body", [])))


def program_to_json(p) -> dict:
    """JSON object of a program (inverse of parse_program)."""
    def node(n):
        if isinstance(n, AccessNode) or hasattr(n, "index_exprs"):
            return {"access": {"tensor": n.tensor, "kind": n.kind,
                               "idx": [str(AffineExpr(tuple(e.terms), e.const)) for e in n.index_exprs]}}
        attrs = (["parallel"] if n.parallel else []) + (["unroll"] if n.unrolled else [])
        if n.vector_width is not None:
            attrs.append(f"vectorize:{n.vector_width}")
        return {"loop": {"var": n.var, "extent": n.extent, "step": n.step, "attrs": attrs,
                         "body": [node(c) for c in n.children]}}
    return {"tensors": [{"name": t.name, "dims": list(t.dims), "elem_bytes": t.elem_bytes,
                         "scope": t.scope} for t in p.tensors],
            "body": [node(n) for n in p.body]}


# -- schedules -------------------------------------------------------------------


@dataclass(frozen=True)
class Tile:
    loop: str
    factor: int


@dataclass(frozen=True)
class Reorder:
    order: tuple


@dataclass(frozen=True)
class Unroll:
    loop: str


@dataclass(frozen=True)
class Vectorize:
    loop: str
    width: int


@dataclass(frozen=True)
class Parallel:
    loop: str


def transform_to_json(t) -> dict:
    name = type(t).__name__
    if name == "Tile":
        return {"tile": {"loop": t.loop, "factor": t.factor}}
    if name == "Reorder":
        return {"reorder": list(t.order)}
    if name == "Unroll":
        return {"unroll": {"loop": t.loop}}
    if name == "Vectorize":
        return {"vectorize": {"loop": t.loop, "width": t.width}}
    if name == "Parallel":
        return {"parallel": {"loop": t.loop}}
    raise ProgramError(f"unknown transform {t!r}")


@dataclass(frozen=True)
class Schedule:
    transforms: tuple = ()

    def to_json(self) -> list:
        return [transform_to_json(t) for t in self.transforms]

    @staticmethod
    def from_json(data: list) -> "Schedule":
        out = []
        for rec in data:
            if "tile" in rec:
                out.append(Tile(rec["tile"]["loop"], int(rec["tile"]["factor"])))
            elif "reorder" in rec:
                out.append(Reorder(tuple(rec["reorder"])))
            elif "unroll" in rec:
                out.append(Unroll(rec["unroll"]["loop"]))
            elif "vectorize" in rec:
                out.append(Vectorize(rec["vectorize"]["loop"], int(rec["vectorize"]["width"])))
            elif "parallel" in rec:
                out.append(Parallel(rec["parallel"]["loop"]))
            else:
                raise ProgramError(f"unknown transform record {rec!r}")
        return Schedule(tuple(out))


def schedule_key(s) -> str:
    """The memo / tie-break key of a schedule: json.dumps(s.to_json()) (ls/es.py:145)."""
    return json.dumps([transform_to_json(t) for t in s.transforms])


# -- schedule spaces ---------------------------------------------------------------


@dataclass(frozen=True)
class SpaceAxis:
    name: str
    choices: tuple


def space_axes(p, space: dict) -> list:
    """Independent choice axes in the reference's fixed order (ls/ir.py:517-547):
    tiles sorted by loop, reorder, vectorize sorted by loop (0 = off), unroll, parallel."""
    axes = []
    for loop, factors in sorted(space.get("tile", {}).items()):
        extent = p.find_loop(loop).extent
        bad = [f for f in factors if f < 1 or extent % f]
        if bad:
            raise ProgramError(f"tile factor {bad[0]} is not a divisor of extent {extent} (loop {loop!r})")
        axes.append(SpaceAxis(f"tile:{loop}", tuple((Tile(loop, f),) for f in sorted(factors))))
    perms = space.get("reorder", [])
    if perms:
        axes.append(SpaceAxis("reorder", tuple((Reorder(tuple(o)),) for o in perms)))
    for loop, widths in sorted(space.get("vectorize", {}).items()):
        extent = p.find_loop(loop).extent
        choices = []
        for w in sorted(widths):
            if w == 0:
                choices.append(())
            elif extent % w:
                raise ProgramError(f"vector width {w} is not a divisor of extent {extent} (loop {loop!r})")
            else:
                choices.append((Vectorize(loop, w),))
        axes.append(SpaceAxis(f"vectorize:{loop}", tuple(choices)))
    for loop in sorted(space.get("unroll", [])):
        p.find_loop(loop)
        axes.append(SpaceAxis(f"unroll:{loop}", ((), (Unroll(loop),))))
    for loop in sorted(space.get("parallel", [])):
        p.find_loop(loop)
        axes.append(SpaceAxis(f"parallel:{loop}", ((), (Parallel(loop),))))
    return axes


# -- failure messages ---------------------------------------------------------------


def failure_message(program, schedule) -> "tuple[str, str] | None":
    """(exception type, message) apply_schedule raises for `schedule`, or None.

    The device reports a failed candidate as a status code; the text the
    reference's exception carries (ls/ir.py:151, 361-470) is rebuilt here for
    the diagnostics of a failed candidate only, by replaying the transforms
    over the loop names, extents and nesting of the program tree.  Scores and
    features always come from the device.
    """
    # loop tree: name -> [extent, parent name | None, [child names and access markers]]
    loops = {}
    top = []

    def add(n, parent):
        if type(n).__name__ != "LoopNode":
            return None
        loops[n.var] = [n.extent, parent, []]
        for ch in n.children:
            nm = add(ch, n.var)
            loops[n.var][2].append(nm if nm is not None else "<access>")
        return n.var

    for n in program.body:
        nm = add(n, None)
        top.append(nm if nm is not None else "<access>")
    names = set(loops)

    def find(v):
        if v not in loops:
            raise ProgramError(f"no loop named {v!r}")
        return loops[v]

    def tile(v, factor):
        node = find(v)
        ext = node[0]
        if factor < 1 or factor > ext:
            raise ProgramError(f"tile factor {factor} out of range for loop {v!r} (extent {ext})")
        inner = v + "_i"
        while inner in names:
            inner += "_"
        names.add(inner)
        loops[inner] = [factor, v, node[2]]
        for ch in node[2]:
            if ch in loops:
                loops[ch][1] = inner
        node[0] = -(-ext // factor)
        node[2] = [inner]

    def depth(v):
        d, p = 0, loops[v][1]
        while p is not None:
            d, p = d + 1, loops[p][1]
        return d

    try:
        for t in schedule.transforms:
            kind = type(t).__name__
            if kind == "Tile":
                tile(t.loop, t.factor)
            elif kind == "Vectorize":
                ext = find(t.loop)[0]
                if ext % t.width != 0:
                    raise ProgramError(f"vectorize width {t.width} does not divide extent {ext} of {t.loop!r}")
                tile(t.loop, t.width)
            elif kind == "Reorder":
                order = tuple(t.order)
                if len(order) < 2:
                    continue
                for v in order:
                    find(v)
                if len(set(order)) != len(order):
                    raise ProgramError(f"reorder {order!r}: missing loops")
                cur = min(order, key=depth)  # stable: the first shallowest name
                for _ in range(len(order) - 1):
                    kids = loops[cur][2]
                    if len(kids) != 1 or kids[0] not in order:
                        raise ProgramError(f"reorder {order!r}: loops do not form a perfect nest chain")
                    cur = kids[0]
                # headers move, the structure stays: extents follow the names
                seq = [min(order, key=depth)]
                for _ in range(len(order) - 1):
                    seq.append(loops[seq[-1]][2][0])
                ext = {v: loops[v][0] for v in order}
                kids_of_last = loops[seq[-1]][2]
                parent_of_first = loops[seq[0]][1]
                for i, v in enumerate(order):
                    loops[v][0] = ext[v]
                    loops[v][1] = parent_of_first if i == 0 else order[i - 1]
                    loops[v][2] = [order[i + 1]] if i + 1 < len(order) else kids_of_last
                for ch in kids_of_last:
                    if ch in loops:
                        loops[ch][1] = order[-1]
                if parent_of_first is not None:
                    pk = loops[parent_of_first][2]
                    pk[pk.index(seq[0])] = order[0]
                else:
                    top[top.index(seq[0])] = order[0]
            else:  # Unroll / Parallel: existence only
                find(t.loop)
    except ProgramError as e:
        return "ProgramError", str(e)
    except ZeroDivisionError as e:
        return "ZeroDivisionError", str(e)
    return None
