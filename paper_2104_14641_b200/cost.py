"""Drop-in batched scoring and ranking (the ``rank`` path).

``score_batch`` is the batched equivalent of running, for every schedule,
apply_schedule + emit_mock_asm + extract_features + score (ls/ir.py:454,
ls/ir.py:557, ls/cost.py:132, ls/cost.py:155) -- the per-candidate closure of
cmd_rank (ls/cli.py:115-119) -- on the device.  ``rank_schedules`` adds the
cmd_rank ordering by (score, input index) (ls/cli.py:124-126).  Failed
candidates are reported as (index, message) like evaluate_population's
``errors`` list (ls/es.py:96-116).
"""

from __future__ import annotations

from collections import OrderedDict
from dataclasses import dataclass, field

import numpy as np

from . import abi
from .arch import CPU_FEATURES, GPU_FEATURES, CostModelError, FeatureVector
from .engine import EngineError, Task, to_device_records
from .pack import PackError, pack_schedules


class CandidateError(ValueError):
    """A candidate failed the way the reference would have raised (see .status)."""

    def __init__(self, status: int):
        super().__init__(abi.STATUS.get(status, f"status {status}"))
        self.status = status


@dataclass
class BatchResult:
    scores: np.ndarray          # f64[n], NaN where failed
    features: "np.ndarray | None"  # f64[n, F]
    status: np.ndarray          # i32[n], 0 = ok (include/loopscout_b200.h)
    feature_names: tuple
    messages: dict = field(default_factory=dict)  # index -> (exception type, text) raised on the host

    @property
    def errors(self) -> list:
        return [(int(i), self.exception(int(i))) for i in np.nonzero(self.status)[0]]

    def exception(self, i: int) -> Exception:
        """The failure of candidate i: the host-side exception when one was recorded, else the
        device status as a CandidateError."""
        if i in self.messages and self.messages[i][0] == "CostModelError":
            return CostModelError(self.messages[i][1])
        return CandidateError(int(self.status[i]))

    def feature_vector(self, i: int) -> FeatureVector:
        return FeatureVector(tuple(zip(self.feature_names, map(float, self.features[i]))))


class _TaskCache:
    """Device tasks per (template, arch, launch, device), LRU-bounded: a task is built once
    (descriptor upload + per-task tables, ~0.1 ms) and reused by every later batch of the shape."""

    def __init__(self, cap: int = 64):
        self.cap = cap
        self.d: "OrderedDict" = OrderedDict()

    def get(self, template, arch, launch, device):
        key = (id(template), id(arch), id(launch), device)
        hit = self.d.get(key)
        if hit is not None and hit[1] is template and hit[2] is arch and hit[3] is launch:
            self.d.move_to_end(key)
            return hit[0]
        task = Task(template.desc(arch, launch), device)
        self.d[key] = (task, template, arch, launch)
        while len(self.d) > self.cap:
            old = self.d.popitem(last=False)[1][0]
            old.close()
        return task


_TASKS = _TaskCache()


def score_batch(program, schedules, arch, launch=None, device: int = 0, features: bool = True) -> BatchResult:
    """Score every schedule on the device (groups by shape, one fused launch per group).

    Per-candidate failures never abort the batch: device status codes for the reference's
    ProgramError/CostModelError classes, and host-side failures of a whole group (a GPU arch
    without a launch record, a shape outside the device class) recorded per candidate with the
    reference's message, like evaluate_population's `errors` (ls/es.py:96-116)."""
    import torch

    n = len(schedules)
    names = CPU_FEATURES if arch.family == "cpu" else GPU_FEATURES
    scores = np.full(n, np.nan)
    feats = np.full((n, len(names)), np.nan) if features else None
    status = np.zeros(n, np.int32)
    messages: dict = {}
    for g in pack_schedules(program, schedules):
        if g.template is None:
            status[g.index] = abi.ST_UNSUPPORTED
            continue
        try:
            task = _TASKS.get(g.template, arch, launch, device)
        except CostModelError as e:  # e.g. a GPU arch without a launch record (ls/cost.py:137-138)
            status[g.index] = abi.ST_UNSUPPORTED
            messages.update({int(i): ("CostModelError", str(e)) for i in g.index})
            continue
        except (EngineError, PackError) as e:
            if isinstance(e, EngineError) and "(-3)" not in str(e):  # only LS_E_UNSUPPORTED is per candidate
                raise
            status[g.index] = abi.ST_UNSUPPORTED
            continue
        d_rec = to_device_records(g.records, device)
        task.prepare_unroll_for(d_rec)
        s, f, st = task.score(d_rec, features=features)
        torch.cuda.synchronize(device)
        st = st.cpu().numpy()
        st = np.where(g.host_status != 0, g.host_status, st)
        status[g.index] = st
        ok = st == 0
        scores[g.index[ok]] = s.cpu().numpy()[ok]
        if features:
            feats[g.index[ok]] = f.cpu().numpy()[ok]
    return BatchResult(scores, feats, status, names, messages)


def _access_order(program) -> list:
    """Tensor names in first-access order (the order CacheModel merges tensor states)."""
    order, stack = [], list(reversed(program.body))
    while stack:
        nd = stack.pop()
        if hasattr(nd, "children"):
            stack.extend(reversed(nd.children))
        elif getattr(nd, "tensor", None) is not None and nd.tensor not in order:
            order.append(nd.tensor)
    return order


def inexact_footprints(program, schedules, arch, launch=None, device: int = 0, diagnostics: "list | None" = None):
    """Per schedule, the cache model's inexact-footprint flag of the scheduled program --
    `analyze(apply_schedule(program, s), cache).node_costs["<root>"].inexact` (ls/cache.py:
    198-202, 228-231) -- computed on the device: 1 inexact, 0 exact, -1 the schedule fails
    apply_schedule (or its shape is outside the device class).  `diagnostics`, if given,
    receives one list per schedule: the model's notes ("inexact footprint for tensor 'A' at
    loop 'i'", innermost loop first)."""
    import torch

    out = np.full(len(schedules), -1, np.int8)
    notes: list = [[] for _ in schedules]
    tensors = [t.name for t in program.tensors]
    rank_of = {nm: j for j, nm in enumerate(_access_order(program))}
    for g in pack_schedules(program, schedules):
        if g.template is None:
            continue
        task = _TASKS.get(g.template, arch, launch, device)
        d_rec = to_device_records(g.records, device)
        f, m, ch = task.inexact_footprints(d_rec, notes=True)
        torch.cuda.synchronize(device)
        f = f.cpu().numpy().astype(np.int16)
        f = np.where((f == 255) | (g.host_status != 0), -1, f)
        out[g.index] = f
        if diagnostics is None:
            continue
        m, ch = m.cpu().numpy().view(np.uint64), ch.cpu().numpy()
        for row, gi in enumerate(g.index):
            if f[row] != 1:
                continue
            chain = [int(x) for x in ch[row] if x != 0xFF]
            for p in range(len(chain) - 1, -1, -1):
                hit = [t for t in range(len(tensors))
                       if (int(m[row, (8 * p + t) // 64]) >> ((8 * p + t) % 64)) & 1]
                for t in sorted(hit, key=lambda t: rank_of.get(tensors[t], len(tensors))):
                    notes[gi].append(f"inexact footprint for tensor {tensors[t]!r} at loop "
                                     f"{g.template.names[chain[p]]!r}")
    if diagnostics is not None:
        diagnostics.extend(notes)
    return out


def rank_schedules(program, schedules, arch, launch=None, device: int = 0):
    """cmd_rank's core: [(index, score, FeatureVector)] ascending by (score, index) + errors."""
    res = score_batch(program, schedules, arch, launch, device)
    ok = np.nonzero(res.status == 0)[0]
    ok = ok[np.lexsort((ok, res.scores[ok]))]  # ties keep input order (ls/cli.py:124-126)
    rows = [(int(i), float(res.scores[i]), res.feature_vector(int(i))) for i in ok]
    return rows, res.errors


def rank_topk(program, schedules, arch, k: int, launch=None, device: int = 0):
    """The k best of a schedule list by (score, input index) -- cmd_rank's order (ls/cli.py:124-126)
    cut at k -- with the fused score + top-k launch per shape group and the library merge across
    groups.  Returns (scores f64[k], indices i64[k] (+inf / -1 padded), valid count)."""
    import torch

    from .engine import topk_merge

    lists = []
    n_valid = 0
    for g in pack_schedules(program, schedules):
        if g.template is None or (g.host_status != 0).any():
            ok = g.host_status == 0 if g.template is not None else np.zeros(len(g.index), bool)
            if not ok.any():
                continue
            g = type(g)(g.template, g.index[ok], g.records[ok], g.host_status[ok])
        try:
            task = _TASKS.get(g.template, arch, launch, device)
        except (CostModelError, EngineError, PackError) as e:
            if isinstance(e, EngineError) and "(-3)" not in str(e):
                raise
            continue
        d_rec = to_device_records(g.records, device)
        task.prepare_unroll_for(d_rec)
        # group-local indices ranked by the fused kernel, mapped to input positions: the group's
        # positions ascend, so (score, local) order == (score, input index) order
        s, i, nv = task.score_topk(d_rec, k)
        loc = i.cpu().numpy()
        glob = np.where(loc >= 0, g.index[np.clip(loc, 0, None)], -1)
        lists.append((s, torch.from_numpy(glob).to(s.device)))
        n_valid += int(nv.item())
    if not lists:
        return np.full(k, np.inf), np.full(k, -1, np.int64), 0
    if len(lists) == 1:
        s, i = lists[0]
    else:
        s, i = topk_merge(torch.cat([x[0] for x in lists]), torch.cat([x[1] for x in lists]), len(lists), k, k)
    return s.cpu().numpy(), i.cpu().numpy(), n_valid


def score(fv, arch) -> float:
    """score (ls/cost.py:155-161) of an already extracted FeatureVector."""
    from .arch import CostModelError
    total = 0.0
    for name, value in fv.values:
        if name not in arch.coefficients:
            raise CostModelError(f"no coefficient for feature {name!r} in arch {arch.name!r}")
        total += arch.coefficients[name] * value
    return total


def rank(candidates, arch) -> list:
    """rank (ls/cost.py:164-168) over precomputed (Schedule, FeatureVector) pairs."""
    scored = sorted(((score(fv, arch), i) for i, (_, fv) in enumerate(candidates)))
    return [i for _, i in scored]


def analyze(program, arch, launch=None, device: int = 0) -> FeatureVector:
    """Features of the program as given (the `analyze` command without --code)."""
    from .ir import Schedule
    res = score_batch(program, [Schedule(())], arch, launch, device)
    if res.status[0]:
        raise CandidateError(int(res.status[0]))
    return res.feature_vector(0)
