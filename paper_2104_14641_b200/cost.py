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

from dataclasses import dataclass

import numpy as np

from . import abi
from .arch import CPU_FEATURES, GPU_FEATURES, FeatureVector
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

    @property
    def errors(self) -> list:
        return [(int(i), CandidateError(int(self.status[i]))) for i in np.nonzero(self.status)[0]]

    def feature_vector(self, i: int) -> FeatureVector:
        return FeatureVector(tuple(zip(self.feature_names, map(float, self.features[i]))))


_TASKS: dict = {}


def _task_for(template, arch, launch, device):
    key = (id(template), arch, launch, device)
    t = _TASKS.get(key)
    if t is None:
        t = (Task(template.desc(arch, launch), device), template)
        _TASKS[key] = t
    return t[0]


def score_batch(program, schedules, arch, launch=None, device: int = 0, features: bool = True) -> BatchResult:
    import torch

    n = len(schedules)
    names = CPU_FEATURES if arch.family == "cpu" else GPU_FEATURES
    scores = np.full(n, np.nan)
    feats = np.full((n, len(names)), np.nan) if features else None
    status = np.zeros(n, np.int32)
    for g in pack_schedules(program, schedules):
        if g.template is None:
            status[g.index] = abi.ST_UNSUPPORTED
            continue
        try:
            task = Task(g.template.desc(arch, launch), device)
        except EngineError as e:
            if "(-3)" not in str(e):  # LS_E_UNSUPPORTED: outside the device class, per candidate
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
        task.close()
    return BatchResult(scores, feats, status, names)


def rank_schedules(program, schedules, arch, launch=None, device: int = 0):
    """cmd_rank's core: [(index, score, FeatureVector)] ascending by (score, index) + errors."""
    import torch

    res = score_batch(program, schedules, arch, launch, device)
    ok = np.nonzero(res.status == 0)[0]
    if len(ok):
        s = torch.from_numpy(res.scores[ok]).cuda(device)
        order = torch.sort(s, stable=True).indices.cpu().numpy()  # ties keep input order
        ok = ok[order]
    rows = [(int(i), float(res.scores[i]), res.feature_vector(int(i))) for i in ok]
    return rows, res.errors


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
