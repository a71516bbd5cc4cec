"""Evolution-strategies search with device-scored populations.

API and trajectory of the reference's ``optimize`` (ls/es.py:119-204): same
EsParams, same centroid start, same SeedSequence/PCG64 noise per generation,
same round-half-even decode, same rank-shaped update, same memo of distinct
schedules keyed by their JSON, same incumbent tie-break (score, JSON key).
What changes is the evaluation: each generation's *new distinct* schedules
are packed into records and scored in one device launch instead of one
Python call chain per candidate.  Scores are bit-identical to the reference,
so the theta trajectory, trace and evaluated table are too.
"""

from __future__ import annotations

import json
from dataclasses import dataclass

import numpy as np

from .engine import EsRun, Task, to_device_records
from .ir import Schedule, space_axes
from .pack import PackError, SpaceTemplate
from .arch import CPU_FEATURES, GPU_FEATURES, FeatureVector


class SearchError(RuntimeError):
    pass


@dataclass(frozen=True)
class EsParams:
    alpha: float = 0.05
    sigma: float = 0.3
    population: int = 32
    iterations: int = 100
    seed: int = 0
    rank_normalize: bool = True

    def __post_init__(self):
        if self.alpha <= 0 or self.sigma <= 0:
            raise ValueError("alpha and sigma must be positive")
        if self.population < 2:
            raise ValueError("population must be >= 2")
        if self.iterations < 1:
            raise ValueError("iterations must be >= 1")


@dataclass(frozen=True)
class ThetaEncoding:
    axes: tuple

    @property
    def dim(self) -> int:
        return len(self.axes)

    def initial(self) -> np.ndarray:
        return np.array([(len(ax.choices) - 1) / 2.0 for ax in self.axes])

    def indices(self, thetas: np.ndarray) -> np.ndarray:
        sizes = np.array([len(ax.choices) for ax in self.axes], np.int64)
        return np.clip(np.rint(np.asarray(thetas, np.float64)), 0, sizes - 1).astype(np.int64)

    def decode(self, theta) -> Schedule:
        out = []
        for i, ax in zip(self.indices(np.asarray(theta).reshape(1, -1))[0], self.axes):
            out.extend(ax.choices[int(i)])
        return Schedule(tuple(out))


def shape_fitness(values: np.ndarray) -> np.ndarray:
    """Centered ranks on [-0.5, 0.5] (ls/es.py:65-71)."""
    n = len(values)
    if n == 1 or np.ptp(values) == 0:
        return np.zeros(n)
    order = np.argsort(np.argsort(values, kind="stable"), kind="stable")
    return order / (n - 1) - 0.5


def es_update(theta: np.ndarray, params: EsParams, values: np.ndarray, noise: np.ndarray,
              diagnostics: "list | None" = None) -> np.ndarray:
    """theta + alpha/(n*sigma) * sum(F_i * eps_i) with the reference's NaN handling (ls/es.py:74-93)."""
    values = np.asarray(values, dtype=float)
    bad = ~np.isfinite(values)
    if bad.any():
        if diagnostics is not None:
            diagnostics.append(f"{int(bad.sum())} non-finite objective values replaced by population minimum")
        fill = values[~bad].min() if (~bad).any() else 0.0
        values = np.where(bad, fill, values)
    weights = shape_fitness(values) if params.rank_normalize else values
    return theta + (params.alpha / (params.population * params.sigma)) * (weights @ noise)


@dataclass
class OptimizeResult:
    best_schedule: Schedule
    best_score: float
    best_features: FeatureVector
    trace: list
    evaluated: dict
    evaluations: int
    diagnostics: list


class _DeviceObjective:
    """Memoised device scoring of space points (the evaluate_schedule cache, ls/es.py:139-160)."""

    def __init__(self, program, space, arch, launch, device):
        import torch
        self.torch = torch
        self.program = program
        self.arch, self.launch = arch, launch
        self.device = device
        self.names = CPU_FEATURES if arch.family == "cpu" else GPU_FEATURES
        try:
            self.st = SpaceTemplate(program, space)
        except PackError:  # e.g. reorder choices over different loop sets: score the decoded
            self.st = None  # schedules as lists (one template per shape, cost.score_batch)
            self.axes = tuple(space_axes(program, space))
            self.sizes = np.array([len(ax.choices) for ax in self.axes], np.int64)
        if self.st is not None:
            self.task = Task(self.st.template.desc(arch, launch), device)
            self.sizes = self.st.sizes
        self.cache: dict = {}   # flat point index -> (key, score, features)
        self.by_key: dict = {}  # json key -> (score, features)

    def schedule_of(self, row) -> Schedule:
        if self.st is not None:
            return self.st.schedule_of(row)
        return Schedule(tuple(t for a, i in enumerate(row) for t in self.axes[a].choices[int(i)]))

    def flat(self, idx: np.ndarray) -> np.ndarray:
        f = np.zeros(len(idx), np.int64)
        for a, n in enumerate(self.sizes):
            f = f * int(n) + idx[:, a]
        return f

    def evaluate(self, idx: np.ndarray, where: str) -> np.ndarray:
        """Scores of rows of choice indices; new distinct points go to the device in one batch."""
        flat = self.flat(idx)
        uniq, first = np.unique(flat, return_index=True)
        order = np.argsort(first, kind="stable")  # first-appearance order, like a serial loop
        uniq, first = uniq[order], first[order]
        is_new = np.array([int(u) not in self.cache for u in uniq], bool)
        new = [int(u) for u in uniq[is_new]]
        if new:
            rows = idx[first[is_new]]
            if self.st is not None:
                recs = self.st.records_from_indices(rows)
                d_rec = to_device_records(recs, self.device)
                self.task.prepare_unroll_for(d_rec)
                s, f, st = self.task.score(d_rec, features=True)
                s, f, st = s.cpu().numpy(), f.cpu().numpy(), st.cpu().numpy()
            else:
                from .cost import score_batch
                res = score_batch(self.program, [self.schedule_of(r) for r in rows], self.arch, self.launch,
                                  self.device)
                s, f, st = res.scores, res.features, res.status
            bad = [j for j in range(len(new)) if st[j]]
            if bad:  # the reference's message: the first failing member in population order
                failing = {new[j]: j for j in bad}
                member = next(m for m, u in enumerate(flat) if int(u) in failing)
                j = failing[int(flat[member])]
                sched = self.schedule_of(rows[j])
                key = json.dumps(sched.to_json())
                from .ir import failure_message
                fm = failure_message(self.program, sched)
                text = fm[1] if fm is not None else f"status {int(st[j])}"
                inner = f"candidate {key} failed: {text}"  # ls/es.py:153-154
                if where == "start":
                    raise SearchError(inner)
                raise SearchError(f"population candidate {member} failed at {where}: {inner}")  # ls/es.py:186-187
            for j, u in enumerate(new):
                key = json.dumps(self.schedule_of(rows[j]).to_json())
                self.cache[u] = (key, float(s[j]), f[j])
                self.by_key[key] = (float(s[j]), f[j])
        return np.array([self.cache[int(u)][1] for u in flat])


def optimize(program, space: dict, arch, params: EsParams, jobs=None, launch=None,
             device: int = 0) -> OptimizeResult:
    """ES search for the lowest-scoring schedule (ls/es.py:130-204), device-scored."""
    axes = tuple(space_axes(program, space))
    if not axes:
        raise SearchError("empty schedule space")
    enc = ThetaEncoding(axes)
    obj = _DeviceObjective(program, space, arch, launch, device)
    diagnostics: list = []
    theta = enc.initial()
    trace: list = []
    children = np.random.SeedSequence(params.seed).spawn(params.iterations)
    obj.evaluate(enc.indices(theta.reshape(1, -1)), "start")
    single = all(len(ax.choices) == 1 for ax in axes)
    best = lambda: min(obj.by_key, key=lambda k: (obj.by_key[k][0], k))  # noqa: E731
    for t in range(params.iterations):
        if single:
            break
        rng = np.random.default_rng(children[t])
        noise = rng.standard_normal((params.population, enc.dim))
        pts = theta + params.sigma * noise
        scores = obj.evaluate(enc.indices(pts), f"iteration {t}")
        theta = es_update(theta, params, -scores, noise, diagnostics)
        trace.append(obj.by_key[best()][0])
    bk = best()
    if not trace:
        trace = [obj.by_key[bk][0]]
    bs, bf = obj.by_key[bk]
    return OptimizeResult(
        best_schedule=Schedule.from_json(json.loads(bk)),
        best_score=bs,
        best_features=FeatureVector(tuple(zip(obj.names, map(float, bf)))),
        trace=trace,
        evaluated={k: v[0] for k, v in obj.by_key.items()},
        evaluations=len(obj.by_key),
        diagnostics=diagnostics,
    )


def _error_text(err: int) -> str:
    from . import abi
    gen, member, st = err >> 40, (err >> 8) & ((1 << 32) - 1), err & 0xFF
    where = "start point" if gen == 0 else f"population candidate {member} failed at iteration {gen - 1}"
    return f"{where}: {abi.STATUS.get(st, st)}"


def optimize_device(program, space: dict, arch, params: EsParams, jobs=None, launch=None, device: int = 0,
                    materialize: bool = True, group=None) -> OptimizeResult:
    """ES search with every generation on the device (throughput mode, include/loopscout_b200.h ls_es_*).

    Same API, EsParams, centroid start, decode, memo of distinct schedules,
    rank-shaped update and incumbent rule as optimize (ls/es.py:130-204); the
    Gaussian noise is Philox4x32-10 + Box-Muller on the device instead of
    numpy's PCG64, so the trajectory is not the reference's (optimize above is
    the exact-trajectory mode).  `jobs` is accepted for API parity and unused.
    materialize=False skips building the evaluated dict (JSON keys) for large runs.
    Under torch.distributed (world > 1 in `group`) the population is sharded over the ranks
    (one GPU each, dist.py); every rank returns the same result, bit-identical to one rank.
    """
    axes = tuple(space_axes(program, space))
    if not axes:
        raise SearchError("empty schedule space")
    st = SpaceTemplate(program, space)
    task = Task(st.template.desc(arch, launch), device)
    try:
        task.set_space(st.space_desc())
        if task.has_unroll:  # block cycles for every body-replication product the space can produce
            if st.size > 1 << 22:
                raise SearchError("device ES: unroll axes over a space above 2^22 points are not supported")
            idx = st.indices_from_points(np.arange(st.size, dtype=np.uint64))
            task.prepare_unroll_for(to_device_records(st.records_from_indices(idx), device))
        world, rank = 1, 0
        try:
            import torch.distributed as dist
            if dist.is_available() and dist.is_initialized():
                world, rank = dist.get_world_size(group), dist.get_rank(group)
        except ImportError:
            pass
        single = all(len(ax.choices) == 1 for ax in axes)
        run = EsRun(task, params.alpha, params.sigma, params.population, params.iterations, params.seed,
                    params.rank_normalize, rank=rank, world=world)
        try:
            if world == 1:
                run.run()
            else:
                from .dist import es_exchange
                run.run_sharded(es_exchange(group), generations=0 if single else None)
            hist, trace, evaluations, err, best = run.result(st.dim)
            pts, scores = run.evaluated()
        finally:
            run.close()
        if world > 1:
            from .dist import es_merge_results
            trace, pts, scores, err, best = es_merge_results(trace, pts, scores, err, best, group)
            evaluations = len(pts)
        if err:
            raise SearchError(_error_text(err))
        key_of = lambda p: json.dumps(st.schedule_of(st.indices_from_points(np.array([p]))[0]).to_json())  # noqa: E731
        # incumbent: min over distinct schedules by (score, JSON key) (ls/es.py:189, 197)
        ties = [int(p) for p, s in zip(pts, scores) if s == best]
        bk = min((key_of(p) for p in ties))
        best_pt = next(p for p in ties if key_of(p) == bk)
        import torch
        dp = torch.tensor([int(best_pt)], dtype=torch.int64, device=f"cuda:{device}")
        _, bf, _ = task.score_points(dp, features=True)
        bf = bf.cpu().numpy()[0]
        names = CPU_FEATURES if arch.family == "cpu" else GPU_FEATURES
        evaluated = {key_of(p): float(s) for p, s in zip(pts, scores)} if materialize else {}
        return OptimizeResult(
            best_schedule=Schedule.from_json(json.loads(bk)),
            best_score=float(best),
            best_features=FeatureVector(tuple(zip(names, map(float, bf)))),
            trace=[float(x) for x in trace] if not single else [float(best)],
            evaluated=evaluated,
            evaluations=evaluations,
            diagnostics=[],
        )
    finally:
        task.close()
