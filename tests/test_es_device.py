"""Device ES (ls_es_*, es.optimize_device) against the numpy restatement (oracle/es_oracle.py)
and the C oracle's scores: noise, decode, memo/evaluations, rank-shaped update, trace, incumbent."""

import json
import sys
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from golden_util import GOLDEN, arch_named, launch

sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "oracle"))
import es_oracle  # noqa: E402
import pyoracle  # noqa: E402


@pytest.fixture(scope="module")
def torch():
    import torch as t
    return t


def _space(name):
    from paper_2104_14641_b200 import ir, workloads as W
    from paper_2104_14641_b200.pack import SpaceTemplate
    if name == "conv56":
        prog = W.program(W.conv2d_json())
        return prog, W.conv_space(512, 1), "x86-avx2"
    r = next(x for x in json.loads((GOLDEN / "es_runs.json").read_text()) if x["name"] == name)
    return ir.parse_program(json.dumps(r["program"])), r["space"], r["arch"]


def _oracle_scores(st, desc, points):
    recs = st.records_from_indices(st.indices_from_points(np.asarray(points, np.uint64)))
    s, _, status = pyoracle.evaluate(desc, recs, nthreads=8)
    assert (status == 0).all()
    return s


@pytest.mark.parametrize("name,pop,iters,sigma,rank", [("matmul32", 512, 6, 0.3, True),
                                                       ("conv_small", 300, 5, 0.8, True),
                                                       ("conv_gpu", 256, 4, 0.6, False),
                                                       ("conv56", 4096, 4, 2.0, True)])
def test_device_es_one_step_parity(torch, name, pop, iters, sigma, rank):
    from paper_2104_14641_b200 import engine as E
    from paper_2104_14641_b200.pack import SpaceTemplate
    prog, space, arch = _space(name)
    st = SpaceTemplate(prog, space)
    desc = st.template.desc(arch_named(arch), launch())
    task = E.Task(desc, 0)
    task.set_space(st.space_desc())
    if task.has_unroll:
        idx = st.indices_from_points(np.arange(st.size, dtype=np.uint64))
        task.prepare_unroll_for(E.to_device_records(st.records_from_indices(idx)))
    alpha, seed = 0.05, 12345
    run = E.EsRun(task, alpha, sigma, pop, iters, seed, rank)
    run.run()
    hist, trace, evals, err, best = run.result(st.dim)
    assert err == 0
    assert np.array_equal(hist[0], [(n - 1) / 2.0 for n in st.sizes])  # ThetaEncoding.initial
    memo = {}

    def score_all(points):
        new = sorted({int(p) for p in points} - memo.keys())
        if new:
            for p, s in zip(new, _oracle_scores(st, desc, new)):
                memo[p] = float(s)
        return np.array([memo[int(p)] for p in points])

    score_all(st.points_from_indices(es_oracle.decode(hist[0][None, :], st.sizes)).astype(np.uint64))
    for g in range(iters):
        eps = run.noise(g, st.dim).cpu().numpy()
        np.testing.assert_allclose(eps, es_oracle.normals(seed, g, pop, st.dim), rtol=1e-13, atol=1e-15)
        pts = st.points_from_indices(es_oracle.decode(hist[g] + sigma * eps, st.sizes)).astype(np.uint64)
        values = -score_all(pts)
        want = es_oracle.es_update(hist[g], alpha, sigma, pop, values, eps, rank)
        np.testing.assert_allclose(hist[g + 1], want, rtol=1e-12, atol=1e-12)
        assert trace[g] == min(memo.values())
    assert evals == len(memo) and best == min(memo.values())
    pts, scores = run.evaluated()
    assert sorted(pts.tolist()) == sorted(memo)
    assert all(memo[int(p)] == s for p, s in zip(pts, scores))  # bit-exact vs the C oracle
    run.close()
    task.close()


def test_optimize_device_api(torch):
    """optimize_device returns the reference's OptimizeResult contract over its own trajectory."""
    from paper_2104_14641_b200.es import EsParams, optimize_device
    from paper_2104_14641_b200.pack import SpaceTemplate
    prog, space, arch = _space("matmul32")
    res = optimize_device(prog, space, arch_named(arch), EsParams(population=64, iterations=10, seed=3),
                          launch=launch())
    assert res.evaluations == len(res.evaluated)
    best_key = min(res.evaluated, key=lambda k: (res.evaluated[k], k))
    assert json.dumps(res.best_schedule.to_json()) == best_key
    assert res.best_score == res.evaluated[best_key] == res.trace[-1]
    assert all(a >= b for a, b in zip(res.trace, res.trace[1:]))
    st = SpaceTemplate(prog, space)
    desc = st.template.desc(arch_named(arch), launch())
    idx = st.indices_from_points(np.arange(st.size, dtype=np.uint64))
    row = next(r for r in idx if json.dumps(st.schedule_of(r).to_json()) == best_key)
    recs = st.records_from_indices(row[None, :])
    s, f, status = pyoracle.evaluate(desc, recs)
    assert status[0] == 0 and s[0] == res.best_score
    assert [v for _, v in res.best_features.values] == f[0].tolist()


def test_optimize_device_single_schedule_space(torch):
    from paper_2104_14641_b200 import workloads as W
    from paper_2104_14641_b200.es import EsParams, optimize_device
    prog = W.program(W.matmul_json(32))
    res = optimize_device(prog, {"tile": {"i": [4]}}, arch_named("x86-avx2"),
                          EsParams(population=8, iterations=3), launch=launch())
    assert res.evaluations == 1 and res.trace == [res.best_score]


def test_optimize_failure_messages_match_reference():
    """es.optimize (exact trajectory) raises the reference's SearchError text when a population
    member's schedule fails: 'population candidate {i} failed at iteration {t}: candidate {key}
    failed: {ProgramError text}' (ls/es.py:153-154, 186-187); successful runs find the same best."""
    import json

    from golden_util import GOLDEN
    from paper_2104_14641_b200.arch import load_arch
    from paper_2104_14641_b200.es import EsParams, SearchError, optimize
    from paper_2104_14641_b200.ir import parse_program
    g = json.loads((GOLDEN / "es_fail.json").read_text())
    prog = parse_program(json.dumps(g["program"]))
    for c in g["cases"]:
        params = EsParams(seed=c["seed"], **g["params"])
        if "error" in c:
            with pytest.raises(SearchError) as ei:
                optimize(prog, c["space"], load_arch("x86-avx2"), params, jobs=1)
            assert [type(ei.value).__name__, str(ei.value)] == c["error"]
        else:
            r = optimize(prog, c["space"], load_arch("x86-avx2"), params, jobs=1)
            assert r.best_score == c["best"] and r.evaluations == c["evaluations"]


@pytest.mark.parametrize("name,pop,sigma", [("conv_small", 2, 0.8), ("conv_small", 777, 0.8),
                                            ("conv_small", 8191, 0.8), ("conv56", 8192, 2.0),
                                            ("conv56", 8193, 2.0), ("conv_small", 40000, 0.8),
                                            ("conv56", 3 * (1 << 16) + 5, 2.0), ("equal", 20000, 1e-9)])
def test_rank_sort_is_stable_argsort(torch, name, pop, sigma):
    """The onesweep rank sort (es_dev.cuh rs_*: multi-tile look-back, partial last tile, heavy
    ties on a small space, every key equal) == numpy's stable argsort of the F keys
    (_shape_fitness, ls/es.py:65-71), every generation's last sort."""
    from paper_2104_14641_b200 import engine as E
    from paper_2104_14641_b200.pack import SpaceTemplate
    if name == "equal":  # odd axis sizes: theta starts on a point and sigma ~0 keeps every member
        # there, so every key is equal (the plan's single copy pass)
        from paper_2104_14641_b200 import workloads as W
        prog, space, arch = W.program(W.matmul_json(32)), {"tile": {"i": [2, 4, 8], "j": [2, 4, 8]}}, "x86-avx2"
    else:
        prog, space, arch = _space(name)
    st = SpaceTemplate(prog, space)
    task = E.Task(st.template.desc(arch_named(arch), launch()), 0)
    task.set_space(st.space_desc())
    for iters in (1, 3):
        run = E.EsRun(task, 0.05, sigma, pop, iters, 99 + iters)
        run.run()
        kin, kout, mem, rk = (x.cpu().numpy() for x in run.sort_state())
        kin = kin.view(np.uint64)
        order = np.argsort(kin, kind="stable")
        assert np.array_equal(mem.astype(np.int64), order)
        ranks = np.empty(pop, np.int64)
        ranks[order] = np.arange(pop)  # argsort(argsort(F, stable), stable): each member's rank
        assert np.array_equal(rk.astype(np.int64), ranks)
        assert np.array_equal(kout.view(np.uint64), kin[order])
        if name == "equal":
            assert (kin == kin[0]).all()
        run.close()
    task.close()
