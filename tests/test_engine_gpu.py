"""CUDA engine parity: the sm_100a kernels through the C-ABI against the oracle and the golden outputs."""

import json

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from golden_util import (ALL_SPACE_FIXTURES, GOLDEN, SPACE_FIXTURES, arch_named, launch, rank_cases, rank_groups, space_case,
                         status_of_error)


@pytest.fixture(scope="module")
def torch():
    import torch as t
    return t


def _engine():
    from paper_2104_14641_b200 import engine
    return engine


PATHS = [1, 2]  # LS_PATH_GENERIC, LS_PATH_TABULATED (include/loopscout_b200.h)


def _set_path(task, path):
    """Force a scoring path; False if the task is not eligible for it."""
    if path in (2, 3) and task.path != 2:
        return False
    task.set_path(path)
    return True


POINT_PATHS = [1, 2, 3]  # + LS_PATH_SPACE (points calls only)


@pytest.mark.parametrize("path", PATHS)
@pytest.mark.parametrize("name", ALL_SPACE_FIXTURES)
def test_space_fixtures_bit_exact(torch, name, path):
    E = _engine()
    st, recs, z = space_case(name)
    for a in z["arches"]:
        a = str(a)
        task = E.Task(st.template.desc(arch_named(a), launch()), 0)
        assert _set_path(task, path), "every BASELINE space is eligible for the tabulated path"
        s, f, status = task.score(E.to_device_records(recs))
        torch.cuda.synchronize()
        assert (status.cpu().numpy() == 0).all()
        np.testing.assert_array_equal(f.cpu().numpy(), z[f"feats_{a}"])
        np.testing.assert_array_equal(s.cpu().numpy(), z[f"scores_{a}"])
        task.close()


def _rank_params():
    return [(c["program"], a) for c in rank_cases()["cases"] for a in c["results"]]


@pytest.mark.parametrize("path", PATHS)
@pytest.mark.parametrize("program,arch", _rank_params())
def test_rank_cases(torch, program, arch, path):
    """Random valid/invalid schedules of every transform kind: scores, features and failure classes."""
    E = _engine()
    case = next(c for c in rank_cases()["cases"] if c["program"] == program)
    res = case["results"][arch]
    prog, groups = rank_groups(case)
    ar = arch_named(arch)
    unsupported = 0
    for g in groups:
        if g.template is None:
            unsupported += len(g.index)
            continue
        task = E.Task(g.template.desc(ar, launch()), 0)
        if not _set_path(task, path):
            task.close()
            continue
        d = E.to_device_records(g.records)
        task.prepare_unroll_for(d)
        s, f, st = task.score(d)
        torch.cuda.synchronize()
        s, f, st = s.cpu().numpy(), f.cpu().numpy(), st.cpu().numpy()
        for r, i in enumerate(g.index):
            want = status_of_error(res["errors"][i])
            assert st[r] == want, (i, case["schedules"][i], res["errors"][i], st[r])
            if want == 0:
                assert s[r] == res["scores"][i], (i, case["schedules"][i])
                assert list(f[r]) == res["features"][i], (i, case["schedules"][i])
        task.close()
    # the only packing limit: more than 8 tile/vectorize parameters in one schedule
    assert unsupported <= 2, unsupported


def test_gemm_top64_matches_reference(torch):
    E = _engine()
    st, recs, z = space_case("gemm1024")
    for a in ("x86-avx2", "aarch64-neon", "nvidia-volta"):
        task = E.Task(st.template.desc(arch_named(a), launch()), 0)
        ts, ti, nv = task.score_topk(E.to_device_records(recs), 64)
        torch.cuda.synchronize()
        ref = sorted(range(len(recs)), key=lambda i: (z[f"scores_{a}"][i], i))[:64]
        assert ti.cpu().tolist() == ref
        np.testing.assert_array_equal(ts.cpu().numpy(), z[f"scores_{a}"][ref])
        assert int(nv.item()) == len(recs)
        task.close()


def _conv_task(arch="x86-avx2", n=1 << 18, seed=3, reorders=512, path=0):
    E = _engine()
    from paper_2104_14641_b200 import workloads as W
    from paper_2104_14641_b200.pack import SpaceTemplate
    st = SpaceTemplate(W.program(W.conv2d_json()), W.conv_space(reorders, 1))
    recs = st.records_from_indices(W.distinct_indices(st.sizes, n, seed))
    task = E.Task(st.template.desc(arch_named(arch), launch()), 0)
    if path:
        task.set_path(path)
    return task, recs


@pytest.mark.parametrize("path", PATHS)
@pytest.mark.parametrize("arch", ["x86-avx2", "nvidia-volta"])
def test_fused_topk_equals_full_sort_large(torch, arch, path):
    """Size-independent property at 2^18: fused top-k == stable sort of the per-candidate scores."""
    E = _engine()
    task, recs = _conv_task(arch, path=path)
    d = E.to_device_records(recs)
    s, _, st = task.score(d, features=False)
    for k in (1, 64, 1000):
        ts, ti, nv = task.score_topk(d, k, base_index=7)
        torch.cuda.synchronize()
        order = torch.sort(s, stable=True).indices[:k]
        assert torch.equal(ti, order + 7)
        assert torch.equal(ts, s[order])
        assert int(nv.item()) == len(recs)


@pytest.mark.parametrize("path", PATHS)
def test_oracle_parity_sample_conv(torch, path):
    """Device vs oracle on a 4096-candidate sample of the bench workload (all three arches)."""
    import pyoracle
    E = _engine()
    for a in ("x86-avx2", "aarch64-neon", "nvidia-volta"):
        task, recs = _conv_task(a, n=4096, seed=11, path=path)
        s, f, st = task.score(E.to_device_records(recs))
        torch.cuda.synchronize()
        rs, rf, rst = pyoracle.evaluate(task.desc, recs, nthreads=8)
        np.testing.assert_array_equal(st.cpu().numpy(), rst)
        np.testing.assert_array_equal(s.cpu().numpy(), rs)
        np.testing.assert_array_equal(f.cpu().numpy(), rf)


def test_shard_merge_equals_single(torch):
    """Multi-GPU merge logic on one device: 4 shards with global bases merge to the 1-shard answer."""
    E = _engine()
    from paper_2104_14641_b200.dist import shard_range
    task, recs = _conv_task(n=1 << 16)
    d = E.to_device_records(recs)
    k = 100
    full_s, full_i, _ = task.score_topk(d, k)
    parts_s, parts_i = [], []
    for r in range(4):
        lo, hi = shard_range(len(recs), r, 4)
        s, i, _ = task.score_topk(d[lo:hi], k, base_index=lo)
        parts_s.append(s)
        parts_i.append(i)
    ms, mi = E.topk_merge(torch.cat(parts_s), torch.cat(parts_i), 4, k, k)
    torch.cuda.synchronize()
    assert torch.equal(mi, full_i) and torch.equal(ms, full_s)


def test_host_buffer_path_equals_device(torch):
    E = _engine()
    task, recs = _conv_task(n=(1 << 20) + 12345, seed=5)
    ds, di, nv = task.score_topk(E.to_device_records(recs), 64)
    torch.cuda.synchronize()
    hs, hi, hnv = task.score_topk_host(recs, 64)
    assert hi.tolist() == di.cpu().tolist() and np.array_equal(hs, ds.cpu().numpy())
    assert hnv == int(nv.item()) == len(recs)


def test_edge_cases(torch):
    E = _engine()
    task, recs = _conv_task(n=10)
    d = E.to_device_records(recs)
    # k larger than n pads with (+inf, -1)
    ts, ti, nv = task.score_topk(d, 16)
    torch.cuda.synchronize()
    assert (ti[10:].cpu().numpy() == -1).all() and np.isinf(ts[10:].cpu().numpy()).all()
    assert int(nv.item()) == 10
    # empty input
    ts, ti, nv = task.score_topk(d[:0], 4)
    torch.cuda.synchronize()
    assert (ti.cpu().numpy() == -1).all() and int(nv.item()) == 0
    # all candidates failing (factor 0 -> tile range) are excluded
    bad = recs.copy()
    bad["param"][:, 0] = 0
    ts, ti, nv = task.score_topk(E.to_device_records(bad), 4)
    _, _, st = task.score(E.to_device_records(bad))
    torch.cuda.synchronize()
    assert int(nv.item()) == 0 and (st.cpu().numpy() == 2).all()


def test_es_runs_match_reference(torch):
    """optimize() with device scoring reproduces the reference's search exactly."""
    from paper_2104_14641_b200 import ir
    from paper_2104_14641_b200.es import EsParams, optimize
    runs = json.loads((GOLDEN / "es_runs.json").read_text())
    for r in runs:
        prog = ir.parse_program(json.dumps(r["program"]))
        res = optimize(prog, r["space"], arch_named(r["arch"]), EsParams(**r["params"]), launch=launch())
        assert res.best_schedule.to_json() == r["best_schedule"], r["name"]
        assert res.best_score == r["best_score"]
        assert [[k, v] for k, v in res.best_features.values] == r["best_features"]
        assert res.trace == r["trace"], r["name"]
        assert res.evaluated == r["evaluated"], r["name"]
        assert res.evaluations == r["evaluations"]


def test_score_batch_api(torch):
    from paper_2104_14641_b200 import ir
    from paper_2104_14641_b200.cost import rank_schedules
    case = next(c for c in rank_cases()["cases"] if c["program"] == "matmul8")
    prog, _ = rank_groups(case)
    scheds = [ir.Schedule.from_json(s) for s in case["schedules"]]
    res = case["results"]["x86-avx2"]
    rows, errors = rank_schedules(prog, scheds, arch_named("x86-avx2"))
    ok = [i for i, e in enumerate(res["errors"]) if e is None]
    want = sorted(ok, key=lambda i: (res["scores"][i], i))
    assert [r[0] for r in rows] == want
    assert sorted(i for i, _ in errors) == [i for i, e in enumerate(res["errors"]) if e is not None]


def _es_space(name):
    from paper_2104_14641_b200 import ir
    from paper_2104_14641_b200.pack import SpaceTemplate
    r = next(x for x in json.loads((GOLDEN / "es_runs.json").read_text()) if x["name"] == name)
    return SpaceTemplate(ir.parse_program(json.dumps(r["program"])), r["space"]), r["arch"]


@pytest.mark.parametrize("path", POINT_PATHS)
@pytest.mark.parametrize("which", ["gemm1024", "conv56", "es:conv_small"])
def test_points_equal_records(torch, which, path):
    """Points API (space-point decode on device) == records API on the same candidates."""
    E = _engine()
    from paper_2104_14641_b200 import workloads as W
    if which.startswith("es:"):
        st, arch = _es_space(which[3:])
        idx = W.distinct_indices(st.sizes, min(4096, st.size), 9)
    else:
        st, _, z = space_case(which)
        arch = "x86-avx2"
        idx = z["idx"]
    for a in (arch, "nvidia-volta"):
        task = E.Task(st.template.desc(arch_named(a), launch()), 0)
        if not _set_path(task, path):
            task.close()
            continue
        task.set_space(st.space_desc())
        if path == 3 and not which.startswith("es:"):
            assert task.points_path == 3, "tile+reorder BASELINE spaces take the space-specialised path"
        recs = st.records_from_indices(idx)
        pts = st.points_from_indices(idx)
        assert np.array_equal(st.indices_from_points(pts), idx)
        d = E.to_device_records(recs)
        task.prepare_unroll_for(d)
        s, f, stt = task.score(d)
        dp = torch.from_numpy(pts.view(np.int32) if pts.dtype == np.uint32 else pts.view(np.int64)).cuda()
        ps, pf, pst = task.score_points(dp)
        torch.cuda.synchronize()
        assert torch.equal(stt, pst)
        ok = stt == 0
        assert torch.equal(s[ok], ps[ok]) and torch.equal(f[ok], pf[ok])
        k = min(64, len(idx))
        ts, ti, nv = task.score_topk(d, k, base_index=3)
        qs, qi, qnv = task.score_topk_points(dp, k, base_index=3)
        hs, hi, hnv = task.score_topk_points_host(pts, k, base_index=3)
        torch.cuda.synchronize()
        assert torch.equal(ti, qi) and torch.equal(ts, qs) and int(nv.item()) == int(qnv.item()) == hnv
        assert hi.tolist() == ti.cpu().tolist() and np.array_equal(hs, ts.cpu().numpy())
        task.close()


def test_points_out_of_range(torch):
    E = _engine()
    st, _, z = space_case("gemm1024")
    task = E.Task(st.template.desc(arch_named("x86-avx2"), launch()), 0)
    task.set_space(st.space_desc())
    pts = np.array([0, st.size - 1, st.size, 2 ** 32 - 1], np.uint32)
    s, f, stt = task.score_points(torch.from_numpy(pts.view(np.int32)).cuda())
    torch.cuda.synchronize()
    assert stt.cpu().tolist()[2:] == [19, 19] and stt.cpu().tolist()[:2] == [0, 0]
    task.close()


@pytest.mark.parametrize("path", POINT_PATHS)
@pytest.mark.parametrize("name", ALL_SPACE_FIXTURES)
def test_space_fixtures_points_bit_exact(torch, name, path):
    """Every BASELINE space through the points API on every points path == the reference's outputs."""
    E = _engine()
    st, _, z = space_case(name)
    pts = st.points_from_indices(z["idx"])
    dp = torch.from_numpy(pts.view(np.int32) if pts.dtype == np.uint32 else pts.view(np.int64)).cuda()
    for a in z["arches"]:
        a = str(a)
        task = E.Task(st.template.desc(arch_named(a), launch()), 0)
        assert _set_path(task, path)
        task.set_space(st.space_desc())
        assert task.points_path == path
        s, f, status = task.score_points(dp)
        torch.cuda.synchronize()
        assert (status.cpu().numpy() == 0).all()
        np.testing.assert_array_equal(f.cpu().numpy(), z[f"feats_{a}"])
        np.testing.assert_array_equal(s.cpu().numpy(), z[f"scores_{a}"])
        ts, ti, nv = task.score_topk_points(dp, 64)
        want = sorted(range(len(pts)), key=lambda q: (z[f"scores_{a}"][q], q))[:64]
        assert ti.cpu().tolist() == want and int(nv.item()) == len(pts)
        task.close()


@pytest.mark.parametrize("reorder", [["i", "i_i", "j"], ["j", "i_i"], ["k", "i"], ["i", "q"]])
def test_space_path_failing_reorders(torch, reorder):
    """Reorder sets that are valid, non-contiguous (REORDER_CHAIN) or name a missing loop (NO_LOOP):
    the space-specialised path reports the same status and scores as the generic record path."""
    import itertools
    E = _engine()
    from paper_2104_14641_b200 import workloads as W
    from paper_2104_14641_b200.pack import SpaceTemplate
    prog = W.program(W.matmul_json(64))
    space = {"tile": {"i": W.divisors(64), "j": [1, 2, 8]},
             "reorder": [list(p) for p in itertools.permutations(reorder)]}
    st = SpaceTemplate(prog, space)
    idx = W.distinct_indices(st.sizes, int(st.size), 3)
    for a in ("x86-avx2", "aarch64-neon", "nvidia-volta"):
        task = E.Task(st.template.desc(arch_named(a), launch()), 0)
        task.set_space(st.space_desc())
        assert task.points_path == 3
        pts = st.points_from_indices(idx)
        dp = torch.from_numpy(pts.view(np.int32)).cuda()
        ps, pf, pst = task.score_points(dp)
        task.set_path(1)
        s, f, stt = task.score(E.to_device_records(st.records_from_indices(idx)))
        torch.cuda.synchronize()
        assert torch.equal(stt, pst)
        ok = stt == 0
        assert torch.equal(s[ok], ps[ok]) and torch.equal(f[ok], pf[ok])
        task.close()


@pytest.mark.parametrize("k", [1, 7, 64, 300, 1024])
def test_topk_selection_ties(torch, k):
    """Radix-selected block lists and merge tree under heavy score ties: equal to a stable sort."""
    E = _engine()
    st, _, z = space_case("gemm1024")
    task = E.Task(st.template.desc(arch_named("x86-avx2"), launch()), 0)
    task.set_space(st.space_desc())
    from paper_2104_14641_b200 import workloads as W
    idx = np.concatenate([W.distinct_indices(st.sizes, 200000, 5)] * 3)  # every score 3x (and more ties)
    pts = st.points_from_indices(idx)
    dp = torch.from_numpy(pts.view(np.int32)).cuda()
    s, _, _ = task.score_points(dp, features=False)
    ts, ti, nv = task.score_topk_points(dp, k, base_index=11)
    torch.cuda.synchronize()
    sc = s.cpu().numpy()
    want = np.lexsort((np.arange(len(sc)), sc))[:k]
    assert (ti.cpu().numpy() - 11).tolist() == want.tolist()
    assert np.array_equal(ts.cpu().numpy(), sc[want])
    task.close()


@pytest.mark.parametrize("n", [97, 100_003, 1 << 20])
def test_pinned_host_points_mapped(torch, n):
    """Pinned host points (read zero-copy through the mapping by the scoring kernel) == the
    device-resident call: identical top-k and valid count, repeatedly (cached staging reuse)."""
    E = _engine()
    from paper_2104_14641_b200 import workloads as W
    from paper_2104_14641_b200.pack import SpaceTemplate
    st = SpaceTemplate(W.program(W.conv2d_json()), W.conv_space(4096, 1))
    from paper_2104_14641_b200.arch import KernelLaunch, load_arch
    task = E.Task(st.template.desc(load_arch("x86-avx2"), KernelLaunch.from_json(W.KERNEL_LAUNCH)), 0)
    task.set_space(st.space_desc())
    assert task.points_path == 3
    pts = st.points_from_indices(W.distinct_indices(st.sizes, n, 31))
    dev = torch.from_numpy(pts.view(np.int32)).cuda()
    pin = torch.from_numpy(pts.view(np.int32)).pin_memory()
    ds, di, dn = task.score_topk_points(dev, 64, base_index=5)
    torch.cuda.synchronize()
    for _ in range(3):
        hs, hi, hn = task.score_topk_points_host(pin, 64, base_index=5)
        assert hi.tolist() == di.cpu().tolist() and np.array_equal(hs, ds.cpu().numpy()) and hn == int(dn.item())
    task.close()


@pytest.mark.gpu
def test_topk_workspace_reuse_across_layouts(torch):
    """One task, one cached workspace: calls alternating k, n (two-stage merge vs merge tree)
    and the records / points entry points each equal a stable sort (self-resetting counters,
    minima slots and published bound survive every layout change)."""
    E = _engine()
    from paper_2104_14641_b200 import workloads as W
    from paper_2104_14641_b200.pack import SpaceTemplate
    st = SpaceTemplate(W.program(W.conv2d_json()), W.conv_space(4096, 1))
    task = E.Task(st.template.desc(arch_named("x86-avx2"), launch()), 0)
    task.set_space(st.space_desc())
    pts_all = st.points_from_indices(W.distinct_indices(st.sizes, 1 << 20, 17))
    for n, k in [(1 << 20, 64), (5000, 16), (1 << 20, 1), (300_000, 200), (1 << 20, 64), (1 << 19, 1024),
                 (77, 5), (1 << 20, 111), (100_003, 97), (1 << 20, 64)]:  # k ~ grid/4: > 256 survivors
        dp = torch.from_numpy(pts_all[:n].view(np.int32)).cuda()
        s, _, stt = task.score_points(dp, features=False)
        ts, ti, nv = task.score_topk_points(dp, k, base_index=3)
        torch.cuda.synchronize()
        sc, ok = s.cpu().numpy(), stt.cpu().numpy() == 0
        ids = np.flatnonzero(ok)
        want = ids[np.lexsort((ids, sc[ids]))][:k]
        assert (ti.cpu().numpy()[:len(want)] - 3).tolist() == want.tolist(), (n, k)
        assert np.array_equal(ts.cpu().numpy()[:len(want)], sc[want]), (n, k)
        assert int(nv.item()) == int(ok.sum())
    task.close()


def test_topk_two_stage_many_survivors(torch):
    """Points ordered by score put a block's whole buffer under the merge bound (hundreds of
    survivors: the streamed merge path of merge_filter_kernel); still equal to a stable sort."""
    E = _engine()
    from paper_2104_14641_b200 import workloads as W
    from paper_2104_14641_b200.pack import SpaceTemplate
    st = SpaceTemplate(W.program(W.conv2d_json()), W.conv_space(4096, 1))
    task = E.Task(st.template.desc(arch_named("x86-avx2"), launch()), 0)
    task.set_space(st.space_desc())
    pts = st.points_from_indices(W.distinct_indices(st.sizes, 1 << 20, 23))
    dp = torch.from_numpy(pts.view(np.int32)).cuda()
    s, _, stt = task.score_points(dp, features=False)
    sc, ok = s.cpu().numpy(), stt.cpu().numpy() == 0
    order = np.lexsort((np.arange(len(sc)), np.where(ok, sc, np.inf)))  # best first, failures last
    dq = torch.from_numpy(pts[order].view(np.int32)).cuda()
    for k in (64, 111):
        ts, ti, nv = task.score_topk_points(dq, k)
        torch.cuda.synchronize()
        assert ti.cpu().tolist() == list(range(k))
        assert np.array_equal(ts.cpu().numpy(), sc[order[:k]])
        assert int(nv.item()) == int(ok.sum())
    task.close()


@pytest.mark.parametrize("mode", ["bound", "tree"])
def test_topk_merge_modes_forced(mode):
    """The bound merge ranked by the scoring grid's last block (forced even where blocks end
    before the bound is out: the last block filters the lists left) and the in-kernel merge tree
    (forced for small k), at several (n, k): each equals a stable sort."""
    import os
    import subprocess
    import sys
    from pathlib import Path
    env = dict(os.environ, LS_MERGE=mode)
    r = subprocess.run([sys.executable, str(Path(__file__).with_name("merge_modes_check.py"))], env=env,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr


@pytest.mark.parametrize("n", [1, 97, 100_003, 1 << 20])
def test_points_3byte_equal_4byte(torch, n):
    """Packed 3-byte points (pack.pack_points) score and rank exactly like 4-byte points: device
    buffers (score + top-k) and pinned host buffers (results written by the kernel into pinned
    host memory)."""
    E = _engine()
    from paper_2104_14641_b200 import workloads as W
    from paper_2104_14641_b200.arch import KernelLaunch, load_arch
    from paper_2104_14641_b200.pack import SpaceTemplate, pack_points
    st = SpaceTemplate(W.program(W.conv2d_json()), W.conv_space(4096, 1))
    task = E.Task(st.template.desc(load_arch("x86-avx2"), KernelLaunch.from_json(W.KERNEL_LAUNCH)), 0)
    task.set_space(st.space_desc())
    pts = st.points_from_indices(W.distinct_indices(st.sizes, n, 53))
    d4 = torch.from_numpy(pts.view(np.int32)).cuda()
    p3 = pack_points(pts, 3)
    d3 = torch.from_numpy(p3).cuda()
    s4, _, st4 = task.score_points(d4, features=False)
    s3, _, st3 = task.score_points(d3, features=False)
    torch.cuda.synchronize()
    assert np.array_equal(s3.cpu().numpy(), s4.cpu().numpy(), equal_nan=True)
    assert np.array_equal(st3.cpu().numpy(), st4.cpu().numpy())
    k = min(64, n)
    a = task.score_topk_points(d4, k, base_index=9)
    b = task.score_topk_points(d3, k, base_index=9)
    torch.cuda.synchronize()
    assert a[1].cpu().tolist() == b[1].cpu().tolist() and int(a[2].item()) == int(b[2].item())
    pin = torch.from_numpy(p3).pin_memory()
    for _ in range(2):
        hs, hi, hn = task.score_topk_points_host(pin, k, base_index=9)
        assert hi.tolist() == a[1].cpu().tolist() and hn == int(a[2].item())
        assert np.array_equal(hs, a[0].cpu().numpy())
    hs, hi, hn = task.score_topk_points_host(p3, k, base_index=9)  # pageable: staged copies
    assert hi.tolist() == a[1].cpu().tolist() and hn == int(a[2].item())
    task.close()


@pytest.mark.parametrize("path", ["staged"])
def test_host_points_paths_forced(path):
    """The host-buffer points call through the staged-copy path (LS_HOST_PATH forces it for
    pinned buffers too) returns the device call's top-k for 3- and 4-byte points."""
    import os
    import subprocess
    import sys
    from pathlib import Path
    env = dict(os.environ, LS_HOST_PATH=path)
    r = subprocess.run([sys.executable, str(Path(__file__).with_name("host_paths_check.py"))], env=env,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr


def test_host_points_default_paths():
    """Default host paths (pinned: mapped zero-copy with block-cooperative aligned loads; pageable:
    staged copies) == the device call."""
    import subprocess
    import sys
    from pathlib import Path
    r = subprocess.run([sys.executable, str(Path(__file__).with_name("host_paths_check.py"))],
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
