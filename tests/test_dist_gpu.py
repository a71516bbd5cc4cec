"""Multi-rank paths on the device: sharded fused top-k + the packed-key all-gather
merge, and the sharded device ES, against the single-rank answers.

This build has one GPU, so the ranks share cuda:0: real processes over torch.distributed (gloo
transport, the device kernels and the library merge on the GPU), and "virtual" shards of one
ES run driven stage by stage in one process with the exchange done by device copies."""

import os
import sys
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent


def _conv_task(reorders=512):
    from paper_2104_14641_b200 import workloads as W
    from paper_2104_14641_b200.arch import KernelLaunch, load_arch
    from paper_2104_14641_b200.engine import Task
    from paper_2104_14641_b200.pack import SpaceTemplate
    st = SpaceTemplate(W.program(W.conv2d_json()), W.conv_space(reorders, 1))
    task = Task(st.template.desc(load_arch("x86-avx2"), KernelLaunch.from_json(W.KERNEL_LAUNCH)), 0)
    task.set_space(st.space_desc())
    return st, task


def _topk_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    sys.path.insert(0, str(ROOT))
    try:
        dist.init_process_group("gloo", rank=rank, world_size=world)
        torch.cuda.set_device(0)
        from paper_2104_14641_b200 import workloads as W
        from paper_2104_14641_b200.dist import gather_topk, shard_range
        st, task = _conv_task()
        n = 300_001
        pts = st.points_from_indices(W.distinct_indices(st.sizes, n, 77))
        out = []
        for k in (1, 64, 300):
            lo, hi = shard_range(n, rank, world)
            d = torch.from_numpy(pts[lo:hi].view(np.int32)).cuda()
            s, i, _ = task.score_topk_points(d, k, base_index=lo)
            gs, gi = gather_topk(s, i, k)
            out.append((k, gs.cpu().numpy().copy(), gi.cpu().numpy().copy()))
        task.close()
        q.put((rank, out))
        dist.destroy_process_group()
    except Exception as e:  # noqa: BLE001
        q.put((rank, repr(e)))


def _spawn(world, target):
    import multiprocessing as mp
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=target, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=400) for _ in ps)
    for p in ps:
        p.join(60)
    return res


@pytest.mark.parametrize("world", [2, 4])
def test_sharded_topk_merge_equals_single(world):
    """world processes score disjoint shards with the fused kernel, gather packed keys and merge with
    the library kernel: every rank holds the single-GPU top-k (scores and indices bit-identical)."""
    import torch
    from paper_2104_14641_b200 import workloads as W
    res = _spawn(world, _topk_worker)
    st, task = _conv_task()
    pts = st.points_from_indices(W.distinct_indices(st.sizes, 300_001, 77))
    d = torch.from_numpy(pts.view(np.int32)).cuda()
    for r in range(world):
        assert not isinstance(res[r], str), res[r]
        for k, gs, gi in res[r]:
            s, i, _ = task.score_topk_points(d, k)
            torch.cuda.synchronize()
            assert gi.tolist() == i.cpu().tolist(), (world, r, k)
            assert np.array_equal(gs, s.cpu().numpy()), (world, r, k)
    task.close()


def test_topk_merge_keys_matches_lists():
    """ls_topk_to_keys + ls_topk_merge_keys == ls_topk_merge == a stable sort, empty slots skipped."""
    import torch
    from paper_2104_14641_b200.engine import topk_merge, topk_merge_keys, topk_to_keys
    rng = np.random.default_rng(3)
    m, k = 8 * 300, 300
    s = np.round(rng.normal(size=m), 2)  # many ties
    i = rng.permutation(10 * m)[:m].astype(np.int64)
    i[::7] = -1  # empty slots
    ds, di = torch.from_numpy(s).cuda(), torch.from_numpy(i).cuda()
    keys = topk_to_keys(ds, di, torch.empty((m, 2), dtype=torch.int64, device="cuda"))
    ks, ki = topk_merge_keys(keys, k)
    ls, li = topk_merge(ds, di, 8, 300, k)
    torch.cuda.synchronize()
    ok = i >= 0
    want = np.lexsort((i[ok], s[ok]))[:k]
    assert ki.cpu().tolist() == i[ok][want].tolist() == li.cpu().tolist()
    assert np.array_equal(ks.cpu().numpy(), s[ok][want]) and np.array_equal(ls.cpu().numpy(), s[ok][want])


def _run_virtual(task, st, G, pop, iters, sigma, seed):
    """G shards of one ES run on this GPU, stage by stage, the all-gathers done by device copies."""
    import torch
    from paper_2104_14641_b200.engine import EsRun
    runs = [EsRun(task, 0.05, sigma, pop, iters, seed, rank=r, world=G) for r in range(G)]
    bufs = [r.shard_buffers() for r in runs]

    def exchange(which):
        per = bufs[0][2] if which == 0 else bufs[0][3]
        for q in range(G):
            for r in range(G):
                if r != q:
                    bufs[q][which][r * per:(r + 1) * per].copy_(bufs[r][which][r * per:(r + 1) * per])

    for r in runs:
        r.begin()
    for _ in range(iters):
        for r in runs:
            r.step(0)
        exchange(0)
        for r in runs:
            r.step(1)
        exchange(1)
        for r in runs:
            r.step(2)
    torch.cuda.synchronize()
    out = [r.result(st.dim) for r in runs]
    ev = [r.evaluated() for r in runs]
    for r in runs:
        r.close()
    return out, ev


@pytest.mark.parametrize("G", [2, 4, 8])
def test_es_sharded_bit_identical(G):
    """theta history bit-identical to the one-rank graph run for G shards; trace = per-generation
    minimum over shards; the union of the shards' distinct schedules = the one-rank evaluated set,
    with identical scores."""
    import torch
    from paper_2104_14641_b200.engine import EsRun
    st, task = _conv_task(64)
    pop, iters, sigma, seed = 1 << 14, 6, 2.0, 11
    one = EsRun(task, 0.05, sigma, pop, iters, seed)
    one.run()
    torch.cuda.synchronize()
    h1, t1, e1, err1, b1 = one.result(st.dim)
    p1, s1 = one.evaluated()
    one.close()
    assert err1 == 0
    out, ev = _run_virtual(task, st, G, pop, iters, sigma, seed)
    for h, t, e, err, b in out:
        assert err == 0
        assert np.array_equal(h, h1)  # bit-identical theta trajectory on every shard
    assert np.array_equal(np.minimum.reduce([o[1] for o in out]), t1)
    assert min(o[4] for o in out) == b1
    union = {}
    for pts, sc in ev:
        for p, s in zip(pts.tolist(), sc.tolist()):
            assert union.setdefault(p, s) == s
    assert union == dict(zip(p1.tolist(), s1.tolist())) and len(union) == e1
    task.close()


def _es_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    sys.path.insert(0, str(ROOT))
    try:
        dist.init_process_group("gloo", rank=rank, world_size=world)
        torch.cuda.set_device(0)
        from paper_2104_14641_b200 import workloads as W
        from paper_2104_14641_b200.arch import load_arch, KernelLaunch
        from paper_2104_14641_b200.es import EsParams, optimize_device
        r = optimize_device(W.program(W.conv2d_json()), W.conv_space(64, 1), load_arch("x86-avx2"),
                            EsParams(population=1 << 12, iterations=5, sigma=2.0, seed=4),
                            launch=KernelLaunch.from_json(W.KERNEL_LAUNCH))
        q.put((rank, (r.best_schedule.to_json(), r.best_score, r.trace, r.evaluations, r.evaluated)))
        dist.destroy_process_group()
    except Exception as e:  # noqa: BLE001
        q.put((rank, repr(e)))


def test_es_optimize_device_distributed_equals_single():
    """optimize_device under torch.distributed (2 ranks, population sharded) == one rank."""
    from paper_2104_14641_b200 import workloads as W
    from paper_2104_14641_b200.arch import load_arch, KernelLaunch
    from paper_2104_14641_b200.es import EsParams, optimize_device
    res = _spawn(2, _es_worker)
    r = optimize_device(W.program(W.conv2d_json()), W.conv_space(64, 1), load_arch("x86-avx2"),
                        EsParams(population=1 << 12, iterations=5, sigma=2.0, seed=4),
                        launch=KernelLaunch.from_json(W.KERNEL_LAUNCH))
    want = (r.best_schedule.to_json(), r.best_score, r.trace, r.evaluations, r.evaluated)
    for rank in range(2):
        assert not isinstance(res[rank], str), res[rank]
        assert res[rank] == want


def test_two_devices_in_one_process():
    """Per-device kernel attributes: tasks on device 1 after device 0 (skipped with one GPU)."""
    import torch
    if torch.cuda.device_count() < 2:
        pytest.skip("one GPU visible")
    from paper_2104_14641_b200 import workloads as W
    from paper_2104_14641_b200.arch import KernelLaunch, load_arch
    from paper_2104_14641_b200.engine import Task
    from paper_2104_14641_b200.pack import SpaceTemplate
    st = SpaceTemplate(W.program(W.conv2d_json()), W.conv_space(512, 1))
    pts = st.points_from_indices(W.distinct_indices(st.sizes, 200_000, 5))
    res = []
    for dev in (0, 1):
        task = Task(st.template.desc(load_arch("x86-avx2"), KernelLaunch.from_json(W.KERNEL_LAUNCH)), dev)
        task.set_space(st.space_desc())
        task.set_path(2)  # the tabulated kernels use the most dynamic shared memory
        d = torch.from_numpy(pts.view(np.int32)).to(f"cuda:{dev}")
        s, i, _ = task.score_topk_points(d, 64)
        torch.cuda.synchronize(dev)
        res.append((s.cpu().numpy(), i.cpu().numpy()))
        task.close()
    assert np.array_equal(res[0][0], res[1][0]) and np.array_equal(res[0][1], res[1][1])


@pytest.mark.gpu
def test_topk_allgather_merge_nccl_single_rank():
    """ls_topk_allgather_merge over a real NCCL communicator (one rank: the all-gather is the
    local copy) == the rank's own k best; the library binds ncclAllGather from the process's
    libnccl.so.2 (torch's)."""
    import ctypes
    import glob
    import os

    import torch

    from paper_2104_14641_b200 import engine as E
    nccl = None
    cands = ["libnccl.so.2"] + glob.glob(os.path.join(os.path.dirname(torch.__file__), "..", "nvidia", "nccl", "lib",
                                                      "libnccl.so*"))
    for name in cands:
        try:
            nccl = ctypes.CDLL(name, mode=ctypes.RTLD_GLOBAL)
            break
        except OSError:
            continue
    if nccl is None:
        pytest.skip("no libnccl.so.2 in this process")
    torch.cuda.init()
    comm = ctypes.c_void_p()
    devs = (ctypes.c_int * 1)(0)
    assert nccl.ncclCommInitAll(ctypes.byref(comm), 1, devs) == 0
    k = 64
    s = torch.sort(torch.rand(k, dtype=torch.float64, device="cuda")).values
    i = torch.arange(100, 100 + k, dtype=torch.int64, device="cuda")
    out_s, out_i = E.topk_allgather_merge(comm.value, 0, 1, s, i, k)
    torch.cuda.synchronize()
    assert torch.equal(out_s, s) and torch.equal(out_i, i)
    nccl.ncclCommDestroy(comm)
