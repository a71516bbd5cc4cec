"""Multi-GPU sharding: one process per GPU, torch.distributed (NCCL) as plumbing.

Scoring.  Candidates are pure functions of (task, record)
(SPEC.md:448-449), so rank r scores the contiguous global range
[r*n/G, (r+1)*n/G) with its own fused score+top-k kernel; the only exchange is
ONE all-gather of k packed 16-byte keys per rank (ls_topk_key: order-preserving
score bits + global index, include/loopscout_b200.h), merged on every rank by the
library's merge kernel.  (score, global index) is a total order, so the merged
list equals the single-GPU list (the reference's cmd_rank order,
ls/cli.py:124-126) for any G.

ES (ls/es.py:130-204).  The population is sharded by member; the F keys and
the fixed-chunk partial sums are all-gathered in place between the device
stages (ls_es_step), so theta is bit-identical for any G (engine.EsRun).

Under the gloo backend (CPU tests, or a host without NCCL) the exchanged bytes
are staged through host memory; the merge still runs in the library.
"""

from __future__ import annotations


def shard_range(n: int, rank: int, world: int) -> tuple:
    return n * rank // world, n * (rank + 1) // world


_BUFS: dict = {}


def _buffers(torch, k: int, world: int, device):
    """Preallocated per (k, world, device): gathered keys [world*k,2] and the merged outputs."""
    key = (k, world, str(device))
    b = _BUFS.get(key)
    if b is None:
        b = (torch.empty((world * k, 2), dtype=torch.int64, device=device),
             torch.empty(k, dtype=torch.float64, device=device),
             torch.empty(k, dtype=torch.int64, device=device))
        _BUFS[key] = b
    return b


def all_gather_inplace(full, per_rank: int, group=None):
    """In-place all-gather of rank slices full[r*per_rank:(r+1)*per_rank] (any 1-D/2-D tensor)."""
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    if world == 1:
        return full
    mine = full[rank * per_rank:(rank + 1) * per_rank]
    if dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(full, mine, group=group)  # in place: NCCL send = recv + r * count
        return full
    host = mine.cpu()
    parts = [host.clone() for _ in range(world)]
    dist.all_gather(parts, host, group=group)
    for r, p in enumerate(parts):
        if r != rank:
            full[r * per_rank:(r + 1) * per_rank].copy_(p.to(full.device))
    return full


def gather_topk(local_scores, local_index, k: int, group=None, stream=None):
    """All-gather every rank's k-list as packed keys and merge to the global k best (identical on
    every rank).  Returns preallocated (scores, index) tensors, overwritten by the next call with
    the same (k, world, device)."""
    import torch
    import torch.distributed as dist

    from .engine import topk_merge_keys, topk_to_keys

    world = dist.get_world_size(group)
    if world == 1:
        return local_scores, local_index
    rank = dist.get_rank(group)
    full, out_s, out_i = _buffers(torch, k, world, local_scores.device)
    topk_to_keys(local_scores, local_index, full[rank * k:(rank + 1) * k], stream=stream)
    all_gather_inplace(full, k, group)
    return topk_merge_keys(full, k, out=(out_s, out_i), stream=stream)


def sharded_score_topk(task, d_records_local, k: int, base_index: int, group=None, stream=None):
    """Fused local score+top-k on this rank's shard, then the cross-rank merge."""
    s, i, nv = task.score_topk(d_records_local, k, base_index=base_index, stream=stream)
    gs, gi = gather_topk(s, i, k, group=group, stream=stream)
    return gs, gi, nv


def es_exchange(group=None):
    """The exchange callable of engine.EsRun.run_sharded over torch.distributed."""
    return lambda full, per_rank: all_gather_inplace(full, per_rank, group)


def es_merge_results(trace, evaluations_pts, evaluations_scores, err: int, best: float, group=None):
    """Whole-search results of a sharded device ES from every rank's local ones: the trace is the
    per-generation minimum over ranks, the evaluated set the union of the ranks' distinct lists
    (first rank first), the failure the earliest (generation, member), the best the minimum."""
    import numpy as np
    import torch.distributed as dist

    if dist.get_world_size(group) == 1:
        return trace, evaluations_pts, evaluations_scores, err, best
    got = [None] * dist.get_world_size(group)
    dist.all_gather_object(got, (np.asarray(trace), np.asarray(evaluations_pts), np.asarray(evaluations_scores),
                                 int(err), float(best)), group=group)
    trace = np.minimum.reduce([g[0] for g in got])
    pts = np.concatenate([g[1] for g in got])
    sc = np.concatenate([g[2] for g in got])
    _, first = np.unique(pts, return_index=True)
    first.sort()
    errs = [g[3] for g in got if g[3]]
    return trace, pts[first], sc[first], (min(errs) if errs else 0), min(g[4] for g in got)
