"""Multi-GPU sharding: contiguous candidate ranges per rank, one all-gather of top-k lists.

Candidates are pure functions of (task, record), so rank r
scores the contiguous global range [r*n/G, (r+1)*n/G) with its own fused
score+top-k kernel; the only exchange is one all-gather of k (score, index)
pairs per rank, merged by the library's merge kernel.  Because the key
(score, global index) is a total order, the merged list equals the
single-GPU list for any G.
"""

from __future__ import annotations


def shard_range(n: int, rank: int, world: int) -> tuple:
    return n * rank // world, n * (rank + 1) // world


def gather_topk(local_scores, local_index, k: int, merge=None, group=None):
    """All-gather every rank's k-list and merge to the global k best (identical on all ranks)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    if world == 1:
        return local_scores, local_index
    gs = torch.empty(world * k, dtype=local_scores.dtype, device=local_scores.device)
    gi = torch.empty(world * k, dtype=local_index.dtype, device=local_index.device)
    dist.all_gather_into_tensor(gs, local_scores.contiguous(), group=group)
    dist.all_gather_into_tensor(gi, local_index.contiguous(), group=group)
    if merge is None:
        from .engine import topk_merge as merge
    return merge(gs, gi, world, k, k)


def sharded_score_topk(task, d_records_local, k: int, base_index: int, group=None, stream=None):
    """Fused local score+top-k on this rank's shard, then the cross-rank merge."""
    s, i, nv = task.score_topk(d_records_local, k, base_index=base_index, stream=stream)
    gs, gi = gather_topk(s, i, k, group=group)
    return gs, gi, nv
