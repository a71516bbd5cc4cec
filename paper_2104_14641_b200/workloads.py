"""Synthetic workloads of BASELINE.json's configs.

Programs are built as canonical program JSON (parse_program) and schedule
spaces as space dicts (space_axes).  Candidate lists are drawn with numpy
seeds as per-axis choice indices, so a batch is a pure function of
(config, n, seed) and the same indices give the reference's own schedules
through ``SpaceTemplate.schedule_of``.
"""

from __future__ import annotations

import itertools
import json

import numpy as np

from .ir import parse_program


def _acc(t, kind, idx):
    return {"access": {"tensor": t, "kind": kind, "idx": list(idx)}}


def _nest(loops, body):
    for var, ext in reversed(loops):
        body = [{"loop": {"var": var, "extent": ext, "body": body}}]
    return body


def divisors(n: int) -> list:
    return [d for d in range(1, n + 1) if n % d == 0]


def matmul_json(m: int, n: int | None = None, k: int | None = None) -> dict:
    """C[i,j] += A[i,k] * B[k,j] over i<m, j<n, k<k (tests/helpers.py:47-56 shape)."""
    n = m if n is None else n
    k = m if k is None else k
    return {"tensors": [{"name": "A", "dims": [m, k]}, {"name": "B", "dims": [k, n]},
                        {"name": "C", "dims": [m, n]}],
            "body": _nest([("i", m), ("j", n), ("k", k)],
                          [_acc("A", "load", ["i", "k"]), _acc("B", "load", ["k", "j"]),
                           _acc("C", "load", ["i", "j"]), _acc("C", "store", ["i", "j"])])}


def batch_matmul_json(b: int, m: int, n: int, k: int) -> dict:
    return {"tensors": [{"name": "A", "dims": [b, m, k]}, {"name": "B", "dims": [b, k, n]},
                        {"name": "C", "dims": [b, m, n]}],
            "body": _nest([("b", b), ("i", m), ("j", n), ("k", k)],
                          [_acc("A", "load", ["b", "i", "k"]), _acc("B", "load", ["b", "k", "j"]),
                           _acc("C", "load", ["b", "i", "j"]), _acc("C", "store", ["b", "i", "j"])])}


def conv2d_json(n=1, oc=64, oh=56, ow=56, ic=64, kh=3, kw=3, stride=1) -> dict:
    """NCHW conv2d on a pre-padded input: O[n,oc,oh,ow] += I[n,ic,s*oh+kh,s*ow+kw] * W[oc,ic,kh,kw]."""
    s = "" if stride == 1 else f"{stride}*"
    ih, iw = stride * (oh - 1) + kh, stride * (ow - 1) + kw
    return {"tensors": [{"name": "I", "dims": [n, ic, ih, iw]}, {"name": "W", "dims": [oc, ic, kh, kw]},
                        {"name": "O", "dims": [n, oc, oh, ow]}],
            "body": _nest([("n", n), ("oc", oc), ("oh", oh), ("ow", ow), ("ic", ic), ("kh", kh), ("kw", kw)],
                          [_acc("I", "load", ["n", "ic", f"{s}oh + kh", f"{s}ow + kw"]),
                           _acc("W", "load", ["oc", "ic", "kh", "kw"]),
                           _acc("O", "load", ["n", "oc", "oh", "ow"]),
                           _acc("O", "store", ["n", "oc", "oh", "ow"])])}


def program(spec: dict):
    return parse_program(json.dumps(spec))


def tiled_chain(loop_order: list, tiled: list) -> list:
    """Loop names of the chain after tiling `tiled` loops in sorted order (each `v` -> v, v_i)."""
    out = []
    for v in loop_order:
        out.append(v)
        if v in tiled:
            out.append(v + "_i")
    return out


def random_perms(names: list, count: int, seed: int) -> list:
    rng = np.random.default_rng(seed)
    seen, out = set(), []
    while len(out) < count:
        p = tuple(names[i] for i in rng.permutation(len(names)))
        if p not in seen:
            seen.add(p)
            out.append(list(p))
    return out


def gemm_space(n: int = 1024) -> dict:
    """Config 1: tile i/j/k by any divisor + any of the 720 chain orders."""
    chain = tiled_chain(["i", "j", "k"], ["i", "j", "k"])
    return {"tile": {v: divisors(n) for v in "ijk"},
            "reorder": [list(p) for p in itertools.permutations(chain)]}


def conv_space(reorders: int = 512, seed: int = 1, shape: dict | None = None) -> dict:
    """Config 2: tile ic/oc/oh/ow by divisors + `reorders` random 11-loop chain orders."""
    sh = dict(n=1, oc=64, oh=56, ow=56, ic=64, kh=3, kw=3)
    sh.update(shape or {})
    chain = tiled_chain(["n", "oc", "oh", "ow", "ic", "kh", "kw"], ["ic", "oc", "oh", "ow"])
    return {"tile": {"ic": divisors(sh["ic"]), "oc": divisors(sh["oc"]),
                     "oh": divisors(sh["oh"]), "ow": divisors(sh["ow"])},
            "reorder": random_perms(chain, reorders, seed)}


def distinct_indices(sizes, n: int, seed: int, start: int = 0) -> np.ndarray:
    """Rows start..start+n-1 of a seeded enumeration of distinct points of a
    mixed-radix space (per-axis choice indices).  Disjoint `start` ranges give
    disjoint points, so shards can be generated independently."""
    sizes = np.asarray(sizes, np.int64)
    total = int(np.prod(sizes))
    if start + n > total:
        raise ValueError(f"space has {total} points, asked for rows up to {start + n}")
    flat = _feistel(total, np.arange(start, start + n, dtype=np.int64), seed)
    out = np.empty((n, len(sizes)), np.int64)
    for a in range(len(sizes) - 1, -1, -1):
        out[:, a] = flat % sizes[a]
        flat = flat // sizes[a]
    return out


def _feistel(total: int, x: np.ndarray, seed: int) -> np.ndarray:
    """A keyed bijection of [0, total) (balanced Feistel on 2^b, cycle-walked)."""
    bits = max(2, int(total - 1).bit_length())
    bits += bits & 1
    half = bits // 2
    mask = np.int64((1 << half) - 1)
    keys = np.random.default_rng(seed).integers(1, 1 << 31, size=4, dtype=np.int64)

    def perm(v):
        l, r = v >> half, v & mask
        for k in keys:
            f = ((r * np.int64(0x9E3779B1) + k) ^ (r >> 3)) & mask
            l, r = r, l ^ f
        return (l << half) | r

    y = perm(x)
    while True:
        bad = y >= total
        if not bad.any():
            return y
        y[bad] = perm(y[bad])


KERNEL_LAUNCH = {"grid_blocks": 160, "threads_per_block": 256, "registers_per_thread": 32,
                 "shared_mem_per_block": 4096}


def bert_tasks(reorders: int = 720) -> list:
    """Config 4: BERT-base (seq 128, batch 8 -> M = 1024 tokens) dense + batch_matmul tasks
    (SURVEY.md §8d1 (4)): (name, program spec, space) with divisor tiles and chain orders."""
    out = []
    for (m, n, k) in ((1024, 768, 768), (1024, 3072, 768), (1024, 768, 3072)):
        chain = tiled_chain(["i", "j", "k"], ["i", "j", "k"])
        perms = [list(p) for p in itertools.permutations(chain)][:reorders]
        out.append((f"dense_{m}_{n}_{k}", matmul_json(m, n, k),
                    {"tile": {"i": divisors(m), "j": divisors(n), "k": divisors(k)}, "reorder": perms}))
    for (b, m, n, k) in ((96, 128, 128, 64), (96, 128, 64, 128)):
        chain = tiled_chain(["b", "i", "j", "k"], ["i", "j", "k"])
        out.append((f"bmm_{b}_{m}_{n}_{k}", batch_matmul_json(b, m, n, k),
                    {"tile": {"i": divisors(m), "j": divisors(n), "k": divisors(k)},
                     "reorder": random_perms(chain, reorders, 10)}))
    return out


def resnet50_tasks(reorders: int = 512) -> list:
    """Config 3: the distinct conv2d / dense layers of ResNet-50 v1.5 at batch 1 (torchvision
    layout: stride on the 3x3 of each bottleneck, 1x1/2 downsamples), SURVEY.md §8d1 (3).
    (name, program spec, space): tile oc/oh/ow/ic by divisors + `reorders` 11-loop orders;
    the dense layer tiles j/k by divisors + every 6-loop order."""
    layers = [("conv1", dict(oc=64, oh=112, ow=112, ic=3, kh=7, kw=7, stride=2))]
    ch_in, hw = 64, 56
    for stage, (width, blocks) in enumerate(((64, 3), (128, 4), (256, 6), (512, 3))):
        out_ch = width * 4
        down = 1 if stage == 0 else 2
        in_hw = hw if stage == 0 else hw * 2
        layers += [(f"s{stage}_reduce_a", dict(oc=width, oh=in_hw, ow=in_hw, ic=ch_in, kh=1, kw=1)),
                   (f"s{stage}_conv3_a", dict(oc=width, oh=hw, ow=hw, ic=width, kh=3, kw=3, stride=down)),
                   (f"s{stage}_expand", dict(oc=out_ch, oh=hw, ow=hw, ic=width, kh=1, kw=1)),
                   (f"s{stage}_downsample", dict(oc=out_ch, oh=hw, ow=hw, ic=ch_in, kh=1, kw=1, stride=down))]
        if blocks > 1:
            layers += [(f"s{stage}_reduce_b", dict(oc=width, oh=hw, ow=hw, ic=out_ch, kh=1, kw=1))]
            if stage > 0:
                layers += [(f"s{stage}_conv3_b", dict(oc=width, oh=hw, ow=hw, ic=width, kh=3, kw=3))]
        ch_in, hw = out_ch, max(7, hw // 2)
    out = []
    chain = tiled_chain(["n", "oc", "oh", "ow", "ic", "kh", "kw"], ["ic", "oc", "oh", "ow"])
    for i, (name, sh) in enumerate(layers):
        spec = conv2d_json(n=1, **sh)
        space = {"tile": {v: divisors(sh[v]) for v in ("ic", "oc", "oh", "ow")},
                 "reorder": random_perms(chain, reorders, 100 + i)}
        out.append((name, spec, space))
    dchain = tiled_chain(["i", "j", "k"], ["j", "k"])
    out.append(("fc1000", matmul_json(1, 1000, 2048),
                {"tile": {"j": divisors(1000), "k": divisors(2048)},
                 "reorder": [list(p) for p in itertools.permutations(dchain)]}))
    return out
