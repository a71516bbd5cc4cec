"""General trees on the device: imperfect nests, sibling loops, accesses at any
level, top-level accesses, deep nests (PTX counter wrap) under Tile / Reorder / Parallel schedules,
bit-exact against the reference's own outputs (tests/golden/tree_rank.json, trees.json)."""

import json

import numpy as np
import pytest

from golden_util import GOLDEN, arch_named, launch, status_of_error

pytestmark = pytest.mark.gpu

TREE_RANK = json.loads((GOLDEN / "tree_rank.json").read_text())
TREE_INLINE = json.loads((GOLDEN / "tree_inline.json").read_text())
TREES = json.loads((GOLDEN / "trees.json").read_text())


@pytest.fixture(scope="module")
def torch():
    import torch as t
    return t


CASES = [(TREE_RANK, c) for c in TREE_RANK["cases"]] + [(TREE_INLINE, c) for c in TREE_INLINE["cases"]]


@pytest.mark.parametrize("fx,case", CASES, ids=[("inline-" if f is TREE_INLINE else "") + c["program"] for f, c in CASES])
def test_scheduled_trees_match_reference(torch, fx, case):
    """Tile / Reorder / Parallel (tree_rank) and + Unroll / Vectorize with unrolled base loops
    (tree_inline: the emission replay + device list scheduler)."""
    from paper_2104_14641_b200 import ir
    from paper_2104_14641_b200.cost import score_batch
    prog = ir.parse_program(json.dumps(fx["programs"][case["program"]]))
    scheds = [ir.Schedule.from_json(s) for s in case["schedules"]]
    for a, res in case["results"].items():
        out = score_batch(prog, scheds, arch_named(a), launch())
        want_st = np.array([status_of_error(e) for e in res["errors"]])
        assert np.array_equal(out.status, want_st), (a, np.nonzero(out.status != want_st)[0][:5])
        ok = want_st == 0
        assert np.array_equal(out.scores[ok], np.array(res["scores"], dtype=float)[ok]), a
        want_f = np.array([f for f, o in zip(res["features"], ok) if o])
        assert np.array_equal(out.features[ok], want_f), a


@pytest.mark.parametrize("name", list(TREES))
def test_unscheduled_trees_match_reference(torch, name):
    from paper_2104_14641_b200 import ir
    from paper_2104_14641_b200.cost import score_batch
    t = TREES[name]
    prog = ir.parse_program(json.dumps(t["program"]))
    for a, feats in t["features"].items():
        out = score_batch(prog, [ir.Schedule(())], arch_named(a), launch())
        assert out.status[0] == 0
        assert out.features[0].tolist() == [v for _, v in feats], a
        assert out.scores[0] == t["scores"][a]


def test_tree_topk_and_points(torch):
    """Fused top-k and the points API on a tree task (the 2MM nest)."""
    from paper_2104_14641_b200 import ir, engine as E
    from paper_2104_14641_b200.pack import SpaceTemplate
    prog = ir.parse_program(json.dumps(TREES["two_mm_64_8"]["program"]))
    space = {"tile": {"k": [1, 2, 4, 8, 16, 32, 64], "l": [1, 2, 4, 8, 16, 32, 64], "i1": [1, 2, 4, 8]},
             "reorder": [["i1_i", "j1"], ["j1", "i1_i"]], "parallel": ["jt"]}
    st = SpaceTemplate(prog, space)
    idx = st.indices_from_points(np.arange(st.size, dtype=np.uint64))
    for a in ("x86-avx2", "nvidia-volta"):
        task = E.Task(st.template.desc(arch_named(a), launch()), 0)
        d = E.to_device_records(st.records_from_indices(idx))
        s, f, status = task.score(d)
        ts, ti, nv = task.score_topk(d, 16)
        task.set_space(st.space_desc())
        pts = st.points_from_indices(idx)
        ps, pf, pst = task.score_points(torch.from_numpy(pts.view(np.int32)).cuda())
        torch.cuda.synchronize()
        sc = s.cpu().numpy()
        assert (status.cpu().numpy() == 0).all() and int(nv.item()) == len(idx)
        assert ti.cpu().tolist() == np.lexsort((np.arange(len(sc)), sc))[:16].tolist()
        assert torch.equal(s, ps) and torch.equal(f, pf)
        task.close()
