"""The cache model's inexact-footprint flag and notes on the device (ls_inexact_footprints) against
the reference's own CacheModel (NodeCost.inexact and its diagnostics, ls/cache.py:198-202) on every
rank-fixture schedule
and 160 schedules of each ResNet-50 task space (tests/golden/inexact.json, oracle/gen_golden.py)."""

import json

import numpy as np
import pytest

from golden_util import GOLDEN, arch_named

pytestmark = pytest.mark.gpu


def test_inexact_flags_match_reference():
    from paper_2104_14641_b200.cost import inexact_footprints
    from paper_2104_14641_b200.ir import Schedule, parse_program
    data = json.loads((GOLDEN / "inexact.json").read_text())
    arch = arch_named("x86-avx2")
    checked = inexact = n_notes = 0
    bad = []
    for case in data["cases"]:
        prog = parse_program(json.dumps(data["programs"][case["program"]]))
        scheds = [Schedule.from_json(s) for s in case["schedules"]]
        notes: list = []
        got = inexact_footprints(prog, scheds, arch, diagnostics=notes)
        for i, (g, nt, w) in enumerate(zip(got.tolist(), notes, case["inexact"])):
            if w is None:
                ok = g == -1
            else:
                ok = g == int(w[0]) and nt == w[1]  # the flag and the notes, in the model's order
                inexact += int(w[0])
                n_notes += len(w[1])
            checked += 1
            if not ok:
                bad.append((case["program"], i, g, w, nt))
    assert checked > 5000 and inexact > 500 and n_notes > 4000
    assert not bad, (len(bad), bad[:3])


def test_inexact_flags_tree_program_unsupported():
    """General trees (sibling loops) are outside the flag kernel: the library says so (LS_E_UNSUPPORTED)."""
    from paper_2104_14641_b200.cost import inexact_footprints
    from paper_2104_14641_b200.engine import EngineError
    from paper_2104_14641_b200.ir import Schedule, parse_program
    fx = json.loads((GOLDEN / "tree_rank.json").read_text())
    case = fx["cases"][0]
    prog = parse_program(json.dumps(fx["programs"][case["program"]]))
    with pytest.raises(EngineError, match="perfect chains"):
        inexact_footprints(prog, [Schedule.from_json(s) for s in case["schedules"][:4]], arch_named("x86-avx2"))


def test_inexact_flags_empty_and_failing():
    """An empty list, and schedules that fail apply_schedule (-1, no notes)."""
    from paper_2104_14641_b200 import workloads as W
    from paper_2104_14641_b200.cost import inexact_footprints
    from paper_2104_14641_b200.ir import Schedule
    prog = W.program(W.matmul_json(32))
    assert inexact_footprints(prog, [], arch_named("x86-avx2")).shape == (0,)
    notes: list = []
    bad = Schedule.from_json([{"tile": {"loop": "nope", "factor": 4}}])
    got = inexact_footprints(prog, [bad, Schedule.from_json([])], arch_named("x86-avx2"), diagnostics=notes)
    assert got.tolist() == [-1, 0] and notes == [[], []]
