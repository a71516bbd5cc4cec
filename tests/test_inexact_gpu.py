"""The cache model's inexact-footprint flag on the device (ls_inexact_footprints) against the
reference's own CacheModel (NodeCost.inexact, ls/cache.py:198-202) on every rank-fixture schedule
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
    checked = inexact = 0
    bad = []
    for case in data["cases"]:
        prog = parse_program(json.dumps(data["programs"][case["program"]]))
        scheds = [Schedule.from_json(s) for s in case["schedules"]]
        got = inexact_footprints(prog, scheds, arch)
        for i, (g, w) in enumerate(zip(got.tolist(), case["inexact"])):
            if w is None:
                ok = g == -1
            else:
                ok = g == int(w)
                inexact += int(w)
            checked += 1
            if not ok:
                bad.append((case["program"], i, g, w))
    assert checked > 5000 and inexact > 500
    assert not bad, (len(bad), bad[:5])
