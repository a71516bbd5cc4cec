"""The CPU oracle against the reference's own outputs (tests/golden, oracle/gen_golden.py).

Pins the oracle before anything is compared against it: bit-exact float64
scores and features on every golden candidate, identical failure classes,
the reference's published cache known-answers, and byte-identical mock text.
"""

import json

import numpy as np
import pytest

import pyoracle
from golden_util import (ALL_SPACE_FIXTURES, SPACE_FIXTURES, arch_named, launch, rank_cases, rank_groups, space_case,
                         status_of_error, GOLDEN)
from paper_2104_14641_b200 import abi, ir
from paper_2104_14641_b200.pack import pack_schedules


def test_descriptor_layout_matches_c():
    import ctypes
    assert pyoracle.sizeof_desc() == ctypes.sizeof(abi.TaskDesc)


@pytest.mark.parametrize("name", ALL_SPACE_FIXTURES)
def test_space_fixtures_bit_exact(name):
    st, recs, z = space_case(name)
    for a in z["arches"]:
        a = str(a)
        d = st.template.desc(arch_named(a), launch())
        sc, fe, status = pyoracle.evaluate(d, recs, nthreads=8)
        assert (status == 0).all()
        np.testing.assert_array_equal(fe, z[f"feats_{a}"])
        np.testing.assert_array_equal(sc, z[f"scores_{a}"])


def test_gemm_top64_matches_reference_order():
    st, recs, z = space_case("gemm1024")
    d = st.template.desc(arch_named("x86-avx2"), launch())
    sc, _, _ = pyoracle.evaluate(d, recs, nthreads=8)
    ref = sorted(range(len(sc)), key=lambda i: (z["scores_x86-avx2"][i], i))[:64]
    got = sorted(range(len(sc)), key=lambda i: (sc[i], i))[:64]
    assert got == ref


def _rank_params():
    return [(c["program"], a) for c in rank_cases()["cases"] for a in c["results"]]


@pytest.mark.parametrize("program,arch", _rank_params())
def test_rank_cases(program, arch):
    case = next(c for c in rank_cases()["cases"] if c["program"] == program)
    res = case["results"][arch]
    prog, groups = rank_groups(case)
    ar = arch_named(arch)
    unpackable = sum(len(g.index) for g in groups if g.template is None)
    assert unpackable <= 2, "more than 8 tile/vectorize parameters is the only packing limit hit here"
    for g in groups:
        if g.template is None:
            continue
        d = g.template.desc(ar, launch())
        sc, fe, st = pyoracle.evaluate(d, g.records)
        for r, i in enumerate(g.index):
            want = status_of_error(res["errors"][i])
            assert st[r] == want, (i, case["schedules"][i], res["errors"][i], st[r])
            if want == 0:
                assert sc[r] == res["scores"][i], (i, case["schedules"][i])
                assert list(fe[r]) == res["features"][i], (i, case["schedules"][i])


def _trees():
    return json.loads((GOLDEN / "trees.json").read_text())


@pytest.mark.parametrize("name", sorted(_trees()))
def test_tree_programs(name):
    e = _trees()[name]
    prog = ir.parse_program(json.dumps(e["program"]))
    g = pack_schedules(prog, [ir.Schedule(())])[0]
    # cache model node costs at the fixture's capacity
    arch = arch_named("x86-avx2")
    d = g.template.desc(arch, launch())
    d.cache_capacity = e["cap"]
    st, nodes, rdfp, rdmov = pyoracle.cache_detail(d, g.records[0])
    assert st == 0
    assert [rdfp, rdmov] == e["nodes"]["<root>"]
    for var, (dfp, dmov) in e["nodes"].items():
        if var == "<root>":
            continue
        assert nodes[g.template.var_id[var]] == (dfp, dmov), var
    for a, feats in e["features"].items():
        d = g.template.desc(arch_named(a), launch())
        sc, fe, st = pyoracle.evaluate(d, g.records)
        assert st[0] == 0
        assert list(fe[0]) == [v for _, v in feats], a
        assert sc[0] == e["scores"][a]


def test_reference_known_answers():
    """Values the reference's own tests assert (tests/test_cache.py:57-68, test_acceptance.py:55-93)."""
    t = _trees()
    assert t["two_mm_64_8"]["nodes"]["jt"] == [9728, 9728]
    assert t["two_mm_64_8"]["nodes"]["it"][1] == 77824
    cache_golden = [
        (4368, 8208), (512, 512), (128, 128), (1104, 2064), (256, 256), (768, 4608), (1728, 1728),
        (512, 512), (512, 512), (1160, 2056), (256, 256), (264, 1088), (4368, 8208), (512, 512),
        (272, 1152), (512, 512), (520, 2112), (512, 512), (3072, 34816), (528, 2176)]
    got = [tuple(t[f"random_nest_{k}"]["nodes"]["<root>"]) for k in range(20)]
    assert got == cache_golden


def test_emit_text_byte_identical():
    cases = json.loads((GOLDEN / "emit.json").read_text())
    assert len(cases) >= 30
    progs = rank_cases()["programs"]
    for c in cases:
        prog = ir.parse_program(json.dumps(progs[c["program"]]))
        g = pack_schedules(prog, [ir.Schedule.from_json(c["schedule"])])[0]
        d = g.template.desc(arch_named("nvidia-volta"), launch())
        tgt = abi.TARGET[c["target"]]
        assert pyoracle.emit_text(d, g.records[0], tgt) == c["text"], (c["program"], c["schedule"])


@pytest.mark.parametrize("fixture", ["tree_rank.json", "tree_inline.json"])
def test_oracle_scheduled_trees(fixture):
    """The C oracle on scheduled tree programs == the reference (tests/golden/tree_*.json)."""
    import json
    from golden_util import GOLDEN, arch_named, launch, status_of_error
    from paper_2104_14641_b200 import ir
    from paper_2104_14641_b200.pack import pack_schedules
    tr = json.loads((GOLDEN / fixture).read_text())
    for case in tr["cases"]:
        prog = ir.parse_program(json.dumps(tr["programs"][case["program"]]))
        scheds = [ir.Schedule.from_json(s) for s in case["schedules"]]
        groups = pack_schedules(prog, scheds)
        for a, res in case["results"].items():
            arch = arch_named(a)
            for g in groups:
                assert g.template is not None
                s, f, st = pyoracle.evaluate(g.template.desc(arch, launch()), g.records)
                for j, i in enumerate(g.index):
                    want = status_of_error(res["errors"][i])
                    assert st[j] == want, (case["program"], a, i)
                    if want == 0:
                        assert s[j] == res["scores"][i]
                        assert f[j].tolist() == res["features"][i]
