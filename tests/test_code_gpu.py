"""f4: external code-text analysis on the device (csrc/code.cu) against the reference's own
extract_features(program, code, arch, launch, diagnostics) on emitted texts, user-style edits of them and the
reference tests' hand-written texts (tests/golden/code_analysis.json, oracle/gen_golden.py)."""

import json
from collections import defaultdict

import pytest

from golden_util import GOLDEN, arch_named, launch

pytestmark = pytest.mark.gpu


def _cases():
    return json.loads((GOLDEN / "code_analysis.json").read_text())


def test_code_features_match_reference():
    from paper_2104_14641_b200 import code as K
    from paper_2104_14641_b200.cost import score
    from paper_2104_14641_b200.ir import parse_program
    cases = _cases()
    groups = defaultdict(list)
    for i, c in enumerate(cases):
        groups[(json.dumps(c["program"], sort_keys=True), c["arch"])].append(i)
    bad, diag_bad = [], []
    checked = n_notes = 0
    for (pj, an), idx in groups.items():
        prog = parse_program(pj)
        arch = arch_named(an)
        notes: list = []
        res = K.code_features(prog, [cases[i]["text"] for i in idx], arch, launch(), diagnostics=notes)
        for i, r, nt in zip(idx, res, notes):
            c = cases[i]
            checked += 1
            if "error" in c:
                if not isinstance(r, Exception) or [type(r).__name__, str(r)] != c["error"]:
                    bad.append((i, c["kind"], an, "error", c["error"], repr(r)))
                continue
            if isinstance(r, Exception):
                bad.append((i, c["kind"], an, "raised", repr(r)))
                continue
            want = [tuple(x) for x in c["features"]]
            got = [(k, v) for k, v in r.values]
            if got != want or score(r, arch) != c["score"]:
                bad.append((i, c["kind"], an, got, want))
            if nt != c["diagnostics"]:  # the notes extract_features appends, in order
                bad.append((i, c["kind"], an, "diagnostics", nt[:4], c["diagnostics"][:4]))
                diag_bad.append(i)
            n_notes += len(nt)
    assert checked == len(cases)
    assert not bad, (len(bad), len(diag_bad), bad[:5])
    assert n_notes > 1000  # the fixture exercises every kind of note


def test_extract_features_drop_in_errors():
    """The single-text drop-in raises the reference's exceptions."""
    from paper_2104_14641_b200 import code as K
    from paper_2104_14641_b200.arch import CostModelError
    from paper_2104_14641_b200.ir import parse_program
    prog = parse_program(json.dumps({"tensors": [{"name": "A", "dims": [8]}], "body": [
        {"loop": {"var": "i", "extent": 8, "body": [{"access": {"tensor": "A", "kind": "load", "idx": ["i"]}}]}}]}))
    with pytest.raises(K.AsmError, match="empty assembly input"):
        K.extract_features(prog, "  # nothing\n", arch_named("x86-avx2"))
    with pytest.raises(CostModelError, match="kernel launch record"):
        K.extract_features(prog, "    ret\n", arch_named("nvidia-volta"))
    fv = K.extract_features(prog, "    mov r1, 0\nb:\n    add r1, r1, 1\n    setp.lt r1, 8\n    bra b\n",
                            arch_named("nvidia-volta"), launch())
    assert dict(fv.values)["workload_per_thread"] > 0
    notes = ["kept"]
    K.extract_features(prog, "    mov r1, 1\nb:\n    mul r1, r1, 2\n    setp.lt r1, 64\n    bra b\n",
                       arch_named("nvidia-volta"), launch(), notes)
    assert notes == ["kept"] + ["loop at b: non-linear induction register r1"] * 2  # count_ptx, thread_cycles
