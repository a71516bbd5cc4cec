"""Loaders for tests/golden (written by oracle/gen_golden.py from the reference)."""

from __future__ import annotations

import json
import tomllib
from functools import lru_cache
from pathlib import Path

import numpy as np

from paper_2104_14641_b200 import arch as A
from paper_2104_14641_b200 import ir
from paper_2104_14641_b200 import workloads as W
from paper_2104_14641_b200.pack import SpaceTemplate, pack_schedules

GOLDEN = Path(__file__).resolve().parent / "golden"

# reference exception -> device status code (include/loopscout_b200.h)
_ERR = [("no loop named", 1), ("tile factor", 2), ("does not divide extent", 3),
        ("ZeroDivisionError", 4), ("missing loops", 5), ("perfect nest chain", 6),
        ("must be finite", 7)]


def status_of_error(err) -> int:
    if err is None:
        return 0
    for key, code in _ERR:
        if key in err:
            return code
    raise AssertionError(f"unmapped reference error {err!r}")


@lru_cache(None)
def rank_cases():
    return json.loads((GOLDEN / "rank_cases.json").read_text())


def arch_named(name: str):
    data = rank_cases()["archs"]
    if name in data:
        return A.arch_from_dict(tomllib.loads(data[name]), name)
    return A.load_arch(name)


def launch():
    return A.KernelLaunch.from_json(W.KERNEL_LAUNCH)


@lru_cache(None)
def space_npz(name: str):
    z = np.load(GOLDEN / f"{name}.npz")
    return {k: z[k] for k in z.files}


def space_case(name: str):
    """(SpaceTemplate, records, golden dict) of a space fixture."""
    z = space_npz(name)
    prog = ir.parse_program(str(z["program"]))
    st = SpaceTemplate(prog, json.loads(str(z["space"])))
    return st, st.records_from_indices(z["idx"]), z


SPACE_FIXTURES = ["gemm1024", "conv56", "dense_1024_768_768", "dense_1024_3072_768",
                  "dense_1024_768_3072", "bmm_96_128_128_64", "bmm_96_128_64_128"]
# configs[2] / configs[3] exactly as bench.py builds them (workloads.resnet50_tasks / bert_tasks)
RESNET_FIXTURES = sorted(p.stem for p in GOLDEN.glob("resnet_*.npz"))
BERT_FIXTURES = sorted(p.stem for p in GOLDEN.glob("bert_*.npz"))
BENCH_FIXTURES = RESNET_FIXTURES + BERT_FIXTURES
ALL_SPACE_FIXTURES = SPACE_FIXTURES + BENCH_FIXTURES


def rank_groups(case):
    spec = rank_cases()["programs"][case["program"]]
    prog = ir.parse_program(json.dumps(spec))
    scheds = [ir.Schedule.from_json(s) for s in case["schedules"]]
    return prog, pack_schedules(prog, scheds)
