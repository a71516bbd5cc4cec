"""Generate tests/golden/* by running the REFERENCE itself (/root/reference).

TEST INFRASTRUCTURE.  Run in the build container only (the reference does not
exist on the GPU box):

    python oracle/gen_golden.py            # writes tests/golden/*.npz|json

Every fixture stores inputs (programs as canonical JSON, schedules as JSON or
per-axis choice indices of a space) and the reference's outputs
(scores, feature vectors, or the exception each candidate raised).
The reference is imported from /root/reference/pkg/src (its numpy version is recorded in tests/golden/README.md).
"""

from __future__ import annotations

import json
import math
import multiprocessing as mp
import random
import sys
import time
from pathlib import Path

import numpy as np

REPO = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(REPO))
sys.path.insert(0, "/root/reference/pkg/src")

import loopscout as L  # noqa: E402  (the reference)

from paper_2104_14641_b200 import workloads as W  # noqa: E402
from paper_2104_14641_b200.pack import SpaceTemplate  # noqa: E402

OUT = REPO / "tests" / "golden"
LAUNCH = W.KERNEL_LAUNCH

# Custom arches that exercise what the shipped TOMLs do not: issue caps,
# unknown-class defaults, 2-wide x86, non-integral PTX costs.
CUSTOM_ARCHS = {
    "bench-x86": """[meta]
name = "bench-x86"
family = "cpu"
target = "cpu-x86"
dialect = "x86-att"
[coefficients]
n_fma = 0.01
n_vload = 0.01
n_vstore = 0.01
est_l1_movement = 8.0
ilp_cycles = 1.0
[cache]
l1_capacity_bytes = 4096
element_bytes = 4
[ilp]
issue_width = 4
default_latency = 1
[ilp.latency]
fma = 4
load = 5
store = 4
move = 1
""",
    "odd-x86": """[meta]
name = "odd-x86"
family = "cpu"
target = "cpu-x86"
dialect = "x86-att"
[coefficients]
n_fma = 0.37
n_vload = 1.3
n_vstore = 0.7
est_l1_movement = 3.1
ilp_cycles = 1.7
[cache]
l1_capacity_bytes = 2048
element_bytes = 4
[ilp]
issue_width = 2
default_latency = 2
[ilp.latency]
fma = 5
load = 3
addq = 1
[ilp.units]
load = 1
fma = 1
""",
    "odd-a64": """[meta]
name = "odd-a64"
family = "cpu"
target = "cpu-aarch64"
dialect = "aarch64"
[coefficients]
n_fma = 0.11
n_vload = 0.9
n_vstore = 1.9
est_l1_movement = 2.5
ilp_cycles = 1.3
[cache]
l1_capacity_bytes = 1024
element_bytes = 2
[ilp]
issue_width = 3
default_latency = 1
[ilp.latency]
fma = 3
load = 6
store = 2
[ilp.units]
store = 1
""",
    "odd-gpu": """[meta]
name = "odd-gpu"
family = "gpu"
target = "gpu-ptx"
dialect = "ptx"
[coefficients]
workload_per_thread = 0.3
sm_underuse = 1.7
warp_slack = 2.9
n_smem_ops_adjusted = 0.13
n_fma = 0.7
n_ld = 1.1
n_st = 0.9
[gpu]
num_sms = 132
max_threads_per_sm = 1536
registers_per_sm = 65536
shared_mem_per_sm_bytes = 65536
[gpu.instr_cost]
fma = 2.5
ld = 7
st = 9
mov = 0.5
add = 1
setp = 1.5
bra = 3
""",
}

_ARCH_CACHE = {}


def ref_arch(name: str):
    if name not in _ARCH_CACHE:
        if name in CUSTOM_ARCHS:
            p = Path(f"/tmp/golden_arch_{name}.toml")
            if not p.exists() or p.read_text() != CUSTOM_ARCHS[name]:
                p.write_text(CUSTOM_ARCHS[name])
            _ARCH_CACHE[name] = L.load_arch(str(p))
        else:
            _ARCH_CACHE[name] = L.load_arch(name)
    return _ARCH_CACHE[name]


def ref_eval(args):
    """One candidate through the reference: (score, features) or (None, error)."""
    prog_json, sched_json, arch_name = args
    prog = L.parse_program(prog_json)
    arch = ref_arch(arch_name)
    launch = L.KernelLaunch.from_json(LAUNCH)
    try:
        s = L.Schedule.from_json(sched_json)
        q = L.apply_schedule(prog, s)
        code = L.emit_mock_asm(q, arch.target)
        fv = L.extract_features(q, code, arch, launch)
        return L.score(fv, arch), [v for _, v in fv.values], None
    except Exception as e:  # noqa: BLE001 - recorded as the golden outcome
        return None, None, f"{type(e).__name__}: {e}"


def run_pool(jobs):
    with mp.Pool(mp.cpu_count()) as pool:
        return pool.map(ref_eval, jobs, chunksize=16)


def space_fixture(name, spec, space, n, seed, arches):
    t0 = time.time()
    prog = W.program(spec)
    st = SpaceTemplate(prog, space)
    idx = W.distinct_indices(st.sizes, n, seed)
    scheds = [st.schedule_of(r).to_json() for r in idx]
    pj = json.dumps(spec)
    out = {"idx": idx, "program": np.array(pj), "space": np.array(json.dumps(space)),
           "arches": np.array(arches)}
    for a in arches:
        res = run_pool([(pj, s, a) for s in scheds])
        assert all(r[2] is None for r in res), [r[2] for r in res if r[2]][:3]
        out[f"scores_{a}"] = np.array([r[0] for r in res], np.float64)
        out[f"feats_{a}"] = np.array([r[1] for r in res], np.float64)
    np.savez_compressed(OUT / f"{name}.npz", **out)
    print(f"{name}: {n} candidates x {len(arches)} arches in {time.time() - t0:.1f}s")


# -- random schedules for the rank path --------------------------------------------


def chain_names(spec):
    out, node = [], spec["body"]
    while len(node) == 1 and "loop" in node[0]:
        out.append(node[0]["loop"]["var"])
        node = node[0]["loop"]["body"]
    return out


def random_schedule(rng: random.Random, prog, kinds="TRVUP"):
    """A random transform list on a (chain) program, valid or not."""
    names = [lp.var for lp in prog.loops()]
    ext = {lp.var: lp.extent for lp in prog.loops()}
    sched = []
    cur = list(names)
    for v in rng.sample(names, rng.randint(0, min(len(names), 4))):
        if "T" not in kinds:
            break
        e = ext[v]
        r = rng.random()
        if r < 0.6:
            f = rng.choice([d for d in range(1, e + 1) if e % d == 0])
        elif r < 0.95:
            f = rng.randint(1, e)
        else:
            f = rng.choice([0, e + 1, e + 7])
        sched.append({"tile": {"loop": v, "factor": f}})
        i = cur.index(v)
        cur.insert(i + 1, v + "_i")
        ext[v + "_i"] = max(f, 1)
        ext[v] = math.ceil(e / max(f, 1))
    if "R" in kinds and len(cur) >= 2 and rng.random() < 0.8:
        r = rng.random()
        if r < 0.7:
            order = rng.sample(cur, len(cur))
        elif r < 0.85:
            a = rng.randint(0, len(cur) - 2)
            b = rng.randint(a + 2, len(cur))
            seg = cur[a:b]
            order = rng.sample(seg, len(seg))
        elif r < 0.92:
            order = rng.sample(cur, min(len(cur), 3))
        elif r < 0.96:
            order = [cur[0], cur[0]] + cur[1:2]
        else:
            order = cur[:2] + ["nope"]
        sched.append({"reorder": order})
    if "V" in kinds and rng.random() < 0.4:
        v = rng.choice(cur)
        e = ext.get(v, 4)
        r = rng.random()
        w = rng.choice([d for d in range(1, e + 1) if e % d == 0]) if r < 0.8 else rng.choice([0, 3, e + 1])
        sched.append({"vectorize": {"loop": v, "width": w}})
        i = cur.index(v)
        cur.insert(i + 1, v + ("_i" if v + "_i" not in cur else "_i_"))
    if "U" in kinds and rng.random() < 0.4:
        small = [v for v in cur if ext.get(v, 99) <= 8] or cur
        sched.append({"unroll": {"loop": rng.choice(small if rng.random() < 0.8 else cur)}})
    if "P" in kinds and rng.random() < 0.4:
        sched.append({"parallel": {"loop": rng.choice(cur)}})
    if rng.random() < 0.03:
        sched.append({"tile": {"loop": "ghost", "factor": 2}})
    return sched


def smem_json(idx="tid", dim=2048, outer=4, elem_bytes=4):
    return {"tensors": [{"name": "S", "dims": [dim], "scope": "shared", "elem_bytes": elem_bytes},
                        {"name": "G", "dims": [dim]}],
            "body": [{"loop": {"var": "i", "extent": outer, "body": [
                {"loop": {"var": "tid", "extent": 32, "attrs": ["parallel"], "body": [
                    {"access": {"tensor": "S", "kind": "load", "idx": [idx]}},
                    {"access": {"tensor": "G", "kind": "load", "idx": ["tid"]}},
                    {"access": {"tensor": "S", "kind": "store", "idx": [idx]}}]}}]}}]}


def smem2d_json():
    return {"tensors": [{"name": "S", "dims": [64, 33], "scope": "shared"},
                        {"name": "T", "dims": [16, 64], "scope": "shared", "elem_bytes": 8},
                        {"name": "G", "dims": [64, 64]}],
            "body": [{"loop": {"var": "r", "extent": 16, "body": [
                {"loop": {"var": "c", "extent": 64, "body": [
                    {"access": {"tensor": "G", "kind": "load", "idx": ["c", "4*r"]}},
                    {"access": {"tensor": "S", "kind": "load", "idx": ["c", "2*r + 1"]}},
                    {"access": {"tensor": "T", "kind": "store", "idx": ["r", "c"]}}]}}]}}]}


RANK_PROGRAMS = {
    "matmul8": W.matmul_json(8),
    "matmul48": W.matmul_json(48),
    "mm_rect": W.matmul_json(24, 40, 12),
    "nested4x8": {"tensors": [{"name": "A", "dims": [32]}, {"name": "B", "dims": [32]}],
                  "body": [{"loop": {"var": "i", "extent": 4, "body": [
                      {"loop": {"var": "j", "extent": 8, "body": [
                          {"access": {"tensor": "A", "kind": "load", "idx": ["8*i + j"]}},
                          {"access": {"tensor": "B", "kind": "store", "idx": ["8*i + j"]}}]}}]}}]},
    "single16": {"tensors": [{"name": "A", "dims": [16]}, {"name": "B", "dims": [16]}],
                 "body": [{"loop": {"var": "i", "extent": 16, "body": [
                     {"access": {"tensor": "A", "kind": "load", "idx": ["i"]}},
                     {"access": {"tensor": "A", "kind": "load", "idx": ["i"]}},
                     {"access": {"tensor": "B", "kind": "store", "idx": ["i"]}}]}}]},
    "conv_small": W.conv2d_json(1, 8, 6, 6, 4, 3, 3),
    "conv_s2": W.conv2d_json(1, 4, 5, 5, 4, 3, 3, stride=2),
    "bmm": W.batch_matmul_json(2, 8, 6, 4),
    "neg_stride": {"tensors": [{"name": "A", "dims": [64]}, {"name": "B", "dims": [64, 8]}],
                   "body": [{"loop": {"var": "i", "extent": 16, "step": 2, "body": [
                       {"loop": {"var": "j", "extent": 8, "body": [
                           {"access": {"tensor": "A", "kind": "load", "idx": ["40 - 2*i + j"]}},
                           {"access": {"tensor": "B", "kind": "store", "idx": ["i", "j"]}},
                           {"access": {"tensor": "B", "kind": "load", "idx": ["i + 1", "j"]}}]}}]}}]},
    "deep9": {"tensors": [{"name": "A", "dims": [8, 8, 8]}, {"name": "B", "dims": [8, 8, 8]}],
              "body": W._nest([(f"l{k}", 2) for k in range(9)],
                              [{"access": {"tensor": t, "kind": kd, "idx": [
                                  f"l{3 * d} + 2*l{3 * d + 1} + 4*l{3 * d + 2}" for d in range(3)]}}
                               for t, kd in (("A", "load"), ("B", "store"))])},
    "smem_tid": smem_json("tid"),
    "smem_32tid": smem_json("32*tid"),
    "smem_2tid": smem_json("2*tid", elem_bytes=2),
    "smem_5tid": smem_json("5*tid + 3", elem_bytes=8),
    "smem_2d": smem2d_json(),
}


def rank_fixture(n_per=120, seed=2024):
    rng = random.Random(seed)
    cases = []
    jobs = []
    for pname, spec in RANK_PROGRAMS.items():
        prog = L.parse_program(json.dumps(spec))
        is_smem = pname.startswith("smem")
        arches = ["nvidia-volta", "odd-gpu"] if is_smem else ["x86-avx2", "aarch64-neon", "nvidia-volta",
                                                               "bench-x86", "odd-x86", "odd-a64", "odd-gpu"]
        scheds = [[]] + [random_schedule(rng, prog) for _ in range(n_per)]
        cases.append({"program": pname, "schedules": scheds, "results": {a: {} for a in arches}})
        for a in arches:
            jobs.extend((json.dumps(spec), s, a) for s in scheds)
    t0 = time.time()
    res = run_pool(jobs)
    k = 0
    nerr = 0
    for c in cases:
        for a, r in c["results"].items():
            outs = res[k:k + len(c["schedules"])]
            k += len(c["schedules"])
            r["scores"] = [o[0] for o in outs]
            r["features"] = [o[1] for o in outs]
            r["errors"] = [o[2] for o in outs]
            nerr += sum(o[2] is not None for o in outs)
    payload = {"programs": RANK_PROGRAMS, "archs": CUSTOM_ARCHS, "launch": LAUNCH, "cases": cases}
    (OUT / "rank_cases.json").write_text(json.dumps(payload, separators=(",", ":")))
    print(f"rank_cases: {len(jobs)} evaluations ({nerr} reference errors) in {time.time() - t0:.1f}s")


# -- general trees (oracle-only class), reference known answers --------------------------


def tree_fixture():
    sys.path.insert(0, "/root/reference/pkg/tests")
    import helpers as H
    from loopscout.ir import serialize_program

    progs = {
        "two_mm_64_8": H.two_mm(64, 8), "two_mm_16_4": H.two_mm(16, 4),
        "interposed": H.build([H.tensor("A", [8]), H.tensor("B", [256])],
                              [H.loop("o", 4, [H.loop("i", 8, [H.acc("A", "load", ["i"])]),
                                               H.loop("j", 256, [H.acc("B", "load", ["j"])]),
                                               H.loop("i2", 8, [H.acc("A", "load", ["i2"])])])]),
        "trace_layout": H.build([H.tensor("A", [2, 2]), H.tensor("B", [2])],
                                [H.loop("i", 2, [H.loop("j", 2, [H.acc("A", "load", ["i", "j"])]),
                                                 H.acc("B", "store", ["i"])])]),
    }
    rng = random.Random(20250823)  # CACHE_GOLDEN's generator (tests/test_acceptance.py:68-93)
    caps = {}
    for k in range(20):
        p, cap = H.random_nest(rng)
        progs[f"random_nest_{k}"] = p
        caps[f"random_nest_{k}"] = cap
    out = {}
    for name, p in progs.items():
        cap = caps.get(name, 4096)
        model = L.analyze(p, L.CacheSpec(cap))
        entry = {"program": json.loads(serialize_program(p)), "cap": cap,
                 "nodes": {k: [v.dfp, v.dmov] for k, v in model.node_costs.items()},
                 "features": {}}
        for a in ("x86-avx2", "aarch64-neon", "nvidia-volta", "odd-x86", "odd-gpu"):
            arch = ref_arch(a)
            fv = L.extract_features(p, L.emit_mock_asm(p, arch.target), arch,
                                    L.KernelLaunch.from_json(LAUNCH))
            entry["features"][a] = [[k, v] for k, v in fv.values]
            entry.setdefault("scores", {})[a] = L.score(fv, arch)
        out[name] = entry
    (OUT / "trees.json").write_text(json.dumps(out, separators=(",", ":")))
    print(f"trees: {len(out)} programs")


def emit_fixture():
    cases = []
    rng = random.Random(7)
    for pname in ("matmul8", "nested4x8", "conv_small", "deep9", "smem_tid"):
        spec = RANK_PROGRAMS[pname]
        prog = L.parse_program(json.dumps(spec))
        for _ in range(6):
            s = random_schedule(rng, prog, kinds="TRVUP")
            try:
                q = L.apply_schedule(prog, L.Schedule.from_json(s))
            except Exception:  # noqa: BLE001
                continue
            for tgt in ("cpu-x86", "cpu-aarch64", "gpu-ptx"):
                text = L.emit_mock_asm(q, tgt)
                if len(text) < 200000:
                    cases.append({"program": pname, "schedule": s, "target": tgt, "text": text})
    (OUT / "emit.json").write_text(json.dumps(cases))
    print(f"emit: {len(cases)} texts")


def es_fixture():
    sys.path.insert(0, "/root/reference/pkg/tests")
    runs = []
    specs = [
        ("matmul16", W.matmul_json(16), {"tile": {"i": [2, 4, 8], "j": [2, 4]}}, "bench-x86",
         dict(seed=7, population=6, iterations=5)),
        ("matmul32", W.matmul_json(32),
         {"tile": {"i": [2, 4, 8, 16], "j": [2, 4, 8, 16], "k": [4, 8]},
          "reorder": [["i", "i_i", "j", "j_i", "k", "k_i"], ["i", "j", "k", "i_i", "j_i", "k_i"]]},
         "x86-avx2", dict(seed=0, population=16, iterations=12)),
        ("conv_small", W.conv2d_json(1, 8, 6, 6, 4, 3, 3),
         {"tile": {"oc": [1, 2, 4, 8], "ow": [1, 2, 3, 6]},
          "reorder": W.random_perms(W.tiled_chain(["n", "oc", "oh", "ow", "ic", "kh", "kw"], ["oc", "ow"]), 24, 3),
          "vectorize": {"ic": [0, 2, 4]}, "unroll": ["kw"], "parallel": ["oc"]},
         "aarch64-neon", dict(seed=3, population=24, iterations=8, sigma=0.8)),
        ("conv_gpu", W.conv2d_json(1, 8, 6, 6, 4, 3, 3),
         {"tile": {"oc": [1, 2, 4, 8], "oh": [1, 2, 3, 6]},
          "reorder": W.random_perms(W.tiled_chain(["n", "oc", "oh", "ow", "ic", "kh", "kw"], ["oc", "oh"]), 16, 5)},
         "nvidia-volta", dict(seed=11, population=20, iterations=6, sigma=0.6, rank_normalize=False)),
    ]
    for name, spec, space, arch_name, kw in specs:
        prog = L.parse_program(json.dumps(spec))
        arch = ref_arch(arch_name)
        params = L.EsParams(**kw)
        res = L.optimize(prog, space, arch, params, jobs=1, launch=L.KernelLaunch.from_json(LAUNCH))
        runs.append({"name": name, "program": spec, "space": space, "arch": arch_name, "params": kw,
                     "best_schedule": res.best_schedule.to_json(), "best_score": res.best_score,
                     "best_features": [[k, v] for k, v in res.best_features.values],
                     "trace": res.trace, "evaluated": res.evaluated, "evaluations": res.evaluations})
    (OUT / "es_runs.json").write_text(json.dumps(runs))
    print(f"es: {len(runs)} optimize runs")


def random_tree_schedule(rng: random.Random, prog, inline=False):
    """A random Tile / Reorder / Parallel (+ Unroll / Vectorize) list on a tree program, valid or not."""
    loops = {lp.var: lp for lp in prog.loops()}
    ext = {v: lp.extent for v, lp in loops.items()}
    kids = {v: [c.var if hasattr(c, "var") else None for c in lp.children] for v, lp in loops.items()}
    sched = []
    names = list(loops)
    for v in rng.sample(names, rng.randint(0, min(len(names), 3))):
        e = ext[v]
        r = rng.random()
        f = rng.choice([d for d in range(1, e + 1) if e % d == 0]) if r < 0.7 else (
            rng.randint(1, e) if r < 0.95 else rng.choice([0, e + 1]))
        sched.append({"tile": {"loop": v, "factor": f}})
        inner = v + "_i"
        while inner in kids:
            inner += "_"
        kids[inner] = kids[v]
        kids[v] = [inner]
        ext[inner] = max(f, 1)
        ext[v] = math.ceil(e / max(f, 1))
    if rng.random() < 0.8:
        if rng.random() < 0.8:  # a single-child chain from a random loop
            v = rng.choice(list(kids))
            seg = [v]
            while len(kids[seg[-1]]) == 1 and kids[seg[-1]][0] is not None and rng.random() < 0.85:
                seg.append(kids[seg[-1]][0])
            if len(seg) >= 2:
                sched.append({"reorder": rng.sample(seg, len(seg))})
        else:  # any set of names (mostly invalid)
            seg = rng.sample(list(kids), min(len(kids), rng.randint(2, 4)))
            if rng.random() < 0.1:
                seg.append("nope")
            sched.append({"reorder": seg})
    for v in rng.sample(list(kids), rng.randint(0, min(2, len(kids)))):
        sched.append({"parallel": {"loop": v}})
    if inline:
        for v in rng.sample(list(kids), rng.randint(0, min(2, len(kids)))):
            r = rng.random()
            if r < 0.5 and ext[v] <= 8:
                sched.append({"unroll": {"loop": v}})
            elif r < 0.9:
                e = ext[v]
                w = rng.choice([d for d in (1, 2, 4, 8) if e % d == 0] + ([3] if rng.random() < 0.2 else []))
                if rng.random() < 0.05:
                    w = 0
                sched.append({"vectorize": {"loop": v, "width": w}})
                inner = v + "_i"
                while inner in kids:
                    inner += "_"
                kids[inner] = kids[v]
                kids[v] = [inner]
                ext[inner] = max(w, 1)
                ext[v] = math.ceil(e / max(w, 1))
            else:
                sched.append({"unroll": {"loop": v}})
    return sched


def tree_rank_fixture(n_per=60, seed=77):
    """Scheduled tree programs (imperfect nests, siblings, top-level accesses, deep nests) through
    the reference: scores / features / errors per arch."""
    sys.path.insert(0, "/root/reference/pkg/tests")
    import helpers as H
    from loopscout.ir import serialize_program
    trees = json.loads((OUT / "trees.json").read_text())
    progs = {k: v["program"] for k, v in trees.items() if k in ("two_mm_64_8", "two_mm_16_4", "interposed",
                                                               "trace_layout") or k.startswith("random_nest_")}
    mixed = H.build([H.tensor("A", [16, 16]), H.tensor("B", [16]), H.tensor("C", [16, 16])],
                    [H.acc("B", "load", ["0"]),
                     H.loop("i", 16, [H.acc("B", "load", ["i"]),
                                      H.loop("j", 16, [H.acc("A", "load", ["i", "j"]),
                                                       H.acc("C", "store", ["j", "i"])]),
                                      H.acc("B", "store", ["i"]),
                                      H.loop("k", 8, [H.acc("C", "load", ["i", "2*k"])])]),
                     H.loop("m", 4, [H.acc("A", "load", ["m", "m"])])])
    progs["mixed_levels"] = json.loads(serialize_program(mixed))
    deep = H.loop("d9", 2, [H.acc("A", "load", ["d0 + d9"]), H.acc("A", "store", ["d1"])])
    for k in range(8, -1, -1):
        deep = H.loop(f"d{k}", 2, [deep] + ([H.loop(f"s{k}", 3, [H.acc("A", "load", [f"s{k}"])])] if k == 3 else []))
    progs["deep_branch"] = json.loads(serialize_program(H.build([H.tensor("A", [32])], [deep])))
    rng = random.Random(seed)
    arches = ["x86-avx2", "aarch64-neon", "nvidia-volta", "odd-x86", "odd-gpu"]
    cases, jobs = [], []
    for pname, spec in progs.items():
        prog = L.parse_program(json.dumps(spec))
        scheds = [[]] + [random_tree_schedule(rng, prog) for _ in range(n_per)]
        cases.append({"program": pname, "schedules": scheds, "results": {a: {} for a in arches}})
        for a in arches:
            jobs.extend((json.dumps(spec), sch, a) for sch in scheds)
    res = run_pool(jobs)
    k = 0
    for c in cases:
        for a, r in c["results"].items():
            outs = res[k:k + len(c["schedules"])]
            k += len(c["schedules"])
            r["scores"] = [o[0] for o in outs]
            r["features"] = [o[1] for o in outs]
            r["errors"] = [o[2] for o in outs]
    (OUT / "tree_rank.json").write_text(json.dumps({"programs": progs, "cases": cases}, separators=(",", ":")))
    print(f"tree_rank: {len(jobs)} evaluations")
    # Unroll / Vectorize on trees (inlined loops: the emission replay path), incl. unrolled base loops
    small = {k: v for k, v in progs.items() if k in ("two_mm_16_4", "interposed", "trace_layout", "mixed_levels",
                                                    "deep_branch") or k in ("random_nest_0", "random_nest_1",
                                                                             "random_nest_2", "random_nest_3")}
    ub = H.build([H.tensor("A", [8, 8]), H.tensor("B", [8])],
                 [H.loop("i", 4, [H.acc("B", "load", ["i"]),
                                  H.loop("j", 2, [H.acc("A", "load", ["i", "j"]),
                                                  H.loop("k", 3, [H.acc("A", "store", ["k", "j"])])],
                                         attrs=("unroll",)),
                                  H.loop("m", 4, [H.acc("B", "store", ["m"])])])])
    small["unrolled_base"] = json.loads(serialize_program(ub))
    cases2, jobs2 = [], []
    for pname, spec in small.items():
        prog = L.parse_program(json.dumps(spec))
        scheds = [[]] + [random_tree_schedule(rng, prog, inline=True) for _ in range(n_per)]
        cases2.append({"program": pname, "schedules": scheds, "results": {a: {} for a in arches}})
        for a in arches:
            jobs2.extend((json.dumps(spec), sch, a) for sch in scheds)
    res = run_pool(jobs2)
    k = 0
    for c in cases2:
        for a, r in c["results"].items():
            outs = res[k:k + len(c["schedules"])]
            k += len(c["schedules"])
            r["scores"] = [o[0] for o in outs]
            r["features"] = [o[1] for o in outs]
            r["errors"] = [o[2] for o in outs]
    (OUT / "tree_inline.json").write_text(json.dumps({"programs": small, "cases": cases2}, separators=(",", ":")))
    print(f"tree_inline: {len(jobs2)} evaluations")


def cli_fixture():
    """Reference CLI outputs (rank --json with failures, search --json --trace, analyze --code with
    notes) on files under golden/cli."""
    import contextlib
    import io
    from loopscout import cli as ref_cli
    d = OUT / "cli"
    d.mkdir(exist_ok=True)
    rc = json.loads((OUT / "rank_cases.json").read_text())
    runs = []
    for pname in ("matmul48", "conv_small", "neg_stride", "deep9"):
        case = next(c for c in rc["cases"] if c["program"] == pname)
        (d / f"{pname}.json").write_text(json.dumps(rc["programs"][pname]))
        (d / f"{pname}_scheds.json").write_text(json.dumps(case["schedules"]))
        for arch in ("x86-avx2", "nvidia-volta"):
            argv = ["rank", str(d / f"{pname}.json"), str(d / f"{pname}_scheds.json"), "--arch", arch, "--json",
                    "--jobs", "1"] + (["--launch", str(d / "launch.json")] if arch == "nvidia-volta" else [])
            runs.append((f"rank_{pname}_{arch}", argv, None))
    (d / "launch.json").write_text(json.dumps(LAUNCH))
    # analyze --code (f4): emitted texts and edited ones (changed loop bounds -> notes), text and JSON output
    mrng = random.Random(5)
    for pname in ("matmul48", "conv_small", "deep9"):
        prog = L.parse_program(json.dumps(rc["programs"][pname]))
        for arch, tgt in (("x86-avx2", "cpu-x86"), ("aarch64-neon", "cpu-aarch64"), ("nvidia-volta", "gpu-ptx")):
            for kind in ("none", "bound"):
                cf = d / f"{pname}_{tgt}_{kind}.s"
                cf.write_text(_mutate(mrng, L.emit_mock_asm(prog, tgt), tgt, kind))
                for js in ((["--json"], []) if kind == "bound" else (["--json"],)):
                    argv = ["analyze", str(d / f"{pname}.json"), "--code", str(cf), "--arch", arch, *js] + \
                        (["--launch", str(d / "launch.json")] if arch == "nvidia-volta" else [])
                    runs.append((f"analyze_{pname}_{tgt}_{kind}{'_json' if js else ''}", argv, None))
    es_runs = json.loads((OUT / "es_runs.json").read_text())
    for r in es_runs:
        (d / f"es_{r['name']}.json").write_text(json.dumps(r["program"]))
        (d / f"es_{r['name']}_space.json").write_text(json.dumps(r["space"]))
        arch = r["arch"]
        arch_arg = str(d / f"{arch}.toml") if arch in CUSTOM_ARCHS else arch
        if arch in CUSTOM_ARCHS:
            (d / f"{arch}.toml").write_text(CUSTOM_ARCHS[arch])
        p = r["params"]
        argv = ["search", str(d / f"es_{r['name']}.json"), str(d / f"es_{r['name']}_space.json"), "--arch", arch_arg,
                "--json", "--jobs", "1", "--top-k", "5", "--seed", str(p.get("seed", 0)),
                "--population", str(p.get("population", 32)), "--iterations", str(p.get("iterations", 100)),
                "--sigma", str(p.get("sigma", 0.3))]
        if p.get("rank_normalize") is False:
            argv.append("--no-rank-normalize")
        if "nvidia" in arch or "gpu" in arch:
            argv += ["--launch", str(d / "launch.json")]
        runs.append((f"search_{r['name']}", argv, f"search_{r['name']}_trace.csv"))
    manifest = []
    for name, argv, trace in runs:
        if trace:
            argv = argv + ["--trace", str(d / trace)]
        buf = io.StringIO()
        with contextlib.redirect_stdout(buf):
            code = ref_cli.main(argv)
        assert code == 0, (name, code)
        (d / f"{name}.out").write_text(buf.getvalue())
        rel = [a.replace(str(d) + "/", "{dir}/") for a in argv]
        manifest.append({"name": name, "argv": rel, "trace": trace})
    (d / "manifest.json").write_text(json.dumps(manifest, indent=1))
    print(f"cli: {len(manifest)} reference CLI runs")


def _mutate(rng: random.Random, text: str, target: str, kind: str) -> str:
    """A user-style edit of an emitted text (the reference decides what it means)."""
    lines = text.splitlines()
    if kind == "comments":
        out = []
        for ln in lines:
            r = rng.random()
            if r < 0.15:
                out.append(ln + ("  # note" if target != "gpu-ptx" else "  // note"))
            elif r < 0.25:
                out.append("")
                out.append(ln)
            elif r < 0.3:
                out.append("\t" + ln.strip() + "   ")
            else:
                out.append(ln)
        return "\n".join(out) + "\n"
    if kind == "extra":
        extra = {"cpu-x86": ["    xorq %rdx, %rdx", "    addq $8, %rsi", "    vmovups %zmm3, (%rdi)",
                             "    vfmadd231ps %zmm4, %zmm5, %zmm6", "    leaq 16(%rax,%rbx,4), %rcx"],
                 "cpu-aarch64": ["    add x3, x3, #1", "    ld1 {v4.4s}, [x5]", "    fmla v6.4s, v4.4s, v5.4s",
                                 "    st1 {v6.4s}, [x7]", "    mul x8, x8, x9"],
                 "gpu-ptx": ["    mov.u32 %r9, 7;", "    ld.global.f32 %f9, [%rd9];", "    fma.rn.f32 %f9, %f9, %f8, %f9;",
                             "    st.shared.f32 [%rd8], %f9;", "    mul.lo.s32 %r8, %r8, 3;"]}[target]
        out = list(lines)
        for _ in range(rng.randint(1, 6)):
            out.insert(rng.randint(0, len(out)), rng.choice(extra))
        return "\n".join(out) + "\n"
    if kind == "bound":
        idx = [i for i, ln in enumerate(lines) if ("cmp" in ln or "setp" in ln) and any(c.isdigit() for c in ln)]
        if idx:
            i = rng.choice(idx)
            import re as _re
            lines[i] = _re.sub(r"(\d+)(?!.*\d)", lambda m: str(int(m.group(1)) + rng.choice((1, 2, -1))), lines[i])
        return "\n".join(lines) + "\n"
    if kind == "join":  # a label and its first instruction on one line
        out, i = [], 0
        while i < len(lines):
            if lines[i].rstrip().endswith(":") and i + 1 < len(lines) and rng.random() < 0.5:
                out.append(lines[i].rstrip() + " " + lines[i + 1].strip())
                i += 2
            else:
                out.append(lines[i])
                i += 1
        return "\n".join(out) + "\n"
    if kind == "upper":
        out = []
        for ln in lines:
            parts = ln.split(None, 1)
            if parts and not parts[0].endswith(":") and rng.random() < 0.3:
                ln = ln.replace(parts[0], parts[0].upper(), 1)
            out.append(ln)
        return "\n".join(out) + "\n"
    if kind == "crlf":
        return "\r\n".join(lines) + "\r\n"
    if kind == "droplabel":
        idx = [i for i, ln in enumerate(lines) if ln.rstrip().endswith(":")]
        if idx:
            del lines[rng.choice(idx)]
        return "\n".join(lines) + "\n"
    return text


def code_fixture():
    """f4: extract_features(program, code, arch, launch) of the reference on emitted texts and on
    user-style edits of them (comments, blank lines, extra instructions, changed loop bounds,
    label + instruction lines, upper-case mnemonics, CRLF, a dropped label), plus the
    reference tests' own hand-written texts."""
    from loopscout.ir import serialize_program
    cases = []
    rng = random.Random(11)
    launch = L.KernelLaunch.from_json(LAUNCH)
    progs = dict(RANK_PROGRAMS)
    arches = {"cpu-x86": ["x86-avx2", "odd-x86"], "cpu-aarch64": ["aarch64-neon"], "gpu-ptx": ["nvidia-volta", "odd-gpu"]}
    for pname in ("matmul8", "nested4x8", "conv_small", "deep9", "smem_tid"):
        prog = L.parse_program(json.dumps(progs[pname]))
        for _ in range(5):
            s = random_schedule(rng, prog, kinds="TRVUP")
            try:
                q = L.apply_schedule(prog, L.Schedule.from_json(s))
            except Exception:  # noqa: BLE001
                continue
            for tgt, anames in arches.items():
                base = L.emit_mock_asm(q, tgt)
                if len(base) > 60000:
                    continue
                for kind in ("none", "comments", "extra", "bound", "join", "upper", "crlf", "droplabel"):
                    text = _mutate(rng, base, tgt, kind)
                    for an in anames:
                        arch = ref_arch(an)
                        entry = {"program": json.loads(serialize_program(q)), "arch": an, "kind": kind,
                                 "text": text}
                        try:
                            diag = []
                            fv = L.extract_features(q, text, arch, launch, diag)
                            entry["features"] = [[k, v] for k, v in fv.values]
                            entry["diagnostics"] = diag
                            entry["score"] = L.score(fv, arch)
                        except Exception as e:  # noqa: BLE001
                            entry["error"] = [type(e).__name__, str(e)]
                        cases.append(entry)
    # hand-written texts in the style of the reference's tests (ls tests/test_ptx.py, test_asm.py)
    single = L.parse_program(json.dumps({"tensors": [{"name": "A", "dims": [64]}],
                                         "body": [{"loop": {"var": "i", "extent": 8, "body": [
                                             {"access": {"tensor": "A", "kind": "load", "idx": ["i"]}}]}}]}))

    def countdown(init, delta, op, bound, body=""):
        return (f"    mov r1, {init}\n" "back:\n" f"{body}" f"    add r1, r1, {delta}\n"
                f"    setp.{op} r1, {bound}\n" "    bra back\n")
    body = "    fma.rn.f32 %f0, %f1, %f2, %f0\n" * 4 + "    ld.global.f32 %f3, [%rd1]\n" * 2
    hand = [countdown(0, 1, "lt", 8), countdown(4, 2, "lt", 16), countdown(0, 1, "le", 7), countdown(0, 2, "ne", 10),
            countdown(0, 3, "ne", 10), countdown(0, 1, "lt", 4, body), countdown(10, -1, "gt", 0, body),
            "    mov r1, 1\nback:\n    mul r1, r1, 2\n    setp.lt r1, 64\n    bra back\n",
            "back:\n    add r1, r1, 1\n    setp.lt r1, 8\n    bra back\n", "    ret\n", "", "   // only a comment\n",
            "    mov r1, 0\nback:\n    add r1, r1, 1\n    setp.lt %p1, r1, 8\n    @%p1 bra back\n    ret\n",
            "    mov r1, 0\nL0: add r1, r1, 1\n    setp.ge r1, 8\n    @!%p1 bra L0\n",
            "    jmp nowhere\n", "@p\n",
            "    mov r1, 0\nback:\n    add r1, r1, 1\n    setp.lt r1, r2\n    bra back\n",  # non-immediate bound
            countdown(10, 1, "lt", 4), countdown(0, 1, "gt", 8, body),  # inconsistent / consistent lt-gt
            "    mov r1, 0\nback:\n    add r1, r1, 3\n    setp r1, 8\n    bra back\n"]  # implicit "ne"
    xhand = ["    movq $0, %r8\n.L1:\n    vmovups (%rax), %zmm0\n    vfmadd231ps %zmm0, %zmm1, %zmm2\n"
             "    vmovups %zmm2, (%rcx)\n    addq $1, %r8\n    cmpq $8, %r8\n    jne .L1\n    ret\n",
             "    mov x0, #0\n.L1:\n    ld1 {v0.4s}, [x1]\n    fmla v2.4s, v0.4s, v1.4s\n    st1 {v2.4s}, [x2]\n"
             "    add x0, x0, #1\n    cmp x0, #8\n    b.ne .L1\n    ret\n",
             "    movq $0, %r8\n.L1:\n    addq $1, %r8\n    cmpq %r9, %r8\n    jne .L1\n    ret\n"]  # no bound
    for text in hand:
        for an in ("nvidia-volta", "odd-gpu"):
            entry = {"program": json.loads(serialize_program(single)), "arch": an, "kind": "hand", "text": text}
            try:
                diag = []
                fv = L.extract_features(single, text, ref_arch(an), launch, diag)
                entry["features"] = [[k, v] for k, v in fv.values]
                entry["diagnostics"] = diag
                entry["score"] = L.score(fv, ref_arch(an))
            except Exception as e:  # noqa: BLE001
                entry["error"] = [type(e).__name__, str(e)]
            cases.append(entry)
    for text, an in ((xhand[0], "x86-avx2"), (xhand[0], "odd-x86"), (xhand[1], "aarch64-neon"), (xhand[2], "x86-avx2")):
        entry = {"program": json.loads(serialize_program(single)), "arch": an, "kind": "hand", "text": text}
        try:
            diag = []
            fv = L.extract_features(single, text, ref_arch(an), launch, diag)
            entry["features"] = [[k, v] for k, v in fv.values]
            entry["diagnostics"] = diag
            entry["score"] = L.score(fv, ref_arch(an))
        except Exception as e:  # noqa: BLE001
            entry["error"] = [type(e).__name__, str(e)]
        cases.append(entry)
    (OUT / "code_analysis.json").write_text(json.dumps(cases, separators=(",", ":")))
    print(f"code: {len(cases)} (program, text, arch) cases, "
          f"{sum('error' in c for c in cases)} raise in the reference")


def inexact_fixture():
    """The cache model's inexact-footprint flag and notes (CacheModel.run -> NodeCost.inexact and
    CacheModel.diagnostics, ls/cache.py:198-202) of the reference on every rank-fixture schedule
    and on 160 schedules of each ResNet-50 task space ([flag, notes]; None: apply_schedule raises)."""
    from loopscout import cache as ref_cache
    from loopscout.ir import serialize_program
    from paper_2104_14641_b200.pack import SpaceTemplate
    rc = json.loads((OUT / "rank_cases.json").read_text())
    programs, cases = {}, []

    def flags(prog, scheds):
        out = []
        for s in scheds:
            try:
                q = L.apply_schedule(prog, L.Schedule.from_json(s))
            except Exception:  # noqa: BLE001
                out.append(None)
                continue
            model = ref_cache.analyze(q, ref_cache.CacheSpec(4096))
            out.append([bool(model.node_costs["<root>"].inexact), list(model.diagnostics)])
        return out
    for case in rc["cases"]:
        name = case["program"]
        programs[name] = rc["programs"][name]
        prog = L.parse_program(json.dumps(programs[name]))
        cases.append({"program": name, "schedules": case["schedules"], "inexact": flags(prog, case["schedules"])})
    rng = np.random.default_rng(8)
    for name, spec, space in W.resnet50_tasks():
        prog = L.parse_program(json.dumps(spec))
        st = SpaceTemplate(W.program(spec), space)
        idx = np.stack([rng.integers(0, n, 160) for n in st.sizes], axis=1)
        scheds = [st.schedule_of(row).to_json() for row in idx]
        programs[f"resnet_{name}"] = json.loads(serialize_program(prog))
        cases.append({"program": f"resnet_{name}", "schedules": scheds, "inexact": flags(prog, scheds)})
    (OUT / "inexact.json").write_text(json.dumps({"programs": programs, "cases": cases}, separators=(",", ":")))
    n = sum(len(c["inexact"]) for c in cases)
    t = sum(sum(1 for f in c["inexact"] if f and f[0]) for c in cases)
    print(f"inexact: {n} schedules, {t} inexact in the reference")


def main():
    OUT.mkdir(parents=True, exist_ok=True)
    for name in CUSTOM_ARCHS:  # write the TOMLs before the pool forks (no write races)
        ref_arch(name)
    which = set(sys.argv[1:]) or {"gemm", "conv", "bert", "rank", "trees", "emit", "es", "cli", "tree_rank",
                                  "resnet", "bertbench", "code", "inexact"}
    if "gemm" in which:
        space_fixture("gemm1024", W.matmul_json(1024), W.gemm_space(1024), 4096, 0,
                      ["x86-avx2", "aarch64-neon", "nvidia-volta"])
    if "conv" in which:
        space_fixture("conv56", W.conv2d_json(), W.conv_space(512, 1), 1024, 0,
                      ["x86-avx2", "aarch64-neon", "nvidia-volta"])
    if "bert" in which:
        for (m, n, k) in ((1024, 768, 768), (1024, 3072, 768), (1024, 768, 3072)):
            sp = {"tile": {"i": W.divisors(m)[:12], "j": W.divisors(n)[:12], "k": W.divisors(k)[:12]},
                  "reorder": W.random_perms(W.tiled_chain(["i", "j", "k"], ["i", "j", "k"]), 120, 9)}
            space_fixture(f"dense_{m}_{n}_{k}", W.matmul_json(m, n, k), sp, 256, 1,
                          ["x86-avx2", "nvidia-volta"])
        for (b, m, n, k) in ((96, 128, 128, 64), (96, 128, 64, 128)):
            sp = {"tile": {"b": W.divisors(b), "i": W.divisors(m), "j": W.divisors(n), "k": W.divisors(k)},
                  "reorder": W.random_perms(W.tiled_chain(["b", "i", "j", "k"], ["b", "i", "j", "k"]), 120, 10)}
            space_fixture(f"bmm_{b}_{m}_{n}_{k}", W.batch_matmul_json(b, m, n, k), sp, 256, 2,
                          ["x86-avx2", "nvidia-volta"])
    if "resnet" in which:
        # configs[2]: every ResNet-50 task space exactly as bench.py builds it (workloads.resnet50_tasks)
        for name, spec, space in W.resnet50_tasks():
            space_fixture(f"resnet_{name}", spec, space, 1024, 3, ["x86-avx2", "aarch64-neon", "nvidia-volta"])
    if "bertbench" in which:
        # configs[3]: the BERT spaces exactly as bench.py builds them (workloads.bert_tasks)
        for name, spec, space in W.bert_tasks():
            space_fixture(f"bert_{name}", spec, space, 1024, 4, ["x86-avx2", "aarch64-neon", "nvidia-volta"])
    if "rank" in which:
        rank_fixture()
    if "trees" in which:
        tree_fixture()
    if "emit" in which:
        emit_fixture()
    if "es" in which:
        es_fixture()
    if "cli" in which:
        cli_fixture()
    if "tree_rank" in which:
        tree_rank_fixture()
    if "code" in which:
        code_fixture()
    if "inexact" in which:
        inexact_fixture()


if __name__ == "__main__":
    main()
