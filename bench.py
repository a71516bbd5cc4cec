#!/usr/bin/env python
"""Throughput of the B200 batched schedule-cost path (BASELINE.json metric).

One step = score + rank (fused top-k) of this rank's batch of packed
candidate records of the ResNet-50 conv2d 56x56x64->64 3x3 search space
(BASELINE config 2), with records resident in HBM; for N>1 one NCCL
all-gather of the per-GPU top-k lists and the merge kernel follow.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

The reference arm (--impl reference) times the CPU restatement of the
reference algorithm (oracle/, C, all host threads) on a bounded sample of the
same workload; see DESIGN.md §6.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "candidate schedules scored+ranked/sec at 1/2/4/8 B200; % HBM roofline; top-k match"
UNIT = "candidates/s"
REORDERS = 4096  # 3136 tile points x 4096 chain orders = 12.8M distinct candidates (>= 8 x 2^20)
RECORD_BYTES = 32
POINT_BYTES = 4
PROFILE_JSON = "ncu_score_topk_r02_space.json"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["b200", "reference"], default="b200")
    ap.add_argument("--n", type=int, default=1 << 20, help="candidates per GPU per step")
    ap.add_argument("--k", type=int, default=64)
    ap.add_argument("--arch", default="x86-avx2")
    ap.add_argument("--no-baseline", action="store_true", help="skip the CPU baseline leg")
    ap.add_argument("--path", type=int, default=0, help="0 auto, 1 generic, 2 tabulated, 3 space-specialised")
    ap.add_argument("--workload", default="conv", choices=["conv", "gemm", "bert", "resnet50-es", "sweep"],
                    help="conv: BASELINE configs[1] (the headline); gemm: configs[0]; bert: configs[3]; "
                         "resnet50-es: configs[2]; sweep: configs[4]")
    ap.add_argument("--population", type=int, default=1 << 20, help="resnet50-es: ES population per generation")
    ap.add_argument("--generations", type=int, default=20, help="resnet50-es: generations per task")
    ap.add_argument("--sigma", type=float, default=2.0, help="resnet50-es: ES sigma")
    ap.add_argument("--es-streams", type=int, default=4, help="resnet50-es: concurrent task streams")
    return ap.parse_args()


def workload(arch_name: str):
    from paper_2104_14641_b200 import workloads as W
    from paper_2104_14641_b200.arch import KernelLaunch, load_arch
    from paper_2104_14641_b200.pack import SpaceTemplate

    st = SpaceTemplate(W.program(W.conv2d_json()), W.conv_space(REORDERS, 1))
    desc = st.template.desc(load_arch(arch_name), KernelLaunch.from_json(W.KERNEL_LAUNCH))
    return st, desc


def records_for(st, start: int, n: int, seed: int = 2104):
    from paper_2104_14641_b200 import workloads as W
    return st.records_from_indices(W.distinct_indices(st.sizes, n, seed, start=start))


def config_dict(args, n):
    return {"workload": "resnet50 conv2d 56x56x64->64 3x3 schedule space (tile ic/oc/oh/ow by divisors x "
                        f"{REORDERS} 11-loop orders = 12.8M points), {n} distinct packed candidates per GPU "
                        f"per step, score + top-{args.k} by (score, index)",
            "config": "BASELINE.json configs[1]", "arch": args.arch, "candidates_per_gpu": n, "k": args.k,
            "candidate_encoding": "space point (uint32 mixed-radix choice indices, 4 B)",
            "l2": "flushed between timed steps (256 MiB write)",
            "step": "one Task.score_topk_points call (Python API -> C-ABI) writing the k best + count into "
                    "preallocated output tensors (out=); steps enqueued back to back, each bracketed by its own "
                    "CUDA events after an L2 flush (device time; see sync_step_ms for host-synchronous calls)"}


# -- CPU baseline (the oracle port of the reference algorithm) ---------------------------------


def cpu_rate(desc, recs, threads: int, k: int = 64):
    """Oracle scoring of `recs` plus the cmd_rank ordering cut at k (ls/cli.py:124-126): the
    (score, index) sort of the valid candidates, timed together."""
    sys.path.insert(0, str(ROOT / "oracle"))
    import pyoracle
    t0 = time.perf_counter()
    s, f, st = pyoracle.evaluate(desc, recs, nthreads=threads)
    ok = np.nonzero(st == 0)[0]
    top = ok[np.lexsort((ok, s[ok]))][:k]
    dt = time.perf_counter() - t0
    return len(recs) / dt, dt, s, st


def calibrate_sample(desc, st, threads: int, target_s: float):
    recs = records_for(st, 0, 2048)
    rate, _, _, _ = cpu_rate(desc, recs, threads)
    return max(2048, int(rate * target_s) // 256 * 256)


def cpu_cores() -> int:
    return len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()


def reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    st, desc = workload(args.arch)
    threads = cpu_cores()
    m = calibrate_sample(desc, st, threads, 2.0)
    for w in range(args.warmup):
        cpu_rate(desc, records_for(st, w * m, m), threads)
    times = []
    for k in range(args.steps):
        total = int(np.prod(st.sizes))
        recs = records_for(st, ((args.warmup + k) * m) % (total - m), m)
        _, dt, _, _ = cpu_rate(desc, recs, threads)
        times.append(dt)
    value = m * args.steps / sum(times)
    sample = (f"{m} candidates per step of the same conv2d workload, oracle/oracle.c (C restatement of "
              f"the reference path) on {threads} threads of a {cpu_model()}, scoring + (score, index) "
              f"sort of the top {args.k}")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * sum(times) / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int64+f64",
            "data": "synthetic", "config": config_dict(args, m),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port", "sample": sample,
                             "cpu_model": cpu_model()},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def points_parity(task, st, desc, pts: np.ndarray, k: int, torch, threads: int) -> dict:
    """Bit-exact check of the device scores, status and top-k of `pts` (one task) against the
    oracle (oracle/oracle.c, run after the timed region)."""
    sys.path.insert(0, str(ROOT / "oracle"))
    import pyoracle
    recs = st.records_from_indices(st.indices_from_points(pts))
    cs, _, cst = pyoracle.evaluate(desc, recs, nthreads=threads)
    d = torch.from_numpy(pts.astype(np.uint32).view(np.int32)).to(task.device)
    gs, _, gst = task.score_points(d, features=False)
    _, ti, _ = task.score_topk_points(d, k)
    torch.cuda.synchronize()
    ok = cst == 0
    want = np.nonzero(ok)[0][np.lexsort((np.nonzero(ok)[0], cs[ok]))][:k]
    return {"sample": int(len(pts)),
            "scores_bit_exact": bool(np.array_equal(np.where(ok, gs.cpu().numpy(), 0.0), np.where(ok, cs, 0.0))),
            "status_equal": bool(np.array_equal(gst.cpu().numpy(), cst)),
            "topk_identical": ti.cpu().numpy()[:len(want)].tolist() == want.tolist()}


def merge_parity(parts: list) -> dict:
    return {"sample": sum(p["sample"] for p in parts),
            "scores_bit_exact": all(p["scores_bit_exact"] for p in parts),
            "status_equal": all(p["status_equal"] for p in parts),
            "topk_identical": all(p["topk_identical"] for p in parts), "per_task": len(parts)}


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def init_dist(torch, dist, local: int):
    """One process per GPU over NCCL.  LS_BENCH_SHARED_GPU=1 (a test hook for the multi-rank code
    paths on a one-GPU box) puts every rank on GPU 0 and uses gloo (NCCL refuses two ranks on one
    device); the exchanged top-k lists are staged through host memory (dist.all_gather_inplace)."""
    if os.environ.get("LS_BENCH_SHARED_GPU") == "1":
        torch.cuda.set_device(0)
        dist.init_process_group("gloo")
    else:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))


# -- clocks -------------------------------------------------------------------------------------


class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 6:
                self.rows.append(parts)

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(2)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[2 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


# -- B200 arm ------------------------------------------------------------------------------------


def _timed(step, steps, flush, stream, torch, sync_each: bool = False):
    """Device time of `steps` calls of step(), each preceded by an L2 flush (outside its events).

    The steps are enqueued back to back (the host runs ahead, as a pipelined caller does), so
    each step's events bracket its device work only; sync_each=True synchronises the host
    before every step instead, exposing the per-call host/launch latency too."""
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    kev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    torch.cuda.synchronize()
    for j in range(steps):
        flush.zero_()
        if sync_each:
            torch.cuda.synchronize()
        ev[j][0].record(stream)
        step(kev[j])
        ev[j][1].record(stream)
    torch.cuda.synchronize()
    try:
        kms = [a.elapsed_time(b) for a, b in kev]
    except (ValueError, RuntimeError):  # the step does not bracket a single kernel
        kms = None
    return [a.elapsed_time(b) for a, b in ev], kms


def b200_arm(args):
    import torch
    import torch.distributed as dist

    from paper_2104_14641_b200.build import build
    from paper_2104_14641_b200.dist import gather_topk
    from paper_2104_14641_b200.engine import Task, to_device_records
    from paper_2104_14641_b200 import workloads as W

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        init_dist(torch, dist, local)
    else:
        torch.cuda.set_device(0)
    if rank == 0:
        build()
    if world > 1:
        dist.barrier()
    dev = torch.cuda.current_device()
    n, k = args.n, args.k
    st, desc = workload(args.arch)
    task = Task(desc, dev)
    if args.path:
        task.set_path(args.path)
    task.set_space(st.space_desc())
    idx = W.distinct_indices(st.sizes, n, 2104, start=rank * n)
    recs = st.records_from_indices(idx)
    pts = st.points_from_indices(idx)
    assert pts.dtype == np.uint32
    d_rec = to_device_records(recs, dev)
    d_pts = torch.from_numpy(pts.view(np.int32)).to(dev)
    base = rank * n
    # the host-buffer (e2e) call ships packed 3-byte points when the space has < 2^24 of them
    # (pack.pack_points; a quarter less over the host link than 4-byte points)
    from paper_2104_14641_b200.pack import pack_points
    e2e_pbytes = 3 if int(np.prod(st.sizes)) <= (1 << 24) else 4
    pinned_pts = (torch.from_numpy(pack_points(pts, 3)) if e2e_pbytes == 3
                  else torch.from_numpy(pts.view(np.int32))).pin_memory()
    pinned_rec = torch.from_numpy(recs.view(np.uint8).reshape(-1, RECORD_BYTES)).pin_memory()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream()

    def make_step(points: bool):
        # steady-state caller: the k best + count land in the same output tensors every step (out=)
        out = (torch.empty(k, dtype=torch.float64, device=dev), torch.empty(k, dtype=torch.int64, device=dev),
               torch.empty(1, dtype=torch.int64, device=dev))

        def step(kev=None):
            if kev:
                kev[0].record(stream)
            if points:
                s, i, nv = task.score_topk_points(d_pts, k, base_index=base, out=out)
            else:
                s, i, nv = task.score_topk(d_rec, k, base_index=base, out=out)
            if kev:
                kev[1].record(stream)
            if world > 1:
                s, i = gather_topk(s, i, k)
            step.out = (s, i, nv)
        return step

    step_p, step_r = make_step(True), make_step(False)
    for _ in range(max(3, args.warmup)):
        step_p()
        step_r()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()

    def max_over_ranks(ms):
        t = torch.tensor([ms], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return t.item()

    # ---- device-resident throughput (value: points; records as a secondary line item) ----
    with ClockSampler(dev) as clk:
        t_soak = time.perf_counter()  # keep the GPU loaded while nvidia-smi starts sampling
        while time.perf_counter() - t_soak < 1.5:
            step_p()
            torch.cuda.synchronize()
        step_ms, kern_ms = _timed(step_p, args.steps, flush, stream, torch)
        rstep_ms, rkern_ms = _timed(step_r, args.steps, flush, stream, torch)
        sync_ms, _ = _timed(step_p, args.steps, flush, stream, torch, sync_each=True)
    if world > 1:
        dist.barrier()
    total_s = max_over_ranks(sum(step_ms)) / 1e3
    sync_step_ms = max_over_ranks(sum(sync_ms)) / args.steps  # host-synchronous call (launch latency exposed)
    value = world * n * args.steps / total_s
    value_rec = world * n * args.steps / (max_over_ranks(sum(rstep_ms)) / 1e3)
    top_i = step_p.out[1].cpu().numpy()
    n_valid = int(step_p.out[2].item())
    same_paths = top_i.tolist() == step_r.out[1].cpu().tolist()

    # ---- end to end through the C-ABI host-buffer calls (H2D + top-k D2H inside the timed region) ----
    def e2e(call, reps):
        for _ in range(2):
            call()
        ms = []
        for _ in range(reps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            a.record(stream)
            hs, hi, hnv = call()
            if world > 1:
                gs, gi = gather_topk(torch.from_numpy(hs).to(dev), torch.from_numpy(hi).to(dev), k)
                hi = gi.cpu().numpy()
            b.record(stream)
            torch.cuda.synchronize()
            ms.append(a.elapsed_time(b))
        return world * n / (max_over_ranks(sum(ms) / len(ms)) / 1e3), hi

    reps = max(3, args.steps // 2)
    h_out = (np.empty(k, np.float64), np.empty(k, np.int64), np.zeros(1, np.int64))
    e2e_value, e2e_top = e2e(lambda: task.score_topk_points_host(pinned_pts, k, base_index=base, out=h_out), reps)
    e2e_top = e2e_top.copy()
    e2e_rec, e2e_rtop = e2e(lambda: task.score_topk_host(pinned_rec, k, base_index=base), reps)

    # ---- roofline of the fused launch ----
    peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) if (ROOT / "MEASURED_PEAKS.json").exists() else {}
    peak = peaks.get("hbm_gbs", 6650.0)
    peak_src = "measured (MEASURED_PEAKS.json hbm_gbs)" if "hbm_gbs" in peaks else "fallback (B200_PROFILING.md)"
    kavg = sum(kern_ms) / len(kern_ms) / 1e3
    alg_bytes = n * POINT_BYTES
    achieved = alg_bytes / kavg / 1e9
    traffic, issue = None, None
    prof = ROOT / "profiles" / PROFILE_JSON
    if prof.exists():
        try:
            pj = json.loads(prof.read_text())
            traffic = pj.get("dram_bytes_per_launch")
            slots = pj.get("warp_issue_slots_per_candidate")
            if slots:
                clk_mhz = peaks.get("sm_max_mhz", 1965.0)
                ceil = 4 * 148 * clk_mhz * 1e6 / slots
                issue = {"bound": "issue", "warp_issue_slots_per_candidate": slots,
                         "ceiling_candidates_per_s": ceil, "achieved_candidates_per_s": n / kavg,
                         "frac": n / kavg / ceil, "source": f"profiles/{PROFILE_JSON} (ncu) + live kernel time"}
        except ValueError:
            pass

    line = None
    if rank == 0:
        # ---- CPU baseline + parity on the same sample ----
        cpu = None
        parity = None
        if not args.no_baseline:
            threads = cpu_cores()
            m = calibrate_sample(desc, st, threads, 10.0)
            sidx = W.distinct_indices(st.sizes, m, 2104)
            sample = st.records_from_indices(sidx)
            rate, dt, cs, cst = cpu_rate(desc, sample, threads)
            cpu = {"value": rate, "unit": UNIT, "cores": threads, "kind": "port", "cpu_model": cpu_model(),
                   "sample": f"{m} candidates of the same workload through oracle/oracle.c (C restatement of "
                             f"the reference path) on {threads} threads, scoring + (score, index) sort of "
                             f"the top {k}, {dt:.1f} s"}
            dsp = torch.from_numpy(st.points_from_indices(sidx).view(np.int32)).to(dev)
            gs, _, gst = task.score_points(dsp, features=False)
            ts, ti, _ = task.score_topk_points(dsp, k)
            torch.cuda.synchronize()
            want = sorted(range(m), key=lambda q: (cs[q], q))[:k]
            parity = {"sample": m, "scores_bit_exact": bool(np.array_equal(gs.cpu().numpy(), cs)),
                      "status_equal": bool(np.array_equal(gst.cpu().numpy(), cst)),
                      "topk_identical": ti.cpu().tolist() == want}
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": total_s * 1e3 / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "int64+f64", "data": "synthetic",
            "config": config_dict(args, n),
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": n * e2e_pbytes,
                    "d2h_bytes_per_step": k * 16 + 8,
                    "path": f"ls_score_topk_points_host (C-ABI): {e2e_pbytes}-byte space points in pinned, mapped "
                            "host memory, read by the scoring kernel over the host link (the H2D transfer inside the "
                            "kernel, no staging copy); the k best + count written by the kernel into pinned host "
                            "memory (no D2H copy)",
                    "topk_equals_device_path": e2e_top.tolist() == top_i.tolist() if world == 1 else None},
            "records_path": {"value": value_rec, "e2e": e2e_rec, "record_bytes": RECORD_BYTES,
                             "path": "ls_score_topk / ls_score_topk_host over 32-byte ls_record (rank path)",
                             "topk_equals_points_path": same_paths and e2e_rtop.tolist() == top_i.tolist()},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic, "peak_source": peak_src,
                         "kernel": "score_topk_kernel<3,4,5,1> (space path: point decode + fused 32-bit walk/closed forms + "
                                   "block radix-select top-k + in-kernel minima-bound merge); one ls_score_topk_points "
                                   "call, one launch",
                         "kernel_ms": kavg * 1e3, "algorithmic_bytes_per_launch": alg_bytes,
                         "note": "instruction-issue bound by design (4 B read per candidate vs thousands of "
                                 "integer ops): see issue_roofline"},
            "issue_roofline": issue,
            "cpu_baseline": cpu, "parity": parity,
            "clocks": clk.summary(),
            # per step: the fused kernel (score + top-k + merge in one launch), and for N > 1 the
            # all-gathered lists' lists_to_keys + merge_keys kernels (the memsets are not ours)
            "gpu_launches": args.steps * (1 + (2 if world > 1 else 0)),
            "sync_step_ms": sync_step_ms,
            "n_valid_per_gpu": n_valid, "path": task.path, "points_path": task.points_path,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    task.close()


# -- extra workloads (BASELINE configs 3-5; the headline is `conv`) ----------------------------------


def _dist_setup(torch, dist):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        init_dist(torch, dist, local)
    else:
        torch.cuda.set_device(0)
    if rank == 0:
        from paper_2104_14641_b200.build import build
        build()
    if world > 1:
        dist.barrier()
    return world, rank, torch.cuda.current_device()


def _max_ms(torch, dist, world, dev, ms):
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return t.item()


def _emit(line, world, dist):
    if int(os.environ.get("RANK", "0")) == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def bert_arm(args):
    """configs[3]: BERT-base dense + batch_matmul tasks, 2^22 distinct candidates per generation
    (spread over the 5 tasks, each sharded across ranks), fused score + top-k per task."""
    import torch
    import torch.distributed as dist
    from paper_2104_14641_b200 import workloads as W
    from paper_2104_14641_b200.arch import KernelLaunch, load_arch
    from paper_2104_14641_b200.dist import gather_topk
    from paper_2104_14641_b200.engine import Task
    from paper_2104_14641_b200.pack import SpaceTemplate
    world, rank, dev = _dist_setup(torch, dist)
    tasks = W.bert_tasks()
    total = 1 << 22
    jobs = []
    for j, (name, spec, space) in enumerate(tasks):
        st = SpaceTemplate(W.program(spec), space)
        n_task = min(total // len(tasks), int(st.size)) // world
        task = Task(st.template.desc(load_arch(args.arch), KernelLaunch.from_json(W.KERNEL_LAUNCH)), dev)
        task.set_space(st.space_desc())
        pts = st.points_from_indices(W.distinct_indices(st.sizes, n_task, 40 + j, start=rank * n_task))
        jobs.append((name, task, torch.from_numpy(pts.view(np.int32)).to(dev), n_task, task.points_path))
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream()
    # the five tasks of a generation run concurrently, one stream each (their launch ramps and
    # merge tails overlap); the step joins them back onto the timing stream
    side = [torch.cuda.Stream(device=dev) for _ in jobs]
    outs = [(torch.empty(args.k, dtype=torch.float64, device=dev), torch.empty(args.k, dtype=torch.int64, device=dev),
             torch.empty(1, dtype=torch.int64, device=dev)) for _ in jobs]

    def step():
        start = torch.cuda.Event()
        start.record(stream)
        for (name, task, d, n_task, _), ss, out in zip(jobs, side, outs):
            ss.wait_event(start)
            task.score_topk_points(d, args.k, base_index=rank * n_task, stream=ss, out=out)
        for ss in side:
            stream.wait_stream(ss)
        if world > 1:
            for s, i, _ in outs:
                gather_topk(s, i, args.k)
    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()
    with ClockSampler(dev) as clk:
        t_soak = time.perf_counter()  # keep the GPU loaded while nvidia-smi starts sampling
        while time.perf_counter() - t_soak < 1.5:
            step()
            torch.cuda.synchronize()
        ms, _ = _timed(lambda kev=None: step(), args.steps, flush, stream, torch)
    per_step = sum(n for _, _, _, n, _ in jobs) * world
    tot = _max_ms(torch, dist, world, dev, sum(ms)) / 1e3
    parity = None
    if rank == 0 and not args.no_baseline:  # bit-exact vs the oracle on 4096 of each task's points
        parts = []
        for j, ((name, spec, space), (_, task, d, n_task, _)) in enumerate(zip(tasks, jobs)):
            st = SpaceTemplate(W.program(spec), space)
            desc = st.template.desc(load_arch(args.arch), KernelLaunch.from_json(W.KERNEL_LAUNCH))
            pts = d[:4096].cpu().numpy().view(np.uint32).astype(np.uint64)
            parts.append(points_parity(task, st, desc, pts, args.k, torch, cpu_cores()))
        parity = merge_parity(parts)
    line = {"metric": METRIC, "value": per_step * args.steps / tot, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": tot * 1e3 / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int64+f64",
            "data": "synthetic",
            "config": {"workload": "BERT-base (seq 128, batch 8) dense 1024x768x768 / 1024x3072x768 / "
                                   "1024x768x3072 + batch_matmul 96x128x128x64 / 96x128x64x128 schedule spaces "
                                   "(divisor tiles x chain orders), 2^22 distinct candidates per generation, "
                                   f"score + top-{args.k} per task (the 5 tasks on concurrent streams)",
                       "config": "BASELINE.json configs[3]",
                       "arch": args.arch, "candidates_per_step": per_step, "k": args.k,
                       "tasks": {name: {"candidates_per_gpu": n, "points_path": pp} for name, _, _, n, pp in jobs},
                       "l2": "flushed between timed steps (256 MiB write)"},
            "clocks": clk.summary(), "gpu_launches": args.steps * len(jobs) * (1 + (2 if world > 1 else 0)),
            "parity": parity}
    for _, task, _, _, _ in jobs:
        task.close()
    _emit(line, world, dist)


def resnet_es_arm(args):
    """configs[2]: the ResNet-50 task set, a `generations`-generation ES per task with every
    generation on the device (Philox noise, decode, memo, scoring, rank sort, update); tasks
    round-robin over ranks."""
    import torch
    import torch.distributed as dist
    from paper_2104_14641_b200 import workloads as W
    from paper_2104_14641_b200.arch import KernelLaunch, load_arch
    from paper_2104_14641_b200.engine import EsRun, Task
    from paper_2104_14641_b200.pack import SpaceTemplate
    world, rank, dev = _dist_setup(torch, dist)
    tasks = W.resnet50_tasks()
    mine = [t for j, t in enumerate(tasks) if j % world == rank]
    runs = []
    for name, spec, space in mine:
        st = SpaceTemplate(W.program(spec), space)
        task = Task(st.template.desc(load_arch(args.arch), KernelLaunch.from_json(W.KERNEL_LAUNCH)), dev)
        task.set_space(st.space_desc())
        run = EsRun(task, 0.05, args.sigma, args.population, args.generations, 2104)
        runs.append((name, st, task, run))
    stream = torch.cuda.current_stream()
    # tasks on concurrent streams (round-robin): one task's latency-bound sort passes and
    # launch gaps overlap another's scoring; the step joins them back onto the timing stream
    side = [torch.cuda.Stream(device=dev) for _ in range(max(1, min(args.es_streams, len(runs))))]

    def step():
        start = torch.cuda.Event()
        start.record(stream)
        for ss in side:
            ss.wait_event(start)
        for j, (_, _, _, run) in enumerate(runs):
            run.run(stream=side[j % len(side)])
        for ss in side:
            stream.wait_stream(ss)
    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    with ClockSampler(dev) as clk:
        ms, _ = _timed(lambda kev=None: step(), args.steps, flush, stream, torch)
    distinct = 0
    paths = {}
    parts = []
    for name, st, task, run in runs:
        _, trace, ev, err, best = run.result(st.dim)
        assert err == 0, (name, err)
        distinct += ev
        paths[name] = task.points_path
        if not args.no_baseline:  # the memo's scores (every distinct schedule scored) vs the oracle
            sys.path.insert(0, str(ROOT / "oracle"))
            import pyoracle
            pts, sc = run.evaluated()
            sel = np.linspace(0, len(pts) - 1, min(len(pts), 1024)).astype(np.int64)
            desc = task.desc
            recs = st.records_from_indices(st.indices_from_points(pts[sel]))
            cs, _, cst = pyoracle.evaluate(desc, recs, nthreads=cpu_cores())
            parts.append({"sample": int(len(sel)), "scores_bit_exact": bool(np.array_equal(sc[sel], cs)),
                          "status_equal": bool((cst == 0).all()),
                          # the incumbent (best score) is the minimum over the evaluated schedules
                          "topk_identical": bool(len(sc) > 0 and float(np.min(sc)) == float(best))})
    parity = merge_parity(parts) if parts else None
    dt = torch.tensor([distinct], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(dt)
    tot = _max_ms(torch, dist, world, dev, sum(ms)) / 1e3
    members = len(tasks) * args.generations * args.population
    line = {"metric": "ES population members scored+ranked/sec (configs[2]: ResNet-50 task set, on-device ES)",
            "value": members * args.steps / tot, "unit": "members/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": tot * 1e3 / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "int64+f64", "data": "synthetic",
            "distinct_schedules_per_s": float(dt.item()) * args.steps / tot,
            "config": {"workload": f"ResNet-50 v1.5 conv/dense task set ({len(tasks)} tasks), "
                                   f"{args.generations}-generation ES per task, population {args.population}, "
                                   f"sigma {args.sigma}, every generation on device (Philox noise, decode, memo, "
                                   "score, onesweep radix rank sort, update; one CUDA graph per generation; "
                                   f"tasks on {len(side)} concurrent streams)",
                       "config": "BASELINE.json configs[2]", "arch": args.arch,
                       "distinct_schedules_per_step": float(dt.item()), "points_paths": paths,
                       "l2": "flushed between timed steps (256 MiB write)"},
            "clocks": clk.summary(), "gpu_launches": args.steps * len(mine) * (1 + 4 * args.generations),
            "parity": parity}
    for _, _, task, run in runs:
        run.close()
        task.close()
    _emit(line, world, dist)


def gemm_arm(args):
    """configs[0]: one GEMM 1024^3 task, 4096 random tile/reorder candidates scored and ranked
    top-64.  `value`: the fused launch over 4096 device-resident points; `e2e`: the reference-facing
    rank API from the reference's own Schedule objects (cost.rank_topk: host packing, H2D of the
    packed records, the fused launch, D2H of the k best; cmd_rank's seam ls/cli.py:106-141)."""
    import torch
    import torch.distributed as dist
    from paper_2104_14641_b200 import cost
    from paper_2104_14641_b200 import workloads as W
    from paper_2104_14641_b200.arch import KernelLaunch, load_arch
    from paper_2104_14641_b200.engine import Task
    from paper_2104_14641_b200.pack import SpaceTemplate
    world, rank, dev = _dist_setup(torch, dist)
    prog = W.program(W.matmul_json(1024))
    st = SpaceTemplate(prog, W.gemm_space(1024))
    arch, launch = load_arch(args.arch), KernelLaunch.from_json(W.KERNEL_LAUNCH)
    desc = st.template.desc(arch, launch)
    task = Task(desc, dev)
    task.set_space(st.space_desc())
    n = 4096
    idx = W.distinct_indices(st.sizes, n, 1024 + rank)
    schedules = [st.schedule_of(row) for row in idx]
    pts = st.points_from_indices(idx)
    d = torch.from_numpy(pts.view(np.int32)).to(dev)
    out = (torch.empty(args.k, dtype=torch.float64, device=dev), torch.empty(args.k, dtype=torch.int64, device=dev),
           torch.empty(1, dtype=torch.int64, device=dev))
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream()

    def step(kev=None):
        task.score_topk_points(d, args.k, out=out)
    for _ in range(max(3, args.warmup)):
        step()
        cost.rank_topk(prog, schedules, arch, args.k, launch, dev)
    torch.cuda.synchronize()
    with ClockSampler(dev) as clk:
        ms, _ = _timed(step, args.steps, flush, stream, torch)
        e2e_ms = []
        for _ in range(args.steps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            a.record(stream)
            rs, ri, rnv = cost.rank_topk(prog, schedules, arch, args.k, launch, dev)
            b.record(stream)
            torch.cuda.synchronize()
            e2e_ms.append(a.elapsed_time(b))
    tot = _max_ms(torch, dist, world, dev, sum(ms)) / 1e3
    e2e_tot = _max_ms(torch, dist, world, dev, sum(e2e_ms)) / 1e3
    # the same rank API over a long list: 2^19 of the space's 958 320 schedules as Schedule objects
    big = None
    if rank == 0:
        bidx = W.distinct_indices(st.sizes, 1 << 19, 77)
        bsched = [st.schedule_of(row) for row in bidx]
        cost.rank_topk(prog, bsched[:4096], arch, args.k, launch, dev)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        cost.rank_topk(prog, bsched, arch, args.k, launch, dev)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        big = {"candidates": len(bsched), "value": len(bsched) / dt, "unit": UNIT, "wall_s": dt,
               "path": "cost.rank_topk over 2^19 Schedule objects (host wall clock: native packer + H2D + fused "
                       "launch + D2H); the host packer bounds it"}
        del bsched
    parity = None
    if rank == 0 and not args.no_baseline:  # every candidate vs the oracle; the rank API's top-k
        sys.path.insert(0, str(ROOT / "oracle"))
        import pyoracle
        cs, _, cst = pyoracle.evaluate(desc, st.records_from_indices(idx), nthreads=cpu_cores())
        ok = np.nonzero(cst == 0)[0]
        want = ok[np.lexsort((ok, cs[ok]))][:args.k]
        gs, _, gst = task.score_points(d, features=False)
        torch.cuda.synchronize()
        parity = {"sample": n, "scores_bit_exact": bool(np.array_equal(gs.cpu().numpy()[ok], cs[ok])),
                  "status_equal": bool(np.array_equal(gst.cpu().numpy(), cst)),
                  "topk_identical": out[1].cpu().tolist()[:len(want)] == want.tolist()
                  and ri.tolist()[:len(want)] == want.tolist()}
    line = {"metric": METRIC, "value": world * n * args.steps / tot, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": tot * 1e3 / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int64+f64",
            "data": "synthetic",
            "config": {"workload": "single GEMM 1024x1024x1024 task: 4096 random tile (divisors of 1024 for i/j/k) "
                                   "x 720 chain-order candidates scored and top-64 ranked",
                       "config": "BASELINE.json configs[0]", "arch": args.arch, "candidates_per_gpu": n,
                       "k": args.k, "l2": "flushed between timed steps (256 MiB write)",
                       "step": "value: one Task.score_topk_points launch over 4096 device-resident points"},
            "e2e": {"value": world * n * args.steps / e2e_tot, "unit": UNIT,
                    "h2d_bytes_per_step": n * RECORD_BYTES, "d2h_bytes_per_step": args.k * 16 + 8,
                    "path": "cost.rank_topk(program, [Schedule] * 4096, arch, 64): the reference's Schedule "
                            "objects packed on the host (native packer), 32-byte records H2D, the fused "
                            "launch, the k best D2H", "ms_per_step": e2e_tot * 1e3 / args.steps},
            "rank_list": big, "clocks": clk.summary(), "gpu_launches": args.steps, "parity": parity}
    task.close()
    _emit(line, world, dist)


def sweep_arm(args):
    """configs[4]: n = 2^20 .. 2^26 distinct conv candidates per step, sharded over the ranks
    (strong scaling per n), fused score + top-k + all-gather merge; one line with every n."""
    import torch
    import torch.distributed as dist
    from paper_2104_14641_b200 import workloads as W
    from paper_2104_14641_b200.arch import KernelLaunch, load_arch
    from paper_2104_14641_b200.dist import gather_topk
    from paper_2104_14641_b200.engine import Task
    from paper_2104_14641_b200.pack import SpaceTemplate
    world, rank, dev = _dist_setup(torch, dist)
    st = SpaceTemplate(W.program(W.conv2d_json()), W.conv_space(21504, 1))  # 3136 x 21504 > 2^26 points
    task = Task(st.template.desc(load_arch(args.arch), KernelLaunch.from_json(W.KERNEL_LAUNCH)), dev)
    task.set_space(st.space_desc())
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream()
    rows = []
    sweep_parity = None
    for e in range(20, 27):
        n = (1 << e) // world
        pts = st.points_from_indices(W.distinct_indices(st.sizes, n, 2104, start=rank * n))
        d = torch.from_numpy(pts.view(np.int32)).to(dev)
        del pts

        def step(kev=None):
            s, i, nv = task.score_topk_points(d, args.k, base_index=rank * n)
            if world > 1:
                gather_topk(s, i, args.k)
        for _ in range(3):
            step()
        torch.cuda.synchronize()
        steps = max(3, args.steps // 4)
        ms, _ = _timed(step, steps, flush, stream, torch)
        tot = _max_ms(torch, dist, world, dev, sum(ms)) / 1e3
        rows.append({"n": 1 << e, "value": (1 << e) * steps / tot, "ms_per_step": tot * 1e3 / steps})
        if e == 26 and rank == 0 and not args.no_baseline:  # bit-exact vs the oracle on a sample
            sample = d[: 1 << 12].cpu().numpy().view(np.uint32).astype(np.uint64)
            desc = st.template.desc(load_arch(args.arch), KernelLaunch.from_json(W.KERNEL_LAUNCH))
            sweep_parity = points_parity(task, st, desc, sample, args.k, torch, cpu_cores())
        del d
    peak = max(r["value"] for r in rows)
    line = {"metric": METRIC, "value": rows[-1]["value"], "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": rows[-1]["ms_per_step"], "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "int64+f64", "data": "synthetic",
            "config": {"workload": "resnet50 conv2d 56x56x64->64 3x3 space with 21504 chain orders (67.4M points); "
                                   "n = 2^20..2^26 distinct candidates per step sharded over the GPUs, "
                                   f"score + top-{args.k}", "config": "BASELINE.json configs[4]", "arch": args.arch,
                       "l2": "flushed between timed steps (256 MiB write)"},
            "sweep": rows, "peak_value": peak, "gpu_launches": sum(max(3, args.steps // 4) for _ in rows),
            "parity": sweep_parity}
    task.close()
    _emit(line, world, dist)


def main():
    args = parse()
    if args.impl == "reference":
        reference_arm(args)
    elif args.workload == "gemm":
        gemm_arm(args)
    elif args.workload == "bert":
        bert_arm(args)
    elif args.workload == "resnet50-es":
        resnet_es_arm(args)
    elif args.workload == "sweep":
        sweep_arm(args)
    else:
        b200_arm(args)


if __name__ == "__main__":
    main()
