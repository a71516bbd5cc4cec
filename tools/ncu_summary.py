"""Summarise an ncu --set full report of the scoring kernel into profiles/*.json.

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep profiles/ncu_score_topk_r01.json [n_candidates [bytes_per_candidate]]

bytes_per_candidate: 4 for space points (the bench headline), 32 for ls_record (default).

Reads the report here (no GPU needed): duration, DRAM bytes per launch (the
`traffic` of bench.py's roofline), issue/occupancy/divergence counters and
the warp-stall breakdown.
"""

import csv
import io
import json
import subprocess
import sys


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units, vals = rows[0], rows[1], rows[2]
    return {n: (v, u) for n, u, v in zip(h, units, vals)}


def num(x):
    try:
        return float(x.replace(",", ""))
    except ValueError:
        return None


def to_bytes(v, u):
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}
    return v * scale.get(u, 1)


def main():
    rep, out = sys.argv[1], sys.argv[2]
    n = int(sys.argv[3]) if len(sys.argv) > 3 else None
    bpc = int(sys.argv[4]) if len(sys.argv) > 4 else 32
    m = raw(rep)
    g = lambda k: num(m[k][0]) if k in m else None  # noqa: E731
    rd = to_bytes(g("dram__bytes_read.sum"), m["dram__bytes_read.sum"][1])
    wr = to_bytes(g("dram__bytes_write.sum"), m["dram__bytes_write.sum"][1])
    dur_ns = g("gpu__time_duration.sum")
    dur_ns *= {"us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6, "s": 1e9, "second": 1e9}.get(
        m["gpu__time_duration.sum"][1], 1.0)
    stalls = {k.replace("smsp__pcsamp_warps_issue_stalled_", ""): g(k) for k in m
              if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")}
    tot = sum(v for v in stalls.values() if v) or 1
    summary = {
        "kernel": m.get("Kernel Name", ("?", ""))[0],
        "grid": m.get("launch__grid_size", ("?", ""))[0],
        "block": m.get("launch__block_size", ("?", ""))[0],
        "duration_us": dur_ns / 1e3 if dur_ns else None,
        "dram_bytes_read": rd, "dram_bytes_write": wr, "dram_bytes_per_launch": rd + wr,
        "registers_per_thread": g("launch__registers_per_thread"),
        "dynamic_smem_per_block": m.get("launch__shared_mem_per_block_dynamic", ("?", ""))[0],
        "achieved_occupancy_pct": g("sm__warps_active.avg.pct_of_peak_sustained_active"),
        "issue_slots_busy_pct": g("sm__inst_issued.avg.pct_of_peak_sustained_active"),
        "ipc_active": g("sm__inst_executed.avg.per_cycle_active"),
        "warp_instructions": g("smsp__inst_executed.sum"),
        "thread_instructions": g("thread_inst_executed"),
        "avg_active_threads_per_warp": g("smsp__thread_inst_executed_per_inst_executed.ratio"),
        "avg_predicated_on_threads_per_warp": g("smsp__thread_inst_executed_pred_on_per_inst_executed.ratio"),
        "dram_throughput_pct": g("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
        "stall_share": {k: round(v / tot, 4) for k, v in sorted(stalls.items(), key=lambda kv: -(kv[1] or 0))
                        if v},
    }
    if n:
        summary["candidates_per_launch"] = n
        summary["algorithmic_bytes_per_launch"] = bpc * n
        wi = (g("smsp__inst_executed.sum") or 0) / n
        summary["warp_issue_slots_per_candidate"] = wi
        summary["thread_instructions_per_candidate"] = (g("thread_inst_executed") or 0) / n
        # issue-bound ceiling: 4 warp-instructions per cycle per SM
        summary["issue_roofline_candidates_per_s"] = 148 * 4 * 1.965e9 / wi if wi else None
        if summary["duration_us"]:
            summary["candidates_per_s_under_ncu"] = n / (summary["duration_us"] * 1e-6)
    with open(out, "w") as f:
        json.dump(summary, f, indent=1)
    print(json.dumps(summary, indent=1))


if __name__ == "__main__":
    main()
