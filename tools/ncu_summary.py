#!/usr/bin/env python
"""Summarise ncu outputs into profiles/ (run here, on the CPU box).

  python tools/ncu_summary.py full  gpurun_out/prof_X.ncu-rep  TAG  [N_traj FLOP_per_traj]
  python tools/ncu_summary.py metrics        (prints the --metrics list for the executed-FLOP counters)
  python tools/ncu_summary.py launches gpurun_out/launches_X.csv TAG
  python tools/ncu_summary.py alias NAME=TAG [NAME=TAG ...]   (point the bench's side-measurement
      entries, e.g. c2_adaptive_f32=exec_c2a_r02y, at a fresh capture in profiles/ncu_summary.json)

full: key metrics of the captured kernel (time, DRAM bytes, pipe / issue
utilisation, occupancy, registers) → profiles/ncu_full_TAG.json, and the
per-launch DRAM traffic into profiles/ncu_summary.json[TAG].
launches: per-kernel launch counts, mean device time and share of the total →
profiles/launches_TAG.json (+ the raw csv copied next to it).
"""
from __future__ import annotations

import csv
import io
import json
import shutil
import subprocess
import sys
from collections import defaultdict
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
PROF = ROOT / "profiles"

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "sm__cycles_elapsed.avg.per_second",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__thread_inst_executed_per_inst_executed.ratio",
        "sm__sass_thread_inst_executed_op_ffma_pred_on.sum", "sm__sass_thread_inst_executed_op_fadd_pred_on.sum",
        "sm__sass_thread_inst_executed_op_fmul_pred_on.sum", "sm__sass_thread_inst_executed_op_dfma_pred_on.sum",
        "smsp__average_warp_latency_issue_stalled.ratio", "local_load", "lts__t_bytes.sum"]


# executed FP thread-instructions; pass with --metrics next to --set full
EXEC_METRICS = ["sm__sass_thread_inst_executed_op_ffma_pred_on.sum", "sm__sass_thread_inst_executed_op_fadd_pred_on.sum",
                "sm__sass_thread_inst_executed_op_fmul_pred_on.sum", "sm__sass_thread_inst_executed_op_ffma2_pred_on.sum",
                "sm__sass_thread_inst_executed_op_fadd2_pred_on.sum", "sm__sass_thread_inst_executed_op_fmul2_pred_on.sum",
                "sm__sass_thread_inst_executed_op_dfma_pred_on.sum", "sm__sass_thread_inst_executed_op_dadd_pred_on.sum",
                "sm__sass_thread_inst_executed_op_dmul_pred_on.sum"]
# FLOPs per thread-instruction: an FMA is 2, an add / mul 1; the packed FP32 forms carry two lanes
EXEC_FLOP = {"ffma": 2, "fadd": 1, "fmul": 1, "ffma2": 4, "fadd2": 2, "fmul2": 2, "dfma": 2, "dadd": 1, "dmul": 1}
KEYS += EXEC_METRICS


def executed_flop(hdr, units, v):
    """(fp32 FLOP, fp64 FLOP, per-op counts) from the executed-instruction counters, or None."""
    counts = {}
    for op in EXEC_FLOP:
        k = f"sm__sass_thread_inst_executed_op_{op}_pred_on.sum"
        if k not in hdr:
            return None
        counts[op] = float(v[hdr.index(k)].replace(",", ""))
    f32 = sum(EXEC_FLOP[o] * counts[o] for o in ("ffma", "fadd", "fmul", "ffma2", "fadd2", "fmul2"))
    f64 = sum(EXEC_FLOP[o] * counts[o] for o in ("dfma", "dadd", "dmul"))
    return f32, f64, counts


def to_bytes(v: str, unit: str) -> float:
    mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(unit, 1)
    return float(v.replace(",", "")) * mult


def full(rep: str, tag: str, n_traj: float | None, flop: float | None):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, vals = rows[0], rows[1], rows[2:]
    out = []
    for v in vals:
        d = {"kernel": v[hdr.index("Kernel Name")] if "Kernel Name" in hdr else None}
        for i, h in enumerate(hdr):
            if any(h == k or h.startswith(k) for k in KEYS) or "pipe_fma" in h or "pipe_fp64" in h:
                d[h] = f"{v[i]} {units[i]}".strip()
        rd = to_bytes(v[hdr.index("dram__bytes_read.sum")], units[hdr.index("dram__bytes_read.sum")])
        wr = to_bytes(v[hdr.index("dram__bytes_write.sum")], units[hdr.index("dram__bytes_write.sum")])
        t_ns = float(v[hdr.index("gpu__time_duration.sum")].replace(",", "")) * \
            {"ns": 1, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6, "nsecond": 1}.get(
                units[hdr.index("gpu__time_duration.sum")], 1)
        d["dram_bytes_per_launch"] = rd + wr
        d["time_ms"] = t_ns / 1e6
        if n_traj and flop:
            d["achieved_tflops_under_ncu"] = n_traj * flop / (t_ns * 1e-9) / 1e12
        ex = executed_flop(hdr, units, v)
        if ex is not None:
            d["executed_fp32_flop"], d["executed_fp64_flop"], d["executed_counts"] = ex
            d["executed_tflops_under_ncu"] = (ex[0] + ex[1]) / (t_ns * 1e-9) / 1e12
            if n_traj:
                d["executed_flop_per_traj"] = (ex[0] + ex[1]) / n_traj
        out.append(d)
    PROF.mkdir(exist_ok=True)
    (PROF / f"ncu_full_{tag}.json").write_text(json.dumps(out, indent=1))
    summ = PROF / "ncu_summary.json"
    s = json.loads(summ.read_text()) if summ.exists() else {}
    s[tag] = {"dram_bytes_per_launch": out[0]["dram_bytes_per_launch"], "time_ms": out[0]["time_ms"],
              "kernel": out[0]["kernel"], "source": f"profiles/ncu_full_{tag}.json"}
    if n_traj:
        s[tag]["traj_per_launch"] = n_traj
    if "executed_fp32_flop" in out[0]:
        s[tag]["executed_flop_per_launch"] = out[0]["executed_fp32_flop"] + out[0]["executed_fp64_flop"]
        s[tag]["executed_source"] = f"profiles/ncu_full_{tag}.json"
    summ.write_text(json.dumps(s, indent=1))
    print(json.dumps(out[0], indent=1))


def launches(path: str, tag: str):
    lines = [ln for ln in Path(path).read_text().splitlines() if not ln.startswith("==")]
    rows = list(csv.DictReader(io.StringIO("\n".join(lines))))
    agg = defaultdict(lambda: [0, 0.0])
    total = 0.0
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        t = float(r["Metric Value"].replace(",", ""))
        name = r["Kernel Name"].split("(")[0][:120]
        agg[name][0] += 1
        agg[name][1] += t
        total += t
    res = [{"kernel": k, "launches": c, "mean_us": s / c / 1e3, "share": s / total} for k, (c, s) in
           sorted(agg.items(), key=lambda kv: -kv[1][1])]
    PROF.mkdir(exist_ok=True)
    (PROF / f"launches_{tag}.json").write_text(json.dumps(res, indent=1))
    shutil.copy(path, PROF / f"launches_{tag}.csv")
    print(json.dumps(res, indent=1))


def alias(pairs):
    summ = PROF / "ncu_summary.json"
    s = json.loads(summ.read_text())
    for pr in pairs:
        name, tag = pr.split("=", 1)
        s[name] = dict(s[tag])
        print(name, "<-", tag, s[name].get("executed_flop_per_launch"))
    summ.write_text(json.dumps(s, indent=1))


if __name__ == "__main__":
    if sys.argv[1] == "alias":
        alias(sys.argv[2:])
    elif sys.argv[1] == "metrics":
        print(",".join(EXEC_METRICS))
    elif sys.argv[1] == "full":
        full(sys.argv[2], sys.argv[3], float(sys.argv[4]) if len(sys.argv) > 4 else None,
             float(sys.argv[5]) if len(sys.argv) > 5 else None)
    else:
        launches(sys.argv[2], sys.argv[3])
