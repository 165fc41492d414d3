#!/usr/bin/env python
"""Summarise ncu captures (gpurun_out/*.ncu-rep) and launch lists (launches.csv) into
profiles/.  Usage: python scripts/ncu_summary.py <round-tag> rep1.ncu-rep[:key] ... [--launches launches.csv]

key = "N<N>_<nx>x<ny>x<nz>" labels the workload; dram bytes per launch are written to
profiles/ncu_op_summary.json (read by bench.py for roofline.traffic)."""
from __future__ import annotations

import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
NCU = "/usr/local/cuda/bin/ncu"

WANT = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "launch__registers_per_thread", "launch__block_size", "launch__grid_size", "launch__occupancy_limit_registers",
    "launch__occupancy_limit_shared_mem", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__throughput.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum", "sm__cycles_elapsed.avg.per_second", "lts__t_sectors_op_red.sum",
    "lts__t_sectors_op_atom.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "lts__t_sector_hit_rate.pct",
    "smsp__average_warp_latency_issue_stalled_long_scoreboard", "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
]


def raw(rep: str):
    out = subprocess.run([NCU, "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if len(rows) < 3:
        return []
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {}
        for h, u, v in zip(hdr, units, r):
            d[h] = (v, u)
        res.append(d)
    return res


def num(v):
    try:
        return float(v.replace(",", ""))
    except (ValueError, AttributeError):
        return None


def main():
    tag = sys.argv[1]
    args = sys.argv[2:]
    launches = None
    if "--launches" in args:
        i = args.index("--launches")
        launches = args[i + 1]
        args = args[:i] + args[i + 2:]
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    summ_path = os.path.join(ROOT, "profiles", "ncu_op_summary.json")
    summ = json.load(open(summ_path)) if os.path.exists(summ_path) else {}
    summ.setdefault("dram_bytes_per_launch", {})
    summ.setdefault("captures", {})
    md = [f"# ncu summary ({tag})\n"]
    for a in args:
        rep, _, key = a.partition(":")
        for k, d in enumerate(raw(rep)):
            name = d.get("Kernel Name", ("?", ""))[0]
            vals = {m: (num(d[m][0]), d[m][1]) for m in WANT if m in d}
            rd = vals.get("dram__bytes_read.sum", (None, ""))
            wr = vals.get("dram__bytes_write.sum", (None, ""))
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
            tot = None
            if rd[0] is not None and wr[0] is not None:
                tot = rd[0] * scale.get(rd[1], 1) + wr[0] * scale.get(wr[1], 1)
            if key:
                summ["dram_bytes_per_launch"][key] = tot
            summ["captures"][f"{tag}:{key or os.path.basename(rep)}:{k}"] = {
                "kernel": name[:120], "dram_bytes": tot, **{m: v[0] for m, v in vals.items()}}
            md.append(f"## {os.path.basename(rep)} [{key}] launch {k}\n\n`{name[:160]}`\n")
            md.append("| metric | value | unit |\n|---|---|---|")
            for m, (v, u) in vals.items():
                md.append(f"| {m} | {v} | {u} |")
            md.append(f"| dram bytes (read+write) | {tot} | byte |\n")
    if launches and os.path.exists(launches):
        with open(launches) as f:
            text = f.read()
        lines = [l for l in text.splitlines() if l.startswith('"')]
        rows = list(csv.reader(io.StringIO("\n".join(lines))))
        if rows:
            hdr = rows[0]
            ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
            agg = {}
            for r in rows[1:]:
                nm = r[ki].split("(")[0][:60]
                v = num(r[vi]) or 0.0
                a = agg.setdefault(nm, [0, 0.0])
                a[0] += 1
                a[1] += v
            tot = sum(v[1] for v in agg.values())
            md.append("## launch list (ncu gpu__time_duration.sum, cold-cache, serialised)\n")
            md.append("| kernel | launches | total ns | share |\n|---|---|---|---|")
            for nm, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
                md.append(f"| `{nm}` | {c} | {t:.0f} | {t / tot:.3f} |")
            summ.setdefault("launch_shares", {})[tag] = {nm: t / tot for nm, (c, t) in agg.items()}
    json.dump(summ, open(summ_path, "w"), indent=1)
    with open(os.path.join(ROOT, "profiles", f"ncu_{tag}.md"), "w") as f:
        f.write("\n".join(md) + "\n")
    print("\n".join(md))


if __name__ == "__main__":
    main()
