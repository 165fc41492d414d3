#!/usr/bin/env python
"""Digest ncu reports on the GPU box (reports are too large to bring back): key metrics, warp
stall reasons (per issued instruction) and the top source lines by stall samples, one text file
per report.  Usage: python scripts/ncu_digest.py out_dir rep1.ncu-rep ..."""
import csv
import io
import os
import subprocess
import sys

NCU = "/usr/local/cuda/bin/ncu"
KEYS = ("gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "launch__registers_per_thread", "launch__block_size", "launch__grid_size",
        "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__throughput.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "lts__t_sector_hit_rate.pct",
        "smsp__inst_executed.sum", "sm__cycles_elapsed.avg.per_second", "launch__shared_mem_per_block_dynamic")


def main():
    out = sys.argv[1]
    os.makedirs(out, exist_ok=True)
    for rep in sys.argv[2:]:
        name = os.path.basename(rep).replace(".ncu-rep", "")
        raw = subprocess.run([NCU, "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
        rows = list(csv.reader(io.StringIO(raw)))
        lines = []
        if len(rows) >= 3:
            hdr, units, vals = rows[0], rows[1], rows[2]
            lines.append("kernel: " + vals[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "")
            for k in KEYS:
                if k in hdr:
                    i = hdr.index(k)
                    lines.append(f"{k} = {vals[i]} {units[i]}")
            st = []
            for i, k in enumerate(hdr):
                if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
                    try:
                        st.append((float(vals[i]), k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
                    except ValueError:
                        pass
            lines.append("warp stalls per issued instruction:")
            for v, k in sorted(st, reverse=True)[:12]:
                lines.append(f"  {k:28s} {v:8.3f}")
        src = subprocess.run([sys.executable, os.path.join(os.path.dirname(__file__), "ncu_lines.py"), rep, "25"],
                             capture_output=True, text=True).stdout
        lines.append("top source lines by stall samples:")
        lines.append(src)
        with open(os.path.join(out, name + ".txt"), "w") as f:
            f.write("\n".join(lines) + "\n")


if __name__ == "__main__":
    main()
