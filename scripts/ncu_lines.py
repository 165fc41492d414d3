#!/usr/bin/env python
"""Per-source-line warp-stall sampling of an ncu report (SASS rows attributed to the CUDA line
above them): python scripts/ncu_lines.py report.ncu-rep [top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 20
out = subprocess.run(["/usr/local/cuda/bin/ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
agg, src, cur = {}, {}, None
for r in rows[3:]:
    if len(r) < 5:
        continue
    if r[0]:
        cur = r[0]
        src[cur] = r[1].strip()[:95]
    try:
        v = float(r[4])
    except ValueError:
        continue
    if not r[0]:
        agg[cur] = agg.get(cur, 0) + v
tot = sum(agg.values()) or 1
for ln, v in sorted(agg.items(), key=lambda kv: -kv[1])[:top]:
    print(f"{v / tot:6.3f} L{ln:>4} {src.get(ln, '')}")
