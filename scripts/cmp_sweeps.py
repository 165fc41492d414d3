#!/usr/bin/env python
"""Side-by-side fraction of peak per N from opbench sweep files: cmp_sweeps.py base.jsonl other.jsonl ..."""
import json
import sys


def load(f):
    d = {}
    for line in open(f):
        try:
            j = json.loads(line)
        except ValueError:
            continue
        if "frac_of_peak" in j:
            d[j["N"]] = j["frac_of_peak"]
    return d


files = sys.argv[1:]
runs = [load(f) for f in files]
print("N  " + " ".join(f"{f.split('/')[-1][:12]:>12s}" for f in files))
for N in sorted(set().union(*runs)):
    print(f"{N:<3d}" + " ".join(f"{r[N]:12.3f}" if N in r else f"{'-':>12s}" for r in runs))
