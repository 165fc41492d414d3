#!/usr/bin/env python
"""Operator-only timing (P:268 methodology: mean of back-to-back applies after warm-up),
per degree N, for kernel tuning.  Prints one JSON line per configuration.

    python scripts/opbench.py --N 7 --box 52,52,52 [--reps 50] [--variant V]
    python scripts/opbench.py --sweep            # C3: ~50 M DOFs for N = 1..15
"""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

# C3 boxes: ~50 M DOFs per degree
C3 = {1: 367, 2: 184, 3: 122, 4: 92, 5: 73, 6: 61, 7: 52, 8: 46, 9: 41, 10: 37, 11: 33, 12: 31, 13: 28, 14: 26, 15: 24}


def run(N, box, reps, peak):
    import torch
    import paper_2202_12477_b200 as hb
    from paper_2202_12477_b200 import ledger
    m = hb.Mesh(*box, N)
    op = hb.Operator(m)
    if int(os.environ.get("HB_BENCH_VARIANT", "0")):
        op.set_variant(int(os.environ["HB_BENCH_VARIANT"]))
    n = op.n_owned
    s = m.sizes
    x = torch.empty(n, dtype=torch.float64, device="cuda")
    op.forcing(2, x)
    y = torch.empty_like(x)
    for _ in range(5):
        op.apply(x, y)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    op.set_profiling(True)
    e0.record()
    for _ in range(reps):
        op.apply(x, y)
    e1.record()
    torch.cuda.synchronize()
    nk, tk = op.kernel_time()
    op.set_profiling(False)
    ms = e0.elapsed_time(e1) / reps
    alg = ledger.op_bytes_fused(n, s["N_L"])
    out = {"N": N, "box": list(box), "N_G": n, "E": s["E_local"], "apply_ms": ms, "kernel_ms": tk * 1e3,
           "kernel_GBps": alg / tk / 1e9, "frac_of_peak": alg / tk / 1e9 / peak,
           "op_GFLOPs": ledger.op_flops(s["E_local"], N) / tk / 1e9,
           "roofline_GFLOPs_at_peak": ledger.op_roofline(N, peak * 1e9),
           "paper_ledger_GBps": ledger.op_bytes_paper(n, s["N_L"]) / tk / 1e9,
           "variant": os.environ.get("HB_AX_VARIANT", "default")}
    print(json.dumps(out), flush=True)
    del op, m


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--N", type=int, default=7)
    ap.add_argument("--box", default="52,52,52")
    ap.add_argument("--reps", type=int, default=50)
    ap.add_argument("--sweep", action="store_true")
    ap.add_argument("--tune", default="", help="variants to try per N, e.g. 0,1,2 (needs an HB_TUNE build)")
    ap.add_argument("--degrees", default="", help="comma list of N for --sweep/--tune (default 1..15)")
    ap.add_argument("--tune-box", default="", help="box for --tune instead of the C3 box, e.g. 16,16,16")
    a = ap.parse_args()
    import __graft_entry__
    __graft_entry__.build()
    pp = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(pp):
        with open(pp) as f:
            peak = json.load(f)["hbm_gbs"]
    else:  # driver-written per pod; B200_PROFILING.md fallback otherwise (as bench.py)
        peak = 6650.0
    degrees = [int(v) for v in a.degrees.split(",")] if a.degrees else list(C3)
    if a.tune:
        for N in degrees:
            n = C3[N]
            tb = tuple(int(v) for v in a.tune_box.split(",")) if a.tune_box else (n, n, n)
            for v in a.tune.split(","):
                os.environ["HB_AX_VN"] = str(N)
                os.environ["HB_AX_VARIANT"] = v
                try:
                    run(N, tb, a.reps, peak)
                except Exception as ex:  # a variant may not launch (resources): report and go on
                    print(json.dumps({"N": N, "variant": v, "error": repr(ex)}), flush=True)
        return
    if a.sweep:
        for N in degrees:
            n = C3[N]
            run(N, (n, n, n), a.reps, peak)
    else:
        run(a.N, tuple(int(v) for v in a.box.split(",")), a.reps, peak)


if __name__ == "__main__":
    main()
