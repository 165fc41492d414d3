#!/usr/bin/env python
"""Time the CG modes beside the fixed-iteration benchmark (one B200): fixed 100 iterations,
tolerance mode (device WHILE-loop graph, stop at r.r <= eps), Jacobi PCG (NEXT #3) in
both modes.  eps = rel^2 * b.b.  Prints one JSON line per (box, N, mode).
    python scripts/bench_modes.py [--rel 1e-8] [--reps 5]"""
import argparse
import json
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2202_12477_b200 as hb  # noqa: E402
from paper_2202_12477_b200 import ledger  # noqa: E402


def timed(fn, reps):
    fn()  # warm-up (graph capture / instantiation)
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        out = fn()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    return min(ts), out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rel", type=float, default=1e-8)
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    for box, N in [((16, 16, 16), 7), ((52, 52, 52), 7), ((24, 24, 24), 15)]:
        m = hb.Mesh(*box, N)
        op = hb.Operator(m, lam=1.0)
        n = op.n_owned
        b = torch.empty(n, dtype=torch.float64, device="cuda")
        op.forcing(1, b)
        bb = op.dot(b, b)
        eps = a.rel * a.rel * bb
        E = box[0] * box[1] * box[2]
        for jac in (False, True):
            op.set_jacobi(jac)
            for mode, its, e in (("fixed", 100, -1.0), ("tolerance", 1000, eps)):
                x = torch.zeros_like(b)
                t, (j, h) = timed(lambda: op.cg(b, x.zero_(), its, e), a.reps)
                gf = ledger.nekbone_flops_per_iter(E, N) * j / t / 1e9
                print(json.dumps({"box": list(box), "N": N, "N_G": n, "precond": "jacobi" if jac else "none",
                                  "mode": mode, "eps_rel": a.rel if e >= 0 else None, "iterations": int(j),
                                  "ms": round(t * 1e3, 3), "us_per_iter": round(t * 1e6 / max(j, 1), 2),
                                  "nekbone_gflops": round(gf, 1),
                                  "rr_final_rel": float(h[j] / h[0]) if len(h) > j else None}), flush=True)
        op.set_jacobi(False)
        del op, m
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
