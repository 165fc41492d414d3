#!/usr/bin/env python
"""Small operator applies and CG solves for compute-sanitizer runs (memcheck / racecheck /
synccheck): P=1 fused and deterministic variants, mass modes, and a loopback group."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import __graft_entry__  # noqa: E402

__graft_entry__.build()
import paper_2202_12477_b200 as hb  # noqa: E402

for N, mm in [(int(v.split(':')[0]), int(v.split(':')[1])) for v in os.environ.get('SAN_CASES', '2:0,3:1,7:0,8:1,15:0').split(',') if v]:
    m = hb.Mesh(2, 2, 1, N, mass_mode=mm)
    op = hb.Operator(m)
    b = torch.empty(op.n_owned, dtype=torch.float64, device="cuda")
    op.forcing(1, b)
    y = torch.empty_like(b)
    op.apply(b, y)
    x = torch.zeros_like(b)
    op.cg(b, x, 3)
    op.cg(b, x, 5, 1e-30)
    op.set_variant(1)
    op.apply(b, y)
    op.cg(b, x, 2)
    if mm == 0:
        op.cg_scattered(b, x, 2)
        try:
            op.set_jacobi(True)  # needs the fused (cooperative) update: absent under HB_FUSED_UPDATE=0
            op.cg(b, x, 2)
        except hb.HBError:
            pass
    torch.cuda.synchronize()
# one multi-wave box per operator kernel family (N = 1 vertex kernel; N = 2 multi-element CTAs;
# N = 7 the bench degree; N = 12 streaming epilogue; N = 15 one uncapped CTA per SM): every CTA
# wraps its grid-stride loop >= 3 times, as at the benchmark sizes
for N in [int(v) for v in os.environ.get("SAN_MULTIWAVE", "").split(",") if v]:
    sh = hb.Operator(hb.Mesh(1, 1, 1, N)).launch_shape()
    need = 3 * sh["grid"] * sh["epb"] + 1
    a = max(2, int(round(need ** (1.0 / 3.0))))
    box = (a, a + 1, -(-need // (a * (a + 1))))
    op = hb.Operator(hb.Mesh(*box, N))
    b = torch.empty(op.n_owned, dtype=torch.float64, device="cuda")
    op.forcing(1, b)
    y = torch.empty_like(b)
    op.apply(b, y)
    x = torch.zeros_like(b)
    op.cg(b, x, 2)
    torch.cuda.synchronize()
    print("multiwave", N, box, sh, flush=True)
meshes = [hb.Mesh(4, 2, 2, 3, P=4, rank=r) for r in range(4)]
ops = [hb.Operator(mm) for mm in meshes]
g = hb.Group(ops)
bs = [torch.ones(o.n_owned, dtype=torch.float64, device="cuda") for o in ops]
xs = [torch.zeros_like(t) for t in bs]
g.cg(bs, xs, 3)
torch.cuda.synchronize()
print("sanitize workload done")
