#!/usr/bin/env python
"""Multi-rank self-test: P processes (torchrun), each with its own hb_comm, run the split
operator (halo exchange || interior A, halo elements, assembly exchange || interior B), a dot,
fixed-mode and tolerance-mode CG; rank 0 compares the assembled results with the CPU oracle.

    torchrun --nproc-per-node P --master-addr 127.0.0.1 --master-port 29511 \
        scripts/multirank_selftest.py [--transport ipc|nccl] [--box 4,3,4] [--N 3]
Ranks use GPU (LOCAL_RANK % device_count).  NCCL refuses two ranks on one GPU; the IPC
peer-memory transport (hb_comm_create_ipc) runs them, so on a one-GPU box this exercises the
real multi-process exchange and allreduce logic.  Prints one JSON line on rank 0."""
import argparse
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--transport", default="ipc", choices=["ipc", "nccl"])
    ap.add_argument("--box", default="4,3,4")
    ap.add_argument("--N", type=int, default=3)
    a = ap.parse_args()
    rank, P = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    lr = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(lr % torch.cuda.device_count())
    dist.init_process_group("gloo")
    import __graft_entry__
    if rank == 0:
        __graft_entry__.build()
    dist.barrier()
    import paper_2202_12477_b200 as hb
    box, N = tuple(int(v) for v in a.box.split(",")), a.N
    out = {"P": P, "transport": a.transport, "box": list(box), "N": N, "ok": False}
    try:
        if a.transport == "nccl":
            uid = [hb.comm_unique_id() if rank == 0 else None]
            dist.broadcast_object_list(uid, src=0)
            comm = hb.Comm(P, rank, uid[0])
        else:
            comm = hb.Comm.create_ipc(P, rank)
        m = hb.Mesh(*box, N, P=P, rank=rank)
        op = hb.Operator(m, comm=comm)
        if a.transport == "ipc":
            recs = [None] * P
            dist.all_gather_object(recs, op.ipc_export())
            op.ipc_connect(recs)
        n = op.n_owned
        b = torch.empty(n, dtype=torch.float64, device="cuda")
        op.forcing(2, b)
        y = torch.empty_like(b)
        op.apply(b, y)
        bb = op.dot(b, b)
        x = torch.zeros_like(b)
        op.forcing(1, b)
        K = 20
        modes = [True, False] if a.transport == "ipc" else [None]
        runs = []
        for direct in modes:  # IPC: direct (peer-memory halo elements) and exchange CG
            if direct is not None:
                op.set_ipc_direct(direct)
            x = torch.zeros_like(b)
            j, hist = op.cg(b, x, K)
            x2 = torch.zeros_like(b)
            j2, hist2 = op.cg(b, x2, 400, eps=1e-12)  # tolerance mode (host-driven loop for P > 1)
            runs.append((j, hist, x.cpu().numpy(), j2, hist2))
        op.apply(b, y)                               # re-apply after the solves: sequence numbers advance
        torch.cuda.synchronize()
        gathered = [None] * P
        dist.all_gather_object(gathered, (m.owned(), y.cpu().numpy(), [r[2] for r in runs]))
        if rank == 0:
            from oracle import basis, cg as ocg, forcing as of, mesh as om, operator as oo
            xg, w, D = basis.basis(N)
            E, NG, NL = om.global_sizes(*box, N)
            gid = om.l2g(*box, N)
            G = om.geometric_factors(E, N, w)
            W = om.weights_W(gid, NG)
            A = lambda v: oo.apply(v, gid, D, G, 1.0, W)
            b2 = of.forcing(range(NG), 2)
            b1 = of.forcing(range(NG), 1)
            yo = A(b1)
            s = oo.apply_abs(b1, gid, D, G, 1.0, W)
            yg = np.zeros(NG)
            for own, yy, _ in gathered:
                yg[own] = yy
            xo, _, ho = ocg.cg(A, b1, max_iters=K)
            _, jo2, ho2 = ocg.cg(A, b1, max_iters=400, eps=1e-12)
            out.update(apply_err=float(np.max(np.abs(yg - yo) / s)),
                       dot_rel=abs(bb - ocg.dot(b2, b2)) / ocg.dot(b2, b2), modes=[])
            ok = out["apply_err"] <= 1e-12
            for mi, (direct, (j, hist, _, j2, hist2)) in enumerate(zip(modes, runs)):
                xgv = np.zeros(NG)
                for own, _, xs in gathered:
                    xgv[own] = xs[mi]
                r = dict(direct=direct, cg_hist_rel=float(np.max(np.abs(hist - np.array(ho)) / np.array(ho))),
                         x_rel=float(np.max(np.abs(xgv - xo)) / np.max(np.abs(xo))), iterations=j,
                         tol_iterations=j2, tol_iterations_oracle=jo2,
                         tol_hist_rel=float(np.max(np.abs(np.array(hist2[:j2]) - np.array(ho2[:j2]))
                                                   / np.array(ho2[:j2]))))
                out["modes"].append(r)
                ok = ok and r["cg_hist_rel"] <= 1e-8 and r["x_rel"] <= 1e-10 and j2 == jo2 and r["tol_hist_rel"] <= 1e-8
            out["ok"] = bool(ok)
    except Exception as ex:
        out["error"] = repr(ex)
    if rank == 0:
        print(json.dumps(out), flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
