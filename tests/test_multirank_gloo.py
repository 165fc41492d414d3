"""Multi-process (gloo, CPU) tests of the multi-rank host logic: every rank builds its
partition with the C library (hb_mesh_*, host only), the ranks exchange plan metadata over
torch.distributed/gloo, and the halo and assembly exchanges of the operator schedule
 are replayed with gloo send/recv using exactly the library's send lists, recv
segments and local indices (the same buffers the NCCL path hands to ncclSend/ncclRecv)."""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, P, port, box, N, seed, q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    try:
        dist.init_process_group("gloo", rank=rank, world_size=P)
        import paper_2202_12477_b200 as hb
        from oracle import mesh as om
        m = hb.Mesh(*box, N, P=P, rank=rank, seed=seed)
        s = m.sizes
        owned, halo = m.owned(), m.halo()
        nbr, sc, rc = m.neighbors()
        sends = {int(nbr[k]): m.send_list(k) for k in range(len(nbr))}
        idx = m.local_index()
        gid = m.l2g()
        meta = dict(owned=owned, halo=halo, nbr=[int(v) for v in nbr], sends=sends,
                    rc=[int(v) for v in rc], E=s["E_local"], grid=s["grid"])
        allm = [None] * P
        dist.all_gather_object(allm, meta)
        errs = []
        # ---- ownership partition and plan symmetry
        cat = np.concatenate([a["owned"] for a in allm])
        E, NG, NL = om.global_sizes(*box, N)
        if not np.array_equal(np.sort(cat), np.arange(NG)):
            errs.append("owned sets do not partition the gids")
        if sum(a["E"] for a in allm) != E:
            errs.append("element counts do not sum to E")
        off = 0
        for k, qn in enumerate(meta["nbr"]):
            other = allm[qn]
            if rank not in other["nbr"]:
                errs.append(f"neighbour asymmetry {rank}-{qn}")
                continue
            seg = halo[off:off + meta["rc"][k]]
            off += meta["rc"][k]
            if not np.array_equal(seg, other["sends"][rank]):
                errs.append(f"recv segment from {qn} != its send list")
            if not np.all(np.isin(seg, other["owned"])):
                errs.append(f"halo gids from {qn} not owned by {qn}")
        if off != len(halo):
            errs.append("recv segments do not cover the halo")
        # ---- halo exchange replay: x[g] = g + 0.5 (any injective function)
        x_own = owned.astype(np.float64) + 0.5
        pos = {int(g): t for t, g in enumerate(owned)}
        reqs, bufs = [], {}
        for k, qn in enumerate(meta["nbr"]):
            send = torch.tensor([x_own[pos[int(g)]] for g in sends[qn]], dtype=torch.float64)
            bufs[qn] = torch.empty(meta["rc"][k], dtype=torch.float64)
            if len(send):
                reqs.append(dist.isend(send, qn))
            if meta["rc"][k]:
                reqs.append(dist.irecv(bufs[qn], qn))
        for r_ in reqs:
            r_.wait()
        x_halo = np.concatenate([bufs[qn].numpy() for qn in meta["nbr"]]) if meta["nbr"] else np.zeros(0)
        if not np.array_equal(x_halo, halo.astype(np.float64) + 0.5):
            errs.append("halo exchange delivered wrong values")
        x_ext = np.concatenate([x_own, x_halo])
        if not np.array_equal(x_ext[idx], gid.astype(np.float64) + 0.5):
            errs.append("local index does not address the gathered values")
        # ---- assembly exchange replay: sum of ones per slot -> global degree counts
        y_ext = np.bincount(idx.ravel(), minlength=len(x_ext)).astype(np.float64)
        y_own, y_halo = y_ext[:len(owned)].copy(), y_ext[len(owned):]
        reqs, rbufs, off = [], {}, 0
        for k, qn in enumerate(meta["nbr"]):
            seg = torch.tensor(y_halo[off:off + meta["rc"][k]])
            off += meta["rc"][k]
            rbufs[qn] = torch.empty(len(sends[qn]), dtype=torch.float64)
            if len(seg):
                reqs.append(dist.isend(seg, qn))
            if len(sends[qn]):
                reqs.append(dist.irecv(rbufs[qn], qn))
        for r_ in reqs:
            r_.wait()
        for qn in meta["nbr"]:
            for g, v in zip(sends[qn], rbufs[qn].numpy()):
                y_own[pos[int(g)]] += v
        counts = om.counts(om.l2g(*box, N), NG)
        if not np.array_equal(y_own, counts[owned].astype(np.float64)):
            errs.append("assembly exchange does not reproduce the degree counts")
        # ---- scalar allreduce (the CG dots): sum over ranks of owned x.x = global x.x
        t = torch.tensor([float(np.dot(x_own, x_own))], dtype=torch.float64)
        dist.all_reduce(t)
        gx = np.arange(NG) + 0.5
        if abs(t.item() - float(np.dot(gx, gx))) > 1e-9 * float(np.dot(gx, gx)):
            errs.append("allreduce of local dots != global dot")
        q.put((rank, errs))
        dist.barrier()
        dist.destroy_process_group()
    except Exception as ex:  # pragma: no cover - surfaced by the parent
        q.put((rank, [f"exception: {ex!r}"]))


@pytest.mark.parametrize("P,box,N,seed", [(2, (4, 3, 2), 3, 0), (2, (3, 3, 3), 2, 7), (4, (4, 4, 2), 2, 1)])
def test_gloo_plans_and_exchanges(P, box, N, seed):
    import __graft_entry__
    __graft_entry__.build()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, P, port, box, N, seed, q)) for r in range(P)]
    for p in procs:
        p.start()
    results = {}
    for _ in range(P):
        rank, errs = q.get(timeout=180)
        results[rank] = errs
    for p in procs:
        p.join(timeout=60)
    assert all(not e for e in results.values()), results
