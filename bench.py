#!/usr/bin/env python
"""hipBone hot-path benchmark on B200 (BASELINE.json metric: CG GFLOP/s in the NekBone count
& operator HBM GB/s vs peak at N=7).

A step = one fixed-iteration CG solve (Alg. 1; 100 iterations) from x0 = 0 on
the synthetic box workload, i.e. every §8(a) row: gather, gradient, metric, divergence,
scatter-add (operator), p.Ap, r/x update + r.r, p update.  Default workload C2 (N=7, 16^3
elements, BASELINE.json configs[1]); with --gpus P > 1 every rank gets a C2-sized block of a
(16 px) x (16 py) x (16 pz) box (weak scaling, C4 shape).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--box 16,16,16] [--N 7]
    torchrun --nproc-per-node N bench.py --gpus N ...

--impl reference times the CPU oracle (oracle/, plain numpy fp64) on a bounded sample of the
same workload -- the tier's reference arm.  Prints ONE JSON line (rank 0).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "CG GFLOP/s (NekBone count) & operator HBM GB/s vs peak at N=7"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--box", default="16,16,16", help="elements per rank (per-rank block for P>1)")
    ap.add_argument("--N", type=int, default=7)
    ap.add_argument("--iters", type=int, default=100)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--no-profile", action="store_true", help="skip the operator-share pass (no roofline)")
    ap.add_argument("--no-c3", action="store_true", help="skip the C3 N=7 operator roofline block")
    ap.add_argument("--variant", type=int, default=0, help="0 fused scatter-add, 1 y_L + CSR (P=1), 2 fused p update (P=1)")
    ap.add_argument("--jacobi", action="store_true", help="Jacobi-preconditioned CG (P=1; not the NekBone FOM)")
    ap.add_argument("--storage", default="assembled", choices=["assembled", "scattered"],
                    help="scattered = NekBone's x_L storage with weighted dots (P=1 experiment, P:112-121)")
    ap.add_argument("--strong", action="store_true",
                    help="--box is the global box, partitioned across the ranks (strong scaling, e.g. C5: --N 15 --box 50,50,48)")
    ap.add_argument("--transport", default="nccl", choices=["nccl", "ipc"],
                    help="P>1 exchanges/allreduces: NCCL, or the IPC peer-memory transport (several ranks may share a GPU)")
    return ap.parse_args()


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self.proc = None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 7:
                self.samples.append(parts)

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.15)
            self.proc.terminate()
            try:
                self.proc.wait(2)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        sm = sorted(float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit())
        mx = max(float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit())
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for s in self.samples for k in range(4) if s[3 + k].lower() == "active"})
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": mx, "reasons": reasons,
                "samples": len(self.samples)}


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def host_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


# --- the oracle on the host's cores.  The oracle runs as it stands (oracle.cg.cg, Alg. 1,
# with oracle.operator's sum-factorised element apply and bincount assembly); with procs > 1
# the element loop of each apply is split into contiguous chunks over forked worker processes
# (harness-level parallelism: every worker calls oracle.operator.local_apply on its chunk, the
# assembly and the CG vector steps stay in the parent).  Nothing here imports the product.
_OW = {}


def _ow_init():
    from threadpoolctl import threadpool_limits
    _OW["lim"] = threadpool_limits(limits=1)  # one core per worker process


def _ow_chunk(rng_):
    from oracle import operator as oo
    lo, hi = rng_
    d = _OW
    u = d["x"][d["gid"][lo:hi]]
    d["yL"][lo:hi] = oo.local_apply(d["D"], d["G"][lo:hi], u) + d["lam"] * d["W"][lo:hi] * u


class OracleCG:
    """Fixed-box oracle problem (c4, c7, c12: lambda = 1, mass mode 0, b = forcing seed 1)."""

    def __init__(self, box, N, procs: int):
        import multiprocessing as mp

        import numpy as np
        from oracle import basis, forcing as of, mesh as om, operator as oo
        self.N, self.box, self.procs = N, box, procs
        x, w, D = basis.basis(N)
        self.E, self.NG, self.NL = om.global_sizes(*box, N)
        gid = om.l2g(*box, N)
        G = om.geometric_factors(self.E, N, w)
        W = om.weights_W(gid, self.NG)
        self.b = of.forcing(range(self.NG), 1)
        self.pool = None
        if procs <= 1:
            self.A = lambda v: oo.apply(v, gid, D, G, 1.0, W)
            return
        xs = np.frombuffer(mp.RawArray("d", self.NG), dtype=np.float64)
        ys = np.frombuffer(mp.RawArray("d", self.E * (N + 1) ** 3), dtype=np.float64).reshape(self.E, -1)
        _OW.update(x=xs, yL=ys, gid=gid, D=D, G=G, W=W, lam=1.0)
        self.pool = mp.get_context("fork").Pool(procs, initializer=_ow_init)  # children inherit _OW
        step = -(-self.E // (4 * procs))
        chunks = [(lo, min(self.E, lo + step)) for lo in range(0, self.E, step)]

        def A(v):
            xs[:] = v
            self.pool.map(_ow_chunk, chunks)
            return oo.assemble(gid, ys, self.NG)
        self.A = A

    def run(self, iters: int) -> float:
        from oracle import cg as ocg
        from threadpoolctl import threadpool_limits
        with threadpool_limits(limits=1):  # the parent's own numpy work: one core
            t0 = time.perf_counter()
            ocg.cg(self.A, self.b, max_iters=iters)
            return time.perf_counter() - t0

    def close(self):
        if self.pool is not None:
            self.pool.close()
            self.pool.join()
            self.pool = None


def cpu_baseline(box, N, seconds: float):
    """The oracle as it stands (plain numpy fp64) on a bounded sample of the same workload:
    k CG iterations of the same box, k chosen to take ~`seconds`, on all the host's cores
    (element chunks over forked processes) and, for reference, on one core."""
    from oracle import ledger as oled
    cores = host_cores()
    out = {}
    for procs in ([cores, 1] if cores > 1 else [1]):
        o = OracleCG(box, N, procs)
        try:
            t1 = o.run(1)
            k = max(1, min(100, int(0.5 * seconds / max(t1, 1e-6))))
            t = o.run(k)
        finally:
            o.close()
        out[procs] = (k, t, oled.nekbone_flops(o.E, N) * k / t / 1e9)
    k, t, gf = out[cores] if cores in out else out[1]
    res = {"value": gf, "unit": "GFLOP/s", "cores": cores if cores in out else 1, "kind": "oracle",
           "model": cpu_model(),
           "sample": (f"{k} CG iterations (of 100) of box {box[0]}x{box[1]}x{box[2]} N={N}, numpy fp64 oracle, "
                      f"element loop over {cores} forked processes"),
           "seconds": round(t, 3), "iterations": k}
    if 1 in out:
        k1, t1, g1 = out[1]
        res["single_core"] = {"value": g1, "iterations": k1, "seconds": round(t1, 3)}
    return res


def run_reference(args):
    """--impl reference: the CPU oracle (oracle/ only; this process never loads the product
    library) on the GPU arm's config, on all the host's cores."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle import ledger as oled
    from oracle import partition as opart
    box = tuple(int(v) for v in args.box.split(","))
    N = args.N
    blk = box
    if args.gpus > 1 and not args.strong:  # the GPU arm's weak-scaling box: per-GPU block x rank grid
        g = opart.rank_grid(args.gpus, 64, 64, 64)
        box = (box[0] * g[0], box[1] * g[1], box[2] * g[2])
    cores = host_cores()
    o = OracleCG(box, N, cores)
    try:
        # each step: a bounded sample of the 100-iteration solve (sized so the run ends in minutes)
        t1 = o.run(1)
        k = max(1, min(args.iters, int(8.0 / max(t1, 1e-6))))
        for _ in range(args.warmup):
            o.run(1)
        times = [o.run(k) for _ in range(args.steps)]
    finally:
        o.close()
    t = sum(times) / len(times)
    gf = oled.nekbone_flops(o.E, N) * k / t / 1e9
    sample = (f"{k} CG iterations per step (of {args.iters}) of box {box[0]}x{box[1]}x{box[2]} N={N}, "
              f"element loop over {cores} forked processes")
    out = {"impl": "reference", "metric": METRIC, "value": gf, "unit": "GFLOP/s", "n_gpus": args.gpus,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3,
           "higher_is_better": True, "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "scaling": "strong" if args.strong else "weak",
           "config": {"workload": f"{'C2' if blk == (16, 16, 16) and N == 7 else 'custom'}: N={N}, "
                                  f"E={box[0]}x{box[1]}x{box[2]}, {args.iters} CG iterations (sampled)",
                      "box": list(box), "N": N, "N_G": o.NG, "lambda": 1.0},
           "cpu_baseline": {"value": gf, "unit": "GFLOP/s", "cores": cores, "kind": "oracle", "sample": sample,
                            "model": cpu_model()},
           "e2e": {"value": gf, "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


def c3_operator_roofline(hb, ledger, peak, peak_src, device_index, reps=50, rounds=5):
    """C3 at N=7 (52^3 elements, 48.6 M DOFs, BASELINE configs[2]) operator roofline by the
    paper's method (c24): `reps` back-to-back hb_op_apply calls after warm-up, the
    operator kernel bracketed by CUDA events on its stream (outside any graph), the mean per
    round, the median of `rounds` rounds; clocks sampled during the rounds."""
    import torch
    box, N = (52, 52, 52), 7
    m = hb.Mesh(*box, N)
    op = hb.Operator(m)
    n = op.n_owned
    s = m.sizes
    x = torch.empty(n, dtype=torch.float64, device="cuda")
    op.forcing(2, x)
    y = torch.empty_like(x)
    for _ in range(5):
        op.apply(x, y)
    torch.cuda.synchronize()
    means = []
    with ClockSampler(device_index) as clk:
        for _ in range(rounds):
            op.set_profiling(True)
            for _ in range(reps):
                op.apply(x, y)
            torch.cuda.synchronize()
            nl, t = op.kernel_time()
            means.append(t)
    op.set_profiling(False)
    med = sorted(means)[len(means) // 2]
    alg = ledger.op_bytes_fused(n, s["N_L"], 0)
    achieved = alg / med / 1e9
    out = {"workload": "C3 N=7: E=52x52x52 box, 48.6 M DOFs, operator apply (mass mode 0, lambda = 1)",
           "bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
           "frac": round(achieved / peak, 4), "peak_source": peak_src,
           "launch_ms": round(med * 1e3, 4), "round_means_ms": [round(v * 1e3, 4) for v in means],
           "timing": f"median of {rounds} means of {reps} back-to-back applies (P:268, c24), kernel events",
           "alg_bytes_per_launch": alg,
           "paper_ledger_gbs": round(ledger.op_bytes_paper(n, s["N_L"]) / med / 1e9, 1),
           "op_gflops": round(ledger.op_flops(s["E_local"], N) / med / 1e9, 1),
           "clocks": clk.summary()}
    del op, m
    torch.cuda.empty_cache()
    return out


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
        return
    import numpy as np
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    ipc = args.transport == "ipc"
    torch.cuda.set_device(local_rank % torch.cuda.device_count() if ipc else local_rank)
    if world > 1:
        if ipc:  # bootstrap only (records, barriers, the max over ranks); the data path is the library's
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))

    import __graft_entry__
    if rank == 0:
        __graft_entry__.build()
    if world > 1:
        dist.barrier()
    import paper_2202_12477_b200 as hb
    from paper_2202_12477_b200 import ledger

    blk = tuple(int(v) for v in args.box.split(","))
    N = args.N
    comm = None
    if world > 1:
        if args.strong:
            box = blk
            grid = hb.rank_grid(world, *box)
        else:
            grid = hb.rank_grid(world, 64, 64, 64)  # rank grid shape only (px >= py >= pz)
            box = (blk[0] * grid[0], blk[1] * grid[1], blk[2] * grid[2])
        if ipc:
            comm = hb.Comm.create_ipc(world, rank)
        else:
            uid = [hb.comm_unique_id() if rank == 0 else None]
            dist.broadcast_object_list(uid, src=0)
            comm = hb.Comm(world, rank, uid[0])
        mesh = hb.Mesh(*box, N, P=world, rank=rank, grid=grid)
    else:
        box = blk
        mesh = hb.Mesh(*box, N)
    op = hb.Operator(mesh, lam=1.0, comm=comm)
    if world > 1 and ipc:
        recs = [None] * world
        dist.all_gather_object(recs, op.ipc_export())
        op.ipc_connect(recs)
    if args.variant:
        op.set_variant(args.variant)
    if args.jacobi:
        op.set_jacobi(True)
    s = mesh.sizes
    n = op.n_owned
    E_glob, NG = s["E_global"], s["N_G"]
    NL_loc, NG_loc_ref = s["N_L"], n
    K = args.iters
    stream = torch.cuda.current_stream()
    b = torch.empty(n, dtype=torch.float64, device="cuda")
    x = torch.zeros_like(b)
    op.forcing(1, b)
    flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device="cuda")  # > 126 MB L2

    def step():
        if args.storage == "scattered":
            op.cg_scattered(b, x, K)
        else:
            op.cg(b, x, K)

    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()

    def timed_steps(nsteps):
        """nsteps CG steps, each bracketed by CUDA events on the launching stream, L2 flushed
        (256 MiB write) before each; returns the mean step time in ms (this rank)."""
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(nsteps)]
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        for t in range(nsteps):
            flush.zero_()
            ev[t][0].record(stream)
            step()
            ev[t][1].record(stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        return sum(a.elapsed_time(bv) for a, bv in ev) / nsteps

    rdev = "cpu" if ipc else "cuda"

    def max_over_ranks(v):
        t = torch.tensor([v], dtype=torch.float64, device=rdev)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return t.item()

    # ---- timed region: K steps, no instrumentation inside the solve
    l0 = op.launch_count()
    with ClockSampler(local_rank) as clk:
        my_ms = timed_steps(args.steps)
    launches = op.launch_count() - l0
    ms = max_over_ranks(my_ms)
    fom = ledger.nekbone_flops_per_iter(E_glob, N) * K / (ms * 1e-3) / 1e9
    gdofs = NG * K / (ms * 1e-3) / 1e9

    # ---- the operator's share of a step, without instrumenting the solve: the same graph with
    # the operator launches removed (vector kernels only, hb_op_set_timing_mode) timed the same
    # way; (step - vector-only step) / K = the operator's in-situ time per iteration, an upper
    # bound (alone, the vector kernels find their vectors in L2), so the fraction below is a
    # lower bound
    vec_ms = None
    if args.storage == "assembled" and not args.no_profile:
        op.set_timing_mode(True)
        for _ in range(2):
            step()
        vec_ms = max_over_ranks(timed_steps(args.steps))
        op.set_timing_mode(False)
        step()  # restore x / the solver state (and re-validate the normal graph)
        torch.cuda.synchronize()

    # ---- end-to-end: same solve through the host-buffer C-ABI call (H2D + D2H inside)
    bh = torch.empty(n, dtype=torch.float64, pin_memory=True)
    bh.copy_(b.cpu())
    xh = torch.empty(n, dtype=torch.float64, pin_memory=True)
    bnp, xnp = bh.numpy(), xh.numpy()
    for _ in range(2 if args.storage == "assembled" else 0):
        op.cg_host(bnp, xnp, K, hist=False)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e2e_ms = []
    for t in range(args.steps if args.storage == "assembled" else 0):
        flush.zero_()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        op.cg_host(bnp, xnp, K, hist=False)
        e2e_ms.append((time.perf_counter() - t0) * 1e3)
    e2e_v = max_over_ranks(sum(e2e_ms) / max(len(e2e_ms), 1))
    e2e_fom = ledger.nekbone_flops_per_iter(E_glob, N) * K / (e2e_v * 1e-3) / 1e9 if e2e_ms else None

    # ---- roofline of the dominant kernel (operator)
    peak, peak_src = peaks()
    roof = None
    roof_apply_s = None
    roof_note = None
    if vec_ms is not None and ms <= vec_ms:
        # no operator share to attribute (ranks time-sliced on one GPU: the exchanges' waits
        # dominate both steps) -- report no roofline rather than a negative one
        roof_note = (f"operator share not measurable: step {ms:.4f} ms <= vector-only step {vec_ms:.4f} ms")
        vec_ms = None
    if vec_ms is not None:
        mean_s = (ms - vec_ms) * 1e-3 / K
        alg_bytes = ledger.op_bytes_fused(n, NL_loc, 0)
        achieved = alg_bytes / mean_s / 1e9
        roof_apply_s = mean_s
        traffic = None
        prof = os.path.join(ROOT, "profiles", "ncu_op_summary.json")
        if world == 1 and os.path.exists(prof):  # captures are single-GPU launches of this workload
            with open(prof) as f:
                pj = json.load(f)
            key = f"N{N}_{blk[0]}x{blk[1]}x{blk[2]}"
            traffic = pj.get("dram_bytes_per_launch", {}).get(key)
        s81 = None  # the paper's 8:1 streaming rate, measured on a B200 by scripts/calib.py
        cal = os.path.join(ROOT, "profiles", "r1_calib_stream8to1.json")
        if os.path.exists(cal):
            with open(cal) as f:
                s81 = json.load(f).get("asymptotic_GBps")
        roof = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                "frac": round(achieved / peak, 4), "traffic": traffic,
                "frac_of_datasheet_7700": round(achieved / 7700.0, 4),
                "frac_of_stream8to1": round(achieved / s81, 4) if s81 else None,
                "kernel": f"operator N={N}" + (" (A + halo + B launches and exchanges of one apply)" if world > 1 else ""),
                "launch_ms": round(mean_s * 1e3, 4),
                "timing": "in-situ share: (CG step - same step without operator launches) / iterations, CUDA events",
                "alg_bytes_per_launch": alg_bytes, "peak_source": peak_src,
                "paper_ledger_gbs": round(ledger.op_bytes_paper(n, NL_loc) / mean_s / 1e9, 1),
                "op_gflops": round(ledger.op_flops(s["E_local"], N) / mean_s / 1e9, 1)}

    measured_bpd = None
    prof = os.path.join(ROOT, "profiles", "ncu_op_summary.json")
    if world == 1 and args.variant == 0 and args.storage == "assembled" and os.path.exists(prof):
        with open(prof) as f:
            dbl = json.load(f).get("dram_bytes_per_launch", {})
        ko, kv = f"N{N}_{blk[0]}x{blk[1]}x{blk[2]}", f"vec_N{N}_{blk[0]}x{blk[1]}x{blk[2]}"
        if ko in dbl and kv in dbl:
            measured_bpd = round((dbl[ko] + dbl[kv]) / NG, 2)

    roof_c3 = None
    if world == 1 and not args.no_c3 and (tuple(blk), N) == ((16, 16, 16), 7):
        roof_c3 = c3_operator_roofline(hb, ledger, peak, peak_src, local_rank)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(box, N, args.cpu_seconds)

    wname = {((16, 16, 16), 7): "C2", ((52, 52, 52), 7): "C3 N=7", ((66, 66, 66), 7): "C4 (1 GPU)",
             ((50, 50, 48), 15): "C5 (1 GPU)"}.get((tuple(blk), N), "custom")
    if rank == 0:
        out = {"metric": METRIC, "value": round(fom, 2), "unit": "GFLOP/s", "n_gpus": world, "steps": args.steps,
               "warmup": max(3, args.warmup), "ms_per_step": round(ms, 4), "higher_is_better": True,
               "scaling": "strong" if args.strong else "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
               "config": {"workload": f"{wname}: N={N}, E={box[0]}x{box[1]}x{box[2]} box, {K} CG iterations per step"
                                      + (f" (strong scaling: fixed box over {world} GPUs)" if world > 1 and args.strong else
                                         f" (weak scaling, {blk[0]}x{blk[1]}x{blk[2]} per GPU)" if world > 1 else ""),
                          "box": list(box), "N": N, "E": E_glob, "N_G": NG, "N_L": E_glob * (N + 1) ** 3,
                          "iterations": K, "lambda": 1.0, "mass_mode": 0, "forcing_seed": 1,
                          "l2": "flushed between steps (256 MiB write); working set > L2",
                          "parallelism": f"element partition p{world}",
                          "transport": (args.transport if world > 1 else None),
                          "assembly_variant": args.variant, "preconditioner": "jacobi" if args.jacobi else "none",
                          "storage": args.storage},
               "gdofs_per_s": round(gdofs, 4),
               "cg_bytes_per_iter_fused": ledger.cg_bytes_fused(NG, E_glob * (N + 1) ** 3),
               # bytes per DOF per CG iteration: this build's algorithmic ledger vs the paper's
               # assembled-storage minimum 108 + 80 N_L/N_G
               "bytes_per_dof_iter": round(ledger.cg_bytes_fused(NG, E_glob * (N + 1) ** 3) / NG, 2),
               "bytes_per_dof_iter_paper": round(ledger.cg_bytes_paper(NG, E_glob * (N + 1) ** 3) / NG, 2),
               # ncu DRAM bytes of one iteration's kernels (operator + vector update, committed
               # capture of this workload) per DOF
               "bytes_per_dof_iter_measured": measured_bpd,
               "cg_gbs_fused_ledger": round(ledger.cg_bytes_fused(NG, E_glob * (N + 1) ** 3) * K / (ms * 1e-3) / 1e9, 1),
               "e2e": ({"value": round(e2e_fom, 2), "unit": "GFLOP/s", "h2d_bytes_per_step": 8 * n,
                        "d2h_bytes_per_step": 8 * n + 48} if e2e_ms else None),
               "gpu_launches": launches,
               "phase_ms_per_iter": ({"operator": round(1e3 * roof_apply_s, 5),
                                      "vector_kernels": round(vec_ms / K, 5),
                                      "sum": round(ms / K, 5)} if vec_ms is not None else None),
               "roofline": roof,
               **({"roofline_note": roof_note} if roof_note else {}),
               "roofline_c3": roof_c3,
               "cpu_baseline": cpu,
               "clocks": clk.summary()}
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
