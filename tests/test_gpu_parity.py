"""GPU parity of the CUDA path (through the C ABI) against the CPU oracle.

Criteria (BASELINE.json north_star):
  * forcing, l2g map, partition: bit-exact;
  * operator: |y_i - o_i| <= 1e-12 * s_i with s = |A| |x| (c17);
  * CG: tolerance mode reaches the same iteration count with ||r|| within 1e-8 relative;
    fixed mode r.r history within 1e-8 relative up to the tolerance-mode stop j*, final x
    within 1e-10 ||x_o||_inf (c18).
"""
import numpy as np
import pytest

from oracle import basis, cg as ocg, forcing as of, mesh as om, operator as oo, partition as opart
from tests.inputs import random_positive, random_spd_factors, uniform_vector

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def hb():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import __graft_entry__
    __graft_entry__.build()
    import paper_2202_12477_b200 as hb
    torch.cuda.set_device(0)
    return hb


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to("cuda")


class OracleProblem:
    def __init__(self, box, N, ext=(2.0, 2.0, 2.0), mass_mode=0, G=None, B=None):
        self.box, self.N = box, N
        self.x, self.w, self.D = basis.basis(N)
        self.E, self.NG, self.NL = om.global_sizes(*box, N)
        self.gid = om.l2g(*box, N)
        self.G = om.geometric_factors(self.E, N, self.w, ext) if G is None else G
        if mass_mode == 0:
            self.M = om.weights_W(self.gid, self.NG)
        else:
            self.M = om.mass_B(self.E, N, self.w, ext) if B is None else B

    def apply(self, v, lam):
        return oo.apply(v, self.gid, self.D, self.G, lam, self.M)

    def scale(self, v, lam):
        if self.N <= 5:
            return oo.apply_abs_explicit(v, self.gid, self.D, self.G, lam, self.M)
        return oo.apply_abs(v, self.gid, self.D, self.G, lam, self.M)


def check_apply(hb, box, N, lam, mass_mode, random_geom, seed=0, ext=(2.0, 2.0, 2.0)):
    G = random_spd_factors(np.prod(box), (N + 1) ** 3, seed=seed + 17, scale=None) if random_geom else None
    B = random_positive((np.prod(box), (N + 1) ** 3), seed + 5) if (random_geom and mass_mode == 1) else None
    o = OracleProblem(box, N, ext, mass_mode, G, B)
    m = hb.Mesh(*box, N, ext=ext, mass_mode=mass_mode)
    if G is not None:
        m.set_geometry(G)
    if B is not None:
        m.set_mass(B)
    op = hb.Operator(m, lam=lam)
    xv = uniform_vector(o.NG, seed + 1)
    y = torch.full((o.NG,), np.nan, dtype=torch.float64, device="cuda")
    op.apply(dev(xv), y)
    torch.cuda.synchronize()
    yo = o.apply(xv, lam)
    s = o.scale(xv, lam)
    err = np.abs(y.cpu().numpy() - yo) / s
    assert np.all(np.isfinite(y.cpu().numpy()))
    assert err.max() <= 1e-12, (box, N, lam, mass_mode, err.max())
    return err.max()


@pytest.mark.parametrize("N", list(range(1, 16)))
def test_apply_all_degrees_random_geometry(hb, N):
    # several CTAs' worth of elements and a ragged tail (E odd, not a multiple of EPB)
    box = (3, 3, 3) if N <= 7 else (3, 2, 1)
    check_apply(hb, box, N, 1.0, 0, True, seed=N)


def _multiwave_box(hb, N, waves=3):
    """A box whose element count is >= `waves` full grid waves of the operator's resident launch
    (every CTA runs its grid-stride loop at least `waves` times) plus a ragged tail."""
    shape = hb.Operator(hb.Mesh(1, 1, 1, N)).launch_shape()
    need = waves * shape["grid"] * shape["epb"] + shape["epb"] // 2 + 1
    a = max(2, int(round(need ** (1.0 / 3.0))))
    c = -(-need // (a * (a + 1)))
    box = (a, a + 1, c)
    E = a * (a + 1) * c
    if shape["epb"] > 1 and E % shape["epb"] == 0:
        box = (a, a + 1, c + 1)
    return box, shape


@pytest.mark.parametrize("N", list(range(1, 16)))
def test_apply_multiwave_random_geometry(hb, N):
    """Every degree at >= 3 grid waves of its resident launch (the grid-stride loop wraps, as
    at the benchmark sizes) with random SPD geometric factors: the whole output vector under
    c17 (scale: the pinned sum-factorised |D|^T|G||D| bound, R5)."""
    box, shape = _multiwave_box(hb, N)
    E = int(np.prod(box))
    assert E >= 3 * shape["grid"] * shape["epb"]
    G = random_spd_factors(E, (N + 1) ** 3, seed=200 + N)
    o = OracleProblem(box, N, G=G)
    m = hb.Mesh(*box, N)
    m.set_geometry(G)
    op = hb.Operator(m, lam=1.0)
    xv = uniform_vector(o.NG, 300 + N)
    y = torch.full((o.NG,), np.nan, dtype=torch.float64, device="cuda")
    op.apply(dev(xv), y)
    yg = y.cpu().numpy()
    assert np.all(np.isfinite(yg))
    yo = o.apply(xv, 1.0)
    s = oo.apply_abs(xv, o.gid, o.D, o.G, 1.0, o.M)
    err = np.abs(yg - yo) / s
    assert err.max() <= 1e-12, (box, N, err.max())
    # a second apply of the same input agrees to rounding (atomic order only)
    op.apply(dev(xv), y)
    assert (np.abs(y.cpu().numpy() - yo) / s).max() <= 1e-12


@pytest.mark.parametrize("N", [1, 2, 3, 4, 6, 7, 9, 15])  # 2, 4: odd slabs; 6: aligned rows
@pytest.mark.parametrize("mass_mode,lam", [(0, 0.0), (0, 2.5), (1, 1.0)])
def test_apply_modes(hb, N, mass_mode, lam):
    box = (2, 3, 1)
    check_apply(hb, box, N, lam, mass_mode, True, seed=100 + N)


@pytest.mark.parametrize("N", [2, 7])
def test_apply_box_geometry_unequal_extents(hb, N):
    check_apply(hb, (4, 1, 2), N, 1.0, 1, False, ext=(1.0, 2.0, 0.5))
    check_apply(hb, (4, 1, 2), N, 1.0, 0, False, ext=(1.0, 2.0, 0.5))


@pytest.mark.parametrize("N", [1, 6, 15])
def test_apply_single_element(hb, N):
    check_apply(hb, (1, 1, 1), N, 1.0, 0, True, seed=3)


def test_forcing_bit_exact(hb):
    for box, N, seed in [((2, 2, 2), 3, 1), ((16, 16, 16), 7, 1), ((5, 3, 2), 4, 123456789)]:
        m = hb.Mesh(*box, N)
        op = hb.Operator(m)
        b = torch.empty(op.n_owned, dtype=torch.float64, device="cuda")
        op.forcing(seed, b)
        bo = of.forcing(range(op.n_owned), seed)
        assert np.array_equal(b.cpu().numpy(), bo)


def test_dot(hb):
    m = hb.Mesh(5, 4, 3, 3)
    op = hb.Operator(m)
    a, b = uniform_vector(op.n_owned, 1), uniform_vector(op.n_owned, 2)
    v = op.dot(dev(a), dev(b))
    assert abs(v - ocg.dot(a, b)) <= 1e-13 * np.abs(a * b).sum()


def test_C2_apply_full(hb):
    """C2 (N=7, 16^3): the whole vector against the oracle (survey golden values too)."""
    box, N = (16, 16, 16), 7
    o = OracleProblem(box, N)
    m = hb.Mesh(*box, N)
    op = hb.Operator(m)
    b = torch.empty(o.NG, dtype=torch.float64, device="cuda")
    op.forcing(1, b)
    y = torch.empty_like(b)
    op.apply(b, y)
    bo = of.forcing(range(o.NG), 1)
    yo = o.apply(bo, 1.0)
    s = o.scale(bo, 1.0)
    yg = y.cpu().numpy()
    assert (np.abs(yg - yo) / s).max() <= 1e-12
    np.testing.assert_allclose([yg[0], yg[o.NG // 2], yg[-1]],
                               [0.13528629240893, -0.60144944969253, 0.96623820349107], rtol=0, atol=1e-13)


def _cg_contract(hist_gpu, hist_o, j_star):
    hg = np.asarray(hist_gpu[: j_star + 1])
    ho = np.asarray(hist_o[: j_star + 1])
    assert (np.abs(hg - ho) / ho).max() <= 1e-8


@pytest.mark.parametrize("box,N,K", [((2, 2, 2), 3, 50), ((16, 16, 16), 7, 100)])
def test_cg_parity(hb, box, N, K):
    o = OracleProblem(box, N)
    A = lambda v: o.apply(v, 1.0)
    bo = of.forcing(range(o.NG), 1)
    bb = ocg.dot(bo, bo)
    eps = 1e-16 * bb
    xo_t, jo, ho_t = ocg.cg(A, bo, max_iters=K, eps=eps)
    m = hb.Mesh(*box, N)
    op = hb.Operator(m)
    b = torch.empty(o.NG, dtype=torch.float64, device="cuda")
    op.forcing(1, b)
    # (i) tolerance mode: same iteration count, ||r|| within 1e-8, stop not ambiguous
    x = torch.zeros_like(b)
    jg, hg = op.cg(b, x, K, eps)
    assert jg == jo, (jg, jo)
    assert abs(np.sqrt(hg[-1]) - np.sqrt(ho_t[-1])) <= 1e-8 * np.sqrt(ho_t[-1])
    assert not (abs(ho_t[-1] / eps - 1) < 1e-6)
    # (ii) fixed mode: history prefix up to j*, final x, true residuals
    x = torch.zeros_like(b)
    jf, hf = op.cg(b, x, K)
    assert jf == K and len(hf) == K + 1
    _cg_contract(hf, ho_t, jo)
    xf = x.cpu().numpy()
    # the K-iteration x against the survey's independent scratch oracle (Appendix A:
    # sum and 2-norm of x after the fixed 50 / 100 iterations, reproducible to ~1e-13)
    g = _appendix_a()["C1" if N == 3 else "C2"]
    assert g["fixed_iters"] == K
    assert abs(xf.sum() - g["fixed_sum_x"]) <= 1e-12 * abs(g["fixed_sum_x"])
    assert abs(np.linalg.norm(xf) - g["fixed_norm_x"]) <= 1e-12 * g["fixed_norm_x"]
    if np.prod(box) <= 8:
        xo, _, _ = ocg.cg(A, bo, max_iters=K)
        assert np.abs(xf - xo).max() <= 1e-10 * np.abs(xo).max()
        xs = (xf, xo)
    else:  # C2: 100 oracle iterations take ~1 min; the oracle x is compared at the tolerance stop
        xs = (xf,)
        x = torch.zeros_like(b)
        op.cg(b, x, jo)
        assert np.abs(x.cpu().numpy() - xo_t).max() <= 1e-10 * np.abs(xo_t).max()
    for xv in xs:  # c18: true residuals of the fixed-mode solutions
        assert np.linalg.norm(bo - A(xv)) <= 1e-10 * np.linalg.norm(bo)


def _appendix_a():
    import json
    import os
    with open(os.path.join(os.path.dirname(__file__), "golden", "appendix_a.json")) as f:
        return json.load(f)


def test_cg_host_path_matches_device_path(hb):
    box, N = (4, 4, 4), 5
    m = hb.Mesh(*box, N)
    op = hb.Operator(m)
    b = torch.empty(op.n_owned, dtype=torch.float64, device="cuda")
    op.forcing(1, b)
    x = torch.zeros_like(b)
    j1, h1 = op.cg(b, x, 20)
    bh = b.cpu().numpy().copy()
    xh = np.zeros_like(bh)
    j2, h2 = op.cg_host(bh, xh, 20)
    assert j1 == j2 == 20
    # fp64 atomics: the two runs differ only in summation order
    assert (np.abs(h1 - h2) / h1).max() <= 1e-10
    assert np.abs(x.cpu().numpy() - xh).max() <= 1e-10 * np.abs(xh).max()


def test_cg_zero_rhs_and_breakdown(hb):
    m = hb.Mesh(2, 2, 2, 3)
    op = hb.Operator(m)
    b = torch.zeros(op.n_owned, dtype=torch.float64, device="cuda")
    x = torch.ones_like(b)
    j, h = op.cg(b, x, 10, 0.0)
    assert j == 0 and h[0] == 0.0 and not x.cpu().numpy().any()
    # lambda < 0 makes A indefinite: tolerance mode must report a breakdown, not loop
    op2 = hb.Operator(m, lam=-100.0)
    bb = torch.empty_like(b)
    op2.forcing(1, bb)
    with pytest.raises(hb.HBError, match="BREAKDOWN"):
        op2.cg(bb, x, 50, 1e-30)


@pytest.mark.parametrize("P", [2, 4, 8])
def test_loopback_group_apply_and_cg(hb, P):
    """P virtual ranks on one GPU (exchanges as device copies): apply equals the oracle,
    CG equals the P=1 oracle within c18."""
    box, N = (4, 4, 4), 3
    o = OracleProblem(box, N)
    Gr = random_spd_factors(o.E, (N + 1) ** 3, seed=9)
    o.G = Gr
    xv = uniform_vector(o.NG, 4)
    yo = o.apply(xv, 1.0)
    s = o.scale(xv, 1.0)
    meshes, ops = [], []
    for r in range(P):
        m = hb.Mesh(*box, N, P=P, rank=r)
        m.set_geometry(Gr[m.elements()])
        meshes.append(m)
        ops.append(hb.Operator(m))
    g = hb.Group(ops)
    xs = [dev(xv[m.owned()]) for m in meshes]
    ys = [torch.full_like(t, np.nan) for t in xs]
    g.apply(xs, ys)
    torch.cuda.synchronize()
    y = np.full(o.NG, np.nan)
    for m, t in zip(meshes, ys):
        y[m.owned()] = t.cpu().numpy()
    assert (np.abs(y - yo) / s).max() <= 1e-12
    # CG with the box geometry
    for m in meshes:
        m.set_geometry(om.geometric_factors(m.sizes["E_local"], N, o.w))
    ops = [hb.Operator(m) for m in meshes]
    g = hb.Group(ops)
    bo = of.forcing(range(o.NG), 1)
    bs = []
    for m, op in zip(meshes, ops):
        t = torch.empty(op.n_owned, dtype=torch.float64, device="cuda")
        op.forcing(1, t)
        assert np.array_equal(t.cpu().numpy(), bo[m.owned()])
        bs.append(t)
    o.G = om.geometric_factors(o.E, N, o.w)
    eps = 1e-16 * ocg.dot(bo, bo)
    xo, jo, ho = ocg.cg(lambda v: o.apply(v, 1.0), bo, max_iters=100, eps=eps)
    xs = [torch.zeros_like(t) for t in bs]
    j, h = g.cg(bs, xs, 100, eps)
    assert j == jo
    _cg_contract(h, ho, jo)
    x = np.zeros(o.NG)
    for m, t in zip(meshes, xs):
        x[m.owned()] = t.cpu().numpy()
    assert np.abs(x - xo).max() <= 1e-10 * np.abs(xo).max()


C3_BOXES = {1: (120, 100, 91), 2: (184, 184, 184), 3: (122, 122, 122), 4: (92, 92, 92), 5: (73, 73, 73),
             6: (61, 61, 61), 7: (52, 52, 52), 8: (46, 46, 46), 9: (41, 41, 41), 10: (37, 37, 37),
             11: (33, 33, 33), 12: (31, 31, 31), 13: (28, 28, 28), 14: (26, 26, 26), 15: (24, 24, 24)}


@pytest.mark.parametrize("box,N", [(C3_BOXES[n], n) for n in range(1, 16)])
def test_full_size_C3_sampled_and_properties(hb, box, N):
    """C3 at full size (~50 M DOFs), the launch configuration bench.py / opbench time:
    sampled entries against the oracle computed one by one (c17 scale from |D|, |G|), plus
    A 1 = lambda 1 and sum(A x) = lambda sum(x) (mass mode 0) over the whole vector."""
    m = hb.Mesh(*box, N)
    op = hb.Operator(m)
    n = op.n_owned
    b = torch.empty(n, dtype=torch.float64, device="cuda")
    op.forcing(2, b)
    y = torch.empty_like(b)
    op.apply(b, y)
    torch.cuda.synchronize()
    rng = np.random.default_rng(N)
    gx = box[0] * N + 1
    sample = np.unique(np.concatenate([rng.integers(0, n, 120), [0, n - 1, n // 2, gx * gx * N, N * gx + N]]))
    xg, w, D = basis.basis(N)
    Ge = om.geometric_factors(1, N, w)[0]
    wrow = lambda e, row: _w_row(row, box, N)
    yo = oo.apply_entries(lambda row: of.forcing(row, 2), sample.tolist(), *box, N, D, lambda e: Ge, 1.0,
                          wrow, om.l2g)
    so = oo.apply_entries(lambda row: np.abs(of.forcing(row, 2)), sample.tolist(), *box, N, np.abs(D),
                          lambda e: np.abs(Ge), 1.0, wrow, om.l2g)
    yg = y.cpu().numpy()[sample]
    assert (np.abs(yg - yo) / so).max() <= 1e-12
    ones = torch.ones(n, dtype=torch.float64, device="cuda")
    op.apply(ones, y)
    assert (y - 1.0).abs().max().item() <= 1e-12
    op.apply(b, y)
    assert abs(y.sum().item() - b.sum().item()) <= 1e-9 * b.abs().sum().item()


def _w_row(row, box, N):
    """W of the slots of one element: 1 / number of elements containing the point."""
    nx, ny, nz = box
    gx, gy = nx * N + 1, ny * N + 1
    X, Y, Z = row % gx, (row // gx) % gy, row // (gx * gy)

    def c(P0, n_el):
        return np.where((P0 % N == 0) & (P0 > 0) & (P0 < n_el * N), 2, 1)
    return 1.0 / (c(X, nx) * c(Y, ny) * c(Z, nz))


def test_stream_bench_runs(hb):
    v = hb.stream_bench(1 << 22, 5)
    assert np.isfinite(v) and v > 1e11


@pytest.mark.parametrize("N,mass_mode", [(4, 1), (7, 0), (2, 1), (11, 1), (12, 0), (13, 0), (13, 1), (14, 0), (15, 0)])
def test_cg_random_geometry_both_mass_modes(hb, N, mass_mode):
    """CG with random SPD geometric factors (cross terms live) and both mass modes: the
    fused p.Ap (element energy + lambda p.p, or + lambda u.B u in mode 1) must give the
    oracle's Alg. 1 iterates (c18)."""
    box = (3, 2, 3)
    E = int(np.prod(box))
    # geometry scaled by the GLL weight products like the real factors, so the
    # problem is as well conditioned as the benchmark's and CG is not in the roundoff regime
    xg, w = basis.gll(N)
    wq = np.einsum("k,j,i->kji", w, w, w).ravel()
    G = random_spd_factors(E, (N + 1) ** 3, seed=31 + N, scale=wq)
    B = random_positive((E, (N + 1) ** 3), 77) if mass_mode == 1 else None
    o = OracleProblem(box, N, mass_mode=mass_mode, G=G, B=B)
    A = lambda v: o.apply(v, 1.0)
    bo = of.forcing(range(o.NG), 1)
    eps = 1e-16 * ocg.dot(bo, bo)
    xo, jo, ho = ocg.cg(A, bo, max_iters=300, eps=eps)
    m = hb.Mesh(*box, N, mass_mode=mass_mode)
    m.set_geometry(G)
    if B is not None:
        m.set_mass(B)
    op = hb.Operator(m)
    b = torch.empty(o.NG, dtype=torch.float64, device="cuda")
    op.forcing(1, b)
    x = torch.zeros_like(b)
    jg, hg = op.cg(b, x, 300, eps)
    assert jg == jo and jo < 100
    _cg_contract(hg, ho, jo - 1)
    assert np.abs(x.cpu().numpy() - xo).max() <= 1e-10 * np.abs(xo).max()
    x = torch.zeros_like(b)
    jf, hf = op.cg(b, x, jo)  # fixed mode, graph path
    _cg_contract(hf, ho, jo - 1)


@pytest.mark.parametrize("box,N,P", [((5, 4, 3), 7, 4), ((6, 3, 5), 2, 6), ((3, 3, 3), 5, 3), ((9, 7, 5), 1, 4),
                                     ((4, 3, 5), 6, 3), ((5, 3, 4), 4, 2)])
def test_loopback_uneven_partitions_cg(hb, box, N, P):
    """Uneven element splits (remainder layers), several neighbour counts, N=2..7: the split
    apply with per-rank compute/communication streams and the loopback transport (the NCCL
    message lists) reproduces the P=1 oracle's CG iterates (c18)."""
    o = OracleProblem(box, N)
    A = lambda v: o.apply(v, 1.0)
    bo = of.forcing(range(o.NG), 1)
    eps = 1e-16 * ocg.dot(bo, bo)
    xo, jo, ho = ocg.cg(A, bo, max_iters=200, eps=eps)
    meshes = [hb.Mesh(*box, N, P=P, rank=r, seed=3) for r in range(P)]
    ops = [hb.Operator(m) for m in meshes]
    g = hb.Group(ops)
    bs, xs = [], []
    for m, op in zip(meshes, ops):
        t = torch.empty(op.n_owned, dtype=torch.float64, device="cuda")
        op.forcing(1, t)
        bs.append(t)
        xs.append(torch.zeros_like(t))
    j, h = g.cg(bs, xs, 200, eps)
    assert j == jo
    _cg_contract(h, ho, jo - 1)
    x = np.zeros(o.NG)
    for m, t in zip(meshes, xs):
        x[m.owned()] = t.cpu().numpy()
    assert np.abs(x - xo).max() <= 1e-10 * np.abs(xo).max()
    # the fixed-iteration group solve (no host checks) agrees too
    xs2 = [torch.zeros_like(t) for t in bs]
    j2, h2 = g.cg(bs, xs2, jo)
    assert j2 == jo
    _cg_contract(h2, ho, jo - 1)


def test_tolerance_mode_device_graph_matches_host_loop(hb):
    """Tolerance mode as one CUDA graph with a WHILE node (device-side loop test, NEXT #1)
    against the host-driven loop: same iteration count, histories equal to c18 tolerance,
    and the oracle's stop index."""
    box, N = (6, 5, 4), 5
    o = OracleProblem(box, N)
    bo = of.forcing(range(o.NG), 1)
    eps = 1e-16 * ocg.dot(bo, bo)
    xo, jo, ho = ocg.cg(lambda v: o.apply(v, 1.0), bo, max_iters=200, eps=eps)
    m = hb.Mesh(*box, N)
    op = hb.Operator(m)
    b = torch.empty(o.NG, dtype=torch.float64, device="cuda")
    op.forcing(1, b)
    res = {}
    for mode in ("1", "0"):
        op.set_tolerance_loop(mode == "1")
        x = torch.zeros_like(b)
        for rep in range(2):  # second run replays the cached graph
            j, h = op.cg(b, x, 200, eps)
        res[mode] = (j, h, x.cpu().numpy())
    assert res["1"][0] == res["0"][0] == jo
    _cg_contract(res["1"][1], ho, jo - 1)
    _cg_contract(res["0"][1], ho, jo - 1)
    assert np.abs(res["1"][2] - xo).max() <= 1e-10 * np.abs(xo).max()
    # max_iters caps the device loop
    op.set_tolerance_loop(True)
    x = torch.zeros_like(b)
    j, h = op.cg(b, x, 7, eps)
    assert j == 7 and len(h) == 8


@pytest.mark.parametrize("N,mass_mode", [(2, 1), (3, 0), (5, 1), (6, 0), (7, 0), (8, 1)])  # 2, 7, 8: factor-pair G layout
def test_jacobi_pcg(hb, N, mass_mode):
    """Jacobi-preconditioned CG (NEXT #3): diag(A) against the oracle's assembled element
    diagonals; PCG iterates (fixed and tolerance modes, device-graph and host loops) against
    the oracle's PCG (c18)."""
    box = (3, 2, 3)
    E = int(np.prod(box))
    xg, w = basis.gll(N)
    wq = np.einsum("k,j,i->kji", w, w, w).ravel()
    G = random_spd_factors(E, (N + 1) ** 3, seed=51 + N, scale=wq)
    B = (random_positive((E, (N + 1) ** 3), 8) * np.exp(2.0 * uniform_vector(E * (N + 1) ** 3, 9)).reshape(E, -1)
         if mass_mode == 1 else None)
    o = OracleProblem(box, N, mass_mode=mass_mode, G=G, B=B)
    d_o = oo.diagonal(o.gid, o.NG, o.D, o.G, 1.0, o.M)
    m = hb.Mesh(*box, N, mass_mode=mass_mode)
    m.set_geometry(G)
    if B is not None:
        m.set_mass(B)
    op = hb.Operator(m)
    op.set_jacobi(True)
    dg = torch.empty(o.NG, dtype=torch.float64, device="cuda")
    op.jacobi_diagonal(dg)
    assert np.max(np.abs(dg.cpu().numpy() - d_o) / d_o) <= 1e-13
    A = lambda v: o.apply(v, 1.0)
    bo = of.forcing(range(o.NG), 1)
    eps = 1e-16 * ocg.dot(bo, bo)
    xo, jo, ho = ocg.pcg(A, bo, 1.0 / d_o, max_iters=300, eps=eps)
    b = torch.empty(o.NG, dtype=torch.float64, device="cuda")
    op.forcing(1, b)
    for mode in ("1", "0"):
        op.set_tolerance_loop(mode == "1")
        x = torch.zeros_like(b)
        j, h = op.cg(b, x, 300, eps)
        assert j == jo
        _cg_contract(h, ho, jo - 1)
        assert np.abs(x.cpu().numpy() - xo).max() <= 1e-10 * np.abs(xo).max()
    x = torch.zeros_like(b)
    jf, hf = op.cg(b, x, jo)
    _cg_contract(hf, ho, jo - 1)
    # switching back gives plain CG again
    op.set_jacobi(False)
    xc, jc, hc = ocg.cg(A, bo, max_iters=300, eps=eps)
    x = torch.zeros_like(b)
    j, h = op.cg(b, x, 300, eps)
    # this random-geometry, exp-varied-mass problem is ill-conditioned for plain CG: rounding-order
    # differences (fp64 RED assembly) grow over 80+ iterations and the oracle's stop is only 9%
    # under eps, so the switch-back is checked on the early history (which already tells plain
    # CG from PCG at iteration 1) and the stop to within one iteration; c18's exact count is
    # enforced on the well-conditioned problems (test_cg_parity, the PCG runs above)
    assert abs(j - jc) <= 1
    _cg_contract(h, hc, min(j, jc, 20))


@pytest.mark.parametrize("N,mass_mode", [(3, 0), (7, 1), (10, 0), (6, 1), (4, 0)])
def test_deterministic_csr_variant(hb, N, mass_mode):
    """Assembly variant 1 (y_L + CSR gather in ascending (e, n) order): operator parity
    (c17), CG parity (c18), and bitwise reproducibility of repeated applies and solves."""
    box = (3, 3, 2)
    E = int(np.prod(box))
    G = random_spd_factors(E, (N + 1) ** 3, seed=61 + N)
    B = random_positive((E, (N + 1) ** 3), 4) if mass_mode == 1 else None
    o = OracleProblem(box, N, mass_mode=mass_mode, G=G, B=B)
    m = hb.Mesh(*box, N, mass_mode=mass_mode)
    m.set_geometry(G)
    if B is not None:
        m.set_mass(B)
    op = hb.Operator(m)
    op.set_variant(1)
    xv = uniform_vector(o.NG, 12)
    xd = dev(xv)
    y1 = torch.empty_like(xd)
    y2 = torch.empty_like(xd)
    op.apply(xd, y1)
    op.apply(xd, y2)
    assert torch.equal(y1, y2)
    yo = o.apply(xv, 1.0)
    s = o.scale(xv, 1.0)
    assert (np.abs(y1.cpu().numpy() - yo) / s).max() <= 1e-12
    b = torch.empty(o.NG, dtype=torch.float64, device="cuda")
    op.forcing(1, b)
    x1, x2 = torch.zeros_like(b), torch.zeros_like(b)
    j1, h1 = op.cg(b, x1, 30)
    j2, h2 = op.cg(b, x2, 30)
    assert np.array_equal(h1, h2) and torch.equal(x1, x2)
    bo = of.forcing(range(o.NG), 1)
    xo, jo, ho = ocg.cg(lambda v: o.apply(v, 1.0), bo, max_iters=30)
    jt = min(30, next((k for k, v in enumerate(ho) if v <= 1e-16 * ho[0]), 30))
    _cg_contract(h1, ho, jt - 1)


@pytest.mark.parametrize("box,N", [((2, 2, 2), 3), ((5, 4, 3), 7), ((3, 2, 2), 6)])
def test_scattered_storage_cg(hb, box, N):
    """NekBone's scattered storage (NEXT #4): CG on x_L = Z x with Z Z^T S_L +
    lambda I and W-weighted dots has the same iterates as the assembled CG (the weighted
    dots equal the assembled ones), so it must match the oracle's Alg. 1 (c18)."""
    o = OracleProblem(box, N)
    A = lambda v: o.apply(v, 1.0)
    bo = of.forcing(range(o.NG), 1)
    eps = 1e-16 * ocg.dot(bo, bo)
    xo, jo, ho = ocg.cg(A, bo, max_iters=200, eps=eps)
    m = hb.Mesh(*box, N)
    op = hb.Operator(m)
    b = torch.empty(o.NG, dtype=torch.float64, device="cuda")
    op.forcing(1, b)
    x = torch.zeros_like(b)
    j, h = op.cg_scattered(b, x, 200, eps)
    assert j == jo
    _cg_contract(h, ho, jo - 1)
    assert np.abs(x.cpu().numpy() - xo).max() <= 1e-10 * np.abs(xo).max()
    x = torch.zeros_like(b)
    jf, hf = op.cg_scattered(b, x, jo)  # fixed mode, captured graph
    assert jf == jo
    _cg_contract(hf, ho, jo - 1)
    with pytest.raises(hb.HBError, match="STATE"):
        hb.Operator(hb.Mesh(*box, N, mass_mode=1)).cg_scattered(b, x, 3)
