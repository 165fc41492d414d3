"""Pins of oracle/basis.py, oracle/mesh.py, oracle/forcing.py, oracle/ledger.py against
closed forms, invariants and cited golden values (tests/golden/)."""
import json
import math
import os

import numpy as np
import pytest

from oracle import basis, forcing, ledger, mesh

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def _num(v):
    if isinstance(v, (int, float)):
        return float(v)
    v = v.replace("sqrt5", str(math.sqrt(5.0)))
    return float(eval(v))  # fractions like "4/3"


# ---------------------------------------------------------------- GLL / D
@pytest.mark.parametrize("N", ["1", "2", "3"])
def test_gll_closed_forms(N):
    g = gold("gll_closed_forms.json")["gll"][N]
    x, w = basis.gll(int(N))
    np.testing.assert_allclose(x, [_num(v) for v in g["nodes"]], rtol=0, atol=2e-16)
    np.testing.assert_allclose(w, [_num(v) for v in g["weights"]], rtol=0, atol=4e-16)


@pytest.mark.parametrize("N", range(1, 16))
def test_gll_quadrature_exactness(N):
    """sum_i w_i x_i^k = int_{-1}^{1} x^k dx for k <= 2N-1 (GLL exactness), and NOT for
    k = 2N (so the rule is Lobatto with N+1 points, not Gauss)."""
    x, w = basis.gll(N)
    assert abs(w.sum() - 2.0) < 1e-14
    for k in range(0, 2 * N):
        exact = 0.0 if k % 2 else 2.0 / (k + 1)
        assert abs(np.dot(w, x ** k) - exact) < 2e-15, (N, k)
    assert abs(np.dot(w, x ** (2 * N)) - 2.0 / (2 * N + 1)) > 1e-10
    # nodes strictly increasing, symmetric, endpoints
    assert np.all(np.diff(x) > 0) and x[0] == -1.0 and x[-1] == 1.0
    assert np.array_equal(x, -x[::-1])


@pytest.mark.parametrize("N", ["1", "2"])
def test_D_closed_forms(N):
    x, w, D = basis.basis(int(N))
    np.testing.assert_allclose(D, gold("gll_closed_forms.json")["D"][N], rtol=0, atol=1e-15)


@pytest.mark.parametrize("N", range(1, 16))
def test_D_differentiates_polynomials(N):
    """D is the unique matrix exact on degree <= N polynomials: D x^k = k x^(k-1)."""
    x, w, D = basis.basis(N)
    for k in range(0, N + 1):
        expect = k * x ** (k - 1) if k > 0 else np.zeros_like(x)
        assert np.max(np.abs(D @ x ** k - expect)) < 5e-13 * max(1, k * k), (N, k)


# ---------------------------------------------------------------- mesh (c7)
@pytest.mark.parametrize("box,N", [((2, 2, 2), 7), ((3, 2, 1), 2), ((1, 1, 1), 1), ((2, 3, 4), 3)])
def test_l2g_counts_and_sizes(box, N):
    E, NG, NL = mesh.global_sizes(*box, N)
    gid = mesh.l2g(*box, N)
    assert gid.shape == (E, (N + 1) ** 3)
    assert len(np.unique(gid)) == NG and gid.min() == 0 and gid.max() == NG - 1
    c = mesh.counts(gid, NG)
    assert set(np.unique(c)) <= {1, 2, 4, 8}
    # closed form: number of gids with count 2^d = product over axes of per-axis factors
    nx, ny, nz = box
    def axis_hist(n):  # points along one axis shared by 1 or 2 elements
        return {1: n * N + 1 - (n - 1), 2: n - 1}
    hist = {}
    for a, ca in axis_hist(nx).items():
        for b, cb in axis_hist(ny).items():
            for d, cd in axis_hist(nz).items():
                hist[a * b * d] = hist.get(a * b * d, 0) + ca * cb * cd
    got = {int(k): int(v) for k, v in zip(*np.unique(c, return_counts=True))}
    assert got == {k: v for k, v in hist.items() if v}


def test_l2g_2x2x2_N7():
    E, NG, NL = mesh.global_sizes(2, 2, 2, 7)
    assert (NG, NL) == (3375, 4096)


@pytest.mark.parametrize("box,N,ext", [((2, 3, 2), 3, (2.0, 1.0, 0.5)), ((3, 1, 2), 4, (1.0, 1.0, 1.0))])
def test_l2g_geometric_consistency(box, N, ext):
    """Slots with equal gid are the same physical point, different gids different points:
    element-local coordinates (origin + (x_i+1) h/2) vs the global point grid."""
    x, w = basis.gll(N)
    nx, ny, nz = box
    gid = mesh.l2g(*box, N)
    X, Y, Z = mesh.node_coords(*box, N, x, ext)
    NP = N + 1
    for e in range(gid.shape[0]):
        ex, ey, ez = mesh.element_coords(e, nx, ny)
        for n in range(NP ** 3):
            i, j, k = n % NP, (n // NP) % NP, n // NP ** 2
            p = (ex * ext[0] + (x[i] + 1) * ext[0] / 2, ey * ext[1] + (x[j] + 1) * ext[1] / 2,
                 ez * ext[2] + (x[k] + 1) * ext[2] / 2)
            g = gid[e, n]
            assert abs(X[g] - p[0]) < 1e-13 and abs(Y[g] - p[1]) < 1e-13 and abs(Z[g] - p[2]) < 1e-13
    pts = np.round(np.stack([X, Y, Z], 1), 12)
    assert len(np.unique(pts, axis=0)) == len(X)


def test_geometry_goldens():
    g = gold("geometry.json")
    for key in ("unit_cube_N1", "box_2x1x1_N1"):
        c = g[key]
        x, w = basis.gll(c["N"])
        G = mesh.geometric_factors(1, c["N"], w, tuple(c["ext"]))
        np.testing.assert_allclose(G[0, :, 0], c["rr"], rtol=1e-15)
        np.testing.assert_allclose(G[0, :, 3], c["ss"], rtol=1e-15)
        np.testing.assert_allclose(G[0, :, 5], c["tt"], rtol=1e-15)
        assert np.all(G[0, :, [1, 2, 4]] == 0.0)
    c = g["unit_cube_N2_centre"]
    x, w = basis.gll(2)
    G = mesh.geometric_factors(1, 2, w, tuple(c["ext"]))
    assert abs(G[0, 1 + 3 * (1 + 3 * 1), 0] - _num(c["rr"])) < 1e-15
    with pytest.raises(ValueError):
        mesh.geometric_factors(1, 2, w, (1.0, 0.0, 1.0))


@pytest.mark.parametrize("box,N", [((3, 3, 3), 7), ((2, 1, 3), 2)])
def test_W_identity(box, N):
    """Z^T W Z = I (reading c1) and adjointness (Zx).y = x.(Z^T y)."""
    from tests.inputs import uniform_vector
    E, NG, NL = mesh.global_sizes(*box, N)
    gid = mesh.l2g(*box, N)
    W = mesh.weights_W(gid, NG)
    xg = uniform_vector(NG, 5)
    back = np.bincount(gid.ravel(), weights=(W * xg[gid]).ravel(), minlength=NG)
    assert np.max(np.abs(back - xg)) <= 1e-15
    yl = uniform_vector(NL, 6).reshape(gid.shape)
    lhs = np.dot(xg[gid].ravel(), yl.ravel())
    rhs = np.dot(xg, np.bincount(gid.ravel(), weights=yl.ravel(), minlength=NG))
    assert abs(lhs - rhs) <= 1e-13 * np.sqrt(NL) * 10


# ---------------------------------------------------------------- forcing (c12)
def test_splitmix64_reference_vectors():
    g = gold("splitmix64.json")
    gamma = 0x9E3779B97F4A7C15
    for k, hexv in enumerate(g["state0_outputs_hex"]):
        assert forcing.splitmix64((k * gamma) % (1 << 64)) == int(hexv, 16)


def test_forcing_range_and_golden():
    a = gold("appendix_a.json")["C1"]
    b = forcing.forcing(range(343), 1)
    np.testing.assert_array_equal(b[:3], np.array(a["b0_2"]))
    assert abs(b.sum() - a["sum_b"]) < 1e-12
    big = forcing.forcing(range(20000), 3)
    assert big.min() >= -1.0 and big.max() < 1.0
    assert abs(big.mean()) < 0.03 and abs(big.var() - 1 / 3) < 0.02
    # value is exactly representable: 2*(h>>11)*2^-53 - 1 is a multiple of 2^-52
    assert np.all((big + 1.0) * 2.0 ** 52 == np.floor((big + 1.0) * 2.0 ** 52))


# ---------------------------------------------------------------- ledger
def test_ledger_goldens():
    g = gold("ledger.json")
    for E, N, v in g["nekbone_flops"]:
        assert ledger.nekbone_flops(E, N) == v
    for E, N, v in g["hipbone_flops"]:
        assert ledger.hipbone_flops(E, N) == v
    for a, b, v in g["operator_bytes"]:
        assert ledger.operator_bytes(a, b) == v
    for a, b, v in g["cg_bytes"]:
        assert ledger.cg_bytes(a, b) == v
    for N, B, v, tol in g["roofline"]:
        assert abs(ledger.roofline(N, B) - v) / v < tol
    assert ledger.roofline(7, 1e12, C=0.0) == 0.0
    for NG, it, P, t, v in g["throughput"]:
        assert ledger.throughput(NG, it, P, t) == v
    for E in (1, 7, 4096):
        for N in range(1, 16):
            assert ledger.hipbone_flops(E, N) < ledger.nekbone_flops(E, N)
