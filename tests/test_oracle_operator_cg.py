"""Pins of oracle/operator.py and oracle/cg.py: closed forms, quadrature exactness,
symmetry/SPD, explicit-vs-sum-factorised, dense brute force, CG vs direct solve,
and the survey's independent Appendix A values."""
import json
import math
import os

import numpy as np
import pytest

from oracle import basis, cg, forcing, mesh, operator
from tests.inputs import random_spd_factors, uniform_vector, random_positive

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def setup(box, N, ext=(2.0, 2.0, 2.0), mass_mode=0):
    x, w, D = basis.basis(N)
    E, NG, NL = mesh.global_sizes(*box, N)
    gid = mesh.l2g(*box, N)
    G = mesh.geometric_factors(E, N, w, ext)
    M = mesh.weights_W(gid, NG) if mass_mode == 0 else mesh.mass_B(E, N, w, ext)
    return x, w, D, gid, G, M, NG


def test_unit_cube_N1_diag_075():
    c = gold("operator_examples.json")["unit_cube_N1"]
    x, w, D, gid, G, M, NG = setup((1, 1, 1), 1, tuple(c["ext"]))
    A = operator.dense(gid, NG, D, G, c["lambda"], M)
    np.testing.assert_allclose(np.diag(A), c["diag"], rtol=0, atol=1e-15)
    np.testing.assert_allclose(A.sum(1), c["row_sum"], rtol=0, atol=1e-15)


@pytest.mark.parametrize("N", [1, 2, 3, 4, 5])
def test_explicit_equals_sumfactorised_random_G(N):
    """Two independent element operators agree with random SPD G (cross terms live)."""
    box = (2, 1, 2)
    x, w, D, gid, G, M, NG = setup(box, N)
    Gr = random_spd_factors(gid.shape[0], (N + 1) ** 3, seed=11 + N)
    Mr = random_positive(gid.shape, seed=3)
    xv = uniform_vector(NG, 2)
    a = operator.apply(xv, gid, D, Gr, 0.7, Mr)
    b = operator.apply_explicit(xv, gid, D, Gr, 0.7, Mr)
    s = operator.apply_abs_explicit(xv, gid, D, Gr, 0.7, Mr)
    assert np.max(np.abs(a - b) / s) < 1e-14


@pytest.mark.parametrize("box", [(1, 1, 1), (2, 1, 1), (1, 2, 2), (2, 2, 2)])
@pytest.mark.parametrize("N", [1, 2, 3, 4])
def test_dense_bruteforce(box, N):
    """Q^T blockdiag(A_L^e) Q (dense) equals the matrix-free apply."""
    x, w, D, gid, G, M, NG = setup(box, N)
    Gr = random_spd_factors(gid.shape[0], (N + 1) ** 3, seed=N)
    A = operator.dense(gid, NG, D, Gr, 1.0, M)
    for t in range(3):
        xv = uniform_vector(NG, 100 + t)
        y = operator.apply(xv, gid, D, Gr, 1.0, M)
        assert np.max(np.abs(y - A @ xv)) <= 1e-12 * np.max(np.abs(A) @ np.abs(xv))


@pytest.mark.parametrize("N", list(range(1, 16)))
def test_constant_eigenvector(N):
    """A 1 = lambda 1 in mass mode 0 (1^T S = 0 and Z^T W Z = I)."""
    x, w, D, gid, G, M, NG = setup((2, 2, 2), N)
    y = operator.apply(np.ones(NG), gid, D, G, 1.0, M)
    assert np.max(np.abs(y - 1.0)) <= 1e-12
    # mode 1: A 1 = lambda Z^T B 1
    x, w, D, gid, G, B, NG = setup((2, 2, 2), N, mass_mode=1)
    y = operator.apply(np.ones(NG), gid, D, G, 1.0, B)
    mass = np.bincount(gid.ravel(), weights=B.ravel(), minlength=NG)
    assert np.max(np.abs(y - mass)) <= 1e-12
    assert abs(mass.sum() - 8.0 * 8.0) < 1e-11  # total volume of the 4x4x4 box


def _poly_integral(p, lo, hi):
    if p < 0:
        return 0.0  # only reached multiplied by a zero derivative factor
    return (hi ** (p + 1) - lo ** (p + 1)) / (p + 1)


@pytest.mark.parametrize("N", [2, 4, 7])
def test_quadrature_exactness_stiffness_and_mass(N):
    """u^T S v = int grad u . grad v and u^T B v = int u v for u = X^a Y^b Z^c,
    v = X^d Y^e Z^f, a..f <= N, a+d, b+e, c+f <= 2N-1 (GLL collocation),
    on a box with unequal extents (pins the metric scaling of G)."""
    box, ext = (2, 1, 2), (1.0, 2.0, 0.5)
    x, w, D, gid, G, B, NG = setup(box, N, ext, mass_mode=1)
    X, Y, Z = mesh.node_coords(*box, N, x, ext)
    L = [box[i] * ext[i] for i in range(3)]
    rng = np.random.default_rng(N)
    for _ in range(6):
        a, b, c = rng.integers(0, N + 1, 3)
        d, e, f = [int(rng.integers(0, min(N, 2 * N - 1 - t) + 1)) for t in (a, b, c)]
        u = X ** a * Y ** b * Z ** c
        v = X ** d * Y ** e * Z ** f
        Sv = operator.apply(v, gid, D, G, 0.0, B)
        Bv = operator.apply(v, gid, D, G, 1.0, B) - Sv
        Ix = [_poly_integral(p, 0.0, L[0]) for p in (a + d, a + d - 2)]
        Iy = [_poly_integral(p, 0.0, L[1]) for p in (b + e, b + e - 2)]
        Iz = [_poly_integral(p, 0.0, L[2]) for p in (c + f, c + f - 2)]
        grad = ((a * d * Ix[1] * Iy[0] * Iz[0] if a * d else 0.0)
                + (b * e * Ix[0] * Iy[1] * Iz[0] if b * e else 0.0)
                + (c * f * Ix[0] * Iy[0] * Iz[1] if c * f else 0.0))
        mass = Ix[0] * Iy[0] * Iz[0]
        scale = max(1.0, abs(grad), np.abs(u).max() * np.abs(Sv).sum())
        assert abs(u @ Sv - grad) <= 1e-13 * scale, (a, b, c, d, e, f)
        assert abs(u @ Bv - mass) <= 1e-13 * max(1.0, abs(mass)), (a, b, c, d, e, f)


def test_cross_terms_affine_element():
    """Sheared affine element x = x0 + J r: G = w w w |det J| J^-1 J^-T (all six factors
    nonzero).  For linear u = a.x, v = b.x:  u^T S v = (a.b) |det J| * 8  (exact), which
    pins the placement of rs, rt, st."""
    N = 3
    x, w, D = basis.basis(N)
    rng = np.random.default_rng(7)
    Jm = np.eye(3) + 0.3 * rng.uniform(-1, 1, (3, 3))
    det = np.linalg.det(Jm)
    Ki = np.linalg.inv(Jm)           # dr/dx
    Gm = Ki @ Ki.T                    # metric (dr_a/dx . dr_b/dx)
    NP = N + 1
    G = np.zeros((1, NP ** 3, 6))
    coords = np.zeros((NP ** 3, 3))
    for k in range(NP):
        for j in range(NP):
            for i in range(NP):
                n = i + NP * (j + NP * k)
                wq = w[i] * w[j] * w[k] * abs(det)
                G[0, n] = wq * np.array([Gm[0, 0], Gm[0, 1], Gm[0, 2], Gm[1, 1], Gm[1, 2], Gm[2, 2]])
                coords[n] = Jm @ np.array([x[i], x[j], x[k]])
    gid = np.arange(NP ** 3)[None, :]
    for _ in range(5):
        av, bv = rng.uniform(-1, 1, 3), rng.uniform(-1, 1, 3)
        u, v = coords @ av, coords @ bv
        Sv = operator.apply(v, gid, D, G, 0.0, np.ones((1, NP ** 3)))
        assert abs(u @ Sv - av @ bv * abs(det) * 8.0) < 1e-13


@pytest.mark.parametrize("N", [2, 4])
def test_symmetry_spd_and_spectrum(N):
    x, w, D, gid, G, M, NG = setup((2, 2, 2), N)
    Gr = random_spd_factors(gid.shape[0], (N + 1) ** 3, seed=9)
    for t in range(20):
        xv, yv = uniform_vector(NG, 200 + t), uniform_vector(NG, 300 + t)
        Ay = operator.apply(yv, gid, D, Gr, 1.0, M)
        Ax = operator.apply(xv, gid, D, Gr, 1.0, M)
        assert abs(xv @ Ay - yv @ Ax) <= 1e-13 * np.linalg.norm(xv) * np.linalg.norm(yv) * 10
        assert xv @ Ax > 0
    A = operator.dense(gid, NG, D, G, 1.0, M)
    ev = np.linalg.eigvalsh(A)
    assert abs(ev[0] - 1.0) < 1e-10            # lambda_min = lambda (c5)
    A0 = operator.dense(gid, NG, D, G, 0.0, M)
    ev0 = np.linalg.eigvalsh(A0)
    assert np.sum(np.abs(ev0) < 1e-10) == 1   # null space = constants


def test_appendix_a_C1_operator_and_cg():
    a = gold("appendix_a.json")["C1"]
    x, w, D, gid, G, M, NG = setup(tuple(a["box"]), a["N"])
    assert NG == a["NG"] and gid.size == a["NL"]
    b = forcing.forcing(range(NG), 1)
    A = lambda v: operator.apply(v, gid, D, G, 1.0, M)
    y = A(b)
    assert abs(y.sum() - a["sum_Ab"]) < 1e-12
    assert abs(np.linalg.norm(y) - a["norm_Ab"]) < 1e-12 * a["norm_Ab"]
    np.testing.assert_allclose([y[0], y[NG // 2], y[-1]], a["Ab_0_mid_last"], rtol=0, atol=1e-13)
    assert abs(cg.dot(b, y) - a["bAb"]) < 1e-12 * a["bAb"]
    xs, j, h = cg.cg(A, b, max_iters=a["fixed_iters"])
    assert j == a["fixed_iters"] and len(h) == j + 1
    assert abs(h[1] - a["rr1"]) < 1e-11 * a["rr1"] and abs(h[10] - a["rr10"]) < 1e-10 * a["rr10"]
    assert abs(h[20] - a["rr20"]) < 1e-4 * a["rr20"]
    assert abs(xs.sum() - a["fixed_sum_x"]) < 1e-12 * abs(a["fixed_sum_x"])
    assert abs(np.linalg.norm(xs) - a["fixed_norm_x"]) < 1e-12 * a["fixed_norm_x"]
    xs, j, h = cg.cg(A, b, max_iters=500, eps=1e-16 * cg.dot(b, b))
    assert j == a["tol_stop"]
    Ad = operator.dense(gid, NG, D, G, 1.0, M)
    assert abs(np.linalg.cond(Ad) - a["kappa"]) < 0.01


def test_cg_direct_solve_and_properties():
    x, w, D, gid, G, M, NG = setup((2, 2, 2), 3)
    A = lambda v: operator.apply(v, gid, D, G, 1.0, M)
    Ad = operator.dense(gid, NG, D, G, 1.0, M)
    b = forcing.forcing(range(NG), 1)
    xd = np.linalg.solve(Ad, b)
    xs, j, h = cg.cg(A, b, max_iters=500, eps=1e-20 * cg.dot(b, b))
    assert np.max(np.abs(xs - xd)) <= 1e-8 * np.max(np.abs(xd))
    assert h[-1] <= 1e-20 * cg.dot(b, b) and all(v > 1e-20 * h[0] for v in h[:-1])
    assert abs(xs.sum() - b.sum()) < 1e-10 * abs(b.sum())   # 1^T A = lambda 1^T -> sum x = sum b / lambda
    # energy-norm error monotone over the first iterations
    errs = []
    for k in range(1, 25):
        xk, _, _ = cg.cg(A, b, max_iters=k)
        e = xk - xd
        errs.append(e @ (Ad @ e))
    assert all(errs[i + 1] <= errs[i] * (1 + 1e-12) for i in range(len(errs) - 1))
    # b = 0 exits at j = 0 in tolerance mode
    xz, j0, _ = cg.cg(A, np.zeros(NG), max_iters=10, eps=0.0)
    assert j0 == 0 and not xz.any()
    # manufactured solution: b = A x*, x* smooth
    X, Y, Z = mesh.node_coords(2, 2, 2, 3, x)
    xstar = np.sin(X) * np.cos(Y) + Z
    xm, _, _ = cg.cg(A, A(xstar), max_iters=500, eps=1e-26)
    assert np.max(np.abs(xm - xstar)) < 1e-10


@pytest.mark.slow
def test_appendix_a_C2_operator_and_tol_cg():
    a = gold("appendix_a.json")["C2"]
    x, w, D, gid, G, M, NG = setup(tuple(a["box"]), a["N"])
    assert NG == a["NG"]
    b = forcing.forcing(range(NG), 1)
    assert abs(cg.dot(b, b) - a["bb"]) < 1e-12 * a["bb"]
    A = lambda v: operator.apply(v, gid, D, G, 1.0, M)
    y = A(b)
    assert abs(np.linalg.norm(y) - a["norm_Ab"]) < 1e-12 * a["norm_Ab"]
    np.testing.assert_allclose([y[0], y[NG // 2], y[-1]], a["Ab_0_mid_last"], rtol=0, atol=1e-13)
    xs, j, h = cg.cg(A, b, max_iters=100, eps=1e-16 * a["bb"])
    assert j == a["tol_stop"]
    assert abs(h[1] - a["rr1"]) < 1e-11 * a["rr1"] and abs(h[10] - a["rr10"]) < 1e-10 * a["rr10"]
    assert abs(h[20] - a["rr20"]) < 1e-4 * a["rr20"]


@pytest.mark.parametrize("mass_mode", [0, 1])
def test_diagonal_and_pcg(mass_mode):
    """Jacobi PCG pins (NEXT #3): oracle diag(A) equals the dense diagonal; PCG with M = I is
    CG (identical iterates); PCG reaches the direct solution and needs fewer iterations than
    CG on a problem with a strongly varying mass term."""
    box, N = (2, 2, 1), 3
    x, w, D, gid, G, M, NG = setup(box, N, mass_mode=mass_mode)
    Gr = random_spd_factors(gid.shape[0], (N + 1) ** 3, seed=41, scale=np.einsum("k,j,i->kji", w, w, w).ravel())
    if mass_mode == 1:
        M = random_positive(gid.shape, 5) * np.exp(3.0 * uniform_vector(gid.size, 6)).reshape(gid.shape)
    Ad = operator.dense(gid, NG, D, Gr, 1.0, M)
    d = operator.diagonal(gid, NG, D, Gr, 1.0, M)
    assert np.max(np.abs(d - np.diag(Ad))) <= 1e-13 * np.max(np.abs(d))
    A = lambda v: operator.apply(v, gid, D, Gr, 1.0, M)
    b = forcing.forcing(range(NG), 1)
    xa, ja, ha = cg.cg(A, b, max_iters=30)
    xb, jb, hb_ = cg.pcg(A, b, np.ones(NG), max_iters=30)
    assert ha == hb_ and np.array_equal(xa, xb)
    eps = 1e-24 * cg.dot(b, b)
    xp, jp, hp = cg.pcg(A, b, 1.0 / d, max_iters=1000, eps=eps)
    xc, jc, hc = cg.cg(A, b, max_iters=1000, eps=eps)
    xd = np.linalg.solve(Ad, b)
    assert np.max(np.abs(xp - xd)) <= 1e-9 * np.max(np.abs(xd))
    if mass_mode == 1:
        assert jp < jc


# ---------------------------------------------------------------- pins of the parity checkers
# apply_abs_explicit / apply_abs give the c17 error scale s (|y_i - o_i| <= 1e-12 s_i) and
# apply_entries the sampled full-size ground truth; each is pinned to something other than
# itself (dense brute force, exact identities, the pinned apply()).

@pytest.mark.parametrize("N", [1, 2, 3])
def test_abs_explicit_single_element_equals_dense(N):
    """One element: no cross-element sums, so s = |A| |x| exactly with the dense A."""
    x, w, D, gid, G, M, NG = setup((1, 1, 1), N)
    Gr = random_spd_factors(1, (N + 1) ** 3, seed=40 + N)
    Mr = random_positive(gid.shape, seed=41)
    A = operator.dense(gid, NG, D, Gr, 0.8, Mr)
    xv = uniform_vector(NG, 42)
    s = operator.apply_abs_explicit(xv, gid, D, Gr, 0.8, Mr)
    np.testing.assert_allclose(s, np.abs(A) @ np.abs(xv), rtol=1e-14, atol=0)


@pytest.mark.parametrize("N", [1, 2, 3, 4])
@pytest.mark.parametrize("geom", ["box", "random"])
def test_abs_explicit_bounds_dense_and_is_elementwise(N, geom):
    """Several elements: s >= |A| |x| entrywise (triangle inequality over the elements sharing
    a node), with equality at element-interior nodes (one contributing slot); s is the sum of
    the single-element scales (assembly is additive)."""
    box = (2, 2, 1)
    x, w, D, gid, G, M, NG = setup(box, N)
    Gr = G if geom == "box" else random_spd_factors(gid.shape[0], (N + 1) ** 3, seed=50 + N)
    A = operator.dense(gid, NG, D, Gr, 1.0, M)
    xv = uniform_vector(NG, 43)
    s = operator.apply_abs_explicit(xv, gid, D, Gr, 1.0, M)
    lower = np.abs(A) @ np.abs(xv)
    assert np.all(s >= lower * (1 - 1e-14))
    counts = np.bincount(gid.ravel(), minlength=NG)
    one = counts == 1
    np.testing.assert_allclose(s[one], lower[one], rtol=1e-13, atol=0)
    parts = sum(operator.apply_abs_explicit(xv, gid[e:e + 1], D, Gr[e:e + 1], 1.0, M[e:e + 1])
                for e in range(gid.shape[0]))
    np.testing.assert_allclose(s, parts, rtol=1e-14, atol=0)


@pytest.mark.parametrize("N", [1, 2, 3, 4, 5, 6])
@pytest.mark.parametrize("geom", ["box", "random"])
def test_abs_sumfactorised_bounds_explicit(N, geom):
    """apply_abs (used as the c17 scale for N > 5) is |D|^T |G| |D| sum-factorised: it equals
    apply() run on |x| with |D|, |G|, |lambda|, |M| (an identity of the sum-factorisation,
    with apply() pinned above), is >= the explicit |S_e||u| scale, and at most 10x it (the
    looseness of the bound, reading R5: measured max 4.1x at N <= 6, 8.0x at N = 15)."""
    box = (2, 2, 1)
    x, w, D, gid, G, M, NG = setup(box, N)
    Gr = G if geom == "box" else random_spd_factors(gid.shape[0], (N + 1) ** 3, seed=60 + N)
    Mr = random_positive(gid.shape, seed=61)
    xv = uniform_vector(NG, 44)
    s1 = operator.apply_abs(xv, gid, D, Gr, -0.9, Mr)
    np.testing.assert_allclose(s1, operator.apply(np.abs(xv), gid, np.abs(D), np.abs(Gr), 0.9, Mr),
                               rtol=1e-14, atol=0)
    s2 = operator.apply_abs_explicit(xv, gid, D, Gr, -0.9, Mr)
    assert np.all(s1 >= s2 * (1 - 1e-14))
    assert np.all(s1 <= 10.0 * s2)


@pytest.mark.parametrize("N,mass_mode", [(3, 0), (4, 1), (2, 0)])
def test_apply_entries_equals_apply(N, mass_mode):
    """apply_entries (full-size sampled ground truth) equals the pinned apply() at EVERY gid
    of a small mesh (corners, edges, faces, interiors), random SPD G, both mass modes."""
    box = (3, 2, 2)
    x, w, D, gid, G, M, NG = setup(box, N, mass_mode=mass_mode)
    Gr = random_spd_factors(gid.shape[0], (N + 1) ** 3, seed=70 + N)
    if mass_mode == 1:
        M = random_positive(gid.shape, seed=71)
    xv = uniform_vector(NG, 72)
    ref = operator.apply(xv, gid, D, Gr, 1.3, M)
    out = operator.apply_entries(lambda row: xv[row], list(range(NG)), *box, N, D, lambda e: Gr[e], 1.3,
                                 lambda e, row: M[e], mesh.l2g)
    np.testing.assert_allclose(out, ref, rtol=0, atol=1e-13 * np.abs(ref).max())
    # with |.| inputs it gives the sum-factorised scale (the full-size test's c17 scale)
    sabs = operator.apply_entries(lambda row: np.abs(xv[row]), list(range(NG)), *box, N, np.abs(D),
                                  lambda e: np.abs(Gr[e]), 1.3, lambda e, row: M[e], mesh.l2g)
    np.testing.assert_allclose(sabs, operator.apply_abs(xv, gid, D, Gr, 1.3, M), rtol=1e-13, atol=0)
