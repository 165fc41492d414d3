"""Structured box mesh: local-to-global map, degree counts, W, B and geometric factors.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

P:55  -- "regular mesh of E hexahedral elements, together with a degree N polynomial
         discretization amounting to (N+1)^3 interpolation points on each element ...
         N_L = E(N+1)^3 ... N_G is strictly smaller than N_L".
P:88  -- S = Z^T S_L Z, Z the N_L x N_G Boolean scatter with one nonzero per row.
P:100-108 -- G^e: "pointwise values of the corresponding entry of the element's metric
         tensor, combined with GLL quadrature weights".
P:154 -- W: "diagonal matrix of the inverse degree weights" (reading c1: Z^T W Z = I).

Conventions: c7 numbering -- element e = ex + nx (ey + ny ez); local
node n = i + (N+1)(j + (N+1) k); global id of grid point (X, Y, Z) is
X + (nx N + 1)(Y + (ny N + 1) Z) with X = ex N + i.  c4 -- element extents h per axis
(default 2, so J = 1 and the metric is the identity).
"""
from __future__ import annotations

import numpy as np

# packed factor order (P:154 packs all factors of a node together; order c-table B3)
FACTORS = ("rr", "rs", "rt", "ss", "st", "tt")


def global_sizes(nx: int, ny: int, nz: int, N: int) -> tuple[int, int, int]:
    E = nx * ny * nz
    NL = E * (N + 1) ** 3
    NG = (nx * N + 1) * (ny * N + 1) * (nz * N + 1)
    return E, NG, NL


def element_coords(e: int, nx: int, ny: int) -> tuple[int, int, int]:
    return e % nx, (e // nx) % ny, e // (nx * ny)


def l2g(nx: int, ny: int, nz: int, N: int, elements=None) -> np.ndarray:
    """gid[e_local][n] (int64) for the listed global elements (default: all, ascending).

    Written as explicit loops over (e, k, j, i) -- the c7 rule verbatim."""
    NP = N + 1
    if elements is None:
        elements = range(nx * ny * nz)
    elements = list(elements)
    gx, gy = nx * N + 1, ny * N + 1
    out = np.empty((len(elements), NP ** 3), dtype=np.int64)
    for le, e in enumerate(elements):
        ex, ey, ez = element_coords(e, nx, ny)
        for k in range(NP):
            for j in range(NP):
                for i in range(NP):
                    X, Y, Z = ex * N + i, ey * N + j, ez * N + k
                    out[le, i + NP * (j + NP * k)] = X + gx * (Y + gy * Z)
    return out


def counts(gid: np.ndarray, NG: int) -> np.ndarray:
    """Global degree count of every gid: number of (e, n) slots mapping to it (diag(Z^T Z))."""
    return np.bincount(gid.ravel(), minlength=NG).astype(np.int64)


def weights_W(gid: np.ndarray, NG: int) -> np.ndarray:
    """W[e][n] = 1 / count(gid[e][n])  (reading c1: Z^T W Z = I)."""
    c = counts(gid, NG)
    return 1.0 / c[gid].astype(np.float64)


def geometric_factors(nelem: int, N: int, w: np.ndarray, ext=(2.0, 2.0, 2.0)) -> np.ndarray:
    """G[e][n][6] packed (rr, rs, rt, ss, st, tt) for axis-aligned box elements.

    For the affine map x = x0 + (h/2) r per axis: J = hx hy hz / 8, dr/dx = 2/hx, so
    G_rr = w_i w_j w_k J (2/hx)^2, G_ss, G_tt likewise, cross terms 0 (
    SURVEY c4/c6)."""
    hx, hy, hz = ext
    if min(hx, hy, hz) <= 0:
        raise ValueError("element extent must be positive")
    NP = N + 1
    J = hx * hy * hz / 8.0
    G = np.zeros((nelem, NP ** 3, 6), dtype=np.float64)
    for k in range(NP):
        for j in range(NP):
            for i in range(NP):
                n = i + NP * (j + NP * k)
                wq = w[i] * w[j] * w[k] * J
                G[:, n, 0] = wq * (2.0 / hx) ** 2
                G[:, n, 3] = wq * (2.0 / hy) ** 2
                G[:, n, 5] = wq * (2.0 / hz) ** 2
    return G


def mass_B(nelem: int, N: int, w: np.ndarray, ext=(2.0, 2.0, 2.0)) -> np.ndarray:
    """B[e][n] = w_i w_j w_k J, the GLL (lumped) mass of mass_mode 1."""
    hx, hy, hz = ext
    NP = N + 1
    J = hx * hy * hz / 8.0
    B = np.zeros((nelem, NP ** 3), dtype=np.float64)
    for k in range(NP):
        for j in range(NP):
            for i in range(NP):
                B[:, i + NP * (j + NP * k)] = w[i] * w[j] * w[k] * J
    return B


def node_coords(nx: int, ny: int, nz: int, N: int, x: np.ndarray, ext=(2.0, 2.0, 2.0)):
    """Physical coordinates of every global id (for manufactured-solution tests).

    Point (X, Y, Z) with X = ex N + i lies at ex hx + (x_i + 1) hx / 2."""
    hx, hy, hz = ext
    gx, gy, gz = nx * N + 1, ny * N + 1, nz * N + 1

    def axis(n_el, h):
        pts = np.empty(n_el * N + 1)
        for e in range(n_el):
            for i in range(N + 1):
                pts[e * N + i] = e * h + (x[i] + 1.0) * h / 2.0
        return pts

    X = axis(nx, hx)
    Y = axis(ny, hy)
    Z = axis(nz, hz)
    g = np.arange(gx * gy * gz)
    return X[g % gx], Y[(g // gx) % gy], Z[g // (gx * gy)]
