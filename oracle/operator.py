"""Screened-Poisson operator A = Z^T (S_L + lambda M_L) Z, matrix-free and dense.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

P:82  (eq:poisson)   A = S + lambda I
P:88  (eq:stiffness) S = Z^T S_L Z
P:94  S_L^e = D^T G^e D
P:98  bold-D = [D (x) I (x) I ; I (x) D (x) I ; I (x) I (x) D]
P:100-108 G^e: symmetric 3x3 block of diagonal matrices (rr, rs, rt, ss, st, tt)
P:154 y_L = (S_L + lambda W) Z x_G,  A x_G = Z^T y_L,  W = inverse degree weights

Direction convention (stated in DESIGN.md): local node n = i + (N+1)(j + (N+1)k), so a
local vector is ordered with k slowest.  In that (k, j, i) Kronecker order
    D_r = I (x) I (x) D   (derivative along i, paired with G_rr),
    D_s = I (x) D (x) I   (along j, G_ss),
    D_t = D (x) I (x) I   (along k, G_tt).
The paper's bold-D lists the same three blocks; which block is called "r" is a naming
choice and does not change S_L^e (G is symmetric and built per axis).

Mass term (reading c3): mass_mode 0 uses M_L = W (the paper's lambda W, so
Z^T lambda W Z = lambda I); mass_mode 1 uses M_L = B = w_i w_j w_k J (GLL mass).

Two independent element operators are provided:
  element_matrix()  -- explicit (N+1)^3 x (N+1)^3 matrix sum_ab D_a^T diag(G_ab) D_b
                       built with np.kron (tiny meshes only);
  local_apply()     -- sum-factorised: three 1-D contractions, pointwise G, three
                       transposed contractions (np.einsum, no blocking or fusion).
Assembly Z^T is np.bincount over the slots in ascending (e, n) order, i.e. a fixed
summation order, so results do not depend on thread counts.
"""
from __future__ import annotations

import numpy as np

# index pairs of the packed factors (rr, rs, rt, ss, st, tt) into the 3x3 metric
_PAIRS = ((0, 0), (0, 1), (0, 2), (1, 1), (1, 2), (2, 2))


def _grad_blocks(D: np.ndarray):
    NP = D.shape[0]
    I = np.eye(NP)
    Dr = np.kron(I, np.kron(I, D))
    Ds = np.kron(I, np.kron(D, I))
    Dt = np.kron(D, np.kron(I, I))
    return Dr, Ds, Dt


def element_matrix(D: np.ndarray, Ge: np.ndarray) -> np.ndarray:
    """Explicit S_L^e = bold-D^T G^e bold-D for one element; Ge is [(N+1)^3][6]."""
    blocks = _grad_blocks(D)
    n = blocks[0].shape[0]
    S = np.zeros((n, n))
    for f, (a, b) in enumerate(_PAIRS):
        g = Ge[:, f]
        S += blocks[a].T @ (g[:, None] * blocks[b])
        if a != b:  # symmetric block: G_ba = G_ab
            S += blocks[b].T @ (g[:, None] * blocks[a])
    return S


def local_apply(D: np.ndarray, G: np.ndarray, u: np.ndarray) -> np.ndarray:
    """Sum-factorised S_L u for all elements. u: [E][(N+1)^3]; G: [E][(N+1)^3][6]."""
    E = u.shape[0]
    NP = D.shape[0]
    U = u.reshape(E, NP, NP, NP)  # [e][k][j][i]
    ur = np.einsum("im,ekjm->ekji", D, U)
    us = np.einsum("jm,ekmi->ekji", D, U)
    ut = np.einsum("km,emji->ekji", D, U)
    g = G.reshape(E, NP, NP, NP, 6)
    grr, grs, grt, gss, gst, gtt = (g[..., f] for f in range(6))
    wr = grr * ur + grs * us + grt * ut
    ws = grs * ur + gss * us + gst * ut
    wt = grt * ur + gst * us + gtt * ut
    y = (np.einsum("mi,ekjm->ekji", D, wr)
         + np.einsum("mj,ekmi->ekji", D, ws)
         + np.einsum("mk,emji->ekji", D, wt))
    return y.reshape(E, NP ** 3)


def assemble(gid: np.ndarray, yL: np.ndarray, NG: int) -> np.ndarray:
    """Z^T y_L: sum of every slot into its global id, ascending (e, n) order."""
    return np.bincount(gid.ravel(), weights=yL.ravel(), minlength=NG)


def apply(x: np.ndarray, gid: np.ndarray, D: np.ndarray, G: np.ndarray,
          lam: float, M: np.ndarray) -> np.ndarray:
    """A x = Z^T (S_L + lambda M_L) Z x, sum-factorised.  M is W or B per slot."""
    u = x[gid]                               # Z x      (scatter)
    y = local_apply(D, G, u) + lam * M * u   # (S_L + lambda M_L) u
    return assemble(gid, y, x.shape[0])      # Z^T y_L  (gather)


def apply_explicit(x: np.ndarray, gid: np.ndarray, D: np.ndarray, G: np.ndarray,
                   lam: float, M: np.ndarray) -> np.ndarray:
    """Same as apply() but with explicit element matrices (tiny meshes)."""
    y = np.zeros(gid.shape)
    for e in range(gid.shape[0]):
        Se = element_matrix(D, G[e])
        u = x[gid[e]]
        y[e] = Se @ u + lam * M[e] * u
    return assemble(gid, y, x.shape[0])


def apply_abs_explicit(x: np.ndarray, gid: np.ndarray, D: np.ndarray, G: np.ndarray,
                       lam: float, M: np.ndarray) -> np.ndarray:
    """s = |A| |x| entrywise via explicit element matrices: the per-entry error scale of
    reading c17 (|y_i - o_i| <= tol * s_i)."""
    y = np.zeros(gid.shape)
    for e in range(gid.shape[0]):
        Se = np.abs(element_matrix(D, G[e]))
        u = np.abs(x[gid[e]])
        y[e] = Se @ u + abs(lam) * np.abs(M[e]) * u
    return assemble(gid, y, x.shape[0])


def apply_abs(x: np.ndarray, gid: np.ndarray, D: np.ndarray, G: np.ndarray,
              lam: float, M: np.ndarray) -> np.ndarray:
    """Upper bound of |A||x| computed sum-factorised with |D|, |G| (>= the explicit
    |A||x|), for meshes too large for explicit element matrices."""
    aD = np.abs(D)
    E = gid.shape[0]
    NP = D.shape[0]
    U = np.abs(x[gid]).reshape(E, NP, NP, NP)
    ur = np.einsum("im,ekjm->ekji", aD, U)
    us = np.einsum("jm,ekmi->ekji", aD, U)
    ut = np.einsum("km,emji->ekji", aD, U)
    g = np.abs(G).reshape(E, NP, NP, NP, 6)
    wr = g[..., 0] * ur + g[..., 1] * us + g[..., 2] * ut
    ws = g[..., 1] * ur + g[..., 3] * us + g[..., 4] * ut
    wt = g[..., 2] * ur + g[..., 4] * us + g[..., 5] * ut
    y = (np.einsum("mi,ekjm->ekji", aD, wr) + np.einsum("mj,ekmi->ekji", aD, ws)
         + np.einsum("mk,emji->ekji", aD, wt)).reshape(E, NP ** 3)
    y += abs(lam) * np.abs(M) * np.abs(x[gid])
    return assemble(gid, y, x.shape[0])


def dense(gid: np.ndarray, NG: int, D: np.ndarray, G: np.ndarray, lam: float,
          M: np.ndarray) -> np.ndarray:
    """Dense A = Q^T blockdiag(S_L^e + lambda M_e) Q with the Boolean Q (N_L x N_G)."""
    if NG > 20000:
        raise ValueError("dense assembly refused for N_G > 20000")
    E, n = gid.shape
    Q = np.zeros((E * n, NG))
    Q[np.arange(E * n), gid.ravel()] = 1.0
    AL = np.zeros((E * n, E * n))
    for e in range(E):
        AL[e * n:(e + 1) * n, e * n:(e + 1) * n] = element_matrix(D, G[e]) + lam * np.diag(M[e])
    return Q.T @ AL @ Q


def apply_entries(x_of, gids, nx, ny, nz, N, D, G_of, lam, M_of, l2g_fn):
    """(A x)[g] for a sample of global ids, computed one by one from the <= 8 elements
    touching g (for full-size parity checks on sampled outputs).

    x_of(gid_array) -> x values; G_of(elem) -> [(N+1)^3][6]; M_of(elem, gid_row) -> [(N+1)^3].
    """
    gx, gy = nx * N + 1, ny * N + 1
    out = np.zeros(len(gids))
    for t, g in enumerate(gids):
        X, Y, Z = g % gx, (g // gx) % gy, g // (gx * gy)
        cand = []
        for ez in {max(0, (Z - 1) // N), min(nz - 1, Z // N)}:
            for ey in {max(0, (Y - 1) // N), min(ny - 1, Y // N)}:
                for ex in {max(0, (X - 1) // N), min(nx - 1, X // N)}:
                    cand.append(ex + nx * (ey + ny * ez))
        total = 0.0
        for e in sorted(set(cand)):
            row = l2g_fn(nx, ny, nz, N, [e])[0]
            hits = np.nonzero(row == g)[0]
            if len(hits) == 0:
                continue
            u = x_of(row)
            y = local_apply(D, G_of(e)[None], u[None])[0] + lam * M_of(e, row) * u
            for n in hits:
                total += y[n]
        out[t] = total
    return out


def diagonal(gid: np.ndarray, NG: int, D: np.ndarray, G: np.ndarray, lam: float, M: np.ndarray) -> np.ndarray:
    """diag(A) = Z^T diag(S_L^e + lambda M_e) (the Jacobi preconditioner of NEXT #3): the
    diagonal of every explicit element matrix, assembled (tiny meshes)."""
    d = np.zeros(gid.shape)
    for e in range(gid.shape[0]):
        d[e] = np.diag(element_matrix(D, G[e])) + lam * M[e]
    return assemble(gid, d, NG)
