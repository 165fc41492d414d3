"""Conjugate Gradient, Algorithm 1 of the paper, written out literally.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

P:57-78 (Alg. 1):
    j = 0; r_0 = b - A x; p = r
    while r_j . r_j > eps:
        alpha = r_j.r_j / p.Ap ; x = x + alpha p ; r_{j+1} = r_j - alpha Ap
        beta = r_{j+1}.r_{j+1} / r_j.r_j ; p = r_{j+1} + beta p ; j = j + 1
P:53  -- NekBone "runs a fixed 100 iterations of the CG method" (fixed mode).
Readings: c13 x_0 = 0; c14 eps is absolute on r.r; c15 guards alpha = 0 when p.Ap == 0
and beta = 0 when r_j.r_j == 0 (fixed mode only, avoids 0/0).
Dots are exactly rounded sums (math.fsum of the fp64 products) -- order independent.
"""
from __future__ import annotations

import math

import numpy as np


def dot(a: np.ndarray, b: np.ndarray) -> float:
    return math.fsum((a * b).tolist())


def cg(apply_A, b: np.ndarray, *, max_iters: int, eps: float | None = None):
    """Returns (x, j, rr_history).  eps=None -> fixed mode (exactly max_iters iterations);
    otherwise tolerance mode: stop when r.r <= eps or j == max_iters."""
    x = np.zeros_like(b)
    r = b - apply_A(x)
    p = r.copy()
    rr = dot(r, r)
    hist = [rr]
    j = 0
    while j < max_iters and (eps is None or rr > eps):
        Ap = apply_A(p)
        pAp = dot(p, Ap)
        alpha = rr / pAp if pAp != 0.0 else 0.0
        x = x + alpha * p
        r = r - alpha * Ap
        rr_new = dot(r, r)
        beta = rr_new / rr if rr != 0.0 else 0.0
        p = r + beta * p
        rr = rr_new
        hist.append(rr)
        j += 1
    return x, j, hist


def pcg(apply_A, b: np.ndarray, minv: np.ndarray, *, max_iters: int, eps: float | None = None):
    """Preconditioned CG (textbook form, e.g. Saad, Iterative Methods, Alg. 9.1) with a
    diagonal preconditioner M^-1 = diag(minv) -- NekBone's "simple diagonal preconditioning"
    (hipBone itself has none).  Alg. 1 with z = M^-1 r:
        alpha = r.z / p.Ap ; x += alpha p ; r -= alpha Ap ; z = M^-1 r
        beta = r'.z' / r.z ; p = z + beta p
    The stopping test stays Alg. 1's r.r > eps; the history records r.r.
    Returns (x, j, rr_history)."""
    x = np.zeros_like(b)
    r = b - apply_A(x)
    z = minv * r
    p = z.copy()
    rz = dot(r, z)
    rr = dot(r, r)
    hist = [rr]
    j = 0
    while j < max_iters and (eps is None or rr > eps):
        Ap = apply_A(p)
        pAp = dot(p, Ap)
        alpha = rz / pAp if pAp != 0.0 else 0.0
        x = x + alpha * p
        r = r - alpha * Ap
        z = minv * r
        rz_new = dot(r, z)
        beta = rz_new / rz if rz != 0.0 else 0.0
        p = z + beta * p
        rz = rz_new
        rr = dot(r, r)
        hist.append(rr)
        j += 1
    return x, j, hist
