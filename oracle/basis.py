"""1-D spectral-element basis: GLL nodes, weights and derivative matrix D.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

P:48  -- "the high-order polynomial basis functions are chosen as the tensor-product
         of Lagrange polynomials, interpolating the Gauss-Legendre-Lobatto (GLL)
         quadrature points".
P:100 -- "D is the (N+1)x(N+1) one-dimensional SEM derivative operator".

The GLL nodes of degree N are x = +-1 and the roots of P_N'(x), i.e. the roots of
(1 - x^2) P_N'(x); the weights are w_i = 2 / (N (N+1) P_N(x_i)^2) (textbook GLL
rule).  D[i][j] = l_j'(x_i), the derivative of the j-th
Lagrange cardinal polynomial evaluated at node i, computed from its product
definition (no closed-form shortcut), so it can be checked by eye.
"""
from __future__ import annotations

import math

import numpy as np


def legendre(N: int, x: float) -> tuple[float, float]:
    """Return (P_N(x), P_{N-1}(x)) by the three-term recurrence
    (k+1) P_{k+1} = (2k+1) x P_k - k P_{k-1}."""
    p_prev, p = 1.0, x  # P_0, P_1
    if N == 0:
        return 1.0, 0.0
    for k in range(1, N):
        p_prev, p = p, ((2 * k + 1) * x * p - k * p_prev) / (k + 1)
    return p, p_prev


def gll(N: int) -> tuple[np.ndarray, np.ndarray]:
    """GLL nodes (ascending) and weights for degree N >= 1.

    Interior nodes: Newton on q(x) = (1 - x^2) P_N'(x) = N (P_{N-1}(x) - x P_N(x)),
    whose derivative is q'(x) = -N (N+1) P_N(x) (Legendre's equation), started from
    the Chebyshev-Gauss-Lobatto points -cos(pi i / N).
    """
    if N < 1:
        raise ValueError("GLL needs N >= 1")
    x = np.array([-math.cos(math.pi * i / N) for i in range(N + 1)], dtype=np.float64)
    for i in range(1, N):
        xi = x[i]
        for _ in range(100):
            pn, pn1 = legendre(N, xi)
            q = N * (pn1 - xi * pn)
            dq = -N * (N + 1) * pn
            step = q / dq
            xi -= step
            if abs(step) < 1e-16:
                break
        x[i] = xi
    x[0], x[N] = -1.0, 1.0
    # symmetrise (the rule is symmetric about 0)
    x = 0.5 * (x - x[::-1])
    w = np.array([2.0 / (N * (N + 1) * legendre(N, xi)[0] ** 2) for xi in x])
    return x, w


def derivative_matrix(x: np.ndarray) -> np.ndarray:
    """D[i][j] = l_j'(x_i) with l_j(x) = prod_{m != j} (x - x_m) / (x_j - x_m).

    Product rule: l_j'(x) = sum_{a != j} [1/(x_j - x_a)] prod_{m != j, a} (x - x_m)/(x_j - x_m).
    Evaluated directly at x = x_i (plain O(n^3) loops per entry)."""
    n = len(x)
    D = np.zeros((n, n), dtype=np.float64)
    for i in range(n):
        for j in range(n):
            s = 0.0
            for a in range(n):
                if a == j:
                    continue
                term = 1.0 / (x[j] - x[a])
                for m in range(n):
                    if m == j or m == a:
                        continue
                    term *= (x[i] - x[m]) / (x[j] - x[m])
                s += term
            D[i, j] = s
    return D


def basis(N: int) -> tuple[np.ndarray, np.ndarray, np.ndarray]:
    x, w = gll(N)
    return x, w, derivative_matrix(x)
