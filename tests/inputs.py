"""Seeded synthetic input generators shared by the oracle side and the CUDA side of the
tests.  Holds NONE of the method's arithmetic: only random numbers and random SPD 3x3
matrices (a valid stand-in for geometric factors), so cross-term bugs in
either implementation are visible.  Recipe documented in DESIGN.md "Input recipe".
"""
from __future__ import annotations

import numpy as np


def rng(seed: int) -> np.random.Generator:
    return np.random.default_rng(seed)


def uniform_vector(n: int, seed: int) -> np.ndarray:
    """i.i.d. uniform [-1, 1) fp64."""
    return rng(seed).uniform(-1.0, 1.0, size=n)


def random_spd_factors(nelem: int, nodes: int, seed: int, scale: np.ndarray | None = None) -> np.ndarray:
    """[nelem][nodes][6] packed (rr, rs, rt, ss, st, tt) of M M^T + I/2, M ~ U[-1/2, 1/2)^{3x3}.

    If ``scale`` ([nodes], positive) is given every node's matrix is multiplied by it
    (tests pass GLL weight products so magnitudes resemble the real factors)."""
    M = rng(seed).uniform(-0.5, 0.5, size=(nelem, nodes, 3, 3))
    S = M @ np.swapaxes(M, -1, -2) + 0.5 * np.eye(3)
    if scale is not None:
        S = S * scale[None, :, None, None]
    return np.stack([S[..., 0, 0], S[..., 0, 1], S[..., 0, 2],
                     S[..., 1, 1], S[..., 1, 2], S[..., 2, 2]], axis=-1).copy()


def random_positive(n_shape, seed: int) -> np.ndarray:
    """uniform [0.5, 1.5) -- e.g. a random positive mass vector."""
    return rng(seed).uniform(0.5, 1.5, size=n_shape)
