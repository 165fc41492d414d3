"""Pseudo-random forcing vector b and the splitmix64 hash used by ownership.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

P:138 -- "The first [kernel] is used only once to populate a pseudo-random initial
         forcing vector".  The paper gives no distribution; reading c12 fixes
         b[g] = 2 * (splitmix64(g XOR seed) >> 11) * 2^-53 - 1, in [-1, 1), per global id
         (rank-count invariant).  Reading c9 uses splitmix64 for ownership.

splitmix64(z): z += 0x9E3779B97F4A7C15; z = (z ^ z>>30) * 0xBF58476D1CE4E5B9;
               z = (z ^ z>>27) * 0x94D049BB133111EB; return z ^ z>>31   (all mod 2^64)
Written here with Python's unbounded ints reduced mod 2^64 (no numpy overflow tricks),
one value at a time -- slow, obviously correct.
"""
from __future__ import annotations

import numpy as np

MASK64 = (1 << 64) - 1


def splitmix64(z: int) -> int:
    z = (z + 0x9E3779B97F4A7C15) & MASK64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
    return z ^ (z >> 31)


def forcing_value(g: int, seed: int) -> float:
    h = splitmix64((g ^ seed) & MASK64)
    return 2.0 * float(h >> 11) * 2.0 ** -53 - 1.0


def forcing(gids, seed: int) -> np.ndarray:
    """b[g] for every g in gids (any iterable of ints)."""
    return np.array([forcing_value(int(g), seed) for g in gids], dtype=np.float64)
