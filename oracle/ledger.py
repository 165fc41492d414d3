"""FLOP / byte / roofline / throughput formulas of the paper (reporting conventions).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Integer formulas, written verbatim.
"""
from __future__ import annotations


def nekbone_flops(E: int, N: int) -> int:
    """eq:nekbone_flops: 12 E (N+1)^4 + 34 E (N+1)^3 per CG iteration."""
    return 12 * E * (N + 1) ** 4 + 34 * E * (N + 1) ** 3


def hipbone_flops(E: int, N: int) -> int:
    """eq:hipbone_flops: 12 E (N+1)^4 + 19 E (N+1)^3 + 10 E N^3."""
    return 12 * E * (N + 1) ** 4 + 19 * E * (N + 1) ** 3 + 10 * E * N ** 3


def operator_flops(E: int, N: int) -> int:
    """12 E (N+1)^4 + 15 E (N+1)^3 (S_L) + 3 E (N+1)^3 (lambda W)."""
    return 12 * E * (N + 1) ** 4 + 18 * E * (N + 1) ** 3


def operator_bytes(NG: int, NL: int) -> int:
    """8 N_G + 68 N_L (perfect caching of x_G)."""
    return 8 * NG + 68 * NL


def cg_bytes(NG: int, NL: int) -> int:
    """108 N_G + 80 N_L per CG iteration."""
    return 108 * NG + 80 * NL


def roofline(N: int, B: float, C: float = float("inf")) -> float:
    """eq:op_perf: R = min(C, (12(N+1)^4 + 18(N+1)^3)/(8N^3 + 68(N+1)^3) B)."""
    return min(C, (12 * (N + 1) ** 4 + 18 * (N + 1) ** 3) / (8 * N ** 3 + 68 * (N + 1) ** 3) * B)


def throughput(NG: int, iters: int, ranks: int, time_s: float) -> float:
    """eq:throughput: DOFs * CG iterations / (ranks * time)."""
    return NG * iters / (ranks * time_s)
