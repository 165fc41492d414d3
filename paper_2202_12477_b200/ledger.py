"""Reporting formulas of the paper (FOM, ledgers, roofline, throughput) plus this build's
own algorithmic byte counts.  Product-side twin of nothing: the oracle has its own copy
that the tests pin; this module is only used for reporting in bench.py.
"""
from __future__ import annotations


def nekbone_flops_per_iter(E: int, N: int) -> int:
    """eq:nekbone_flops, the FOM convention."""
    NP = N + 1
    return E * (12 * NP ** 4 + 34 * NP ** 3)


def hipbone_flops_per_iter(E: int, N: int) -> int:
    """eq:hipbone_flops."""
    NP = N + 1
    return E * (12 * NP ** 4 + 19 * NP ** 3) + 10 * E * N ** 3


def op_flops(E: int, N: int) -> int:
    """12 E(N+1)^4 + 18 E(N+1)^3 per operator application."""
    NP = N + 1
    return E * (12 * NP ** 4 + 18 * NP ** 3)


def op_bytes_paper(NG: int, NL: int) -> int:
    """8 N_G + 68 N_L (x read with perfect reuse + index + 6 G + W + y_L write)."""
    return 8 * NG + 68 * NL


def op_bytes_fused(NG: int, NL: int, mass_mode: int = 0) -> int:
    """This build's fused gather-apply-scatter-add kernel, algorithmic minimum:
    x read 8 N_G (perfect reuse) + int32 index 4 N_L + six G 48 N_L + assembled output
    read-modify-write 16 N_G (initialised to lambda x by the p-update); mass mode 1 adds
    the B stream 8 N_L.  See DESIGN.md "Operator kernel"."""
    return 24 * NG + 52 * NL + (8 * NL if mass_mode == 1 else 0)


def cg_bytes_paper(NG: int, NL: int) -> int:
    """108 N_G + 80 N_L per CG iteration."""
    return 108 * NG + 80 * NL


def cg_bytes_fused(NG: int, NL: int, mass_mode: int = 0) -> int:
    """This build per CG iteration: operator (24 N_G + 52 N_L, p.Ap fused in as the element
    energy) + the vector update (x, p, r, Ap read; x, r, p, Ap written: 64 N_G; the
    r.r-dependent p update re-reads r and p, counted once more: 80 N_G)."""
    return op_bytes_fused(NG, NL, mass_mode) + 80 * NG


def op_roofline(N: int, B: float, C: float = float("inf")) -> float:
    """eq:op_perf."""
    NP = N + 1
    return min(C, (12 * NP ** 4 + 18 * NP ** 3) / (8 * N ** 3 + 68 * NP ** 3) * B)


def throughput(NG: int, iters: int, ranks: int, seconds: float) -> float:
    """eq:throughput: DOFs * iterations / (ranks * time)."""
    return NG * iters / (ranks * seconds)
