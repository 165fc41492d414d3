"""B200-native hipBone hot path (arXiv 2202.12477): matrix-free assembled SEM screened-Poisson
operator + preconditioner-free CG, behind the C ABI include/hipbone_b200.h.

Python surface = a thin ctypes binding (``hipbone.py``); every step of the path runs in the
library's sm_100a kernels.  The package never imports ``oracle/``.
"""
from .hipbone import (Comm, Group, HBError, Mesh, Operator, comm_unique_id, gll, rank_grid,  # noqa: F401
                      stream_bench, version, EXPORTED, LIB_PATH)
from . import ledger  # noqa: F401
