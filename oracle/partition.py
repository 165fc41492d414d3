"""Element partition, ownership of shared DOFs, halo/interior split and exchange plans.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Brute force over the whole global
mesh (tiny meshes only) -- every rule written as literally as possible.

P:167 -- "partitioning the mesh evenly among the P processes".
P:190-192 -- halo node: node contained in elements owned by different processes;
         halo element: contains >= 1 halo node; interior element: all others.
P:201 -- owner of a halo node "chosen randomly, but fairly, from among the owners of
         the halo elements of which this node is a part"; interior kernel on "half of
         the interior elements".
P:203 -- the other half of the interior elements after the halo elements.
Readings: c8 rank grid minimising total cut area, ties px>=py>=pz, then
lexicographically largest; remainder layers to the lowest ranks; rank order
r = rx + px (ry + py rz); local elements ascending global e.  c9 owner =
sorted_sharers[splitmix64(splitmix64(seed) XOR g) mod k].  c10 A = first ceil(I/2)
interior elements.  c11 halo segment ordered by (owner rank, gid); send lists mirror it.
"""
from __future__ import annotations

import math

import numpy as np

from .forcing import splitmix64
from .mesh import element_coords, l2g


def rank_grid(P: int, nx: int, ny: int, nz: int) -> tuple[int, int, int]:
    best = None
    for px in range(1, P + 1):
        for py in range(1, P + 1):
            for pz in range(1, P + 1):
                if px * py * pz != P or px > nx or py > ny or pz > nz:
                    continue
                area = (px - 1) * ny * nz + (py - 1) * nx * nz + (pz - 1) * nx * ny
                ordered = px >= py >= pz
                key = (area, 0 if ordered else 1, -px, -py, -pz)
                if best is None or key < best[0]:
                    best = (key, (px, py, pz))
    if best is None:
        raise ValueError(f"no rank grid for P={P} with px<=nx={nx}, py<=ny={ny}, pz<=nz={nz}")
    return best[1]


def axis_owner(n: int, p: int) -> list[int]:
    """owner[q] of each of the n element layers when split over p ranks; the first n % p
    ranks get one extra layer."""
    out = []
    for q in range(p):
        out += [q] * (n // p + (1 if q < n % p else 0))
    return out


def element_rank(nx, ny, nz, grid) -> np.ndarray:
    px, py, pz = grid
    ox, oy, oz = axis_owner(nx, px), axis_owner(ny, py), axis_owner(nz, pz)
    E = nx * ny * nz
    er = np.empty(E, dtype=np.int64)
    for e in range(E):
        ex, ey, ez = element_coords(e, nx, ny)
        er[e] = ox[ex] + px * (oy[ey] + py * oz[ez])
    return er


def owner_of(g: int, sharers_sorted, seed: int) -> int:
    """Owner of global id g among its sharing ranks ("randomly, but fairly"; reading c9):
    sorted_sharers[splitmix64(splitmix64(seed) XOR g) mod k]; a node with one sharer is its own."""
    if len(sharers_sorted) == 1:
        return sharers_sorted[0]
    return sharers_sorted[splitmix64(splitmix64(seed) ^ g) % len(sharers_sorted)]


def build(nx, ny, nz, N, P, seed=0, grid=None):
    """Per-rank partition data for every rank (dict list)."""
    if grid is None:
        grid = rank_grid(P, nx, ny, nz)
    er = element_rank(nx, ny, nz, grid)
    gid_all = l2g(nx, ny, nz, N)
    sharers: dict[int, set] = {}
    for e in range(gid_all.shape[0]):
        for g in gid_all[e]:
            sharers.setdefault(int(g), set()).add(int(er[e]))
    owner = {g: owner_of(g, sorted(s), seed) for g, s in sharers.items()}
    ranks = []
    for r in range(P):
        mine = [e for e in range(gid_all.shape[0]) if er[e] == r]
        halo_e, interior = [], []
        for e in mine:
            if any(len(sharers[int(g)]) > 1 for g in gid_all[e]):
                halo_e.append(e)
            else:
                interior.append(e)
        nA = math.ceil(len(interior) / 2)
        A, B = interior[:nA], interior[nA:]
        order = A + halo_e + B
        referenced = sorted({int(g) for e in mine for g in gid_all[e]})
        owned = sorted(g for g, o in owner.items() if o == r)
        halo = sorted((g for g in referenced if owner[g] != r), key=lambda g: (owner[g], g))
        ext = owned + halo
        pos = {g: t for t, g in enumerate(ext)}
        gid_local = gid_all[order] if order else np.zeros((0, (N + 1) ** 3), dtype=np.int64)
        idx = np.array([[pos[int(g)] for g in row] for row in gid_local], dtype=np.int64).reshape(
            gid_local.shape)
        neighbors = sorted({q for e in mine for g in gid_all[e] for q in sharers[int(g)]} - {r})
        recv = {q: [g for g in halo if owner[g] == q] for q in neighbors}
        send = {}
        for q in neighbors:
            q_refs = {int(g) for e in range(gid_all.shape[0]) if er[e] == q for g in gid_all[e]}
            send[q] = sorted(g for g in owned if g in q_refs)
        ranks.append(dict(grid=grid, elements=order, owner=owner, nA=len(A), nH=len(halo_e), nB=len(B),
                          owned=owned, halo=halo, gid=gid_local, idx=idx,
                          neighbors=neighbors, recv=recv, send=send))
    return ranks
