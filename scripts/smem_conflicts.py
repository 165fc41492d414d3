#!/usr/bin/env python
"""Offline shared-memory bank-conflict model of the line-owner kernel (ax_lines.cuh) for
multi-element CTAs (N <= 6): every phase's access pattern for all warps of a CTA, 64-bit
accesses (a double at word w uses bank pair w mod 16; a warp is served as two half-warps),
elements at offsets le * SLAB (odd slabs allowed).  Thread t -> (element le, column c) is
blocked (le = t / (N+1)^2) or interleaved (le = t % EPB, LinesShape::ILV).  Searches
(P1, P2, SLAB) minimising the wavefront count, per mapping.

    python scripts/smem_conflicts.py [2,3,4,5]  # current table vs best found per mapping
"""
import itertools
import sys

PAD = {1: (2, 5, 12), 2: (3, 18, 57), 3: (4, 19, 76), 4: (5, 25, 137), 5: (9, 54, 324), 6: (7, 52, 370)}


def epb(N):
    NP2 = (N + 1) ** 2
    return 128 // NP2 if N == 5 else max(1, 64 // NP2)


def wavefronts(N, P1, P2, SLAB, inter=False):
    NP = N + 1
    NP2 = NP * NP
    E = epb(N)
    block = E * NP2
    total = 0

    def lec(t):
        return (t % E, t // E) if inter else divmod(t, NP2)
    # patterns: (name, function(thread) -> list over loop index m of word addresses)
    def col(t, m):   # column owner (i,j) = (ca,cb), node k = m
        le, c = lec(t)
        ca, cb = c % NP, c // NP
        return le * SLAB + m * P2 + cb * P1 + ca
    def row(t, m):   # row owner (j,k) = (ca,cb): (m, ca, cb)
        le, c = lec(t)
        ca, cb = c % NP, c // NP
        return le * SLAB + cb * P2 + ca * P1 + m
    def sln(t, m):   # s-line owner (i,k) = (ca,cb): (ca, m, cb)
        le, c = lec(t)
        ca, cb = c % NP, c // NP
        return le * SLAB + cb * P2 + m * P1 + ca
    # per apply: col x (P1 write, P3 rd+wr x2, P5 rd x3) ~ 8, row x 4 (P2 rd, wr; P4 rd, wr), sln x 4
    weights = {col: 8, row: 4, sln: 4}
    for f, wgt in weights.items():
        for w0 in range(0, block, 32):
            threads = list(range(w0, min(w0 + 32, block)))
            for m in range(NP):
                for half in (threads[:16], threads[16:]):
                    if not half:
                        continue
                    banks = {}
                    for t in half:
                        a = f(t, m)
                        banks.setdefault(a % 16, set()).add(a)
                    total += wgt * max(len(v) for v in banks.values())
    return total


def search(N, inter=False):
    NP = N + 1
    best = None
    for P1 in range(NP, NP + 9):
        for P2 in range(NP * P1, NP * P1 + 17):
            base = NP * P2
            for SLAB in range(base, base + 34):
                c = wavefronts(N, P1, P2, SLAB, inter)
                key = (c, SLAB, P2, P1)
                if best is None or key < best[0]:
                    best = (key, (P1, P2, SLAB))
    return best


if __name__ == "__main__":
    Ns = [int(v) for v in sys.argv[1].split(",")] if len(sys.argv) > 1 else list(PAD)
    for N in Ns:
        cur = wavefronts(N, *PAD[N])
        (cb, Sb, P2b, P1b), _ = search(N)
        (ci, Si, P2i, P1i), _ = search(N, True)
        print(f"N={N} EPB={epb(N)} table {PAD[N]} wavefronts={cur}  best blocked ({P1b},{P2b},{Sb}) {cb}  "
              f"best interleaved ({P1i},{P2i},{Si}) {ci}", flush=True)
