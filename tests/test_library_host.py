"""CPU-only checks of the C-ABI library: it loads, exports every symbol the header
declares, and its host-side setup (GLL basis, rank grid, l2g map, partition, ownership,
halo/interior classification, exchange plans, geometry, mass) matches the oracle -- the
maps and partition bit-exactly (BASELINE.json north_star).  No compute call needs a GPU."""
import os
import re

import numpy as np
import pytest

from oracle import basis, mesh as omesh, partition as opart

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def hb():
    import __graft_entry__
    __graft_entry__.build()
    import paper_2202_12477_b200 as hb
    return hb


def test_exports_every_declared_symbol(hb):
    hdr = open(os.path.join(ROOT, "include", "hipbone_b200.h")).read()
    declared = set(re.findall(r"^\s*(?:int|const char\*)\s+(hb_\w+)\s*\(", hdr, re.M))
    assert len(declared) >= 30
    import ctypes
    lib = ctypes.CDLL(hb.LIB_PATH)
    for name in declared:
        assert hasattr(lib, name), name
    assert declared == set(hb.EXPORTED)
    assert hb.version() == 1


@pytest.mark.parametrize("N", range(1, 16))
def test_gll_matches_oracle(hb, N):
    x, w, D = hb.gll(N)
    ox, ow, oD = basis.basis(N)
    assert np.max(np.abs(x - ox)) < 4e-16
    assert np.max(np.abs(w - ow)) < 2e-15
    assert np.max(np.abs(D - oD)) < 1e-12 * max(1.0, np.abs(oD).max())


def test_rank_grid(hb):
    for P, box, g in [(1, (2, 2, 2), (1, 1, 1)), (8, (4, 4, 4), (2, 2, 2)), (6, (6, 1, 1), (6, 1, 1)),
                      (2, (132, 66, 66), (2, 1, 1)), (4, (132, 132, 66), (2, 2, 1)), (8, (50, 50, 48), (2, 2, 2))]:
        assert hb.rank_grid(P, *box) == g
        assert hb.rank_grid(P, *box) == opart.rank_grid(P, *box)
    for P in range(1, 13):
        for box in [(3, 2, 2), (5, 4, 1), (2, 2, 2), (7, 3, 5)]:
            try:
                o = opart.rank_grid(P, *box)
            except ValueError:
                with pytest.raises(hb.HBError):
                    hb.rank_grid(P, *box)
                continue
            assert hb.rank_grid(P, *box) == o


@pytest.mark.parametrize("box,N,P,seed", [((2, 2, 2), 3, 1, 0), ((4, 4, 4), 3, 2, 0), ((3, 2, 2), 2, 4, 5),
                                          ((2, 2, 2), 1, 8, 0), ((5, 3, 2), 2, 3, 1), ((4, 3, 3), 4, 6, 7),
                                          ((2, 1, 1), 1, 2, 0), ((6, 5, 4), 2, 8, 3)])
def test_partition_bit_exact(hb, box, N, P, seed):
    ranks = opart.build(*box, N, P, seed=seed)
    for r in range(P):
        m = hb.Mesh(*box, N, P=P, rank=r, seed=seed)
        o = ranks[r]
        s = m.sizes
        assert s["grid"] == o["grid"]
        assert (s["n_intA"], s["n_halo_elems"], s["n_intB"]) == (o["nA"], o["nH"], o["nB"])
        assert np.array_equal(m.elements(), np.array(o["elements"], dtype=np.int64))
        assert np.array_equal(m.owned(), np.array(o["owned"], dtype=np.int64))
        assert np.array_equal(m.halo(), np.array(o["halo"], dtype=np.int64))
        assert np.array_equal(m.l2g(), o["gid"])
        assert np.array_equal(m.local_index(), o["idx"].astype(np.int32))
        nbr, sc, rc = m.neighbors()
        assert list(nbr) == o["neighbors"]
        for q, rank_q in enumerate(nbr):
            assert np.array_equal(m.send_list(q), np.array(o["send"][int(rank_q)], dtype=np.int64))
            assert rc[q] == len(o["recv"][int(rank_q)])


def test_l2g_and_sizes_match_oracle_single_rank(hb):
    for box, N in [((3, 2, 4), 5), ((1, 1, 1), 15), ((16, 16, 16), 7)]:
        m = hb.Mesh(*box, N)
        E, NG, NL = omesh.global_sizes(*box, N)
        assert (m.sizes["E_local"], m.sizes["N_G"], m.sizes["N_L"], m.sizes["n_owned"]) == (E, NG, NL, NG)
        if NL < 100000:
            assert np.array_equal(m.l2g(), omesh.l2g(*box, N))
            assert np.array_equal(m.local_index(), omesh.l2g(*box, N).astype(np.int32))


@pytest.mark.parametrize("N,ext,mode", [(3, (2.0, 2.0, 2.0), 0), (4, (1.0, 2.0, 0.5), 1), (7, (2.0, 2.0, 2.0), 1)])
def test_geometry_and_mass_match_oracle(hb, N, ext, mode):
    box = (2, 3, 2)
    m = hb.Mesh(*box, N, ext=ext, mass_mode=mode)
    x, w = basis.gll(N)
    E, NG, NL = omesh.global_sizes(*box, N)
    G = omesh.geometric_factors(E, N, w, ext)
    assert np.max(np.abs(m.geometry() - G)) <= 4e-16 * np.abs(G).max()
    if mode == 0:
        assert np.array_equal(m.mass(), omesh.weights_W(omesh.l2g(*box, N), NG))
    else:
        B = omesh.mass_B(E, N, w, ext)
        assert np.max(np.abs(m.mass() - B)) <= 4e-16 * B.max()


def test_error_paths(hb):
    with pytest.raises(hb.HBError, match="HB_ERR_ARG"):
        hb.Mesh(2, 2, 2, 0)
    with pytest.raises(hb.HBError, match="HB_ERR_ARG"):
        hb.Mesh(2, 2, 2, 16)
    with pytest.raises(hb.HBError, match="HB_ERR_ARG"):
        hb.Mesh(2, 2, 2, 3, P=2, rank=2)
    with pytest.raises(hb.HBError, match="HB_ERR_GEOMETRY"):
        hb.Mesh(2, 2, 2, 3, ext=(1.0, -1.0, 1.0))
    with pytest.raises(hb.HBError, match="HB_ERR_CONFIG"):
        hb.Mesh(2, 2, 2, 3, P=7)
    with pytest.raises(hb.HBError, match="HB_ERR_STATE"):
        hb.Mesh(2, 2, 2, 3, mass_mode=0).set_mass(np.ones(8 * 64))
    with pytest.raises(hb.HBError, match="HB_ERR_ARG"):
        hb.gll(0)
    # IPC communicator: argument checks happen before any CUDA call
    for P, r in ((0, 0), (2, 2), (2, -1), (33, 0)):
        with pytest.raises(hb.HBError, match="HB_ERR_ARG"):
            hb.Comm.create_ipc(P, r)
    c = hb.Comm.create_ipc(1, 0)  # P = 1: valid, needs no driver entry points
    assert c.ipc


def test_set_geometry_roundtrip(hb):
    m = hb.Mesh(2, 1, 1, 2)
    from tests.inputs import random_spd_factors
    G = random_spd_factors(2, 27, seed=1)
    m.set_geometry(G)
    assert np.array_equal(m.geometry(), G)
