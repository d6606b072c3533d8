"""Host-side indexing of the product library (no GPU): the C ABI's
tsv_index_global_nodes must equal the reference's index_global_nodes /
global_dof bit for bit, and pass the reference's own known-answer tests
(proj/tests/test_global.cpp:61-101)."""
from __future__ import annotations

import ctypes as C

import numpy as np
import pytest

from paper_2411_12690_b200 import native


def product_index(rows, cols, q):
    L = native.load()
    qa = (C.c_uint32 * 3)(*([q] * 3 if np.isscalar(q) else q))
    nd = C.c_uint64()
    lat = (C.c_uint32 * 3)()
    assert L.tsv_index_global_nodes(rows, cols, qa, C.byref(nd), lat, None, None, None) == 0
    lx, ly, lz = lat
    nol = np.empty(lx * ly * lz, np.int32)
    lon = np.empty((nd.value // 3, 3), np.uint32)
    qq = [q] * 3 if np.isscalar(q) else list(q)
    n = 3 * (np.prod(qq) - np.prod([v - 2 for v in qq]))
    dm = np.empty((rows * cols, n), np.uint32)
    assert L.tsv_index_global_nodes(rows, cols, qa, None, None, nol.ctypes.data_as(C.c_void_p),
                                    lon.ctypes.data_as(C.c_void_p), dm.ctypes.data_as(C.c_void_p)) == 0
    return nd.value, (lx, ly, lz), nol, lon, dm


def surface_rank(q, ijk):
    rank = 0
    for i in range(q):
        for j in range(q):
            for k in range(q):
                if 0 < i < q - 1 and 0 < j < q - 1 and 0 < k < q - 1:
                    continue
                if (i, j, k) == ijk:
                    return rank
                rank += 1
    raise KeyError(ijk)


def test_known_answers_from_reference_tests(native_lib):
    # 1x1 keeps every reduced dof (test_global.cpp:64-67)
    for q in (2, 3, 4, 5, 7):
        nd, *_ = product_index(1, 1, q)
        assert nd == 3 * (q ** 3 - (q - 2) ** 3)
    # 2x1 (q=2) shares one face of 4 nodes (:69-72)
    assert product_index(1, 2, 2)[0] == 2 * 24 - 4 * 3
    # corner shared by 4 blocks maps to one dof (:74-91)
    nd, lat, nol, lon, dm = product_index(2, 2, 2)
    cells = {(0, 0): (1, 1, 0), (0, 1): (0, 1, 0), (1, 0): (1, 0, 0), (1, 1): (0, 0, 0)}
    dofs = {dm[r * 2 + c, 3 * surface_rank(2, ijk)] for (r, c), ijk in cells.items()}
    assert len(dofs) == 1
    # q=4, 2x2: lattice 7x7x4 minus 4 block interiors of 2x2x2 (:94-101)
    nd, lat, *_ = product_index(2, 2, 4)
    assert nd // 3 == 7 * 7 * 4 - 4 * 8


@pytest.mark.parametrize("rows,cols,q", [(1, 1, 3), (3, 3, 5), (4, 5, 5), (2, 7, 6), (5, 3, (3, 4, 5))])
def test_matches_oracle_restatement(native_lib, oracle_libs, rows, cols, q):
    _, orcpy = oracle_libs
    nd, lat, nol, lon, dm = product_index(rows, cols, q)
    nol_o, lon_o, lat_o = orcpy.index_global_nodes(rows, cols, q)
    assert tuple(lat) == tuple(lat_o)
    assert np.array_equal(nol, nol_o) and np.array_equal(lon, lon_o)
    qq = (q, q, q) if np.isscalar(q) else q
    dm_o = np.empty_like(dm)
    import ctypes
    orcpy.lib().orc_dof_map(rows, cols, *qq, nol_o.ctypes.data_as(ctypes.c_void_p),
                            dm_o.ctypes.data_as(ctypes.c_void_p))
    assert np.array_equal(dm, dm_o)


def test_matches_reference_index(native_lib, oracle_libs):
    """Against the reference library itself (oracle/_ref) on a real ROM layout."""
    refpy, _ = oracle_libs
    rom = refpy.build_rom(5e-6, 50e-6, 0.5e-6, 15e-6, 4, 4, 3, 0)
    for rows, cols in [(1, 1), (2, 3), (4, 4)]:
        s = refpy.RefSession(rom, None, rows, cols, bc_mode=1)
        nd, lat, nol, lon, dm = product_index(rows, cols, 3)
        nol_r, lon_r = s.lattice()
        assert nd == s.N
        assert np.array_equal(nol, nol_r) and np.array_equal(lon, lon_r)
        assert np.array_equal(dm, s.dof_map())


def test_survey_global_dof_counts(native_lib):
    from paper_2411_12690_b200 import configs
    expect = [1806, 17115, 269970, 3835221, 6384015]
    for cfg, n in zip(configs.CONFIGS, expect):
        nd, *_ = product_index(cfg.rows, cfg.cols, cfg.q) if cfg.B <= 1024 else (cfg.lattice_dofs(),)
        assert nd == n == cfg.lattice_dofs()


def test_invalid_layout_rejected(native_lib):
    L = native.load()
    qa = (C.c_uint32 * 3)(1, 3, 3)
    assert L.tsv_index_global_nodes(2, 2, qa, None, None, None, None, None) != 0
    qa = (C.c_uint32 * 3)(3, 3, 3)
    assert L.tsv_index_global_nodes(0, 2, qa, None, None, None, None, None) != 0
