"""MRST .rom files written by the product are read by the reference's own
load_rom and vice versa (rom.cpp:257-377)."""
from __future__ import annotations

import numpy as np
import pytest

from conftest import RomObj
from paper_2411_12690_b200.api import Error, ReducedOrderModel, load_rom, save_rom


@pytest.fixture(scope="module")
def small_ref_rom(oracle_libs):
    refpy, _ = oracle_libs
    return refpy.build_rom(5e-6, 50e-6, 0.5e-6, 15e-6, 4, 3, 3, 0)


def test_reference_file_round_trips_through_product(tmp_path, small_ref_rom, oracle_libs):
    refpy, _ = oracle_libs
    p = str(tmp_path / "a.rom")
    small_ref_rom.save(p)
    rom = load_rom(p)
    assert rom.fingerprint == small_ref_rom.fingerprint
    assert np.array_equal(rom.basis, small_ref_rom.Phi) and np.array_equal(rom.a_element, small_ref_rom.K)
    q = str(tmp_path / "b.rom")
    save_rom(rom, q)
    assert open(p, "rb").read() == open(q, "rb").read()  # byte-identical
    back = refpy.load_rom(q)
    assert np.array_equal(back.Phi, small_ref_rom.Phi) and back.fingerprint == small_ref_rom.fingerprint


def test_corrupt_files_rejected(tmp_path, small_ref_rom):
    p = tmp_path / "c.rom"
    small_ref_rom.save(str(p))
    data = bytearray(p.read_bytes())
    bad = tmp_path / "bad.rom"
    bad.write_bytes(b"XXXX" + bytes(data[4:]))
    with pytest.raises(Error, match="bad magic"):
        load_rom(str(bad))
    data2 = bytearray(data)
    data2[20] ^= 1  # header byte -> fingerprint mismatch
    bad.write_bytes(bytes(data2))
    with pytest.raises(Error, match="fingerprint"):
        load_rom(str(bad))
    bad.write_bytes(bytes(data[:-8]))
    with pytest.raises(Error, match="corrupt length"):
        load_rom(str(bad))


def _desc_of(r):
    """RomDesc over an oracle RefRom (keeps the arrays alive on the object)."""
    import ctypes as C
    from paper_2411_12690_b200 import native
    d = native.RomDesc()
    d.q[:] = list(r.q)
    d.geometry[:] = list(r.geom)
    r._g = [np.ascontiguousarray(g) for g in (r.gx, r.gy, r.gz)]
    d.grid_len[:] = [len(g) for g in r._g]
    for a in range(3):
        d.grid[a] = r._g[a].ctypes.data_as(C.c_void_p)
    for i in range(3):
        for j in range(3):
            d.materials[i][j] = float(r.mats[i, j])
    d.a_element, d.b_element, d.basis, d.thermal = [a.ctypes.data_as(C.c_void_p) for a in (r.K, r.b_el, r.Phi, r.u_T)]
    return d


def test_native_writer_is_byte_identical(tmp_path, small_ref_rom, native_lib):
    import ctypes as C
    from paper_2411_12690_b200 import native
    L = native.load()
    p, q = str(tmp_path / "ref.rom"), str(tmp_path / "native.rom")
    small_ref_rom.save(p)
    err = C.create_string_buffer(256)
    assert L.tsv_save_rom_file(C.byref(_desc_of(small_ref_rom)), small_ref_rom.kind, q.encode(), err, 256) == 0, err.value
    assert open(p, "rb").read() == open(q, "rb").read()


@pytest.mark.gpu
def test_native_ingest_matches_array_upload(tmp_path, small_ref_rom, native_lib):
    from paper_2411_12690_b200.api import ArrayLayout, GpuGlobalStage, IterOptions
    from conftest import RomObj
    path = str(tmp_path / "a.rom")
    small_ref_rom.save(path)
    g1, g2 = GpuGlobalStage(0), GpuGlobalStage(0)
    assert g1.load_rom_file(path) == 0
    g2.set_rom(0, ReducedOrderModel.from_arrays(RomObj(small_ref_rom), 0))
    for g in (g1, g2):
        g.set_layout(ArrayLayout(2, 3, None, [-250.0], small_ref_rom.geom[3], small_ref_rom.geom[1]))
        g.set_bc("bottom_pin_321")
    u1 = g1.solve_global(IterOptions(1e-12)).u
    u2 = g2.solve_global(IterOptions(1e-12)).u
    assert np.array_equal(u1, u2)
    bad = tmp_path / "bad.rom"
    bad.write_bytes(b"XXXX" + open(path, "rb").read()[4:])
    with pytest.raises(Error, match="bad magic"):
        g1.load_rom_file(str(bad))
