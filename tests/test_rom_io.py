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
