"""Product local stage (GPU build_rom) against the reference's build_rom
(oracle/_ref) on identical inputs. The ROM is an input of the hot path; the
parity tests feed the reference ROM to both sides, the bench uses this one."""
from __future__ import annotations

import numpy as np
import pytest

from conftest import RomObj, ref_rom, rel_l2
from paper_2411_12690_b200 import configs
from paper_2411_12690_b200.api import build_config_rom

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("ci,kind", [(0, 0), (0, 1), (2, 0), (3, 0), (4, 1)])
def test_config_rom_matches_reference(oracle_libs, native_lib, ci, kind):
    """The ROMs the bench consumes (config 2: 24^3 mesh, q = 6; config 3:
    20^3, q = 7; config 4's dummy) against the reference's build_rom."""
    refpy, _ = oracle_libs
    cfg = configs.get(ci)
    r = ref_rom(cfg, kind, refpy)
    g = build_config_rom(cfg, kind)
    assert g.fingerprint == r.fingerprint            # same SHA-256 header (rom.cpp:110-132)
    assert np.array_equal(g.element_material, r.elem_mat)
    assert rel_l2(g.basis, r.Phi) <= 1e-9
    assert rel_l2(g.thermal, r.u_T) <= 1e-9
    assert rel_l2(g.a_element, r.K) <= 1e-9
    assert rel_l2(g.b_element, r.b_el) <= 1e-9


def test_small_rom_matches_reference(oracle_libs, native_lib):
    refpy, _ = oracle_libs
    cfg = configs.TsvConfig("tiny", 1, 1, m_xy=6, m_z=5, q=3, points=8, d=5e-6, h=50e-6, t=0.5e-6, p=15e-6)
    r = refpy.build_rom(cfg.d, cfg.h, cfg.t, cfg.p, cfg.m_xy, cfg.m_z, cfg.q, 0, cfg.liner_e)
    g = build_config_rom(cfg, 0)
    assert g.fingerprint == r.fingerprint
    assert rel_l2(g.a_element, r.K) <= 1e-10 and rel_l2(g.basis, r.Phi) <= 1e-10
