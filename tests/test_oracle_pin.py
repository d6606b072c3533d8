"""Pin the CPU restatement (oracle/tsv_oracle.c) before trusting it.

1. Against the committed golden fixtures produced by the reference itself
   (tests/golden/make_golden.py runs the unmodified tsvstress sources).
2. Against the live reference library (oracle/_ref) on a config-0-sized
   mixed array: operator, load, three preconditioners, recovery.
"""
from __future__ import annotations

import glob
import os

import numpy as np
import pytest

from conftest import ROOT, rel_l2, stress_errors

GOLDEN = sorted(glob.glob(os.path.join(ROOT, "tests", "golden", "*.npz")))


class _Rom:
    def __init__(self, z, tag):
        self.K, self.b_el, self.Phi, self.u_T = z[f"{tag}_K"], z[f"{tag}_b_el"], z[f"{tag}_Phi"], z[f"{tag}_u_T"]
        self.gx, self.gy, self.gz = z[f"{tag}_gx"], z[f"{tag}_gy"], z[f"{tag}_gz"]
        self.elem_mat, self.mats = z[f"{tag}_elem_mat"], z[f"{tag}_mats"]


def golden_system(orcpy, z):
    roms = [_Rom(z, "tsv"), _Rom(z, "dummy") if "dummy_K" in z else None]
    kinds = z["kinds"] if z["kinds"].size else None
    q = int(z["mesh"][2])
    return orcpy.OracleSystem(roms, int(z["rows"]), int(z["cols"]), q, kinds=kinds, delta_t=z["delta_t"],
                              bc_mode=int(z["bc_mode"]))


def rotation_free(d, lon, p, q):
    v = np.zeros((len(lon), 3))
    v[:, 0] = -p * lon[:, 1] / (q - 1)
    v[:, 1] = p * lon[:, 0] / (q - 1)
    v = v.ravel()
    return d - (d @ v) / (v @ v) * v


@pytest.mark.parametrize("path", GOLDEN, ids=[os.path.basename(p) for p in GOLDEN])
def test_oracle_reproduces_reference_golden(oracle_libs, path):
    _, orcpy = oracle_libs
    z = np.load(path)
    o = golden_system(orcpy, z)
    assert np.array_equal(o.dof_map, z["dof_map"])                 # bit-exact index
    assert np.array_equal(o.constrained, z["constrained"])
    assert np.array_equal(o.rhs(), z["load"])                       # bit-exact lifted load
    u, it, rr = o.solve(tol=1e-12, precond=1)
    d = u - z["u"]
    if int(z["bc_mode"]) == 0:  # literal BC: compare modulo the free z-rotation
        d = rotation_free(d, o.lon, float(z["geometry"][3]), int(z["mesh"][2]))
    assert np.linalg.norm(d) / np.linalg.norm(z["u"]) <= 1e-10
    assert abs(it - int(z["iterations"])) <= 2
    s = o.recover(z["u"], 8)
    mx, _ = stress_errors(s, z["stress"])
    assert mx.max() <= 1e-13                                          # same arithmetic as the reference


@pytest.fixture(scope="module")
def live(oracle_libs):
    refpy, orcpy = oracle_libs
    r = refpy.build_rom(5e-6, 50e-6, 0.5e-6, 15e-6, 8, 8, 4, 0)
    dm = refpy.build_rom(5e-6, 50e-6, 0.5e-6, 15e-6, 8, 8, 4, 1)
    rng = np.random.default_rng(11)
    kinds = (rng.random(12) < 0.35).astype(np.uint8)
    dts = -270.0 + 40.0 * rng.random(12)
    s = refpy.RefSession(r, dm, 3, 4, kinds=kinds, delta_t=dts, bc_mode=1)
    from conftest import RomObj
    o = orcpy.OracleSystem([RomObj(r), RomObj(dm)], 3, 4, 4, kinds=kinds, delta_t=dts, bc_mode=1)
    return s, o


def test_oracle_matches_live_reference(live):
    s, o = live
    assert np.array_equal(o.dof_map, s.dof_map())
    nol, lon = s.lattice()
    assert np.array_equal(o.nol, nol) and np.array_equal(o.lon, lon)
    b, cm, _ = s.rhs()
    assert np.array_equal(o.constrained, cm) and np.array_equal(o.rhs(), b)
    x = np.random.default_rng(1).standard_normal(s.N)
    assert rel_l2(o.apply(x), s.apply(x)) <= 1e-14
    for pc in (0, 1, 2):
        u_r, it_r, _ = s.iterate(1e-12, 10000, pc)
        u_o, it_o, _ = o.solve(tol=1e-12, precond=pc)
        assert rel_l2(u_o, u_r) <= 1e-10 and abs(it_o - it_r) <= 2
    u_r, _, _ = s.iterate(1e-12)
    assert np.array_equal(o.recover(u_r, 8), s.recover(u_r, 8))   # bit-exact recovery
    assert np.array_equal(o.recover(u_r, 1), s.recover(u_r, 1))


def test_oracle_no_convergence_matches_reference(live, oracle_libs):
    refpy, orcpy = oracle_libs
    s, o = live
    with pytest.raises(refpy.RefNoConvergence) as er:
        s.iterate(1e-14, 4)
    with pytest.raises(orcpy.OracleCGError) as eo:
        o.solve(tol=1e-14, max_it=4)
    assert eo.value.status == 2 and eo.value.iterations == er.value.iterations
    assert rel_l2(eo.value.x, er.value.u) <= 1e-12


def test_config_generators():
    from paper_2411_12690_b200 import configs
    g = configs.MT19937_64(5489)
    for _ in range(9999):
        g()
    assert g() == 9981545732273789042  # the C++ standard's known answer for mt19937_64
    c3, c4 = configs.get(3), configs.get(4)
    dt = c3.delta_t()
    assert dt.shape == (10000,) and dt.min() >= -270.0 and dt.max() < -230.0
    k = c4.kinds()
    assert k.shape == (40000,) and 0.18 < k.mean() < 0.22
    assert [c.lattice_dofs() for c in configs.CONFIGS] == [1806, 17115, 269970, 3835221, 6384015]


# ---------------------------------------------------------------- Schwarz64
# The FP64 two-level Schwarz PCG oracle (oracle/schwarz64.py) is the CPU
# solution the GPU is compared with at configs 3/4; pin it against the live
# reference's own Jacobi-PCG (CSR path) before trusting it there.

def test_schwarz64_matches_live_reference_mixed(live):
    from oracle.schwarz64 import Schwarz64
    s, o = live
    u_r, it_r, _ = s.iterate(1e-12)
    S = Schwarz64(o, 4, s=2)
    u_o, it_o, rr = S.solve(tol=1e-12)
    assert rr <= 1e-12
    assert rel_l2(u_o, u_r) <= 1e-10
    b, _, _ = s.rhs()
    assert rel_l2(s.apply(u_o), b) <= 1e-11      # residual under the reference's CSR operator
    assert it_o < it_r


def test_schwarz64_operator_is_symmetric_positive(live):
    """M^-1 is a fixed SPD matrix (what plain CG needs)."""
    from oracle.schwarz64 import Schwarz64
    _, o = live
    S = Schwarz64(o, 4, s=2)
    rng = np.random.default_rng(3)
    x, y = rng.standard_normal(o.N), rng.standard_normal(o.N)
    mx, my = S.apply(x), S.apply(y)
    assert abs(x @ my - y @ mx) <= 1e-12 * abs(x @ my)
    assert x @ mx > 0 and y @ my > 0
    assert np.array_equal(S.apply(x), mx)          # deterministic


@pytest.mark.parametrize("ci", [0, 1])
def test_schwarz64_matches_live_reference_configs(oracle_libs, ci):
    from conftest import RomObj, ref_rom
    from oracle.schwarz64 import Schwarz64
    from paper_2411_12690_b200 import configs
    refpy, orcpy = oracle_libs
    cfg = configs.get(ci)
    r = ref_rom(cfg, 0, refpy)
    s = refpy.RefSession(r, None, cfg.rows, cfg.cols, delta_t=cfg.delta_t(), bc_mode=1)
    o = orcpy.OracleSystem([RomObj(r)], cfg.rows, cfg.cols, cfg.q, delta_t=cfg.delta_t(), bc_mode=1)
    u_r, it_r, _ = s.iterate(1e-12)
    u_o, it_o, rr = Schwarz64(o, cfg.q).solve(tol=1e-12)
    assert rr <= 1e-12 and rel_l2(u_o, u_r) <= 1e-10 and it_o < it_r / 5
