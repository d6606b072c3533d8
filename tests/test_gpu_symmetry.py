"""The mirror-symmetric contraction path (csrc/symmetry.hpp, csrc/sym.cuh)
against the reference's CPU path and against the plain DMMA path.

The reference's ROMs are mirror-symmetric to rounding, so K6 runs on the
8-irrep path in every other GPU test already; here the K1 irrep path (on by
default for the large configs only) is forced on small arrays with
TSV_SYM_K1=1 and compared with the reference CSR operator, the reference
solve and the plain path (TSV_SYM=0).
"""
from __future__ import annotations

import numpy as np
import pytest

from conftest import RomObj, ref_rom, rel_l2, stress_errors
from paper_2411_12690_b200 import configs
from paper_2411_12690_b200.api import ArrayLayout, GpuGlobalStage, IterOptions, ReducedOrderModel

pytestmark = pytest.mark.gpu
TOL, U_TOL, S_TOL = 1e-12, 1e-10, 1e-8


def stage(roms, rows, cols, kinds, dts, cfg, env, monkeypatch, bc="bottom_pin_321"):
    for k in ("TSV_SYM", "TSV_SYM_K1", "TSV_SYM_CORR", "TSV_SYM_K1_FUSED", "TSV_SYM_K1_MF", "TSV_K1_VERIFY", "TSV_SYM_K1_PIPE"):
        monkeypatch.delenv(k, raising=False)
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    g = GpuGlobalStage(0)
    g.set_roms(*[ReducedOrderModel.from_arrays(RomObj(r), i) if r is not None else None for i, r in enumerate(roms)])
    g.set_layout(ArrayLayout(rows, cols, kinds, dts, cfg.p, cfg.h))
    g.set_bc(bc)
    return g


@pytest.fixture(scope="module")
def case(oracle_libs, native_lib):
    refpy, _ = oracle_libs
    cfg = configs.get(0)
    rng = np.random.default_rng(11)
    rows, cols = 5, 6
    kinds = (rng.random(rows * cols) < 0.3).astype(np.uint8)
    dts = -270.0 + 40.0 * rng.random(rows * cols)
    roms = (ref_rom(cfg, 0, refpy), ref_rom(cfg, 1, refpy))
    sess = refpy.RefSession(roms[0], roms[1], rows, cols, kinds=kinds, delta_t=dts, bc_mode=1)
    return cfg, roms, rows, cols, kinds, dts, sess


def test_reference_roms_are_symmetric(case, monkeypatch):
    cfg, roms, rows, cols, kinds, dts, _ = case
    g = stage(roms, rows, cols, kinds, dts, cfg, {}, monkeypatch)
    s = g.symmetry()
    assert s["recovery"] and sum(s["irrep_dofs"]) == cfg.n
    assert max(s["defect_k"]) <= 1e-13 and max(s["defect_phi"]) <= 1e-13
    g.close()
    g = stage(roms, rows, cols, kinds, dts, cfg, {"TSV_SYM": "0"}, monkeypatch)
    s = g.symmetry()
    assert not s["recovery"] and not s["operator"]
    g.close()


# the irrep K1 variants: the fused kernel with 16 / 24 / 32 rows per CTA, and the multi-kernel path
K1_VARIANTS = {
    "fused16": {"TSV_SYM_K1": "1"},
    "fused24": {"TSV_SYM_K1": "1", "TSV_SYM_K1_MF": "3"},
    "fused32": {"TSV_SYM_K1": "1", "TSV_SYM_K1_MF": "4"},
    "pipe16": {"TSV_SYM_K1": "1", "TSV_SYM_K1_PIPE": "1"},  # two row buffers, one CTA per SM
    "panels": {"TSV_SYM_K1": "1", "TSV_SYM_K1_FUSED": "0"},
    "fused16_dmma_check": {"TSV_SYM_K1": "1", "TSV_K1_VERIFY": "0"},  # A x of the check on the plain DMMA K1
}


@pytest.mark.parametrize("variant", list(K1_VARIANTS))
def test_irrep_operator_matches_reference_csr(case, monkeypatch, variant):
    cfg, roms, rows, cols, kinds, dts, sess = case
    g = stage(roms, rows, cols, kinds, dts, cfg, K1_VARIANTS[variant], monkeypatch)
    s = g.symmetry()
    assert s["operator"] and s["fused"] == (variant != "panels") and s["correction"] == (variant == "panels")
    gp = stage(roms, rows, cols, kinds, dts, cfg, {"TSV_SYM": "0"}, monkeypatch)
    rng = np.random.default_rng(5)
    for _ in range(3):
        x = rng.standard_normal(sess.N)
        y_ref = sess.apply(x)
        y_sym, y_plain = g.apply(x), gp.apply(x)
        assert rel_l2(y_sym, y_ref) <= 1e-13
        assert rel_l2(y_plain, y_ref) <= 1e-13
        assert rel_l2(y_sym, y_plain) <= 1e-13
    g.close()
    gp.close()


@pytest.mark.parametrize("variant", ["fused16", "fused24", "fused16_dmma_check", "pipe16", "panels"])
@pytest.mark.parametrize("precond", ["diagonal", "schwarz2"])
def test_irrep_path_solve_and_recovery_parity(case, monkeypatch, precond, variant):
    cfg, roms, rows, cols, kinds, dts, sess = case
    u_ref, _, _ = sess.iterate(TOL)
    s_ref = sess.recover(u_ref, 8)
    g = stage(roms, rows, cols, kinds, dts, cfg, K1_VARIANTS[variant], monkeypatch)
    sol = g.solve_global(IterOptions(TOL, 100000, precond))
    assert sol.relative_residual <= TOL
    assert rel_l2(sol.u, u_ref) <= U_TOL
    mx, l2 = stress_errors(g.recover(8), s_ref)
    assert mx.max() <= S_TOL and l2.max() <= S_TOL
    # one block's displacement field (K6 alone) against the reference
    for cell in (0, rows * cols - 1):
        g.set_solution(u_ref)
        assert rel_l2(g.block_field(cell), sess.block_field(u_ref, cell)) <= 1e-12
    g.close()


def test_irrep_recovery_equals_plain_recovery(case, monkeypatch):
    cfg, roms, rows, cols, kinds, dts, sess = case
    u_ref, _, _ = sess.iterate(TOL)
    out = []
    for env in ({}, {"TSV_SYM": "0"}):
        g = stage(roms, rows, cols, kinds, dts, cfg, env, monkeypatch)
        g.set_solution(u_ref)
        out.append((g.recover(8), g.recover(1)))
        g.close()
    for a, b in zip(out[0], out[1]):
        mx, _ = stress_errors(a, b)
        assert mx.max() <= 1e-11


def test_asymmetric_rom_takes_the_plain_path(case, oracle_libs, monkeypatch):
    """A ROM without the mirror symmetry (K_r perturbed) is detected and
    runs on the plain DMMA path; the operator still matches the oracle."""
    _, orcpy = oracle_libs
    cfg, roms, rows, cols, kinds, dts, _ = case
    rng = np.random.default_rng(3)

    def bent(r):
        o = RomObj(r)
        E = rng.standard_normal(o.K.shape)
        o.K = o.K + 1e-7 * np.abs(o.K).max() * (E + E.T)
        return o

    r2 = [bent(r) for r in roms]
    for k in ("TSV_SYM", "TSV_SYM_K1", "TSV_SYM_CORR", "TSV_SYM_K1_FUSED", "TSV_SYM_K1_MF", "TSV_K1_VERIFY", "TSV_SYM_K1_PIPE"):
        monkeypatch.delenv(k, raising=False)
    monkeypatch.setenv("TSV_SYM_K1", "1")
    g = GpuGlobalStage(0)
    g.set_roms(ReducedOrderModel.from_arrays(r2[0], 0), ReducedOrderModel.from_arrays(r2[1], 1))
    g.set_layout(ArrayLayout(rows, cols, kinds, dts, cfg.p, cfg.h))
    g.set_bc("bottom_pin_321")
    s = g.symmetry()
    assert not s["recovery"] and not s["operator"] and max(s["defect_k"]) > 1e-12
    o = orcpy.OracleSystem(r2, rows, cols, cfg.q, kinds=kinds, delta_t=dts, bc_mode=1)
    x = rng.standard_normal(o.N)
    assert rel_l2(g.apply(x), o.apply(x)) <= 1e-13
    g.close()
