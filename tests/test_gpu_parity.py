"""GPU parity through the C ABI against the reference's own CPU path
(oracle/_ref: the unmodified tsvstress sources) on identical seeded inputs.

Bars (BASELINE.json north_star):
  * indexing (dof map, lattice, constrained set): bit-exact
  * lifted load vector: bit-exact (same summation order)
  * interface displacements: rel L2 <= 1e-10, both sides CG to 1e-12
  * stresses: per component max|d|/max|ref| <= 1e-8 (and the L2 analogue)
"""
from __future__ import annotations

import numpy as np
import pytest

from conftest import RomObj, ref_rom, rel_l2, stress_errors
from paper_2411_12690_b200 import configs
from paper_2411_12690_b200.api import (ArrayLayout, BreakdownError, Error, GpuGlobalStage, IterOptions,
                                       NoConvergence, ReducedOrderModel)

pytestmark = pytest.mark.gpu

U_TOL = 1e-10
S_TOL = 1e-8
BC_MODE = {"bottom_pin": 0, "bottom_pin_321": 1, "clamped": 2, "none": 3}


def make_case(refpy, cfg, rows=None, cols=None, kinds=None, dts=None, bc="bottom_pin_321"):
    rows = rows or cfg.rows
    cols = cols or cfg.cols
    r_tsv = ref_rom(cfg, 0, refpy)
    need_dummy = kinds is not None and np.any(kinds)
    r_dum = ref_rom(cfg, 1, refpy) if need_dummy else None
    dts = np.atleast_1d(cfg.delta_t() if dts is None else dts)
    sess = refpy.RefSession(r_tsv, r_dum, rows, cols, kinds=kinds, delta_t=dts, bc_mode=BC_MODE[bc])
    g = GpuGlobalStage(0)
    g.set_roms(ReducedOrderModel.from_arrays(RomObj(r_tsv), 0),
               ReducedOrderModel.from_arrays(RomObj(r_dum), 1) if r_dum is not None else None)
    g.set_layout(ArrayLayout(rows, cols, kinds, dts, cfg.p, cfg.h))
    g.set_bc(bc)
    return sess, g


@pytest.fixture(scope="module")
def cfg0(oracle_libs, native_lib):
    refpy, _ = oracle_libs
    return make_case(refpy, configs.get(0))


@pytest.fixture(scope="module")
def mixed(oracle_libs, native_lib):
    """4x5 array, 2 block kinds, per-block dT (configs 3/4 features at config-0 size)."""
    refpy, _ = oracle_libs
    cfg = configs.get(0)
    rng = np.random.default_rng(7)
    kinds = (rng.random(20) < 0.3).astype(np.uint8)
    dts = -270.0 + 40.0 * rng.random(20)
    return make_case(refpy, cfg, 4, 5, kinds, dts)


def test_index_bitexact(cfg0):
    sess, g = cfg0
    assert np.array_equal(g.dof_map(), sess.dof_map())
    nol_g, lon_g = g.lattice()
    nol_r, lon_r = sess.lattice()
    assert np.array_equal(nol_g, nol_r) and np.array_equal(lon_g, lon_r)
    b_r, cm_r, _ = sess.rhs()
    assert np.array_equal(g.constrained(), cm_r)
    assert np.array_equal(g.load(), b_r)  # bit-exact lifted load


def test_apply_matches_lifted_csr(cfg0):
    sess, g = cfg0
    x = np.random.default_rng(3).standard_normal(sess.N)
    assert rel_l2(g.apply(x), sess.apply(x)) <= 1e-13


@pytest.mark.parametrize("precond", ["diagonal", "none", "block_diagonal"])
def test_solve_matches_reference(cfg0, precond):
    sess, g = cfg0
    pc = {"none": 0, "diagonal": 1, "block_diagonal": 2}[precond]
    u_r, it_r, rr_r = sess.iterate(1e-12, 10000, pc)
    sol = g.solve_global(IterOptions(1e-12, 10000, precond))
    assert sol.relative_residual <= 1e-12
    assert rel_l2(sol.u, u_r) <= U_TOL
    assert abs(sol.iterations - it_r) <= max(3, it_r // 50)
    # independent residual check with the reference's CSR operator
    b_r, _, _ = sess.rhs()
    assert rel_l2(sess.apply(sol.u), b_r) <= 1e-11
    assert not sol.direct_fallback


def test_solve_is_bitwise_deterministic(cfg0):
    _, g = cfg0
    a = g.solve_global(IterOptions(1e-12)).u
    b = g.solve_global(IterOptions(1e-12)).u
    assert np.array_equal(a, b)


def test_recover_gauss_points(cfg0):
    sess, g = cfg0
    u_r, _, _ = sess.iterate(1e-12)
    s_ref = sess.recover(u_r, 8)
    g.set_solution(u_r)
    s_gpu = g.recover(8)
    mx, l2 = stress_errors(s_gpu, s_ref)
    assert mx.max() <= S_TOL and l2.max() <= S_TOL, (mx, l2)


def test_end_to_end_stress(cfg0):
    sess, g = cfg0
    u_r, _, _ = sess.iterate(1e-12)
    s_ref = sess.recover(u_r, 8)
    g.solve_global(IterOptions(1e-12), copy_out=False)
    s_gpu = g.recover(8)
    mx, l2 = stress_errors(s_gpu, s_ref)
    assert mx.max() <= S_TOL and l2.max() <= S_TOL, (mx, l2)


def test_recover_resident_and_ranges(cfg0):
    sess, g = cfg0
    g.solve_global(IterOptions(1e-12), copy_out=False)
    full = g.recover(8)
    g.recover_resident(8)
    assert np.array_equal(g.copy_stress(0, 9, 8), full)
    assert np.array_equal(g.recover(8, 4, 7), full[4:7])


def test_block_field_matches_reconstruct(cfg0):
    sess, g = cfg0
    u_r, _, _ = sess.iterate(1e-12)
    g.set_solution(u_r)
    for cell in (0, 4, 8):
        assert rel_l2(g.block_field(cell), sess.block_field(u_r, cell)) <= 1e-13


def test_mixed_kinds_and_per_block_dt(mixed):
    sess, g = mixed
    assert np.array_equal(g.dof_map(), sess.dof_map())
    b_r, _, _ = sess.rhs()
    assert np.array_equal(g.load(), b_r)
    x = np.random.default_rng(5).standard_normal(sess.N)
    assert rel_l2(g.apply(x), sess.apply(x)) <= 1e-13
    u_r, it_r, _ = sess.iterate(1e-12)
    sol = g.solve_global(IterOptions(1e-12))
    assert rel_l2(sol.u, u_r) <= U_TOL
    s_ref = sess.recover(u_r, 8)
    s_gpu = g.recover(8)
    mx, l2 = stress_errors(s_gpu, s_ref)
    assert mx.max() <= S_TOL and l2.max() <= S_TOL
    s_ref1 = sess.recover(u_r, 1)
    mx1, _ = stress_errors(g.recover(1), s_ref1)
    assert mx1.max() <= S_TOL


def test_literal_bc_parity_modulo_rotation(oracle_libs, native_lib):
    """Literal 'bottom u_z = 0 + one corner' leaves the z-rotation free
    (SURVEY.md Appendix A.3): compare modulo v = (-y, x, 0)."""
    refpy, _ = oracle_libs
    cfg = configs.get(0)
    sess, g = make_case(refpy, cfg, bc="bottom_pin")
    u_r, _, _ = sess.iterate(1e-12)
    sol = g.solve_global(IterOptions(1e-12))
    _, lon = sess.lattice()
    q = cfg.q
    x = cfg.p * lon[:, 0] / (q - 1)
    y = cfg.p * lon[:, 1] / (q - 1)
    v = np.zeros((len(lon), 3))
    v[:, 0], v[:, 1] = -y, x
    v = v.ravel()
    d = sol.u - u_r
    d -= (d @ v) / (v @ v) * v
    assert np.linalg.norm(d) / np.linalg.norm(u_r) <= U_TOL
    mx, _ = stress_errors(g.recover(8), sess.recover(u_r, 8))
    assert mx.max() <= S_TOL


def test_clamped_bc_matches_reference(oracle_libs, native_lib):
    refpy, _ = oracle_libs
    sess, g = make_case(refpy, configs.get(0), 2, 2, bc="clamped")
    b_r, cm_r, _ = sess.rhs()
    assert np.array_equal(g.constrained(), cm_r) and np.array_equal(g.load(), b_r)
    u_r, _, _ = sess.iterate(1e-12)
    assert rel_l2(g.solve_global(IterOptions(1e-12)).u, u_r) <= U_TOL


def test_zero_load_gives_zero_solution(oracle_libs, native_lib):
    refpy, _ = oracle_libs
    _, g = make_case(refpy, configs.get(0), 2, 2, dts=[0.0])
    sol = g.solve_global(IterOptions(1e-12))
    assert sol.iterations == 0 and not np.any(sol.u)
    assert not np.any(g.recover(8))


def test_no_convergence_returns_best_iterate(cfg0):
    sess, g = cfg0
    with pytest.raises(NoConvergence) as ei:
        g.solve_global(IterOptions(1e-14, 5))
    best = ei.value.best
    assert best.iterations == 5 and best.relative_residual > 1e-14
    # the reference returns the same best iterate (linalg.cpp:354-360)
    with pytest.raises(refpy_noconv(sess)) as er:
        sess.iterate(1e-14, 5)
    assert rel_l2(best.u, er.value.u) <= 1e-9
    assert abs(best.relative_residual - er.value.relres) <= 1e-6 * er.value.relres


def refpy_noconv(sess):
    from oracle.refpy import RefNoConvergence
    return RefNoConvergence


def test_invalid_inputs_fail_loudly(cfg0, oracle_libs):
    sess, g = cfg0
    with pytest.raises(Error):
        g.solve_global(IterOptions(0.0))
    with pytest.raises(Error):
        g.solve_global(IterOptions(1e-12, 0))
    with pytest.raises(Error):
        g.set_layout(ArrayLayout(3, 3, None, [-250.0, 1.0], 15e-6, 50e-6))  # bad delta_t length
    with pytest.raises(Error):
        g.set_layout(ArrayLayout(3, 3, None, [-250.0], 10e-6, 50e-6))  # pitch != model
    g.set_layout(ArrayLayout(3, 3, None, [-250.0], 15e-6, 50e-6))
    g.set_bc("bottom_pin_321")
    with pytest.raises(Error):
        g.set_dirichlet([5, 5], [0.0, 1.0])  # conflicting duplicate (fem.cpp:62-80)


def test_nan_load_is_a_breakdown(oracle_libs, native_lib):
    refpy, _ = oracle_libs
    _, g = make_case(refpy, configs.get(0), 2, 2, dts=[float("nan")])
    with pytest.raises(BreakdownError):
        g.solve_global(IterOptions(1e-12))
