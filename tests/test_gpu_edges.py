"""Edge shapes and inputs against the reference's CPU path (oracle/_ref):
a single block, one row, one column, an all-dummy array, a constant vs a
per-block dT, checkerboard kinds — every preconditioner including the
two-level Schwarz (whose coarse lattice degenerates on these shapes), plus
the cut plane on a ragged array. Bars as in test_gpu_parity.py."""
from __future__ import annotations

import numpy as np
import pytest

from conftest import rel_l2, stress_errors
from paper_2411_12690_b200 import configs
from paper_2411_12690_b200.api import IterOptions

pytestmark = pytest.mark.gpu

CASES = {
    "1x1": (1, 1, None, None),
    "1x6": (1, 6, None, None),
    "5x1": (5, 1, None, None),
    "2x2_all_dummy": (2, 2, np.ones(4, np.uint8), None),
    "3x4_const_dt": (3, 4, None, np.array([-180.0])),
    "3x4_checkerboard_dt": (3, 4, (np.indices((3, 4)).sum(axis=0) % 2).astype(np.uint8).ravel(),
                            -270.0 + 10.0 * np.arange(12)),
}


@pytest.fixture(scope="module", params=list(CASES))
def case(request, oracle_libs, native_lib):
    from test_gpu_parity import make_case
    refpy, _ = oracle_libs
    rows, cols, kinds, dts = CASES[request.param]
    sess, g = make_case(refpy, configs.get(0), rows, cols, kinds, dts)
    u_r, it_r, _ = sess.iterate(1e-12)
    return request.param, sess, g, u_r, it_r


def test_index_and_load_bitexact(case):
    _, sess, g, _, _ = case
    b_r, cm_r, _ = sess.rhs()
    assert np.array_equal(g.constrained(), cm_r)
    assert np.array_equal(g.load(), b_r)


@pytest.mark.parametrize("precond", ["diagonal", "block_diagonal", "none", "schwarz2"])
def test_solve(case, precond):
    name, sess, g, u_r, it_r = case
    sol = g.solve_global(IterOptions(1e-12, 20000, precond))
    assert sol.relative_residual <= 1e-12, name
    assert rel_l2(sol.u, u_r) <= 1e-10, name
    if precond == "schwarz2" and it_r > 60:
        assert sol.iterations < it_r, name


# A homogeneous all-dummy (all-Si) array under uniform dT expands stress-free:
# sigma is round-off (~1e-4 Pa) on both sides, so the relative bar is taken
# against max(max|ref|, a thermal-stress floor) -- alpha E |dT| is ~1e8 Pa here.
STRESS_FLOOR = 1e6


def _stress_err(s, r):
    d = np.abs(s.reshape(-1, 7) - r.reshape(-1, 7)).max(axis=0)
    return d / np.maximum(np.abs(r.reshape(-1, 7)).max(axis=0), STRESS_FLOOR)


def test_stress(case):
    name, sess, g, u_r, _ = case
    g.solve_global(IterOptions(1e-12, 20000, "schwarz2"))
    assert _stress_err(g.recover(8), sess.recover(u_r, 8)).max() <= 1e-8, name
    assert _stress_err(g.recover(1), sess.recover(u_r, 1)).max() <= 1e-8, name
    if name != "2x2_all_dummy":
        mx, l2 = stress_errors(g.recover(8), sess.recover(u_r, 8))
        assert mx.max() <= 1e-8 and l2.max() <= 1e-8, name


def test_cutplane_ragged(case):
    name, sess, g, u_r, _ = case
    if name not in ("1x6", "5x1"):
        pytest.skip("cut plane on the ragged shapes only")
    g.set_solution(u_r)
    c = g.cutplane_von_mises(13)
    r = sess.cutplane(u_r, 13)
    assert np.abs(c - r).max() <= 1e-8 * np.abs(r).max()


# ------------------------------------------------- round-2 advisor cases
@pytest.mark.parametrize("pc", ["none", "diagonal", "block_diagonal"])
@pytest.mark.parametrize("max_it", [1, 2])
def test_no_convergence_best_is_initial_guess(oracle_libs, native_lib, pc, max_it):
    """When no iterate beats the initial residual, the reference returns
    best_x = x0 = 0 with relres 1 (linalg.cpp:316-317, 354-355); the GPU's
    best-iterate replay must not run an update in that case."""
    from test_gpu_parity import make_case
    from paper_2411_12690_b200.api import NoConvergence
    refpy, _ = oracle_libs
    sess, g = make_case(refpy, configs.get(0))
    pcn = {"none": 0, "diagonal": 1, "block_diagonal": 2}[pc]
    with pytest.raises(refpy.RefNoConvergence) as er:
        sess.iterate(1e-12, max_it, pcn)
    assert er.value.relres == 1.0 and not np.any(er.value.u)       # the reference's best is x0
    with pytest.raises(NoConvergence) as eg:
        g.solve_global(IterOptions(1e-12, max_it, pc))
    best = eg.value.best
    assert best.best_iterations == 0 and best.relative_residual == 1.0
    assert not np.any(best.u)


@pytest.mark.parametrize("q", [(5, 4, 3), (4, 5, 6), (3, 3, 5)])
def test_schwarz2_anisotropic_node_layout(oracle_libs, native_lib, q):
    """NodeLayout with different node counts per axis (config.cpp:293-295):
    the two-level Schwarz coarse space steps by s (n_x - 1) along x,
    s (n_y - 1) along y and (n_z - 1) along z."""
    from conftest import RomObj
    from paper_2411_12690_b200.api import ArrayLayout, GpuGlobalStage, ReducedOrderModel
    refpy, _ = oracle_libs
    r = refpy.build_rom(5e-6, 50e-6, 0.5e-6, 15e-6, 8, 8, q, 0)
    rows, cols = 7, 9     # the coarse lattice has s > 1 only with TSV_AS_S; the default s = 1 path
    sess = refpy.RefSession(r, None, rows, cols, bc_mode=1)
    u_r, it_r, _ = sess.iterate(1e-12, 100000)
    for s in ("1", "2", "3"):
        import os
        os.environ["TSV_AS_S"] = s
        try:
            g = GpuGlobalStage(0)
            g.set_roms(ReducedOrderModel.from_arrays(RomObj(r), 0), None)
            g.set_layout(ArrayLayout(rows, cols, None, np.array([-250.0]), 15e-6, 50e-6))
            g.set_bc("bottom_pin_321")
            assert np.array_equal(g.dof_map(), sess.dof_map())
            sol = g.solve_global(IterOptions(1e-12, 10000, "schwarz2"))
            info = g.precond_setup("schwarz2")
        finally:
            del os.environ["TSV_AS_S"]
        assert info["super_block"] == int(s)
        assert sol.relative_residual <= 1e-12
        assert rel_l2(sol.u, u_r) <= 1e-10, (q, s)
        assert sol.iterations < it_r
        g.close()
