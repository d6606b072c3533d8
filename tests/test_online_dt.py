"""Online dT update (tsv_set_delta_t): the reference's online stage takes a
new temperature field per call (ArrayLayout::delta_t, global.hpp:16-32);
only the thermal load (global_stage.cpp:135-142) and the recovery's
dT_b u_T term (:215-230) depend on it. The GPU keeps index, BCs and the
preconditioner and must give bit-identical results to a fresh layout."""
from __future__ import annotations

import numpy as np
import pytest

from conftest import rel_l2, stress_errors
from paper_2411_12690_b200 import configs
from paper_2411_12690_b200.api import ArrayLayout, Error, IterOptions

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("pc", ["schwarz2", "diagonal"])
def test_set_delta_t_equals_fresh_layout(oracle_libs, native_lib, pc):
    from test_gpu_parity import make_case
    refpy, _ = oracle_libs
    cfg = configs.get(0)
    rng = np.random.default_rng(21)
    kinds = (rng.random(20) < 0.3).astype(np.uint8)
    dt1 = -270.0 + 40.0 * rng.random(20)
    dt2 = -270.0 + 40.0 * rng.random(20)
    _, g = make_case(refpy, cfg, 4, 5, kinds, dt1)
    opts = IterOptions(1e-12, 10000, pc)
    g.solve_global(opts)
    g.recover(8)
    g.set_delta_t(dt2)                                   # online update
    sol = g.solve_global(opts)
    s_upd = g.recover(8)
    sess2, g2 = make_case(refpy, cfg, 4, 5, kinds, dt2)  # fresh layout with dt2
    sol2 = g2.solve_global(opts)
    assert np.array_equal(g.load(), g2.load())
    assert np.array_equal(sol.u, sol2.u) and sol.iterations == sol2.iterations
    assert np.array_equal(s_upd, g2.recover(8))
    u_r, _, _ = sess2.iterate(1e-12)
    assert rel_l2(sol.u, u_r) <= 1e-10
    mx, _ = stress_errors(s_upd, sess2.recover(u_r, 8))
    assert mx.max() <= 1e-8
    # uniform dT (one entry) through the same path
    g.set_delta_t([-250.0])
    sess3, _ = make_case(refpy, cfg, 4, 5, kinds, np.array([-250.0]))
    b3, _, _ = sess3.rhs()
    assert np.array_equal(g.load(), b3)


def test_set_delta_t_validation(oracle_libs, native_lib):
    from test_gpu_parity import make_case
    refpy, _ = oracle_libs
    _, g = make_case(refpy, configs.get(0))
    with pytest.raises(Error, match="delta_t must have one entry or rows\\*cols entries"):
        g.set_delta_t(np.zeros(5))
    from paper_2411_12690_b200.api import GpuGlobalStage
    with pytest.raises(Error, match="no layout set"):
        GpuGlobalStage(0).set_delta_t([-250.0])
