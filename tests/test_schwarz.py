"""Two-level additive Schwarz preconditioner (new option): same solution as
the reference's Jacobi-PCG within the parity bar, with far fewer iterations."""
from __future__ import annotations

import numpy as np
import pytest

from conftest import rel_l2, stress_errors
from paper_2411_12690_b200 import configs
from paper_2411_12690_b200.api import IterOptions

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("case", ["cfg0", "mixed", "cfg1"])
def test_schwarz2_matches_reference(oracle_libs, native_lib, case):
    from test_gpu_parity import make_case
    refpy, _ = oracle_libs
    cfg = configs.get(0)
    if case == "cfg0":
        sess, g = make_case(refpy, cfg)
    elif case == "cfg1":
        sess, g = make_case(refpy, configs.get(1))
    else:
        rng = np.random.default_rng(7)
        kinds = (rng.random(20) < 0.3).astype(np.uint8)
        sess, g = make_case(refpy, cfg, 4, 5, kinds, -270.0 + 40.0 * rng.random(20))
    u_r, it_r, _ = sess.iterate(1e-12)
    sol = g.solve_global(IterOptions(1e-12, 10000, "schwarz2"))
    assert sol.relative_residual <= 1e-12
    b_r, _, _ = sess.rhs()
    assert rel_l2(sess.apply(sol.u), b_r) <= 1e-11      # residual under the reference's CSR operator
    assert rel_l2(sol.u, u_r) <= 1e-10
    assert sol.iterations < it_r / 3
    mx, _ = stress_errors(g.recover(8), sess.recover(u_r, 8))
    assert mx.max() <= 1e-8
    # deterministic
    assert np.array_equal(g.solve_global(IterOptions(1e-12, 10000, "schwarz2")).u, sol.u)


@pytest.mark.parametrize("case", ["cfg0", "mixed"])
def test_tensor_core_local_solve_matches_fp64(oracle_libs, native_lib, monkeypatch, case):
    """The TF32 tcgen05 local solves (default) against the FP64 DMMA ones
    (TSV_AS_LOCAL_F64=1): M^-1 r agrees to TF32 accuracy, and both PCG runs
    converge to the same u within the parity bar."""
    from test_gpu_parity import make_case
    refpy, _ = oracle_libs
    cfg = configs.get(0)
    rng = np.random.default_rng(11)
    kinds = (rng.random(20) < 0.3).astype(np.uint8) if case == "mixed" else None
    out = {}
    monkeypatch.setenv("TSV_SMALL_PCG", "0")  # the graph path (the persistent small-array path is FP64 only)
    for mode in ("f64", "tf32"):
        if mode == "f64":
            monkeypatch.setenv("TSV_AS_LOCAL_F64", "1")
        else:
            monkeypatch.delenv("TSV_AS_LOCAL_F64", raising=False)
        if case == "mixed":
            sess, g = make_case(refpy, cfg, 4, 5, kinds, -270.0 + 40.0 * np.random.default_rng(3).random(20))
        else:
            sess, g = make_case(refpy, cfg)
        r = np.random.default_rng(5).standard_normal(g.index().dof_count)
        z = g.precond_apply(r, "schwarz2")
        sol = g.solve_global(IterOptions(1e-12, 10000, "schwarz2"))
        out[mode] = (z, sol)
        u_r, _, _ = sess.iterate(1e-12)
        assert rel_l2(sol.u, u_r) <= 1e-10
    z64, s64 = out["f64"]
    z32, s32 = out["tf32"]
    assert 0 < rel_l2(z32, z64) <= 2e-3
    assert abs(s32.iterations - s64.iterations) <= max(3, s64.iterations // 10)


def test_residual_replacement_and_compensated_x(oracle_libs, native_lib, monkeypatch):
    """The Schwarz loop's compensated x and its one mid-solve residual
    replacement (r := b - A x, direction kept) leave the answer within the bar
    of the reference, with and without them; the replacement is taken exactly
    once when the recursive residual crosses its threshold, and never with
    TSV_REPLACE_AT=0 or on the reference's preconditioners."""
    from conftest import RomObj, ref_rom
    from paper_2411_12690_b200.api import ArrayLayout, GpuGlobalStage, ReducedOrderModel
    refpy, _ = oracle_libs
    cfg = configs.get(1)
    r = ref_rom(cfg, 0, refpy)
    sess = refpy.RefSession(r, None, cfg.rows, cfg.cols, delta_t=cfg.delta_t(), bc_mode=1)
    u_ref, _, _ = sess.iterate(1e-12)
    for k in ("TSV_REPLACE_AT", "TSV_COMP_X", "TSV_VERIFY_MARGIN"):
        monkeypatch.delenv(k, raising=False)
    g = GpuGlobalStage(0)
    g.set_roms(ReducedOrderModel.from_arrays(RomObj(r), 0))
    g.set_layout(ArrayLayout(cfg.rows, cfg.cols, cfg.kinds(), cfg.delta_t(), cfg.p, cfg.h))
    g.set_bc("bottom_pin_321")
    monkeypatch.setenv("TSV_SMALL_PCG", "0")  # the graph loop (the persistent small-array kernel has no replacement)
    seen = {}
    for name, env in (("default", {}), ("early", {"TSV_REPLACE_AT": "1e-3"}), ("never", {"TSV_REPLACE_AT": "0"}),
                      ("plain_x", {"TSV_COMP_X": "0"})):
        for k in ("TSV_REPLACE_AT", "TSV_COMP_X"):
            monkeypatch.delenv(k, raising=False)
        for k, v in env.items():
            monkeypatch.setenv(k, v)
        s = g.solve_global(IterOptions(1e-12, 10000, "schwarz2"))
        assert s.relative_residual <= 1e-12 and rel_l2(s.u, u_ref) <= 1e-10, name
        seen[name] = (s.iterations, s.restarts, s.replacements)
    assert seen["default"][2] == 1 and seen["early"][2] == 1
    assert seen["never"][2] == 0 and seen["plain_x"][2] == 0
    # the replacement costs no iterations where the check passed anyway
    assert abs(seen["default"][0] - seen["never"][0]) <= 2
    for k in ("TSV_REPLACE_AT", "TSV_COMP_X"):
        monkeypatch.delenv(k, raising=False)
    sj = g.solve_global(IterOptions(1e-12, 100000, "diagonal"))
    assert sj.replacements == 0 and rel_l2(sj.u, u_ref) <= 1e-10
    g.close()
