"""K1 on the int8 tensor cores (Ozaki digit split, tcgen05.mma kind::i8):
the operator product agrees with the FP64 DMMA product to FP64 round-off,
and a full PCG on it converges to the reference's u within the parity bar."""
from __future__ import annotations

import numpy as np
import pytest

from conftest import rel_l2
from paper_2411_12690_b200 import configs
from paper_2411_12690_b200.api import IterOptions

pytestmark = pytest.mark.gpu


def _case(refpy, mixed):
    from test_gpu_parity import make_case
    cfg = configs.get(0)
    if not mixed:
        return make_case(refpy, cfg)
    rng = np.random.default_rng(13)
    kinds = (rng.random(20) < 0.3).astype(np.uint8)
    return make_case(refpy, cfg, 4, 5, kinds, -270.0 + 40.0 * rng.random(20))


@pytest.mark.parametrize("digits", [9, 10])
@pytest.mark.parametrize("mixed", [False, True])
def test_int8_operator_matches_fp64(oracle_libs, native_lib, monkeypatch, digits, mixed):
    refpy, _ = oracle_libs
    sess, g = _case(refpy, mixed)
    rng = np.random.default_rng(digits)
    n = g.index().dof_count
    xs = [rng.standard_normal(n), rng.standard_normal(n) * np.exp(rng.uniform(-20, 20, n))]
    monkeypatch.delenv("TSV_K1_OZAKI", raising=False)
    ref = [g.apply(x) for x in xs]
    monkeypatch.setenv("TSV_K1_OZAKI", str(digits))
    for x, y64 in zip(xs, ref):
        y = g.apply(x)
        assert rel_l2(y, y64) <= 1e-14
        # and against the reference's CSR operator
        assert rel_l2(y, sess.apply(x)) <= 1e-13


def test_int8_operator_solve_matches_reference(oracle_libs, native_lib, monkeypatch):
    refpy, _ = oracle_libs
    sess, g = _case(refpy, True)
    monkeypatch.setenv("TSV_K1_OZAKI", "10")
    u_r, it_r, _ = sess.iterate(1e-12)
    for pc in ("diagonal", "schwarz2"):
        sol = g.solve_global(IterOptions(1e-12, 10000, pc))
        assert sol.relative_residual <= 1e-12
        assert rel_l2(sol.u, u_r) <= 1e-10


def test_hybrid_verification_matches_fp64_check(oracle_libs, native_lib, monkeypatch):
    """Schwarz PCG with the A x of the true-residual check on int8
    (TSV_K1_VERIFY=10: the default when the irrep K1 carries the iteration,
    opt-in on the plain DMMA path) against the FP64 DMMA check: the same
    answer within the bar, two more (early-exit) launches per iteration."""
    refpy, _ = oracle_libs
    sess, g = _case(refpy, True)
    u_r, _, _ = sess.iterate(1e-12)
    monkeypatch.setenv("TSV_K1_VERIFY", "10")
    a = g.solve_global(IterOptions(1e-12, 10000, "schwarz2"))
    monkeypatch.setenv("TSV_K1_VERIFY", "0")
    b = g.solve_global(IterOptions(1e-12, 10000, "schwarz2"))
    for s in (a, b):
        assert s.relative_residual <= 1e-12 and rel_l2(s.u, u_r) <= 1e-10
    assert a.kernel_launches > b.kernel_launches  # the int8 verification kernels are in the graph
