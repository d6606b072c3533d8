"""The default B200 code paths against their simpler variants, on the same
inputs (GPU):

- K6 split (dense DMMA GEMM over the interior basis rows, (face, component)
  GEMMs over the surface rows) vs one dense GEMM (TSV_K6_DENSE) and vs the
  CSR surface path (TSV_K6_CSR): the same recovered stress to rounding;
- the symmetric packed-tile coarse solve of the Schwarz preconditioner vs the
  dense FP32 GEMV (TSV_AS_COARSE_DENSE) and the FP64 one (TSV_AS_COARSE_F64):
  M r agrees to FP32 rounding, and the PCG converges to the same u;
- the split z = z_l + P z_c (tsv_precond_apply returns the assembled z):
  M is symmetric to TF32 rounding, r1.(M r2) = r2.(M r1).
"""
from __future__ import annotations

import numpy as np
import pytest

from conftest import rel_l2, stress_errors
from paper_2411_12690_b200 import configs
from paper_2411_12690_b200.api import IterOptions

pytestmark = pytest.mark.gpu


def _mixed(refpy):
    from test_gpu_parity import make_case
    rng = np.random.default_rng(5)
    kinds = (rng.random(20) < 0.3).astype(np.uint8)
    return make_case(refpy, configs.get(0), 4, 5, kinds, -270.0 + 40.0 * rng.random(20))


@pytest.mark.parametrize("variant", ["TSV_K6_DENSE", "TSV_K6_CSR"])
def test_k6_split_matches_dense(oracle_libs, native_lib, monkeypatch, variant):
    refpy, _ = oracle_libs
    out = {}
    for mode in ("default", variant):
        monkeypatch.delenv("TSV_K6_DENSE", raising=False)
        monkeypatch.delenv("TSV_K6_CSR", raising=False)
        if mode != "default":
            monkeypatch.setenv(mode, "1")
        sess, g = _mixed(refpy)  # the split is decided when the ROM is set
        sol = g.solve_global(IterOptions(1e-12, 10000, "diagonal"))
        out[mode] = (sol.u, g.recover(8), g.block_field(7))
        g.close()
    u0, s0, f0 = out["default"]
    u1, s1, f1 = out[variant]
    assert np.array_equal(u0, u1)  # the solve does not depend on the recovery path
    mx, l2 = stress_errors(s0, s1)
    assert mx.max() <= 1e-12 and l2.max() <= 1e-12
    assert rel_l2(f0, f1) <= 1e-13


@pytest.mark.parametrize("variant", ["TSV_AS_COARSE_DENSE", "TSV_AS_COARSE_F64"])
def test_symmetric_coarse_matches_dense(oracle_libs, native_lib, monkeypatch, variant):
    refpy, _ = oracle_libs
    r = np.random.default_rng(2)
    res = {}
    for mode in ("default", variant):
        monkeypatch.delenv("TSV_AS_COARSE_DENSE", raising=False)
        monkeypatch.delenv("TSV_AS_COARSE_F64", raising=False)
        if mode != "default":
            monkeypatch.setenv(mode, "1")
        sess, g = _mixed(refpy)
        n = g.index().dof_count
        rv = r.standard_normal(n) if mode == "default" else res["default"][0]
        z = g.precond_apply(rv)
        sol = g.solve_global(IterOptions(1e-12, 10000, "schwarz2"))
        res[mode] = (rv, z, sol.u)
        g.close()
    _, z0, u0 = res["default"]
    _, z1, u1 = res[variant]
    assert rel_l2(z0, z1) <= 1e-5  # FP32 inverse storage, different summation order
    assert rel_l2(u0, u1) <= 1e-10


def test_schwarz_preconditioner_is_symmetric(oracle_libs, native_lib):
    refpy, _ = oracle_libs
    sess, g = _mixed(refpy)
    n = g.index().dof_count
    rng = np.random.default_rng(9)
    r1, r2 = rng.standard_normal(n), rng.standard_normal(n)
    a = r1 @ g.precond_apply(r2)
    b = r2 @ g.precond_apply(r1)
    assert abs(a - b) <= 1e-3 * max(abs(a), abs(b))  # TF32 operands of the local solves
    # positive definite on these samples
    assert r1 @ g.precond_apply(r1) > 0 and r2 @ g.precond_apply(r2) > 0
    g.close()


def test_nonzero_dirichlet_lifting_rigid_translation(oracle_libs, native_lib):
    """Non-zero prescribed values (b_f -= A_fc g, b_c = g; fem.cpp:223-260):
    lifting every constrained u_z of the 3-2-1 set by delta is a rigid
    translation, so u = u_0 + delta e_z and the stress is unchanged."""
    refpy, _ = oracle_libs
    sess, g = _mixed(refpy)
    u0 = g.solve_global(IterOptions(1e-12, 10000, "schwarz2")).u
    s0 = g.recover(8)
    mask = g.constrained().astype(bool)
    dofs = np.nonzero(mask)[0].astype(np.uint32)
    delta = 1e-7
    vals = np.where(dofs % 3 == 2, delta, 0.0)
    g.set_dirichlet(dofs, vals)
    u1 = g.solve_global(IterOptions(1e-12, 10000, "schwarz2")).u
    shift = np.zeros_like(u0)
    shift[2::3] = delta
    assert rel_l2(u1, u0 + shift) <= 1e-9
    assert np.abs(u1[dofs] - vals).max() <= 1e-10 * np.abs(u1).max()  # u_c = g
    mx, _ = stress_errors(g.recover(8), s0)
    assert mx.max() <= 1e-7
    g.close()


def test_programmatic_dependent_launch_is_bitwise_neutral(oracle_libs, native_lib, monkeypatch):
    """PDL only changes when CTAs are scheduled, never what they compute:
    the Schwarz solve is bitwise identical with TSV_NO_PDL=1."""
    refpy, _ = oracle_libs
    out = []
    for flag in (None, "1"):
        if flag:
            monkeypatch.setenv("TSV_NO_PDL", flag)
        else:
            monkeypatch.delenv("TSV_NO_PDL", raising=False)
        sess, g = _mixed(refpy)
        sol = g.solve_global(IterOptions(1e-12, 10000, "schwarz2"))
        out.append((sol.u, sol.iterations))
        g.close()
    assert out[0][1] == out[1][1]
    assert np.array_equal(out[0][0], out[1][0])


def test_recover_into_pinned_host_memory(oracle_libs, native_lib):
    """tsv_host_alloc result buffers (the bench e2e path) receive the same
    stress as a pageable numpy array, across the double-buffered D2H."""
    import ctypes as C
    from paper_2411_12690_b200.api import PinnedArray
    refpy, _ = oracle_libs
    sess, g = _mixed(refpy)
    g.solve_global(IterOptions(1e-12, 10000, "schwarz2"))
    s_np = g.recover(8)
    pin = PinnedArray(s_np.shape)
    rc = g._L.tsv_recover(g._h, 8, 0, s_np.shape[0], pin.array.ctypes.data_as(C.c_void_p))
    assert rc == 0
    assert np.array_equal(pin.array, s_np)
    pin.close()
    g.close()
