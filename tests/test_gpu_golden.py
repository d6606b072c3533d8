"""GPU path against the committed golden fixtures of the reference
(tests/golden/*.npz, produced by the unmodified tsvstress sources)."""
from __future__ import annotations

import glob
import os

import numpy as np
import pytest

from conftest import ROOT, rel_l2, stress_errors
from paper_2411_12690_b200.api import ArrayLayout, GpuGlobalStage, IterOptions, ReducedOrderModel

pytestmark = pytest.mark.gpu
GOLDEN = sorted(glob.glob(os.path.join(ROOT, "tests", "golden", "*.npz")))
BC = {0: "bottom_pin", 1: "bottom_pin_321", 2: "clamped"}


def rom_of(z, tag, kind):
    return ReducedOrderModel(q=(int(z["mesh"][2]),) * 3, geometry=tuple(z["geometry"]),
                             grid=(z[f"{tag}_gx"], z[f"{tag}_gy"], z[f"{tag}_gz"]),
                             materials=z[f"{tag}_mats"][:, :3], a_element=z[f"{tag}_K"], b_element=z[f"{tag}_b_el"],
                             basis=z[f"{tag}_Phi"], thermal=z[f"{tag}_u_T"], element_material=z[f"{tag}_elem_mat"],
                             fingerprint=bytes(z[f"{tag}_fingerprint"]), kind=kind)


@pytest.mark.parametrize("path", GOLDEN, ids=[os.path.basename(p) for p in GOLDEN])
def test_gpu_reproduces_reference_golden(native_lib, path):
    z = np.load(path)
    g = GpuGlobalStage(0)
    g.set_roms(rom_of(z, "tsv", 0), rom_of(z, "dummy", 1) if "dummy_K" in z else None)
    kinds = z["kinds"] if z["kinds"].size else None
    d, h, t, p = z["geometry"]
    g.set_layout(ArrayLayout(int(z["rows"]), int(z["cols"]), kinds, z["delta_t"], p, h))
    g.set_bc(BC[int(z["bc_mode"])])
    assert np.array_equal(g.dof_map(), z["dof_map"])
    assert np.array_equal(g.constrained(), z["constrained"])
    assert np.array_equal(g.load(), z["load"])
    sol = g.solve_global(IterOptions(1e-12))
    d_u = sol.u - z["u"]
    if int(z["bc_mode"]) == 0:
        _, lon = g.lattice()
        q = int(z["mesh"][2])
        v = np.zeros((len(lon), 3))
        v[:, 0], v[:, 1] = -p * lon[:, 1] / (q - 1), p * lon[:, 0] / (q - 1)
        v = v.ravel()
        d_u = d_u - (d_u @ v) / (v @ v) * v
    assert np.linalg.norm(d_u) / np.linalg.norm(z["u"]) <= 1e-10
    assert abs(sol.iterations - int(z["iterations"])) <= 3
    g.set_solution(z["u"])
    mx, l2 = stress_errors(g.recover(8), z["stress"])
    assert mx.max() <= 1e-8 and l2.max() <= 1e-8
    g.close()
