"""Cut-plane von Mises output (§8(f) 1): the reference's own
cutplane_von_mises and StressGrid CSV format."""
from __future__ import annotations

import numpy as np
import pytest

from conftest import ROOT
from paper_2411_12690_b200.api import save_stress_grid_csv


def test_csv_writer_is_byte_identical_to_reference(oracle_libs, tmp_path):
    refpy, _ = oracle_libs
    rng = np.random.default_rng(3)
    rows, cols, res, pitch = 2, 3, 5, 15e-6
    vals = rng.random(rows * cols * res * res) * 1e8
    a, b = str(tmp_path / "ours.csv"), str(tmp_path / "ref.csv")
    save_stress_grid_csv(vals, rows, cols, pitch, a)
    refpy.stress_grid_save_csv(vals, rows, cols, res, pitch, b)
    assert open(a, "rb").read() == open(b, "rb").read()


@pytest.mark.gpu
@pytest.mark.parametrize("res", [100, 17])
def test_gpu_cutplane_matches_reference(oracle_libs, native_lib, res):
    from test_gpu_parity import make_case
    from paper_2411_12690_b200 import configs
    refpy, _ = oracle_libs
    cfg = configs.get(0)
    rng = np.random.default_rng(7)
    kinds = (rng.random(12) < 0.3).astype(np.uint8)
    dts = -270.0 + 40.0 * rng.random(12)
    sess, g = make_case(refpy, cfg, 3, 4, kinds, dts)
    u, _, _ = sess.iterate(1e-12)
    ref = sess.cutplane(u, res)
    g.set_solution(u)
    gpu = g.cutplane_von_mises(res)
    assert gpu.shape == ref.shape
    assert np.abs(gpu - ref).max() <= 1e-8 * np.abs(ref).max()
