"""tsvstress_b200 (paper_2411_12690_b200/_lib): the reference's `local` and
`solve` commands (cli.cpp:62-113) over the C ABI, reading the reference's run
configuration format (config.cpp) and writing .rom files, the StressGrid CSV
and the JSON-lines run log.

CPU: the configuration reader (defaults, validation messages, the
default_grading restatement and the ROM fingerprint, pinned against the
reference library) and the fingerprint check against ROM files.
GPU: `local` + `solve` end to end; the CSV against the reference's own
pipeline (load_rom of the written files, solve_global, cutplane_von_mises,
StressGrid::save_csv) on the same config."""
from __future__ import annotations

import json
import os
import subprocess

import numpy as np
import pytest

from conftest import ROOT

CLI = os.path.join(ROOT, "paper_2411_12690_b200", "_lib", "tsvstress_b200")

DEMO = """# 2x3 array, mixed kinds, per-cell dT (the reference's demo_4x4.conf keys)
geometry.d = 5e-6
geometry.h = 50e-6
geometry.t = 0.5e-6
geometry.p = 15e-6
grid.target = 3e-6
grid.res = 9
layout.rows = 2
layout.cols = 3
layout.kinds = tdt;dtt
layout.delta_t = -250, -240, -230; -220, -210, -200
interpolation.nx = 4
interpolation.ny = 4
interpolation.nz = 4
bc.type = clamped
solver.tolerance = 1e-12
solver.max_iterations = 10000
solver.precond = diagonal
threads = 2
rom.tsv = tsv.rom
rom.dummy = dummy.rom
output.grid_csv = stress_grid.csv
output.run_log = run_log.jsonl
"""


def run(args, cwd):
    return subprocess.run([CLI, *args], cwd=cwd, capture_output=True, text=True, timeout=900)


@pytest.fixture
def demo(tmp_path, native_lib):
    (tmp_path / "demo.conf").write_text(DEMO)
    return tmp_path


def test_default_grading_and_fingerprint_match_reference(demo, oracle_libs):
    refpy, _ = oracle_libs
    out = run(["grid", "--config", "demo.conf"], demo)
    assert out.returncode == 0, out.stderr
    lines = out.stdout.strip().splitlines()
    ours = [np.array([float(v) for v in lines[a].split()[1:]]) for a in range(3)]
    ref, fp = refpy.default_grading(5e-6, 50e-6, 0.5e-6, 15e-6, 3e-6, 4)
    for a in range(3):
        assert np.array_equal(ours[a], ref[a])  # bit-exact grid lines
    assert lines[3] == "fingerprint " + fp.hex()


@pytest.mark.parametrize("edit,message", [
    ("bogus.key = 1", "config: bogus.key: unknown key"),
    ("layout.kinds = tdx;dtt", "unknown cell kind 'x'"),
    ("layout.delta_t = 1, 2; 3", "each row needs 3 values"),
    ("solver.precond = jacobi", "'jacobi' is not one of none|diagonal|block|schwarz2"),
    ("grid.res = 0", "config: grid.res: must lie in [1, 4096]"),
    ("geometry.p = 5e-6", "config: geometry.p: pitch must exceed d + 2t"),
    ("bc.type = submodel", "submodel boundary fields are outside the GPU online stage"),
])
def test_config_validation(demo, edit, message):
    (demo / "demo.conf").write_text(DEMO + edit + "\n")
    out = run(["solve", "--config", "demo.conf"], demo)
    assert out.returncode == 1 and message in out.stderr, out.stderr


def test_rom_fingerprint_mismatch_is_rejected(demo):
    """A valid .rom of another configuration (here a 1-cell grid, q = 2)."""
    from paper_2411_12690_b200.api import ReducedOrderModel, save_rom
    n, nf = 24, 24
    grid = (np.array([0.0, 15e-6]), np.array([0.0, 15e-6]), np.array([0.0, 50e-6]))
    mats = np.array([[110e9, 0.35, 17e-6], [71e9, 0.16, 0.5e-6], [130e9, 0.28, 2.8e-6]])
    rom = ReducedOrderModel(q=(2, 2, 2), geometry=(5e-6, 50e-6, 0.5e-6, 15e-6), grid=grid, materials=mats,
                            a_element=np.eye(n), b_element=np.zeros(n), basis=np.zeros((nf, n)), thermal=np.zeros(nf),
                            element_material=np.zeros(1, np.uint8), fingerprint=b"", kind=0)
    save_rom(rom, str(demo / "tsv.rom"))
    save_rom(rom, str(demo / "dummy.rom"))
    out = run(["solve", "--config", "demo.conf"], demo)
    assert out.returncode == 1 and "was built for a different configuration" in out.stderr, out.stderr


def test_missing_rom_file(demo):
    out = run(["solve", "--config", "demo.conf"], demo)
    assert out.returncode == 1 and "tsv.rom" in out.stderr


@pytest.mark.gpu
def test_local_then_solve_matches_reference_pipeline(demo, oracle_libs):
    refpy, _ = oracle_libs
    out = run(["local", "--config", "demo.conf"], demo)
    assert out.returncode == 0, out.stderr
    assert "wrote tsv.rom" in out.stdout and "wrote dummy.rom" in out.stdout
    out = run(["solve", "--config", "demo.conf", "--out", "gpu.csv"], demo)
    assert out.returncode == 0, out.stderr
    assert "reduced dofs = " in out.stdout and "wrote gpu.csv" in out.stdout
    log = [json.loads(l) for l in (demo / "run_log.jsonl").read_text().splitlines()]
    assert [e["command"] for e in log] == ["local", "solve"]
    assert set(log[1]) == {"command", "wall_s", "peak_mem_bytes", "dofs", "iterations"} and log[1]["iterations"] > 0
    # the reference pipeline on the files `local` wrote
    r_tsv = refpy.load_rom(str(demo / "tsv.rom"))
    r_dum = refpy.load_rom(str(demo / "dummy.rom"))
    kinds = np.array([0, 1, 0, 1, 0, 0], np.uint8)
    dts = np.array([-250, -240, -230, -220, -210, -200], np.float64)
    sess = refpy.RefSession(r_tsv, r_dum, 2, 3, kinds=kinds, delta_t=dts, bc_mode=2)
    u, _, _ = sess.iterate(1e-12)
    grid = sess.cutplane(u, 9)
    refpy.stress_grid_save_csv(grid, 2, 3, 9, 15e-6, str(demo / "ref.csv"))
    a = (demo / "gpu.csv").read_text().splitlines()
    b = (demo / "ref.csv").read_text().splitlines()
    assert a[0] == b[0] and len(a) == len(b)
    ga = np.array([[float(v) for v in l.split(",")] for l in a[1:]])
    gb = np.array([[float(v) for v in l.split(",")] for l in b[1:]])
    assert np.array_equal(ga[:, :6], gb[:, :6])  # indices and coordinates bit-exact
    assert np.abs(ga[:, 6] - gb[:, 6]).max() <= 1e-8 * np.abs(gb[:, 6]).max()
    # the Schwarz preconditioner through the CLI gives the same grid
    out = run(["solve", "--config", "demo.conf", "--out", "gpu_s2.csv", "--precond", "schwarz2"], demo)
    assert out.returncode == 0, out.stderr
    gs = np.array([[float(v) for v in l.split(",")] for l in (demo / "gpu_s2.csv").read_text().splitlines()[1:]])
    assert np.abs(gs[:, 6] - gb[:, 6]).max() <= 1e-8 * np.abs(gb[:, 6]).max()
