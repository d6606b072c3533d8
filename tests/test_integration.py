"""The drop-in: the reference's own online-stage objects (RomSet,
ArrayLayout, DirichletSet, IterOptions from /root/reference/proj/include)
handed to the GPU stage through include/tsvstress_b200/global_gpu.hpp
(oracle/integration_demo.cpp, built against the reference headers)."""
from __future__ import annotations

import json
import os
import subprocess

import pytest

from conftest import ROOT

DEMO = os.path.join(ROOT, "oracle", "_ref", "integration_demo")


def test_cpp_header_compiles_standalone(tmp_path):
    src = tmp_path / "t.cpp"
    src.write_text('#include "tsvstress_b200/global_gpu.hpp"\nint main() { return 0; }\n')
    subprocess.run(["g++", "-std=c++17", "-fsyntax-only", "-I", os.path.join(ROOT, "include"), str(src)], check=True)


@pytest.mark.gpu
def test_reference_objects_drive_the_gpu_stage(oracle_libs, native_lib):
    if not os.path.exists(DEMO):
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "integration"], check=True)
    out = subprocess.run([DEMO], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stdout + out.stderr
    r = json.loads(out.stdout.strip().splitlines()[-1])
    assert r["du_rel_l2"] <= 1e-10 and r["vm_rel_err"] <= 1e-8
    assert r["cutplane_rel_err"] <= 1e-8                       # GPU cut plane vs cutplane_von_mises
    assert r["du_rel_l2_schwarz2"] <= 1e-10                    # two-level Schwarz through the C++ layer
    assert r["iterations_schwarz2"] < r["iterations_ref"]
