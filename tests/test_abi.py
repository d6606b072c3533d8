"""The C-ABI library loads without a GPU and exports every symbol the
public header declares; the product path refuses to run without it."""
from __future__ import annotations

import ctypes
import os
import re

from conftest import ROOT


def declared_symbols():
    hdr = open(os.path.join(ROOT, "include", "tsv_b200.h")).read()
    hdr = re.sub(r"/\*.*?\*/", "", hdr, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:int|void|const char \*)\s*(tsv_\w+)\s*\(", hdr, flags=re.M)))


def test_header_declares_expected_api():
    from paper_2411_12690_b200 import native
    assert set(declared_symbols()) == set(native.EXPORTS)


def test_library_exports_every_declared_symbol(native_lib):
    lib = ctypes.CDLL(os.path.join(ROOT, "paper_2411_12690_b200", "_lib", "libtsv_b200.so"))
    for name in declared_symbols():
        assert hasattr(lib, name), name
    assert lib.tsv_abi_version() == 1


def test_library_is_sm100a_only(native_lib):
    import subprocess
    so = os.path.join(ROOT, "paper_2411_12690_b200", "_lib", "libtsv_b200.so")
    out = subprocess.run(["cuobjdump", "--list-elf", so], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert not re.search(r"sm_(?!100a)\d+", out)


def test_dmma_in_gemm_sass(native_lib):
    """FP64 tensor-core path: the K1/K6 kernel must contain DMMA."""
    import subprocess
    so = os.path.join(ROOT, "paper_2411_12690_b200", "_lib", "libtsv_b200.so")
    sass = subprocess.run(["cuobjdump", "-sass", so], capture_output=True, text=True).stdout
    assert "DMMA.8x8x4" in sass


def test_missing_library_fails_loudly(tmp_path):
    import pytest
    from paper_2411_12690_b200 import native
    saved = native._lib
    native._lib = None
    try:
        with pytest.raises(RuntimeError, match="not built"):
            native.load(str(tmp_path / "nope.so"))
    finally:
        native._lib = saved
