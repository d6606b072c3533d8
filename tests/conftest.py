"""Shared fixtures. `-m "not gpu"` runs the oracle/host/ABI checks on CPU;
`-m gpu` runs the parity tests through the C ABI on a B200.

ROMs (the local-stage output, an INPUT of the hot path) come from the
reference's own build_rom (oracle/_ref, compiled from the unmodified
sources) and are cached under ~/.cache/tsv_b200_roms/ in the reference's MRST format.
"""
from __future__ import annotations

import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
CACHE = os.environ.get("TSV_ROM_CACHE", os.path.join(os.path.expanduser("~"), ".cache", "tsv_b200_roms"))  # outside the repo: not shipped to the GPU box


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200); runs through the C ABI")
    config.addinivalue_line("markers", "slow: long-running (large configs)")


def _have_gpu():
    try:
        import ctypes
        cudart = ctypes.CDLL("libcuda.so.1")
        n = ctypes.c_int()
        return cudart.cuInit(0) == 0 and cudart.cuDeviceGetCount(ctypes.byref(n)) == 0 and n.value > 0
    except OSError:
        return False


HAVE_GPU = _have_gpu()


def pytest_collection_modifyitems(config, items):
    if HAVE_GPU:
        return
    skip = pytest.mark.skip(reason="no CUDA GPU in this container")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)


def _make_oracle():
    need = [os.path.join(ROOT, "oracle", "_ref", "libtsvref.so"), os.path.join(ROOT, "oracle", "_build", "libtsvoracle.so")]
    if all(os.path.exists(p) for p in need) and not os.path.isdir("/root/reference"):
        return  # GPU box: prebuilt oracle travelled with the snapshot
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "-j8"], check=True,
                   stdout=subprocess.DEVNULL)


@pytest.fixture(scope="session")
def oracle_libs():
    _make_oracle()
    from oracle import orcpy, refpy
    return refpy, orcpy


@pytest.fixture(scope="session")
def native_lib():
    from paper_2411_12690_b200 import build, native
    if os.path.isdir(os.path.join(ROOT, "paper_2411_12690_b200", "csrc")) and os.environ.get("TSV_NO_BUILD") != "1":
        try:
            build.build()
        except (RuntimeError, FileNotFoundError, subprocess.CalledProcessError):
            pass  # GPU box without nvcc on PATH: use the travelled .so
    return native.load()


def ref_rom(cfg, kind, refpy):
    """Reference build_rom output for a config (cached .rom)."""
    os.makedirs(CACHE, exist_ok=True)
    path = os.path.join(CACHE, f"{cfg.name}_{'tsv' if kind == 0 else 'dummy'}.rom")
    if os.path.exists(path):
        return refpy.load_rom(path)
    r = refpy.build_rom(cfg.d, cfg.h, cfg.t, cfg.p, cfg.m_xy, cfg.m_z, cfg.q, kind, cfg.liner_e)
    r.save(path + ".tmp")
    os.replace(path + ".tmp", path)
    return r


class RomObj:
    """Attribute view used by the oracle (K, b_el, Phi, ...) over a RefRom."""

    def __init__(self, r):
        self.__dict__.update(dict(K=r.K, b_el=r.b_el, Phi=r.Phi, u_T=r.u_T, gx=r.gx, gy=r.gy, gz=r.gz,
                                  elem_mat=r.elem_mat, mats=r.mats, geom=r.geom, q=r.q,
                                  fingerprint=r.fingerprint, kind=r.kind))


def rel_l2(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)


def stress_errors(s_gpu, s_ref):
    """Per component (xx..zx, vm): max|d| / max|ref| and the L2 analogue."""
    g = s_gpu.reshape(-1, 7)
    r = s_ref.reshape(-1, 7)
    d = g - r
    mx = np.abs(d).max(axis=0) / np.maximum(np.abs(r).max(axis=0), 1e-300)
    l2 = np.linalg.norm(d, axis=0) / np.maximum(np.linalg.norm(r, axis=0), 1e-300)
    return mx, l2
