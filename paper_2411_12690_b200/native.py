"""ctypes binding of the C ABI (include/tsv_b200.h) -> _lib/libtsv_b200.so.

There is no fallback: if the native library is missing or fails to load,
every entry point raises. The product path is the CUDA path.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("TSV_B200_LIB") or os.path.join(HERE, "_lib", "libtsv_b200.so")

TSV_OK, TSV_EINVAL, TSV_ENOCONV, TSV_EBREAKDOWN, TSV_ECUDA, TSV_ENOMEM, TSV_ESTATE = range(7)

# Every symbol include/tsv_b200.h declares (checked by tests/test_abi.py).
EXPORTS = [
    "tsv_ctx_create", "tsv_ctx_destroy", "tsv_last_error", "tsv_abi_version", "tsv_set_rom", "tsv_set_layout", "tsv_set_delta_t",
    "tsv_set_dirichlet", "tsv_set_bc", "tsv_index_global_nodes", "tsv_get_index", "tsv_get_dof_map", "tsv_get_lattice",
    "tsv_get_constrained", "tsv_get_load", "tsv_apply", "tsv_precond_apply", "tsv_precond_setup", "tsv_debug_coarse", "tsv_solve", "tsv_set_solution", "tsv_recover",
    "tsv_recover_resident", "tsv_copy_stress", "tsv_cutplane", "tsv_block_field", "tsv_profile_apply", "tsv_get_timing", "tsv_get_symmetry",
    "tsv_rom_dims", "tsv_rom_fingerprint", "tsv_rom_file_info", "tsv_build_rom", "tsv_load_rom_file", "tsv_save_rom_file", "tsv_host_register", "tsv_host_unregister", "tsv_host_alloc", "tsv_host_free", "tsv_fp64_peak",
]


class RomDesc(C.Structure):
    _fields_ = [
        ("q", C.c_uint32 * 3),
        ("geometry", C.c_double * 4),
        ("grid_len", C.c_uint32 * 3),
        ("grid", C.c_void_p * 3),
        ("materials", (C.c_double * 3) * 3),
        ("element_material", C.c_void_p),
        ("a_element", C.c_void_p),
        ("b_element", C.c_void_p),
        ("basis", C.c_void_p),
        ("thermal", C.c_void_p),
        ("fingerprint", C.c_uint8 * 32),
    ]


class IterOptionsC(C.Structure):
    _fields_ = [("tolerance", C.c_double), ("max_iterations", C.c_int), ("precond", C.c_int)]


class SolveInfo(C.Structure):
    _fields_ = [("iterations", C.c_int), ("relative_residual", C.c_double), ("direct_fallback", C.c_int),
                ("best_iterations", C.c_int), ("solve_ms", C.c_double), ("loop_ms", C.c_double), ("restarts", C.c_int),
                ("replacements", C.c_int), ("kernel_launches", C.c_uint64)]


class PrecondInfo(C.Structure):
    _fields_ = [("setup_ms", C.c_double), ("ntypes", C.c_int), ("coarse_dofs", C.c_int),
                ("super_block", C.c_int), ("local_rows", C.c_int)]


class LocalDesc(C.Structure):
    _fields_ = [("q", C.c_uint32 * 3), ("geometry", C.c_double * 4), ("grid_len", C.c_uint32 * 3),
                ("grid", C.c_void_p * 3), ("materials", (C.c_double * 3) * 3), ("kind", C.c_int)]


class RomOut(C.Structure):
    _fields_ = [("a_element", C.c_void_p), ("b_element", C.c_void_p), ("basis", C.c_void_p),
                ("thermal", C.c_void_p), ("element_material", C.c_void_p), ("fingerprint", C.c_uint8 * 32),
                ("build_ms", C.c_double)]


class Timing(C.Structure):
    _fields_ = [("solve_ms", C.c_double), ("recover_ms", C.c_double), ("apply_ms_avg", C.c_double),
                ("kernel_launches", C.c_uint64), ("stress_ms", C.c_double), ("stress_launches", C.c_int),
                ("reserved_", C.c_int)]


class SymmetryInfo(C.Structure):
    _fields_ = [("recovery_symmetric", C.c_int), ("operator_symmetric", C.c_int), ("defect_correction", C.c_int),
                ("irrep_dofs", C.c_int * 8), ("defect_k", C.c_double * 2), ("defect_phi", C.c_double * 2),
                ("operator_fused", C.c_int), ("reserved_", C.c_int)]


_lib = None


def load(path: str = LIB_PATH):
    """Load the native library (raises if it is missing: no CPU fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise RuntimeError(
            f"native library not built: {path}. Run `python -m paper_2411_12690_b200.build` "
            "(the GPU path has no CPU fallback)")
    L = C.CDLL(path)
    vp, i, u32, u64, sz, d = C.c_void_p, C.c_int, C.c_uint32, C.c_uint64, C.c_size_t, C.c_double
    P = C.POINTER
    sig = {
        "tsv_ctx_create": (i, [i, P(vp)]),
        "tsv_ctx_destroy": (None, [vp]),
        "tsv_last_error": (C.c_char_p, [vp]),
        "tsv_abi_version": (i, []),
        "tsv_set_rom": (i, [vp, i, P(RomDesc)]),
        "tsv_set_layout": (i, [vp, u32, u32, vp, vp, sz, d, d]),
        "tsv_set_delta_t": (i, [vp, vp, sz]),
        "tsv_set_dirichlet": (i, [vp, sz, vp, vp]),
        "tsv_set_bc": (i, [vp, i]),
        "tsv_index_global_nodes": (i, [u32, u32, vp, P(u64), vp, vp, vp, vp]),
        "tsv_get_index": (i, [vp, P(u64), P(u64), vp, P(u32)]),
        "tsv_get_dof_map": (i, [vp, vp]),
        "tsv_get_lattice": (i, [vp, vp, vp]),
        "tsv_get_constrained": (i, [vp, vp]),
        "tsv_get_load": (i, [vp, vp]),
        "tsv_apply": (i, [vp, vp, vp]),
        "tsv_precond_apply": (i, [vp, i, vp, vp]),
        "tsv_debug_coarse": (i, [vp, P(i), vp, vp, vp]),
        "tsv_precond_setup": (i, [vp, i, vp]),
        "tsv_solve": (i, [vp, P(IterOptionsC), vp, P(SolveInfo)]),
        "tsv_set_solution": (i, [vp, vp]),
        "tsv_recover": (i, [vp, i, u64, u64, vp]),
        "tsv_recover_resident": (i, [vp, i]),
        "tsv_copy_stress": (i, [vp, u64, u64, vp]),
        "tsv_cutplane": (i, [vp, u32, vp]),
        "tsv_block_field": (i, [vp, u64, vp]),
        "tsv_profile_apply": (i, [vp, i, P(d)]),
        "tsv_get_timing": (i, [vp, P(Timing)]),
        "tsv_get_symmetry": (i, [vp, P(SymmetryInfo)]),
        "tsv_host_register": (i, [vp, sz]),
        "tsv_host_unregister": (i, [vp]),
        "tsv_host_alloc": (i, [sz, C.POINTER(vp)]),
        "tsv_host_free": (i, [vp]),
        "tsv_fp64_peak": (i, [i, P(d), P(d)]),
        "tsv_load_rom_file": (i, [vp, i, C.c_char_p, P(i), C.c_char_p, sz]),
        "tsv_save_rom_file": (i, [P(RomDesc), i, C.c_char_p, C.c_char_p, sz]),
        "tsv_rom_fingerprint": (i, [P(LocalDesc), vp]),
        "tsv_rom_file_info": (i, [C.c_char_p, P(i), vp, C.c_char_p, sz]),
        "tsv_rom_dims": (i, [P(LocalDesc), P(u64), P(u64), P(u64)]),
        "tsv_build_rom": (i, [i, P(LocalDesc), P(RomOut), C.c_char_p, sz]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    _lib = L
    return L
