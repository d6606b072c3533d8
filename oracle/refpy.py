"""ORACLE TEST INFRASTRUCTURE — ctypes binding of oracle/_ref/libtsvref.so.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs may import this module. It drives the reference's
own C++ sources (compiled unmodified from /root/reference/proj/src by
oracle/Makefile) through oracle/ref_shim.cpp.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_ref", "libtsvref.so")

_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"reference oracle not built: {LIB_PATH} (run `make -C oracle ref`)")
        L = C.CDLL(LIB_PATH)
        vp, d, i, u32, u64, i64 = C.c_void_p, C.c_double, C.c_int, C.c_uint32, C.c_uint64, C.c_int64
        P = C.POINTER
        L.ref_last_error.restype = C.c_char_p
        L.ref_rom_build.restype = vp
        L.ref_rom_build.argtypes = [d, d, d, d, i, i, i, i, d, i]
        L.ref_rom_build3.restype = vp
        L.ref_rom_build3.argtypes = [d, d, d, d, i, i, i, i, i, i, d, i]
        L.ref_rom_load.restype = vp
        L.ref_rom_load.argtypes = [C.c_char_p]
        L.ref_rom_save.argtypes = [vp, C.c_char_p]
        L.ref_rom_free.argtypes = [vp]
        L.ref_rom_dims.argtypes = [vp, P(i64)]
        L.ref_rom_copy.argtypes = [vp] + [vp] * 11
        L.ref_session_create.restype = vp
        L.ref_session_create.argtypes = [vp, vp, u32, u32, vp, vp, u64, d, d, i]
        L.ref_session_free.argtypes = [vp]
        L.ref_session_info.argtypes = [vp, P(i64), vp]
        L.ref_session_dof_map.argtypes = [vp, vp]
        L.ref_session_lattice.argtypes = [vp, vp, vp]
        L.ref_session_rhs.argtypes = [vp, vp, vp, vp]
        L.ref_session_apply.argtypes = [vp, vp, vp, i]
        L.ref_session_solve.argtypes = [vp, d, i, i, i, vp, P(i), P(d), P(i), P(d)]
        L.ref_session_iterate.argtypes = [vp, d, i, i, i, vp, P(i), P(d)]
        L.ref_session_recover.argtypes = [vp, vp, i, u64, u64, vp, i]
        L.ref_session_cutplane.argtypes = [vp, vp, u32, vp, i]
        L.ref_session_block_field.argtypes = [vp, vp, u64, vp]
        _lib = L
    return _lib


def _ptr(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


class RefError(RuntimeError):
    pass


class RefNoConvergence(RefError):
    def __init__(self, msg, u, iterations, relres):
        super().__init__(msg)
        self.u, self.iterations, self.relres = u, iterations, relres


def _err():
    return lib().ref_last_error().decode()


@dataclass
class RefRom:
    """A reference ReducedOrderModel (rom.hpp:57-72) plus the arrays the
    GPU context needs, copied out once."""
    handle: int
    n: int
    n_fine: int
    n_elem: int
    cells: tuple
    q: tuple
    kind: int
    K: np.ndarray = field(repr=False)
    b_el: np.ndarray = field(repr=False)
    Phi: np.ndarray = field(repr=False)
    u_T: np.ndarray = field(repr=False)
    gx: np.ndarray = field(repr=False)
    gy: np.ndarray = field(repr=False)
    gz: np.ndarray = field(repr=False)
    elem_mat: np.ndarray = field(repr=False)
    mats: np.ndarray = field(repr=False)   # [3,5] E, nu, alpha, lambda, mu
    geom: np.ndarray = field(repr=False)   # d, h, t, p
    fingerprint: bytes = b""

    def __del__(self):
        if self.handle and _lib is not None:
            _lib.ref_rom_free(self.handle)
            self.handle = 0

    def save(self, path):
        if lib().ref_rom_save(self.handle, path.encode()) != 0:
            raise RefError(_err())


def _wrap_rom(h):
    if not h:
        raise RefError(_err())
    dims = (C.c_int64 * 10)()
    lib().ref_rom_dims(h, dims)
    n, nf, ne, cx, cy, cz, qx, qy, qz, kind = [int(v) for v in dims]
    K = np.empty((n, n)); b = np.empty(n); Phi = np.empty((nf, n)); uT = np.empty(nf)
    gx = np.empty(cx + 1); gy = np.empty(cy + 1); gz = np.empty(cz + 1)
    em = np.empty(ne, np.uint8); mats = np.empty((3, 5)); geom = np.empty(4); fp = np.empty(32, np.uint8)
    st = lib().ref_rom_copy(h, _ptr(K), _ptr(b), _ptr(Phi), _ptr(uT), _ptr(gx), _ptr(gy), _ptr(gz),
                            _ptr(em), _ptr(mats), _ptr(geom), _ptr(fp))
    if st != 0:
        raise RefError(_err())
    return RefRom(h, n, nf, ne, (cx, cy, cz), (qx, qy, qz), kind, K, b, Phi, uT, gx, gy, gz, em, mats,
                  geom, bytes(fp))


def build_rom(d, h, t, p, m_xy, m_z, q, kind=0, liner_e=71.7e9, threads=0):
    """rom::build_rom (rom.cpp:134-253) on a uniform grid."""
    if threads <= 0:
        threads = os.cpu_count() or 1
    if not np.isscalar(q):  # NodeLayout (n_x, n_y, n_z)
        return _wrap_rom(lib().ref_rom_build3(d, h, t, p, m_xy, m_z, *[int(v) for v in q], kind, liner_e, threads))
    return _wrap_rom(lib().ref_rom_build(d, h, t, p, m_xy, m_z, q, kind, liner_e, threads))


def load_rom(path):
    return _wrap_rom(lib().ref_rom_load(path.encode()))


class RefSession:
    """index_global_nodes -> assemble_global -> lifting on the reference."""

    def __init__(self, tsv: RefRom | None, dummy: RefRom | None, rows, cols, kinds=None, delta_t=(-250.0,),
                 pitch=None, height=None, bc_mode=1):
        any_rom = tsv or dummy
        self.rom_tsv, self.rom_dummy = tsv, dummy
        self.rows, self.cols = rows, cols
        self.kinds = None if kinds is None else np.ascontiguousarray(kinds, np.uint8)
        self.delta_t = np.ascontiguousarray(delta_t, np.float64)
        pitch = any_rom.geom[3] if pitch is None else pitch
        height = any_rom.geom[1] if height is None else height
        self.h = lib().ref_session_create(tsv.handle if tsv else None, dummy.handle if dummy else None,
                                          rows, cols, _ptr(self.kinds), _ptr(self.delta_t),
                                          len(self.delta_t), pitch, height, bc_mode)
        if not self.h:
            raise RefError(_err())
        info = (C.c_int64 * 8)()
        tm = np.zeros(3)
        lib().ref_session_info(self.h, info, _ptr(tm))
        (self.N, self.nnz, self.lat_x, self.lat_y, self.lat_z, self.node_count, self.n,
         self.n_constrained) = [int(v) for v in info]
        self.timings = {"index": tm[0], "assemble": tm[1], "lift": tm[2]}

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.ref_session_free(self.h)
            self.h = None

    @property
    def B(self):
        return self.rows * self.cols

    def dof_map(self):
        out = np.empty((self.B, self.n), np.uint32)
        lib().ref_session_dof_map(self.h, _ptr(out))
        return out

    def lattice(self):
        nol = np.empty(self.lat_x * self.lat_y * self.lat_z, np.int32)
        lon = np.empty((self.node_count, 3), np.uint32)
        lib().ref_session_lattice(self.h, _ptr(nol), _ptr(lon))
        return nol, lon

    def rhs(self):
        b = np.empty(self.N); cm = np.zeros(self.N, np.uint8); vals = np.zeros(self.N)
        lib().ref_session_rhs(self.h, _ptr(b), _ptr(cm), _ptr(vals))
        return b, cm, vals

    def apply(self, x, threads=0):
        x = np.ascontiguousarray(x, np.float64)
        y = np.empty(self.N)
        if lib().ref_session_apply(self.h, _ptr(x), _ptr(y), threads or (os.cpu_count() or 1)) != 0:
            raise RefError(_err())
        return y

    def solve(self, tol=1e-12, max_it=10000, precond=1, threads=0):
        """solve_global (global_stage.cpp:187-205) incl. its LDLT fallback."""
        u = np.empty(self.N); it = C.c_int(); rr = C.c_double(); fb = C.c_int(); wall = C.c_double()
        st = lib().ref_session_solve(self.h, tol, max_it, precond, threads or (os.cpu_count() or 1), _ptr(u),
                                     C.byref(it), C.byref(rr), C.byref(fb), C.byref(wall))
        if st != 0:
            raise RefError(_err())
        return u, it.value, rr.value, bool(fb.value), wall.value

    def iterate(self, tol=1e-12, max_it=10000, precond=1, threads=0):
        """linalg::iterative_solve (CG, no direct fallback)."""
        u = np.empty(self.N); it = C.c_int(); rr = C.c_double()
        st = lib().ref_session_iterate(self.h, tol, max_it, precond, threads or (os.cpu_count() or 1), _ptr(u),
                                       C.byref(it), C.byref(rr))
        if st == 2:
            raise RefNoConvergence(_err(), u, it.value, rr.value)
        if st != 0:
            raise RefError(_err())
        return u, it.value, rr.value

    def recover(self, u, points=8, cell_begin=0, cell_end=None, threads=0):
        cell_end = self.B if cell_end is None else cell_end
        rom = self.rom_tsv or self.rom_dummy
        out = np.empty((cell_end - cell_begin, rom.n_elem, points, 7))
        u = np.ascontiguousarray(u, np.float64)
        st = lib().ref_session_recover(self.h, _ptr(u), points, cell_begin, cell_end, _ptr(out),
                                       threads or (os.cpu_count() or 1))
        if st != 0:
            raise RefError(_err())
        return out

    def cutplane(self, u, res=100, threads=0):
        out = np.empty((self.B, res, res))
        u = np.ascontiguousarray(u, np.float64)
        if lib().ref_session_cutplane(self.h, _ptr(u), res, _ptr(out), threads or (os.cpu_count() or 1)) != 0:
            raise RefError(_err())
        return out

    def block_field(self, u, cell):
        rom = self.rom_tsv or self.rom_dummy
        out = np.empty(rom.n_fine)
        u = np.ascontiguousarray(u, np.float64)
        if lib().ref_session_block_field(self.h, _ptr(u), cell, _ptr(out)) != 0:
            raise RefError(_err())
        return out


def index_dof_map(rows, cols, q):
    """The reference's index_global_nodes / global_dof (no assembly)."""
    L = lib()
    L.ref_index.restype = C.c_int64
    L.ref_index.argtypes = [C.c_uint32, C.c_uint32, C.c_uint32, C.c_void_p]
    nd = L.ref_index(rows, cols, q, None)
    if nd < 0:
        raise RefError(_err())
    n = 3 * (q ** 3 - (q - 2) ** 3)
    out = np.empty((rows * cols, n), np.uint32)
    L.ref_index(rows, cols, q, _ptr(out))
    return nd, out


def stress_grid_save_csv(values, rows, cols, res, pitch, path):
    """The reference's StressGrid::save_csv on given values."""
    L = lib()
    L.ref_stress_grid_save_csv.argtypes = [C.c_void_p, C.c_uint32, C.c_uint32, C.c_uint32, C.c_double, C.c_char_p]
    v = np.ascontiguousarray(values, np.float64)
    if L.ref_stress_grid_save_csv(_ptr(v), rows, cols, res, pitch, path.encode()) != 0:
        raise RefError(_err())


def default_grading(d, h, t, p, target, q=4):
    """The reference's default_grading + rom_fingerprint (default materials)."""
    L = lib()
    L.ref_default_grading.argtypes = [C.c_double] * 5 + [C.c_uint32, C.c_uint32] + [C.c_void_p] * 5
    cap = 4096
    axes = [np.empty(cap) for _ in range(3)]
    ln = np.zeros(3, np.uint32)
    fp = np.zeros(32, np.uint8)
    if L.ref_default_grading(d, h, t, p, target, q, cap, *(_ptr(a) for a in axes), _ptr(ln), _ptr(fp)) != 0:
        raise RefError(_err())
    return [axes[a][:ln[a]].copy() for a in range(3)], bytes(fp)
