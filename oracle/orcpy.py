"""ORACLE TEST INFRASTRUCTURE — ctypes binding of the C restatement
(oracle/tsv_oracle.c -> oracle/_build/libtsvoracle.so).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
import this module. ``OracleSystem`` takes the same ROM arrays the GPU path
receives and restates index_global_nodes / assemble_global + lifting /
cg_solve / recovery of the reference matrix-free (see tsv_oracle.h).
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_build", "libtsvoracle.so")
_lib = None

MAX_KINDS = 2


class _System(C.Structure):
    _fields_ = [("B", C.c_size_t), ("n", C.c_size_t), ("N", C.c_size_t),
                ("dof_map", C.c_void_p), ("kinds", C.c_void_p), ("delta_t", C.c_void_p),
                ("K", C.c_void_p * 2), ("b_el", C.c_void_p * 2), ("constrained", C.c_void_p),
                ("g", C.c_void_p), ("threads", C.c_int)]


class _Recovery(C.Structure):
    _fields_ = [("n_fine", C.c_size_t), ("cx", C.c_uint32), ("cy", C.c_uint32), ("cz", C.c_uint32),
                ("gx", C.c_void_p * 2), ("gy", C.c_void_p * 2), ("gz", C.c_void_p * 2),
                ("Phi", C.c_void_p * 2), ("u_T", C.c_void_p * 2), ("elem_mat", C.c_void_p * 2),
                ("lame", C.c_double * 18)]


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"C oracle not built: {LIB_PATH} (run `make -C oracle`)")
        L = C.CDLL(LIB_PATH)
        vp, sz, u32 = C.c_void_p, C.c_size_t, C.c_uint32
        L.orc_surface_nodes.restype = sz
        L.orc_surface_nodes.argtypes = [u32, u32, u32, vp]
        L.orc_index_global_nodes.restype = sz
        L.orc_index_global_nodes.argtypes = [u32, u32, u32, u32, u32, vp, vp]
        L.orc_dof_map.argtypes = [u32, u32, u32, u32, u32, vp, vp]
        L.orc_bc_mask.restype = sz
        L.orc_bc_mask.argtypes = [C.c_int, sz, vp, u32, u32, vp]
        L.orc_apply.argtypes = [vp, u32, u32, vp, vp]
        L.orc_rhs.argtypes = [vp, u32, u32, vp]
        L.orc_lifted_diagonal.argtypes = [vp, vp]
        L.orc_lifted_node_blocks.argtypes = [vp, vp]
        L.orc_cg_solve.restype = C.c_int
        L.orc_cg_solve.argtypes = [vp, u32, u32, vp, C.c_double, C.c_int, C.c_int, vp,
                                   C.POINTER(C.c_int), C.POINTER(C.c_double)]
        L.orc_recover.argtypes = [vp, vp, vp, C.c_int, sz, sz, vp]
        _lib = L
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def surface_nodes(q):
    qx, qy, qz = (q, q, q) if np.isscalar(q) else q
    cnt = lib().orc_surface_nodes(qx, qy, qz, None)
    out = np.empty((cnt, 3), np.uint32)
    lib().orc_surface_nodes(qx, qy, qz, _p(out))
    return out


def index_global_nodes(rows, cols, q):
    qx, qy, qz = (q, q, q) if np.isscalar(q) else q
    lat_x, lat_y, lat_z = cols * (qx - 1) + 1, rows * (qy - 1) + 1, qz
    nol = np.empty(lat_x * lat_y * lat_z, np.int32)
    cnt = lib().orc_index_global_nodes(rows, cols, qx, qy, qz, None, None)
    lon = np.empty((cnt, 3), np.uint32)
    lib().orc_index_global_nodes(rows, cols, qx, qy, qz, _p(nol), _p(lon))
    return nol, lon, (lat_x, lat_y, lat_z)


class OracleCGError(RuntimeError):
    def __init__(self, status, x, iterations, relres):
        super().__init__({2: "no convergence", 3: "breakdown (NaN/Inf or p'Ap <= 0)"}.get(status, "error"))
        self.status, self.x, self.iterations, self.relres = status, x, iterations, relres


class OracleSystem:
    """Matrix-free restatement of the lifted reduced system.

    roms: list indexed by kind (0 tsv, 1 dummy) of dicts/objects exposing
    K, b_el, Phi, u_T, gx, gy, gz, elem_mat, mats ([3,5] E,nu,alpha,lambda,mu).
    """

    def __init__(self, roms, rows, cols, q, kinds=None, delta_t=(-250.0,), bc_mode=1, g=None, threads=0):
        self.rows, self.cols, self.B = rows, cols, rows * cols
        self.roms = roms
        self.nol, self.lon, (self.lat_x, self.lat_y, self.lat_z) = index_global_nodes(rows, cols, q)
        self.N = 3 * len(self.lon)
        qx, qy, qz = (q, q, q) if np.isscalar(q) else q
        r0 = next(r for r in roms if r is not None)
        self.n = r0.K.shape[0]
        self.dof_map = np.empty((self.B, self.n), np.uint32)
        lib().orc_dof_map(rows, cols, qx, qy, qz, _p(self.nol), _p(self.dof_map))
        self.kinds = None if kinds is None else np.ascontiguousarray(kinds, np.uint8)
        dt = np.asarray(delta_t, np.float64)
        self.delta_t = np.ascontiguousarray(np.full(self.B, dt[0]) if dt.size == 1 else dt)
        self.constrained = np.zeros(self.N, np.uint8)
        self.n_constrained = lib().orc_bc_mask(bc_mode, len(self.lon), _p(self.lon), self.lat_x, self.lat_z,
                                               _p(self.constrained))
        self.g = None if g is None else np.ascontiguousarray(g, np.float64)
        self._keep = []
        s = _System()
        s.B, s.n, s.N = self.B, self.n, self.N
        s.dof_map, s.kinds, s.delta_t = _p(self.dof_map), _p(self.kinds), _p(self.delta_t)
        for k in range(MAX_KINDS):
            r = roms[k] if k < len(roms) and roms[k] is not None else r0
            K = np.ascontiguousarray(r.K, np.float64); b = np.ascontiguousarray(r.b_el, np.float64)
            self._keep += [K, b]
            s.K[k], s.b_el[k] = _p(K), _p(b)
        s.constrained, s.g = _p(self.constrained), _p(self.g)
        s.threads = threads or (os.cpu_count() or 1)
        self._s = s

    def apply(self, x):
        x = np.ascontiguousarray(x, np.float64)
        y = np.empty(self.N)
        lib().orc_apply(C.byref(self._s), self.rows, self.cols, _p(x), _p(y))
        return y

    def rhs(self):
        b = np.empty(self.N)
        lib().orc_rhs(C.byref(self._s), self.rows, self.cols, _p(b))
        return b

    def diagonal(self):
        d = np.empty(self.N)
        lib().orc_lifted_diagonal(C.byref(self._s), _p(d))
        return d

    def node_blocks(self):
        m = np.empty((self.N // 3, 3, 3))
        lib().orc_lifted_node_blocks(C.byref(self._s), _p(m))
        return m

    def solve(self, b=None, tol=1e-12, max_it=10000, precond=1):
        b = self.rhs() if b is None else np.ascontiguousarray(b, np.float64)
        x = np.empty(self.N); it = C.c_int(); rr = C.c_double()
        st = lib().orc_cg_solve(C.byref(self._s), self.rows, self.cols, _p(b), tol, max_it, precond, _p(x),
                                C.byref(it), C.byref(rr))
        if st != 0:
            raise OracleCGError(st, x, it.value, rr.value)
        return x, it.value, rr.value

    def recover(self, u, points=8, cell_begin=0, cell_end=None):
        cell_end = self.B if cell_end is None else cell_end
        r0 = next(r for r in self.roms if r is not None)
        rc = _Recovery()
        rc.n_fine = r0.Phi.shape[0]
        rc.cx, rc.cy, rc.cz = len(r0.gx) - 1, len(r0.gy) - 1, len(r0.gz) - 1
        keep = []
        lame = np.zeros((2, 3, 3))
        for k in range(MAX_KINDS):
            r = self.roms[k] if k < len(self.roms) and self.roms[k] is not None else r0
            arrs = [np.ascontiguousarray(a) for a in (r.gx, r.gy, r.gz, r.Phi, r.u_T)]
            em = np.ascontiguousarray(r.elem_mat, np.uint8)
            keep += arrs + [em]
            rc.gx[k], rc.gy[k], rc.gz[k], rc.Phi[k], rc.u_T[k] = [_p(a) for a in arrs]
            rc.elem_mat[k] = _p(em)
            lame[k, :, 0] = r.mats[:, 3]; lame[k, :, 1] = r.mats[:, 4]; lame[k, :, 2] = r.mats[:, 2]
        for i, v in enumerate(lame.ravel()):
            rc.lame[i] = v
        E = rc.cx * rc.cy * rc.cz
        out = np.empty((cell_end - cell_begin, E, points, 7))
        u = np.ascontiguousarray(u, np.float64)
        lib().orc_recover(C.byref(self._s), C.byref(rc), _p(u), points, cell_begin, cell_end, _p(out))
        return out
