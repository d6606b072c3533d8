"""ORACLE TEST INFRASTRUCTURE — not product code.

An independent FP64 CPU solve of the lifted reduced system for the large
configs (3: 3.8 M DoFs, 4: 6.4 M DoFs), where the reference's own
Jacobi-PCG needs ~12-21k iterations and its CSR assembly ~100-120 GB.

Control flow: the reference's cg_solve (linalg.cpp:292-362: x0 = 0,
unpreconditioned stopping test, true-residual check + restart, p'Ap
breakdown, best iterate), run by the C restatement
(oracle/tsv_oracle.c:orc_cg_solve_pc) with the operator restated from
assemble_global + apply_dirichlet_lifting (global_stage.cpp:121-145,
fem.cpp:223-260). Only the preconditioner differs from the reference: an
exact FP64 two-level additive Schwarz operator, a FIXED SPD matrix

    M^-1 = sum_b R_b^T A_b^-1 R_b  +  P A_c^-1 P^T

  * A_b = R_b A R_b^T, the lifted matrix restricted to block b's interface
    DoFs, assembled here from K_r of every block sharing a DoF with b and
    factorised by LAPACK Cholesky, one per distinct (3x3 neighbourhood of
    kinds, constrained pattern) key: exact, no type approximation;
  * P: trilinear interpolation from the corners of s x s super-blocks
    (x, y) and the bottom/top lattice planes (z), zero on constrained DoFs;
    A_c = P^T A P formed per block in FP64 and factorised by LAPACK.

It shares no code with the product (paper_2411_12690_b200/csrc/schwarz.cuh,
tc_local.cuh: TF32 local solves on tcgen05, FP32 coarse inverse, neighbour
type approximation) and no precision shortcut. It is pinned against the
live reference (oracle/_ref) on configs 0-1 and the mixed two-kind array in
tests/test_oracle_pin.py, and against the reference at config 2 on the GPU
box (tests/test_gpu_configs.py).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
import this module.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np
import scipy.linalg as sla
import scipy.sparse as sp

from . import orcpy

_PC_FN = C.CFUNCTYPE(None, C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_double))


def _lib():
    L = orcpy.lib()
    if not hasattr(L, "_pc_bound"):
        L.orc_cg_solve_pc.restype = C.c_int
        L.orc_cg_solve_pc.argtypes = [C.c_void_p, C.c_uint32, C.c_uint32, C.c_void_p, C.c_double, C.c_int,
                                      _PC_FN, C.c_void_p, C.c_int, C.c_void_p, C.POINTER(C.c_int),
                                      C.POINTER(C.c_double)]
        L.orc_residual_ld.argtypes = [C.c_void_p, C.c_uint32, C.c_uint32, C.c_void_p, C.c_void_p, C.c_void_p]
        L._pc_bound = True
    return L


def choose_super_block(rows, cols, max_coarse=12000):
    """Smallest s with 6 (ceil(cols/s)+1)(ceil(rows/s)+1) <= max_coarse."""
    s = 1
    while 6 * (-(-cols // s) + 1) * (-(-rows // s) + 1) > max_coarse:
        s += 1
    return s


class Schwarz64:
    """Exact FP64 two-level additive Schwarz operator for an orcpy.OracleSystem."""

    def __init__(self, o: "orcpy.OracleSystem", q, s: int | None = None, max_coarse: int = 12000,
                 sparse_coarse: bool = False):
        qx, qy, qz = (q, q, q) if np.isscalar(q) else q
        self.o = o
        rows, cols, B, n, N = o.rows, o.cols, o.B, o.n, o.N
        dm = o.dof_map.astype(np.int64)
        kinds = np.zeros(B, np.int64) if o.kinds is None else o.kinds.astype(np.int64)
        K = [np.ascontiguousarray(r.K, np.float64) if r is not None else None for r in o.roms]
        K = [k if k is not None else K[0] for k in K] + [K[0]] * (2 - len(K))
        cm = o.constrained.astype(bool)
        self.s = s or choose_super_block(rows, cols, max_coarse)

        # ---- local solves: one exact inverse per distinct neighbourhood key
        kg = np.full((rows + 2, cols + 2), -1, np.int64)
        kg[1:-1, 1:-1] = kinds.reshape(rows, cols)
        keys = {}
        self.type_of = np.empty(B, np.int64)
        reps = []
        for b in range(B):
            r, c = divmod(b, cols)
            k = (kg[r:r + 3, c:c + 3].tobytes(), cm[dm[b]].tobytes())
            t = keys.get(k)
            if t is None:
                t = keys[k] = len(reps)
                reps.append(b)
            self.type_of[b] = t
        loc = np.full(N, -1, np.int64)
        self.ainv = []
        for b in reps:
            r, c = divmod(b, cols)
            loc[dm[b]] = np.arange(n)
            A = np.zeros((n, n))
            for rr in range(max(0, r - 1), min(rows, r + 2)):
                for cc in range(max(0, c - 1), min(cols, c + 2)):
                    bb = rr * cols + cc
                    li = loc[dm[bb]]
                    sel = np.nonzero(li >= 0)[0]
                    if sel.size:
                        A[np.ix_(li[sel], li[sel])] += K[kinds[bb]][np.ix_(sel, sel)]
            loc[dm[b]] = -1
            c_b = cm[dm[b]]
            A[c_b, :] = 0.0
            A[:, c_b] = 0.0
            A[c_b, c_b] = 1.0  # lifted unit rows (fem.cpp:240-247)
            self.ainv.append(sla.cho_solve(sla.cho_factor(A, lower=True), np.eye(n)))
        self.groups = [np.nonzero(self.type_of == t)[0] for t in range(len(reps))]
        self.dm = dm
        self.dm_flat = dm.ravel()

        # ---- coarse space: trilinear on s x s super-blocks, linear in z
        sb = self.s
        SX, SY = -(-cols // sb), -(-rows // sb)
        stx, sty = sb * (qx - 1), sb * (qy - 1)
        lat_x, lat_y = o.lat_x, o.lat_y
        vx = np.minimum(np.arange(SX + 1) * stx, lat_x - 1)
        vy = np.minimum(np.arange(SY + 1) * sty, lat_y - 1)
        self.Nc = Nc = 2 * (SX + 1) * (SY + 1) * 3
        lon = o.lon.astype(np.int64)
        gx, gy, gz = lon[:, 0], lon[:, 1], lon[:, 2]
        cx = np.minimum(gx // stx, SX - 1)
        cy = np.minimum(gy // sty, SY - 1)
        tx = (gx - vx[cx]) / (vx[cx + 1] - vx[cx])
        ty = (gy - vy[cy]) / (vy[cy + 1] - vy[cy])
        tz = gz / (qz - 1)
        nodes = len(lon)
        rows_i, cols_i, vals = [], [], []
        for k in range(8):
            w = (tx if k & 1 else 1 - tx) * (ty if k & 2 else 1 - ty) * (tz if k & 4 else 1 - tz)
            vid = ((k >> 2) * (SY + 1) + cy + ((k >> 1) & 1)) * (SX + 1) + cx + (k & 1)
            for comp in range(3):
                dof = 3 * np.arange(nodes) + comp
                keep = (w != 0.0) & ~cm[dof]
                rows_i.append(dof[keep]); cols_i.append(3 * vid[keep] + comp); vals.append(w[keep])
        P = sp.csr_matrix((np.concatenate(vals), (np.concatenate(rows_i), np.concatenate(cols_i))), shape=(N, Nc))
        self.P, self.PT = P, P.T.tocsr()
        # A_c = sum_b (P[d_b])^T K_b P[d_b]  (P is zero on constrained rows,
        # so the lifting's masks drop out); identical P[d_b] share one product
        Ac = sp.lil_matrix((Nc, Nc)) if sparse_coarse else np.zeros((Nc, Nc))
        acc = [] if sparse_coarse else None
        cache = {}
        for b in range(B):
            Pb = P[dm[b]].tocoo()
            cidx, inv = np.unique(Pb.col, return_inverse=True)
            W = np.zeros((n, cidx.size))
            W[Pb.row, inv] = Pb.data
            key = (int(kinds[b]), W.tobytes())
            G = cache.get(key)
            if G is None:
                G = cache[key] = W.T @ (K[kinds[b]] @ W)
            if sparse_coarse:
                acc.append((np.repeat(cidx, cidx.size), np.tile(cidx, cidx.size), G.ravel()))
            else:
                Ac[np.ix_(cidx, cidx)] += G
        if sparse_coarse:  # experiments with large coarse spaces (s = 1): SuperLU instead of dense Cholesky
            import scipy.sparse.linalg as spla
            ri, ci, vv = (np.concatenate(t) for t in zip(*acc))
            Acs = sp.csc_matrix((vv, (ri, ci)), shape=(Nc, Nc))
            self.coarse_lu = spla.splu(Acs)
            self.coarse = None
            return
        # coarse DoFs that every block leaves empty (none in practice) stay identity
        empty = np.nonzero(np.diag(Ac) == 0.0)[0]
        Ac[empty, empty] = 1.0
        self.coarse = sla.cho_factor(Ac, lower=True)

    def apply(self, r):
        """z = M^-1 r."""
        R = r[self.dm]
        Z = np.empty_like(R)
        for t, idx in enumerate(self.groups):
            Z[idx] = R[idx] @ self.ainv[t]
        z = np.bincount(self.dm_flat, weights=Z.ravel(), minlength=self.o.N)
        if self.coarse is None:
            return z + self.P @ self.coarse_lu.solve(self.PT @ r)
        L = self.coarse[0]  # lower Cholesky factor (two TRSVs: LAPACK potrs is ~20x slower here)
        y = sla.solve_triangular(L, self.PT @ r, lower=True, check_finite=False)
        z += self.P @ sla.solve_triangular(L, y, lower=True, trans="T", check_finite=False)
        return z

    def solve(self, b=None, tol=1e-12, max_it=2000, exact_residual=True):
        """cg_solve (linalg.cpp:292-362) preconditioned by this operator.
        Returns (x, iterations, relres); raises orcpy.OracleCGError like
        OracleSystem.solve. exact_residual: the true-residual check
        (linalg.cpp:321-330) evaluates b - A x in long double
        (orc_residual_ld) instead of FP64; at configs 3/4 the FP64 rounding
        of A x is itself ~tol |b|."""
        o = self.o
        b = o.rhs() if b is None else np.ascontiguousarray(b, np.float64)
        N = o.N

        def pc(_ctx, rp, zp):
            r = np.ctypeslib.as_array(rp, shape=(N,))
            z = np.ctypeslib.as_array(zp, shape=(N,))
            z[:] = self.apply(r)

        cb = _PC_FN(pc)
        x = np.empty(N)
        it = C.c_int()
        rr = C.c_double()
        st = _lib().orc_cg_solve_pc(C.byref(o._s), o.rows, o.cols, b.ctypes.data_as(C.c_void_p), tol, max_it, cb,
                                    None, 1 if exact_residual else 0, x.ctypes.data_as(C.c_void_p), C.byref(it),
                                    C.byref(rr))
        if st != 0:
            raise orcpy.OracleCGError(st, x, it.value, rr.value)
        return x, it.value, rr.value

    def true_residual(self, x, b=None):
        """|b - A x| / |b| with A x in long double (orc_residual_ld)."""
        o = self.o
        b = o.rhs() if b is None else np.ascontiguousarray(b, np.float64)
        x = np.ascontiguousarray(x, np.float64)
        r = np.empty(o.N)
        _lib().orc_residual_ld(C.byref(o._s), o.rows, o.cols, b.ctypes.data_as(C.c_void_p),
                               x.ctypes.data_as(C.c_void_p), r.ctypes.data_as(C.c_void_p))
        return float(np.linalg.norm(r) / np.linalg.norm(b))
