"""Compare the GPU two-level Schwarz z = M^-1 r with a numpy restatement
(exact local A_b^-1 per block + trilinear super-block coarse space)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
S = int(sys.argv[1]) if len(sys.argv) > 1 else 1
os.environ["TSV_AS_S"] = str(S)
import numpy as np, scipy.sparse as sp, scipy.sparse.linalg as spla
from oracle import refpy, orcpy
from conftest import RomObj
from paper_2411_12690_b200.api import GpuGlobalStage, ArrayLayout, ReducedOrderModel
q, side = 5, 6
r = refpy.build_rom(5e-6, 50e-6, 0.5e-6, 15e-6, 16, 16, q, 0)
K = r.K; n = K.shape[0]
o = orcpy.OracleSystem([RomObj(r)], side, side, q, delta_t=[-250.0], bc_mode=1)
N = o.N; dm = o.dof_map.astype(np.int64); B = side * side
I = np.repeat(dm, n, axis=1).ravel(); J = np.tile(dm, (1, n)).ravel(); V = np.tile(K.ravel(), B)
A = sp.csr_matrix((V, (I, J)), shape=(N, N)); cm = o.constrained.astype(bool)
Dm = sp.diags((~cm).astype(float)); A = (Dm @ A @ Dm + sp.diags(cm.astype(float))).tocsr()
step = S * (q - 1); SX = -(-side // S); SY = SX; nxn = SX + 1
rowsP, colsP, valsP = [], [], []
for node, (gx, gy, gz) in enumerate(o.lon.astype(int)):
    cx = min(gx // step, SX - 1); cy = min(gy // step, SY - 1)
    x0, x1 = cx * step, min((cx + 1) * step, o.lat_x - 1); y0, y1 = cy * step, min((cy + 1) * step, o.lat_y - 1)
    tx, ty, tz = (gx - x0) / (x1 - x0), (gy - y0) / (y1 - y0), gz / (q - 1)
    for c in range(8):
        w = (tx if c & 1 else 1 - tx) * (ty if c & 2 else 1 - ty) * (tz if c & 4 else 1 - tz)
        if w == 0: continue
        cnode = (((c >> 2) & 1) * (SY + 1) + cy + ((c >> 1) & 1)) * nxn + cx + (c & 1)
        for comp in range(3):
            f = 3 * node + comp
            if not cm[f]: rowsP.append(f); colsP.append(3 * cnode + comp); valsP.append(w)
Nc = nxn * (SY + 1) * 6
P = sp.csr_matrix((valsP, (rowsP, colsP)), shape=(N, Nc))
Ac = (P.T @ A @ P).toarray(); zr = np.abs(Ac).sum(1) == 0; Ac[zr, zr] = 1.0
Ainv = [np.linalg.inv(A[dm[b]][:, dm[b]].toarray()) for b in range(B)]
rv = np.random.default_rng(0).standard_normal(N); rv[cm] = 0.0
zl = np.zeros(N)
for b in range(B): np.add.at(zl, dm[b], Ainv[b] @ rv[dm[b]])
zc = P @ np.linalg.solve(Ac, P.T @ rv)
zp = zl + zc; zp[cm] = rv[cm]
g = GpuGlobalStage(0)
g.set_rom(0, ReducedOrderModel.from_arrays(RomObj(r), 0))
g.set_layout(ArrayLayout(side, side, None, [-250.0], r.geom[3], r.geom[1]))
g.set_bc("bottom_pin_321")
zg = g.precond_apply(rv)
print(f"S={S} |zg-zp|/|zp| = {np.linalg.norm(zg - zp) / np.linalg.norm(zp):.3e}   local part |zl|={np.linalg.norm(zl):.3e} coarse |zc|={np.linalg.norm(zc):.3e}")
# which part differs: project
d = zg - zp
print("  diff on free dofs:", np.linalg.norm(d[~cm]), " |zg - zl|/|zc| =", np.linalg.norm(zg - zl) / np.linalg.norm(zc), " |zg - zc|/|zl| =", np.linalg.norm(zg - zc) / np.linalg.norm(zl))
import ctypes as C
nc = C.c_int()
g._L.tsv_debug_coarse(g._h, C.byref(nc), None, None, None)
rcg = np.empty(nc.value); zcg = np.empty(nc.value); aig = np.empty((nc.value, nc.value))
g._L.tsv_debug_coarse(g._h, None, rcg.ctypes.data_as(C.c_void_p), zcg.ctypes.data_as(C.c_void_p), aig.ctypes.data_as(C.c_void_p))
rcp = P.T @ rv
print("  Nc gpu/proto", nc.value, Nc, " rc rel diff", np.linalg.norm(rcg - rcp) / np.linalg.norm(rcp))
Aci = np.linalg.inv(Ac)
print("  Ac^-1 rel diff", np.linalg.norm(aig - Aci) / np.linalg.norm(Aci), " zc(gpu) vs Aci@rcg", np.linalg.norm(zcg - Aci @ rcg) / np.linalg.norm(Aci @ rcg))
Acg = np.linalg.inv(aig)
print("  Ac diff", np.linalg.norm(Acg - Ac) / np.linalg.norm(Ac), " diag ratio sample", (np.diag(Acg) / np.diag(Ac))[:12])
