"""Python mirror of the reference's online-stage API (tsvstress::global,
proj/include/tsvstress/global.hpp:16-125, linalg.hpp:117-141), backed by
the B200 C ABI. Names, argument meaning and error behaviour follow the
reference so the parity tests read like its own tests:

    ReducedOrderModel  rom.hpp:57-72         RomSet        global.hpp:36-43
    ArrayLayout        global.hpp:16-32      GlobalIndex   global.hpp:47-62
    IterOptions        linalg.hpp:120-129    GlobalSolution global.hpp:91-96
    Error              core.hpp:14-16        NoConvergence linalg.hpp:137-141
    GpuGlobalStage.index_global_nodes / apply_global_bcs / solve_global /
    gather + reconstruct + evaluate_stress (recover) on one GPU.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

from . import native
from .native import (TSV_EBREAKDOWN, TSV_ENOCONV, TSV_OK, IterOptionsC, PrecondInfo, RomDesc, SolveInfo, Timing)

PRECOND = {"none": 0, "diagonal": 1, "block_diagonal": 2, "schwarz2": 3}
BC = {"bottom_pin": 0, "bottom_pin_321": 1, "clamped": 2, "none": 3}
POINTS = {"gauss": 8, "centroid": 1}


class Error(RuntimeError):
    """tsvstress::Error."""


class BreakdownError(Error):
    """CG breakdown: "NaN/Inf breakdown" or "p'Ap <= 0" (linalg.cpp:217, :333-334)."""


class NoConvergence(Error):
    """linalg::NoConvergence carrying the best iterate (linalg.hpp:137-141)."""

    def __init__(self, msg, best: "GlobalSolution"):
        super().__init__(msg)
        self.best = best


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


@dataclass
class ReducedOrderModel:
    """One macro-element: K_r (a_element), b_element, Phi (basis), u_T
    (thermal), plus the unit-block description recovery needs."""
    q: tuple                       # NodeLayout (n_x, n_y, n_z)
    geometry: tuple                # d, h, t, p
    grid: tuple                    # (x, y, z) grid lines
    materials: np.ndarray          # [3, 3] E, nu, alpha per MaterialId
    a_element: np.ndarray = field(repr=False)
    b_element: np.ndarray = field(repr=False)
    basis: np.ndarray = field(repr=False)
    thermal: np.ndarray = field(repr=False)
    element_material: Optional[np.ndarray] = field(default=None, repr=False)
    fingerprint: bytes = b"\0" * 32
    kind: int = 0

    @property
    def reduced_dofs(self):
        return self.a_element.shape[0]

    @property
    def fine_dofs(self):
        return self.basis.shape[0]

    @property
    def cells(self):
        return tuple(len(g) - 1 for g in self.grid)

    @classmethod
    def from_arrays(cls, obj, kind=None):
        """From any object exposing the oracle-style attribute names
        (K, b_el, Phi, u_T, gx, gy, gz, elem_mat, mats, geom, q, fingerprint)."""
        return cls(q=tuple(int(v) for v in obj.q), geometry=tuple(float(v) for v in obj.geom),
                   grid=(obj.gx, obj.gy, obj.gz), materials=np.asarray(obj.mats)[:, :3].copy(),
                   a_element=obj.K, b_element=obj.b_el, basis=obj.Phi, thermal=obj.u_T,
                   element_material=obj.elem_mat, fingerprint=bytes(obj.fingerprint),
                   kind=int(obj.kind if kind is None else kind))


@dataclass
class ArrayLayout:
    rows: int = 1
    cols: int = 1
    kinds: Optional[np.ndarray] = None     # None = all tsv; 1 = dummy
    delta_t: Sequence[float] = (-250.0,)
    pitch: float = 0.0
    height: float = 0.0

    @property
    def cell_count(self):
        return self.rows * self.cols


@dataclass
class IterOptions:
    tolerance: float = 1e-10
    max_iterations: int = 10000
    precond: str = "diagonal"


@dataclass
class GlobalSolution:
    u: Optional[np.ndarray]
    iterations: int = 0
    relative_residual: float = 0.0
    direct_fallback: bool = False
    best_iterations: int = 0
    solve_ms: float = 0.0
    kernel_launches: int = 0
    loop_ms: float = 0.0
    restarts: int = 0
    replacements: int = 0


@dataclass
class GlobalIndex:
    lat_x: int
    lat_y: int
    lat_z: int
    node_count: int
    dof_count: int
    reduced_dofs: int


class GpuGlobalStage:
    """One GPU context: ROMs and the array resident in HBM."""

    def __init__(self, device: int = 0):
        self._L = native.load()
        h = C.c_void_p()
        rc = self._L.tsv_ctx_create(device, C.byref(h))
        if rc != TSV_OK:
            raise Error(f"tsv_ctx_create failed with status {rc} (CUDA device {device} unavailable?)")
        self._h = h
        self._keep = []
        self.layout: Optional[ArrayLayout] = None
        self.roms = [None, None]

    def close(self):
        if getattr(self, "_h", None):
            self._L.tsv_ctx_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    # -------------------------------------------------------------- errors
    def _check(self, rc, what=""):
        if rc == TSV_OK:
            return
        msg = self._L.tsv_last_error(self._h).decode()
        if rc == TSV_EBREAKDOWN:
            raise BreakdownError(msg)
        raise Error(f"{what}: {msg}" if what else msg)

    # ------------------------------------------------------------- set-up
    def set_rom(self, kind: int, rom: ReducedOrderModel):
        d = RomDesc()
        d.q[:] = [int(v) for v in rom.q]
        d.geometry[:] = [float(v) for v in rom.geometry]
        grids = [np.ascontiguousarray(g, np.float64) for g in rom.grid]
        d.grid_len[:] = [len(g) for g in grids]
        for a in range(3):
            d.grid[a] = _p(grids[a])
        mats = np.asarray(rom.materials, np.float64)
        for i in range(3):
            for j in range(3):
                d.materials[i][j] = float(mats[i, j])
        em = None if rom.element_material is None else np.ascontiguousarray(rom.element_material, np.uint8)
        arrs = [np.ascontiguousarray(a, np.float64) for a in (rom.a_element, rom.b_element, rom.basis, rom.thermal)]
        d.element_material = _p(em)
        d.a_element, d.b_element, d.basis, d.thermal = [_p(a) for a in arrs]
        d.fingerprint[:] = list(bytes(rom.fingerprint)[:32].ljust(32, b"\0"))
        self._check(self._L.tsv_set_rom(self._h, kind, C.byref(d)), "set_rom")
        self.roms[kind] = rom

    def load_rom_file(self, path: str, slot: int = -1) -> int:
        """Ingest a reference .rom file (MRST v1) natively into a RomSet slot
        (slot -1 = the file's kind); returns the kind stored in the file."""
        kind = C.c_int()
        err = C.create_string_buffer(512)
        rc = self._L.tsv_load_rom_file(self._h, slot, path.encode(), C.byref(kind), err, 512)
        if rc != TSV_OK:
            raise Error(f"load_rom: {err.value.decode()}")
        return kind.value

    def set_roms(self, tsv: Optional[ReducedOrderModel] = None, dummy: Optional[ReducedOrderModel] = None):
        if tsv is not None:
            self.set_rom(0, tsv)
        if dummy is not None:
            self.set_rom(1, dummy)

    def set_layout(self, layout: ArrayLayout):
        kinds = None if layout.kinds is None else np.ascontiguousarray(layout.kinds, np.uint8)
        dt = np.ascontiguousarray(np.atleast_1d(np.asarray(layout.delta_t, np.float64)))
        self._check(self._L.tsv_set_layout(self._h, layout.rows, layout.cols, _p(kinds), _p(dt), dt.size,
                                           float(layout.pitch), float(layout.height)), "set_layout")
        self.layout = layout

    def set_delta_t(self, delta_t):
        """New per-block temperature change only (1 or rows*cols entries);
        keeps index, BCs and preconditioner (tsv_set_delta_t)."""
        dt = np.ascontiguousarray(np.atleast_1d(np.asarray(delta_t, np.float64)))
        self._check(self._L.tsv_set_delta_t(self._h, _p(dt), dt.size), "set_delta_t")
        if getattr(self, "layout", None) is not None:
            self.layout.delta_t = dt

    def set_bc(self, kind: str = "bottom_pin_321"):
        self._check(self._L.tsv_set_bc(self._h, BC[kind]), "set_bc")

    def set_dirichlet(self, dofs, values):
        dofs = np.ascontiguousarray(dofs, np.uint32)
        values = np.ascontiguousarray(values, np.float64)
        self._check(self._L.tsv_set_dirichlet(self._h, dofs.size, _p(dofs), _p(values)), "set_dirichlet")

    # -------------------------------------------------------------- index
    def index(self) -> GlobalIndex:
        nd, nn, nr = C.c_uint64(), C.c_uint64(), C.c_uint32()
        lat = (C.c_uint32 * 3)()
        self._check(self._L.tsv_get_index(self._h, C.byref(nd), C.byref(nn), lat, C.byref(nr)))
        return GlobalIndex(lat[0], lat[1], lat[2], nn.value, nd.value, nr.value)

    def dof_map(self):
        ix = self.index()
        out = np.empty((self.layout.cell_count, ix.reduced_dofs), np.uint32)
        self._check(self._L.tsv_get_dof_map(self._h, _p(out)))
        return out

    def lattice(self):
        ix = self.index()
        nol = np.empty(ix.lat_x * ix.lat_y * ix.lat_z, np.int32)
        lon = np.empty((ix.node_count, 3), np.uint32)
        self._check(self._L.tsv_get_lattice(self._h, _p(nol), _p(lon)))
        return nol, lon

    def constrained(self):
        out = np.empty(self.index().dof_count, np.uint8)
        self._check(self._L.tsv_get_constrained(self._h, _p(out)))
        return out

    def load(self):
        out = np.empty(self.index().dof_count)
        self._check(self._L.tsv_get_load(self._h, _p(out)))
        return out

    # ------------------------------------------------------------ compute
    def apply(self, x):
        x = np.ascontiguousarray(x, np.float64)
        y = np.empty_like(x)
        self._check(self._L.tsv_apply(self._h, _p(x), _p(y)), "apply")
        return y

    def precond_apply(self, r, precond: str = "schwarz2"):
        r = np.ascontiguousarray(r, np.float64)
        z = np.empty_like(r)
        self._check(self._L.tsv_precond_apply(self._h, PRECOND[precond], _p(r), _p(z)), "precond_apply")
        return z

    def precond_setup(self, precond: str = "schwarz2") -> dict:
        """Build the preconditioner for the current layout now; returns its
        set-up time and (Schwarz) shape."""
        info = PrecondInfo()
        self._check(self._L.tsv_precond_setup(self._h, PRECOND[precond], C.byref(info)), "precond_setup")
        return {"setup_ms": info.setup_ms, "ntypes": info.ntypes, "coarse_dofs": info.coarse_dofs,
                "super_block": info.super_block, "local_rows": info.local_rows}

    def solve_global(self, opts: IterOptions = IterOptions(), copy_out: bool = True) -> GlobalSolution:
        o = IterOptionsC(float(opts.tolerance), int(opts.max_iterations), PRECOND[opts.precond])
        info = SolveInfo()
        u = np.empty(self.index().dof_count) if copy_out else None
        rc = self._L.tsv_solve(self._h, C.byref(o), _p(u), C.byref(info))
        sol = GlobalSolution(u, info.iterations, info.relative_residual, bool(info.direct_fallback),
                             info.best_iterations, info.solve_ms, info.kernel_launches, info.loop_ms, info.restarts,
                             info.replacements)
        if rc == TSV_ENOCONV:
            raise NoConvergence(self._L.tsv_last_error(self._h).decode(), sol)
        self._check(rc, "solve_global")
        return sol

    def set_solution(self, u):
        u = np.ascontiguousarray(u, np.float64)
        self._check(self._L.tsv_set_solution(self._h, _p(u)), "set_solution")

    def _elems(self):
        r = self.roms[0] or self.roms[1]
        cx, cy, cz = r.cells
        return cx * cy * cz

    def recover(self, points: int = 8, cell_begin: int = 0, cell_end: Optional[int] = None):
        cell_end = self.layout.cell_count if cell_end is None else cell_end
        out = np.empty((cell_end - cell_begin, self._elems(), points, 7))
        self._check(self._L.tsv_recover(self._h, points, cell_begin, cell_end, _p(out)), "recover")
        return out

    def recover_resident(self, points: int = 8):
        self._check(self._L.tsv_recover_resident(self._h, points), "recover_resident")

    def copy_stress(self, cell_begin, cell_end, points):
        out = np.empty((cell_end - cell_begin, self._elems(), points, 7))
        self._check(self._L.tsv_copy_stress(self._h, cell_begin, cell_end, _p(out)), "copy_stress")
        return out

    def cutplane_von_mises(self, res: int = 100) -> np.ndarray:
        """cutplane_von_mises (global_stage.cpp:245-274) on the GPU:
        StressGrid values [cell, py, px] at z = h/2."""
        out = np.empty((self.layout.cell_count, res, res))
        self._check(self._L.tsv_cutplane(self._h, res, _p(out)), "cutplane_von_mises")
        return out

    def block_field(self, cell: int):
        r = self.roms[0] or self.roms[1]
        out = np.empty(r.fine_dofs)
        self._check(self._L.tsv_block_field(self._h, cell, _p(out)), "block_field")
        return out

    def profile_apply(self, reps: int = 20) -> float:
        ms = C.c_double()
        self._check(self._L.tsv_profile_apply(self._h, reps, C.byref(ms)), "profile_apply")
        return ms.value

    def symmetry(self) -> dict:
        """Which contractions run on the mirror-symmetric (8 irrep) path."""
        t = native.SymmetryInfo()
        self._check(self._L.tsv_get_symmetry(self._h, C.byref(t)))
        return dict(recovery=bool(t.recovery_symmetric), operator=bool(t.operator_symmetric),
                    correction=bool(t.defect_correction), fused=bool(t.operator_fused), irrep_dofs=list(t.irrep_dofs),
                    defect_k=list(t.defect_k), defect_phi=list(t.defect_phi))

    def timing(self) -> Timing:
        t = Timing()
        self._check(self._L.tsv_get_timing(self._h, C.byref(t)))
        return t


class PinnedArray:
    """A numpy array in page-locked host memory (tsv_host_alloc / cudaHostAlloc):
    the destination for tsv_recover / tsv_copy_stress at full PCIe rate.
    `.array` is the view; `close()` (or garbage collection) frees it."""

    def __init__(self, shape, dtype=np.float64):
        self._L = native.load()
        self.dtype = np.dtype(dtype)
        n = int(np.prod(shape)) * self.dtype.itemsize
        self._ptr = C.c_void_p()
        rc = self._L.tsv_host_alloc(max(n, 1), C.byref(self._ptr))
        if rc != 0:
            raise Error(f"tsv_host_alloc({n} bytes) failed ({rc})")
        buf = (C.c_char * max(n, 1)).from_address(self._ptr.value)
        self.array = np.frombuffer(buf, dtype=self.dtype, count=int(np.prod(shape))).reshape(shape)

    def close(self):
        if self._ptr is not None and self._ptr.value:
            self.array = None
            self._L.tsv_host_free(self._ptr)
            self._ptr = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def build_rom(q, geometry, grid, materials, kind: int = 0, device: int = 0) -> ReducedOrderModel:
    """One-shot local stage on the GPU (rom::build_rom, rom.cpp:134-253):
    the ROM of one unit block. Input of the online stage; timed separately
    (``ReducedOrderModel.build_ms``)."""
    L = native.load()
    d = native.LocalDesc()
    d.q[:] = [int(v) for v in (q if not np.isscalar(q) else (q, q, q))]
    d.geometry[:] = [float(v) for v in geometry]
    grids = [np.ascontiguousarray(g, np.float64) for g in grid]
    d.grid_len[:] = [len(g) for g in grids]
    for a in range(3):
        d.grid[a] = _p(grids[a])
    mats = np.asarray(materials, np.float64)
    for i in range(3):
        for j in range(3):
            d.materials[i][j] = float(mats[i, j])
    d.kind = int(kind)
    n, nf, cells = C.c_uint64(), C.c_uint64(), C.c_uint64()
    rc = L.tsv_rom_dims(C.byref(d), C.byref(n), C.byref(nf), C.byref(cells))
    if rc != TSV_OK:
        raise Error(f"build_rom: invalid descriptor (status {rc})")
    K = np.empty((n.value, n.value)); b = np.empty(n.value); Phi = np.empty((nf.value, n.value))
    uT = np.empty(nf.value); em = np.empty(cells.value, np.uint8)
    out = native.RomOut()
    out.a_element, out.b_element, out.basis, out.thermal, out.element_material = \
        _p(K), _p(b), _p(Phi), _p(uT), _p(em)
    err = C.create_string_buffer(512)
    rc = L.tsv_build_rom(device, C.byref(d), C.byref(out), err, 512)
    if rc != TSV_OK:
        raise Error(f"build_rom: {err.value.decode()}")
    rom = ReducedOrderModel(q=tuple(d.q), geometry=tuple(geometry), grid=tuple(grids), materials=mats[:, :3].copy(),
                            a_element=K, b_element=b, basis=Phi, thermal=uT, element_material=em,
                            fingerprint=bytes(out.fingerprint), kind=int(kind))
    rom.build_ms = out.build_ms
    return rom


def build_config_rom(cfg, kind: int = 0, device: int = 0) -> ReducedOrderModel:
    """ROM of a configs.TsvConfig unit block on its uniform grid."""
    # linspace with exact end points, as tsvstress::linspace (core.cpp:14-22)
    grid = tuple(np.array([0.0] + [a + (b - a) * i / m for i in range(1, m)] + [b]) for (a, b, m) in
                 ((0.0, cfg.p, cfg.m_xy), (0.0, cfg.p, cfg.m_xy), (0.0, cfg.h, cfg.m_z)))
    return build_rom(cfg.q, (cfg.d, cfg.h, cfg.t, cfg.p), grid, cfg.materials(), kind, device)


# ------------------------------------------------------------ .rom files
# The reference's "MRST" v1 little-endian format (rom.cpp:257-377): magic,
# version, kind byte, header (geometry, grid lines, materials, layout), the
# SHA-256 of the header, then the column-major basis, thermal, a_element,
# b_element.
_MAGIC = b"MRST"


def _rom_header(rom: ReducedOrderModel) -> bytes:
    import struct
    out = bytearray()
    out += struct.pack("<4d", *[float(v) for v in rom.geometry])
    for g in rom.grid:
        g = np.ascontiguousarray(g, "<f8")
        out += struct.pack("<I", len(g)) + g.tobytes()
    mats = np.asarray(rom.materials, np.float64)
    for i in range(3):
        out += struct.pack("<B3d", i, *[float(v) for v in mats[i, :3]])
    out += struct.pack("<3I", *[int(v) for v in rom.q])
    return bytes(out)


def save_rom(rom: ReducedOrderModel, path: str) -> None:
    """save_rom (rom.cpp:262-303)."""
    import hashlib
    import struct
    hdr = _rom_header(rom)
    fp = hashlib.sha256(hdr).digest()
    with open(path, "wb") as f:
        f.write(_MAGIC + struct.pack("<IB", 1, int(rom.kind)) + hdr + fp)
        f.write(np.asfortranarray(np.asarray(rom.basis, "<f8")).tobytes(order="F"))
        for a in (rom.thermal, rom.a_element, rom.b_element):
            f.write(np.ascontiguousarray(a, "<f8").tobytes())


def load_rom(path: str) -> ReducedOrderModel:
    """load_rom (rom.cpp:305-377): validates magic, version, kind, the
    header fingerprint and the body length."""
    import hashlib
    import struct
    data = open(path, "rb").read()
    if data[:4] != _MAGIC:
        raise Error(f"load_rom: {path} is not a ROM file (bad magic)")
    version, kind = struct.unpack_from("<IB", data, 4)
    if version != 1:
        raise Error(f"load_rom: {path} has unsupported format version {version}")
    if kind > 1:
        raise Error("load_rom: invalid block kind byte")
    pos = 9
    geom = struct.unpack_from("<4d", data, pos); pos += 32
    grid = []
    for _ in range(3):
        (ln,) = struct.unpack_from("<I", data, pos); pos += 4
        if ln < 2 or ln > 100000000:
            raise Error("load_rom: corrupt grid axis length")
        grid.append(np.frombuffer(data, "<f8", ln, pos).copy()); pos += 8 * ln
    mats = np.zeros((3, 3))
    for i in range(3):
        mid, e, nu, al = struct.unpack_from("<B3d", data, pos); pos += 25
        if mid != i:
            raise Error("load_rom: material table out of order")
        mats[i] = (e, nu, al)
    q = struct.unpack_from("<3I", data, pos); pos += 12
    fp = data[pos:pos + 32]
    if hashlib.sha256(data[9:pos]).digest() != fp:
        raise Error(f"load_rom: {path} fingerprint does not match its header (corrupt file)")
    pos += 32
    nf = 3 * len(grid[0]) * len(grid[1]) * len(grid[2])
    n = 3 * (q[0] * q[1] * q[2] - (q[0] - 2) * (q[1] - 2) * (q[2] - 2))
    body = (nf * n + nf + n * n + n) * 8
    if len(data) - pos != body:
        raise Error(f"load_rom: {path}: corrupt length (body is {len(data) - pos} bytes, expected {body})")
    basis = np.frombuffer(data, "<f8", nf * n, pos).reshape(n, nf).T.copy(); pos += 8 * nf * n
    thermal = np.frombuffer(data, "<f8", nf, pos).copy(); pos += 8 * nf
    K = np.frombuffer(data, "<f8", n * n, pos).reshape(n, n).copy(); pos += 8 * n * n
    b = np.frombuffer(data, "<f8", n, pos).copy()
    return ReducedOrderModel(q=tuple(q), geometry=tuple(geom), grid=tuple(grid), materials=mats, a_element=K,
                             b_element=b, basis=basis, thermal=thermal, element_material=None, fingerprint=fp,
                             kind=kind)


def save_stress_grid_csv(values, rows: int, cols: int, pitch: float, path: str) -> None:
    """StressGrid::save_csv (stress_grid.cpp:36-50): the reference's CSV,
    block_row,block_col,px,py,x,y,von_mises with %.17g numbers."""
    v = np.asarray(values, np.float64).reshape(rows, cols, -1)
    res = int(round(np.sqrt(v.shape[2])))
    v = v.reshape(rows, cols, res, res)
    local = [(q + 0.5) * pitch / res for q in range(res)]
    with open(path, "w", newline="\n") as f:
        f.write("block_row,block_col,px,py,x,y,von_mises\n")
        for r in range(rows):
            for c in range(cols):
                for py in range(res):
                    y = r * pitch + local[py]
                    for px in range(res):
                        x = c * pitch + local[px]
                        f.write("%d,%d,%d,%d,%.17g,%.17g,%.17g\n" % (r, c, px, py, x, y, v[r, c, py, px]))
