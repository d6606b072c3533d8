"""Where the e2e step's time goes (config 3 default): host phases of
set_layout/set_bc, preconditioner set-up, solve with u read back, recovery
into pinned host memory, and the raw pinned D2H bandwidth."""
import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2411_12690_b200 import configs, native
from paper_2411_12690_b200.api import ArrayLayout, GpuGlobalStage, IterOptions, build_config_rom

ci = int(sys.argv[1]) if len(sys.argv) > 1 else 3
pc = sys.argv[2] if len(sys.argv) > 2 else "schwarz2"
cfg = configs.get(ci)
L = native.load()
g = GpuGlobalStage(0)
g.set_roms(build_config_rom(cfg, 0), build_config_rom(cfg, 1) if cfg.dummy_seed else None)
kinds, dt = cfg.kinds(), cfg.delta_t()
from paper_2411_12690_b200.api import PinnedArray
pinned = PinnedArray((cfg.B, cfg.elements, cfg.points, 7))
out = pinned.array
opts = IterOptions(1e-12, 100000, pc)
for rep in range(3):
    t = {}
    t0 = time.perf_counter()
    g.set_layout(ArrayLayout(cfg.rows, cfg.cols, kinds, dt, cfg.p, cfg.h))
    t["set_layout"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    g.set_bc("bottom_pin_321")
    t["set_bc"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    g.precond_setup(pc)
    t["precond_setup"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    s = g.solve_global(opts, copy_out=True)
    t["solve(u->host)"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    L.tsv_recover(g._h, cfg.points, 0, cfg.B, out.ctypes.data_as(C.c_void_p))
    t["recover(->pinned)"] = time.perf_counter() - t0
    t["recover_dev_ms"] = g.timing().recover_ms / 1e3
    print(rep, {k: round(v * 1e3, 1) for k, v in t.items()}, "ms; iters", s.iterations, flush=True)
out = None
pinned.close()
import torch
d = torch.empty(1 << 31, dtype=torch.uint8, device="cuda")
h = torch.empty(1 << 31, dtype=torch.uint8, pin_memory=True)
for _ in range(2):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    h.copy_(d, non_blocking=True)
    torch.cuda.synchronize()
    print("raw pinned D2H GB/s", round(2.147 / (time.perf_counter() - t0), 1))
