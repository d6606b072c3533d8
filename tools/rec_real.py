"""Recovery timing with the real (local-stage) ROM: python tools/rec_real.py CFG [REPS]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2411_12690_b200 import configs
from paper_2411_12690_b200.api import GpuGlobalStage, ArrayLayout, build_config_rom
cfg = configs.get(int(sys.argv[1]) if len(sys.argv) > 1 else 3)
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 4
g = GpuGlobalStage(0)
g.set_roms(build_config_rom(cfg, 0), build_config_rom(cfg, 1) if cfg.dummy_seed else None)
g.set_layout(ArrayLayout(cfg.rows, cfg.cols, cfg.kinds(), cfg.delta_t(), cfg.p, cfg.h))
g.set_bc("bottom_pin_321")
g.set_solution(np.random.default_rng(0).standard_normal(g.index().dof_count) * 1e-7)
for _ in range(reps):
    g.recover_resident(cfg.points)
    print(cfg.name, "recover_ms", round(g.timing().recover_ms, 3), flush=True)
g.close()
