"""Config-3 recovery only (synthetic ROM), for ncu."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from tools.quick_perf import synth_rom
from paper_2411_12690_b200 import configs
from paper_2411_12690_b200.api import GpuGlobalStage, ArrayLayout
cfg = configs.get(int(sys.argv[1]) if len(sys.argv) > 1 else 3)
g = GpuGlobalStage(0)
g.set_roms(synth_rom(cfg, 0), synth_rom(cfg, 1) if cfg.dummy_seed else None)
g.set_layout(ArrayLayout(cfg.rows, cfg.cols, cfg.kinds(), cfg.delta_t(), cfg.p, cfg.h))
g.set_bc("bottom_pin_321")
g.set_solution(np.random.default_rng(0).standard_normal(g.index().dof_count) * 1e-7)
for _ in range(int(os.environ.get("REPS", "1"))):
    g.recover_resident(cfg.points)
    print("recover_ms", g.timing().recover_ms, flush=True)
g.close()
