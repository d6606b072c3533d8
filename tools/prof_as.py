"""Config-3 Schwarz-PCG iterations (synthetic SPD ROM), for ncu."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tools.quick_perf import synth_rom
from paper_2411_12690_b200 import configs
from paper_2411_12690_b200.api import GpuGlobalStage, ArrayLayout, IterOptions, NoConvergence
cfg = configs.get(int(sys.argv[1]) if len(sys.argv) > 1 else 3)
g = GpuGlobalStage(0)
g.set_roms(synth_rom(cfg, 0), synth_rom(cfg, 1) if cfg.dummy_seed else None)
g.set_layout(ArrayLayout(cfg.rows, cfg.cols, cfg.kinds(), cfg.delta_t(), cfg.p, cfg.h))
g.set_bc("bottom_pin_321")
try:
    g.solve_global(IterOptions(1e-30, 8, "schwarz2"), copy_out=False)
except NoConvergence:
    pass
g.close()
