"""Recovery time at a config with / without the K7-beside-K6 overlap (resident recovery, third call)."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2411_12690_b200 import configs
from paper_2411_12690_b200.api import GpuGlobalStage, ArrayLayout, IterOptions, build_config_rom
ci = int(sys.argv[1]) if len(sys.argv) > 1 else 3
cfg = configs.get(ci)
g = GpuGlobalStage(0)
g.set_roms(build_config_rom(cfg, 0), build_config_rom(cfg, 1) if cfg.dummy_seed else None)
g.set_layout(ArrayLayout(cfg.rows, cfg.cols, cfg.kinds(), cfg.delta_t(), cfg.p, cfg.h))
g.set_bc("bottom_pin_321")
s = g.solve_global(IterOptions(1e-12, 100000, "schwarz2"), copy_out=False)
ts = []
for _ in range(5):
    g.recover_resident(cfg.points)
    ts.append(round(g.timing().recover_ms, 3))
print(json.dumps({"config": ci, "iterations": s.iterations, "solve_ms": round(s.solve_ms, 2), "recover_ms": ts}))
g.close()
