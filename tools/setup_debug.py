"""Per-phase breakdown (TSV_DEBUG=1, device-synchronised ticks) of the
Schwarz set-up and the host phases of set_layout / set_bc at a config."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2411_12690_b200 import configs
from paper_2411_12690_b200.api import ArrayLayout, GpuGlobalStage, build_config_rom
cfg = configs.get(int(sys.argv[1]) if len(sys.argv) > 1 else 3)
g = GpuGlobalStage(0)
g.set_roms(build_config_rom(cfg, 0), build_config_rom(cfg, 1) if cfg.dummy_seed else None)
for rep in range(3):
    t0 = time.perf_counter()
    g.set_layout(ArrayLayout(cfg.rows, cfg.cols, cfg.kinds(), cfg.delta_t(), cfg.p, cfg.h))
    t1 = time.perf_counter()
    g.set_bc("bottom_pin_321")
    t2 = time.perf_counter()
    g.precond_setup("schwarz2")
    t3 = time.perf_counter()
    print(f"rep {rep}: set_layout {1e3*(t1-t0):.1f} set_bc {1e3*(t2-t1):.1f} precond {1e3*(t3-t2):.1f} ms", file=sys.stderr, flush=True)
