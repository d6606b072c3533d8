"""K1 alone at a config (the layout's default K1 path; env switches pick variants): time per launch."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2411_12690_b200 import configs
from paper_2411_12690_b200.api import GpuGlobalStage, ArrayLayout, build_config_rom
ci = int(sys.argv[1]) if len(sys.argv) > 1 else 3
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
cfg = configs.get(ci)
g = GpuGlobalStage(0)
g.set_roms(build_config_rom(cfg, 0), build_config_rom(cfg, 1) if cfg.dummy_seed else None)
g.set_layout(ArrayLayout(cfg.rows, cfg.cols, cfg.kinds(), cfg.delta_t(), cfg.p, cfg.h))
g.set_bc("bottom_pin_321")
print(json.dumps({"config": ci, "sym": g.symmetry()["fused"], "k1_ms": g.profile_apply(reps)}))
g.close()
