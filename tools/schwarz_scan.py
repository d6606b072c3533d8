"""Two-level Schwarz iterations vs array size and super-block size (config-3 ROM)."""
import sys, os, json, subprocess
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if len(sys.argv) > 1 and sys.argv[1] == "child":
    side, s = int(sys.argv[2]), sys.argv[3]
    os.environ["TSV_AS_S"] = s
    import numpy as np
    from paper_2411_12690_b200 import configs
    from paper_2411_12690_b200.api import GpuGlobalStage, ArrayLayout, IterOptions, build_config_rom
    cfg = configs.get(3)
    rom = build_config_rom(cfg, 0)
    g = GpuGlobalStage(0)
    g.set_roms(rom)
    g.set_layout(ArrayLayout(side, side, None, [-250.0], cfg.p, cfg.h))
    g.set_bc("bottom_pin_321")
    g.solve_global(IterOptions(1e-12, 100000, "schwarz2"))
    sol = g.solve_global(IterOptions(1e-12, 100000, "schwarz2"))
    print(json.dumps(dict(per_it=round(sol.loop_ms / sol.iterations, 3), side=side, s=int(s), iterations=sol.iterations, restarts=sol.restarts, ms=round(sol.solve_ms, 1))), flush=True)
else:
    for side, s in [(100, 2), (100, 3), (100, 4), (50, 2), (50, 3)]:
        subprocess.run([sys.executable, __file__, "child", str(side), str(s)])
