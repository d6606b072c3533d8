"""Jacobi vs two-level Schwarz on a config with the real (GPU local stage) ROM."""
import sys, os, json, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2411_12690_b200 import configs
from paper_2411_12690_b200.api import GpuGlobalStage, ArrayLayout, IterOptions, build_config_rom
for ci in [int(a) for a in sys.argv[1:]] or [3]:
    cfg = configs.get(ci)
    g = GpuGlobalStage(0)
    g.set_roms(build_config_rom(cfg, 0), build_config_rom(cfg, 1) if cfg.dummy_seed else None)
    g.set_layout(ArrayLayout(cfg.rows, cfg.cols, cfg.kinds(), cfg.delta_t(), cfg.p, cfg.h))
    g.set_bc("bottom_pin_321")
    out = {}
    for pc in (["schwarz2", "diagonal"] if "--jacobi" in sys.argv else ["schwarz2"]):
        t = time.perf_counter()
        s1 = g.solve_global(IterOptions(1e-12, 100000, pc))
        t1 = time.perf_counter() - t
        s2 = g.solve_global(IterOptions(1e-12, 100000, pc))
        out[pc] = dict(iterations=s2.iterations, restarts=s2.restarts, relres=s2.relative_residual, solve_ms=round(s2.solve_ms, 2),
                       first_call_s=round(t1, 3), per_it_ms=round(s2.loop_ms / max(1, s2.iterations), 4))
        out[pc + "_u"] = s2.u
    if "diagonal" in out:
        out["rel_diff"] = float(np.linalg.norm(out["schwarz2_u"] - out["diagonal_u"]) / np.linalg.norm(out["diagonal_u"]))
    g.recover_resident(cfg.points)
    rec = g.timing().recover_ms
    print(cfg.name, json.dumps({k: v for k, v in out.items() if not k.endswith("_u")} | {"recover_ms": rec}), flush=True)
    g.close()
