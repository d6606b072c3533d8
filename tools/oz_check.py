"""int8 Ozaki K1 vs the FP64 DMMA K1 on the same operator (tsv_apply):
relative differences for random and solution-like vectors, per digit count."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2411_12690_b200 import configs
from paper_2411_12690_b200.api import GpuGlobalStage, ArrayLayout, IterOptions, build_config_rom

for ci in [int(a) for a in sys.argv[1:]] or [1]:
    cfg = configs.get(ci)
    g = GpuGlobalStage(0)
    g.set_roms(build_config_rom(cfg, 0), build_config_rom(cfg, 1) if cfg.dummy_seed else None)
    g.set_layout(ArrayLayout(cfg.rows, cfg.cols, cfg.kinds(), cfg.delta_t(), cfg.p, cfg.h))
    g.set_bc("bottom_pin_321")
    os.environ.pop("TSV_K1_OZAKI", None)
    u = g.solve_global(IterOptions(1e-12, 100000, "schwarz2")).u
    rng = np.random.default_rng(1)
    vecs = {"random": rng.standard_normal(u.size), "solution": u, "mixed_scale": u * (1 + 1e6 * (rng.random(u.size) < 0.01))}
    out = {}
    for name, x in vecs.items():
        os.environ.pop("TSV_K1_OZAKI", None)
        y64 = g.apply(x)
        for s in (9, 10):
            os.environ["TSV_K1_OZAKI"] = str(s)
            y = g.apply(x)
            out[f"{name}/s{s}"] = float(np.linalg.norm(y - y64) / np.linalg.norm(y64))
            out[f"{name}/s{s}/max"] = float(np.max(np.abs(y - y64)) / np.max(np.abs(y64)))
    os.environ.pop("TSV_K1_OZAKI", None)
    b = g.load()
    r64 = np.linalg.norm(b - g.apply(u)) / np.linalg.norm(b)
    res = {"fp64": float(r64)}
    for s in (9, 10):
        os.environ["TSV_K1_OZAKI"] = str(s)
        res[f"s{s}"] = float(np.linalg.norm(b - g.apply(u)) / np.linalg.norm(b))
    out["true_relres_of_u"] = res
    print(cfg.name, json.dumps(out), flush=True)
    os.environ.pop("TSV_K1_OZAKI", None)
    g.close()
