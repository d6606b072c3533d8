"""Quick K1 / CG-iteration / recovery timing with synthetic ROM values
(perf only, not parity): python tools/quick_perf.py 3 4"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2411_12690_b200 import configs  # noqa: E402
from paper_2411_12690_b200.api import ArrayLayout, GpuGlobalStage, IterOptions, NoConvergence, ReducedOrderModel  # noqa: E402


def synth_rom(cfg, seed=0):
    rng = np.random.default_rng(seed)
    n, nf = cfg.n, cfg.n_fine
    A = rng.standard_normal((n, n))
    K = A @ A.T / n + np.eye(n)
    grid = (np.linspace(0, cfg.p, cfg.m_xy + 1), np.linspace(0, cfg.p, cfg.m_xy + 1), np.linspace(0, cfg.h, cfg.m_z + 1))
    return ReducedOrderModel(q=(cfg.q,) * 3, geometry=(cfg.d, cfg.h, cfg.t, cfg.p), grid=grid, materials=cfg.materials(),
                             a_element=K, b_element=rng.standard_normal(n), basis=rng.standard_normal((nf, n)) * 1e-3,
                             thermal=rng.standard_normal(nf) * 1e-3)


def iterate(g, its):
    try:
        return g.solve_global(IterOptions(1e-30, its), copy_out=False)
    except NoConvergence as e:
        return e.best


if __name__ == "__main__":
    for ci in [int(a) for a in sys.argv[1:]] or [1, 2, 3, 4]:
        cfg = configs.get(ci)
        g = GpuGlobalStage(0)
        t = time.time()
        g.set_roms(synth_rom(cfg, 0), synth_rom(cfg, 1) if cfg.dummy_seed else None)
        g.set_layout(ArrayLayout(cfg.rows, cfg.cols, cfg.kinds(), cfg.delta_t(), cfg.p, cfg.h))
        g.set_bc("bottom_pin_321")
        setup = time.time() - t
        ms = g.profile_apply(20)
        iterate(g, 32)
        s = iterate(g, 400)
        per_it = s.loop_ms / max(1, s.iterations)
        g.recover_resident(cfg.points)
        g.recover_resident(cfg.points)
        t_rec = g.timing().recover_ms
        flops = 2.0 * cfg.n ** 2 * cfg.B
        rflops = 2.0 * cfg.n_fine * cfg.n * cfg.B
        out_bytes = cfg.B * cfg.elements * cfg.points * 56
        print(cfg.name, json.dumps(dict(setup_s=round(setup, 3), k1_ms=round(ms, 4), k1_tflops=round(flops / ms / 1e9, 2),
                                        iter_ms=round(per_it, 4), vec_ms=round(per_it - ms, 4), recover_ms=round(t_rec, 2),
                                        recover_tflops=round(rflops / t_rec / 1e9, 2),
                                        recover_out_GBps=round(out_bytes / t_rec / 1e6, 1))), flush=True)
        g.close()
