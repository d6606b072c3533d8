"""Quick K1 / recovery timing with synthetic ROM values (perf only, not parity)."""
import sys, os, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2411_12690_b200 import configs
from paper_2411_12690_b200.api import GpuGlobalStage, ReducedOrderModel, ArrayLayout, IterOptions

def synth_rom(cfg, seed=0):
    rng = np.random.default_rng(seed)
    n, nf = cfg.n, cfg.n_fine
    A = rng.standard_normal((n, n)); K = A @ A.T / n + np.eye(n)
    grid = (np.linspace(0, cfg.p, cfg.m_xy + 1), np.linspace(0, cfg.p, cfg.m_xy + 1), np.linspace(0, cfg.h, cfg.m_z + 1))
    return ReducedOrderModel(q=(cfg.q,)*3, geometry=(cfg.d, cfg.h, cfg.t, cfg.p), grid=grid, materials=cfg.materials(),
        a_element=K, b_element=rng.standard_normal(n), basis=rng.standard_normal((nf, n)) * 1e-3,
        thermal=rng.standard_normal(nf) * 1e-3)

if __name__ == '__main__':
    res = {}
    for ci in [int(a) for a in sys.argv[1:]] or [1, 2, 3, 4]:
        cfg = configs.get(ci)
        g = GpuGlobalStage(0)
        t = time.time()
        g.set_roms(synth_rom(cfg, 0), synth_rom(cfg, 1) if cfg.dummy_seed else None)
        g.set_layout(ArrayLayout(cfg.rows, cfg.cols, cfg.kinds(), cfg.delta_t(), cfg.p, cfg.h))
        g.set_bc("bottom_pin_321")
        setup = time.time() - t
        ms = g.profile_apply(20)
        flops = 2.0 * cfg.n ** 2 * cfg.B
        sol = g.solve_global(IterOptions(1e-12, 50))  if False else None
        try:
            s = g.solve_global(IterOptions(1e-30, 40), copy_out=False)
        except Exception as e:
            s = e.best
        per_it = s.solve_ms / max(1, s.iterations)
        g.recover_resident(cfg.points)
        t_rec = g.timing().recover_ms
        rflops = 2.0 * cfg.n_fine * cfg.n * cfg.B
        out_bytes = cfg.B * cfg.elements * cfg.points * 56
        res[cfg.name] = dict(setup_s=setup, k1_ms=ms, k1_tflops=flops / ms / 1e9, iter_ms=per_it, iters=s.iterations,
                             recover_ms=t_rec, recover_tflops=rflops / t_rec / 1e9, recover_out_GBps=out_bytes / t_rec / 1e6)
        print(cfg.name, json.dumps(res[cfg.name]), flush=True)
        g.close()
