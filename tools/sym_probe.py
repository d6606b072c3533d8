"""Irrep (mirror-symmetric) K1 variants at a config against the plain DMMA path: operator agreement on a random and
on the smooth solution vector, a bounded Schwarz solve (iterations, restarts, residual), K1 launch time and recovery
time (second call)."""
import sys, os, json, subprocess
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

VARIANTS = {
    "plain": {"TSV_SYM": "0"},
    "fused16": {},
    "fused24": {"TSV_SYM_K1_MF": "3"},
    "fused32": {"TSV_SYM_K1_MF": "4"},
    "fused16_dmma_check": {"TSV_K1_VERIFY": "0"},
    "panels": {"TSV_SYM_K1_FUSED": "0"},
}


def child(ci, max_it, name):
    from paper_2411_12690_b200 import configs
    from paper_2411_12690_b200.api import GpuGlobalStage, ArrayLayout, IterOptions, NoConvergence, build_config_rom
    cfg = configs.get(ci)
    g = GpuGlobalStage(0)
    g.set_roms(build_config_rom(cfg, 0), build_config_rom(cfg, 1) if cfg.dummy_seed else None)
    g.set_layout(ArrayLayout(cfg.rows, cfg.cols, cfg.kinds(), cfg.delta_t(), cfg.p, cfg.h))
    g.set_bc("bottom_pin_321")
    s = g.symmetry()
    out = {"variant": name, "sym": {k: s[k] for k in ("recovery", "operator", "fused", "correction")}}
    N = g.load().size
    x = np.random.default_rng(1).standard_normal(N)
    np.save(f"/tmp/ax_rand_{name}.npy", g.apply(x))
    try:
        s = g.solve_global(IterOptions(1e-12, max_it, "schwarz2"))
        conv = True
    except NoConvergence as e:
        s = e.best
        conv = False
    s = g.solve_global(IterOptions(1e-12, max_it, "schwarz2")) if conv else s
    out["solve"] = dict(converged=conv, iterations=s.iterations, restarts=s.restarts, relres=s.relative_residual,
                        per_it_ms=round(s.loop_ms / max(1, s.iterations), 4), solve_ms=round(s.solve_ms, 2))
    np.save(f"/tmp/u_{name}.npy", s.u)
    u = np.load("/tmp/u_plain.npy") if os.path.exists("/tmp/u_plain.npy") else s.u
    np.save(f"/tmp/ax_u_{name}.npy", g.apply(u))
    out["k1_ms"] = round(g.profile_apply(20), 5)
    g.recover_resident(cfg.points)
    g.recover_resident(cfg.points)
    out["recover_ms"] = round(g.timing().recover_ms, 3)
    print(json.dumps(out), flush=True)
    g.close()


if __name__ == "__main__":
    if sys.argv[1] == "child":
        child(int(sys.argv[2]), int(sys.argv[3]), sys.argv[4])
    else:
        ci, max_it = int(sys.argv[1]), int(sys.argv[2])
        names = sys.argv[3:] or list(VARIANTS)
        if "plain" not in names:
            names = ["plain"] + names
        for name in names:
            env = dict(os.environ, **VARIANTS[name])
            subprocess.run([sys.executable, __file__, "child", str(ci), str(max_it), name], env=env, check=False)
        rl = lambda a, b: float(np.linalg.norm(a - b) / np.linalg.norm(b))
        for name in names[1:]:
            for k in ("ax_rand", "ax_u", "u"):
                try:
                    a, b = np.load(f"/tmp/{k}_{name}.npy"), np.load(f"/tmp/{k}_plain.npy")
                    print(name, k, "vs plain rel_l2 %.3e abs %.3e" % (rl(a, b), float(np.linalg.norm(a - b))))
                except Exception as e:
                    print(name, k, "missing", e)
