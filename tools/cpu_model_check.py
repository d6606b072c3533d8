#!/usr/bin/env python3
"""Validate bench.py's CPU-baseline extrapolation against a FULL run of the
reference's CSR path (oracle/_ref, the unmodified tsvstress sources).

At config 3 the reference arm cannot run in full inside a bench (CSR
assembly ~120 GB and ~21k Jacobi iterations: hours), so bench.py times a
bounded side x side sub-array sample and extrapolates per block
(bench.cpu_sample). This tool runs that same sample model at config 2 AND
the whole config-2 pipeline (index + assemble + lift, Jacobi cg_solve to
1e-12, Gauss-point recovery of every block) in one process on the same
cores, and writes both to a JSON file (committed under profiles/) that the
reference arm quotes.

    python tools/cpu_model_check.py [--config 2] [--side 10] [--out profiles/r2/cpu_model_check_cfg2.json]
"""
from __future__ import annotations

import argparse
import json
import os
import platform
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--side", type=int, default=10)
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r2", "cpu_model_check_cfg2.json"))
    a = ap.parse_args()
    import bench
    from oracle import refpy
    from paper_2411_12690_b200 import configs
    cfg = configs.get(a.config)
    threads = bench.host_threads()
    t0 = time.perf_counter()
    rom = refpy.build_rom(cfg.d, cfg.h, cfg.t, cfg.p, cfg.m_xy, cfg.m_z, cfg.q, 0, cfg.liner_e, threads)
    t_rom = time.perf_counter() - t0

    # the full pipeline (what the reference's acceptance driver times)
    t0 = time.perf_counter()
    s = refpy.RefSession(rom, None, cfg.rows, cfg.cols, delta_t=cfg.delta_t(), bc_mode=1)
    t_setup = time.perf_counter() - t0
    t0 = time.perf_counter()
    u, iters, relres = s.iterate(1e-12, 1000000, 1, threads)
    t_solve = time.perf_counter() - t0
    t0 = time.perf_counter()
    chunk = 64
    for c0 in range(0, cfg.B, chunk):
        s.recover(u, cfg.points, c0, min(cfg.B, c0 + chunk), threads)
    t_rec = time.perf_counter() - t0
    full = t_setup + t_solve + t_rec
    del s

    # the bench's bounded-sample model at the measured iteration count
    samples = [bench.cpu_sample(cfg, rom, None, iters, a.side, threads) for _ in range(3)]
    pred = [cfg.B / x["value"] for x in samples]
    out = {
        "config": cfg.name, "blocks": cfg.B, "cores": threads, "cpu": cpu_model(),
        "reference_rom_build_s": t_rom,
        "full_run": {"index_assemble_lift_s": t_setup, "cg_s": t_solve, "iterations": iters, "relres": relres,
                     "s_per_iteration": t_solve / iters, "recovery_s": t_rec, "total_s": full,
                     "blocks_per_s": cfg.B / full},
        "sample_model": {"side": a.side, "predicted_total_s": pred, "predicted_blocks_per_s": [cfg.B / p for p in pred],
                         "sample": samples[-1]["sample"]},
        "model_error": [p / full - 1.0 for p in pred],
    }
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    json.dump(out, open(a.out, "w"), indent=1)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
