#!/usr/bin/env python3
"""Experiment (CPU, FP64 Schwarz oracle): the reference's cg_solve control
flow (linalg.cpp:292-362) with A p formed directly, against the same loop
with the product's split recurrence

    A p_new = A z_l + A P z_c + beta A p_old,   p_new = z_l + P z_c + beta p_old

(z = z_l + P z_c the two-level Schwarz output; A z_l is what K1 computes, A P z_c
comes from per-block (K_b P_b) z_c products), which lets the coarse solve run
beside K1 instead of before it. Reports iterations, restarts and the final
true residual (long-double A x).

    python tools/ap_recurrence_check.py --config 2
"""
from __future__ import annotations

import argparse
import os
import sys
import time

import numpy as np
import scipy.linalg as sla

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def cg(o, S, b, tol, max_it, split, true_res):
    N = o.N
    L = S.coarse[0]

    def parts(r):
        R = r[S.dm]
        Z = np.empty_like(R)
        for t, idx in enumerate(S.groups):
            Z[idx] = R[idx] @ S.ainv[t]
        zl = np.bincount(S.dm_flat, weights=Z.ravel(), minlength=N)
        y = sla.solve_triangular(L, S.PT @ r, lower=True, check_finite=False)
        zc = sla.solve_triangular(L, y, lower=True, trans="T", check_finite=False)
        return zl, zc

    norm_b = np.sqrt(b @ b)
    x = np.zeros(N)
    r = b.copy()
    zl, zc = parts(r)
    z = zl + S.P @ zc
    p = z.copy()
    ap = (o.apply(zl) + o.apply(S.P @ zc)) if split else o.apply(p)
    rho = r @ z
    res = np.sqrt(r @ r)
    it = restarts = 0
    while it < max_it:
        if res <= tol * norm_b:
            r = b - o.apply(x)
            res = np.sqrt(r @ r)
            if true_res(x) <= tol:
                break
            restarts += 1
            zl, zc = parts(r)
            z = zl + S.P @ zc
            p = z.copy()
            ap = (o.apply(zl) + o.apply(S.P @ zc)) if split else o.apply(p)
            rho = r @ z
        pap = p @ ap
        alpha = rho / pap
        x += alpha * p
        r -= alpha * ap
        zl, zc = parts(r)
        z = zl + S.P @ zc
        rho_n = r @ z
        beta = rho_n / rho
        rho = rho_n
        if split:
            ap = o.apply(zl) + o.apply(S.P @ zc) + beta * ap
            p = z + beta * p
        else:
            p = z + beta * p
            ap = o.apply(p)
        res = np.sqrt(r @ r)
        it += 1
    return x, it, restarts


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--s", type=int, default=None)
    a = ap.parse_args()
    from conftest import RomObj, ref_rom
    from oracle import orcpy, refpy
    from oracle.schwarz64 import Schwarz64
    from paper_2411_12690_b200 import configs
    cfg = configs.get(a.config)
    r = ref_rom(cfg, 0, refpy)
    rd = ref_rom(cfg, 1, refpy) if cfg.dummy_seed is not None else None
    o = orcpy.OracleSystem([RomObj(r), RomObj(rd) if rd is not None else None], cfg.rows, cfg.cols, cfg.q,
                           kinds=cfg.kinds(), delta_t=cfg.delta_t(), bc_mode=1)
    b = o.rhs()
    S = Schwarz64(o, cfg.q, s=a.s)
    u_ref, it_ref, _ = S.solve(b, tol=1e-12)
    for split in (False, True):
        t = time.time()
        x, it, rs = cg(o, S, b, 1e-12, 600, split, lambda x: S.true_residual(x, b))
        print(f"split={split}: {it} iterations, {rs} restarts, true residual {S.true_residual(x, b):.2e}, "
              f"|x-u_oracle|/|u| {np.linalg.norm(x - u_ref) / np.linalg.norm(u_ref):.2e} ({time.time() - t:.1f}s); "
              f"oracle {it_ref} it", flush=True)


if __name__ == "__main__":
    main()
