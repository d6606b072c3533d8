#!/usr/bin/env python3
"""Experiment (CPU, FP64 Schwarz oracle machinery): PCG iteration counts at a
config for super-block sizes s and a quantised dense coarse inverse
(fp64 / fp32 / fp16 with a per-64x64-tile scale / bf16), all else exact.

    python tools/coarse_quant_scan.py --config 3 --s 2 3 --quant fp64 fp32 fp16t bf16
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


def quantise(A, how, T=64):
    if how == "fp64":
        return A
    if how == "fp32":
        return A.astype(np.float32).astype(np.float64)
    if how == "bf16":
        b = A.astype(np.float32).view(np.uint32)
        b = ((b + 0x7FFF + ((b >> 16) & 1)) & 0xFFFF0000).astype(np.uint32)
        return b.view(np.float32).astype(np.float64)
    if how == "fp16t":  # fp16 values scaled per T x T tile by the tile's max |a| (fp32 scale)
        out = np.empty_like(A)
        n = A.shape[0]
        for i in range(0, n, T):
            for j in range(0, n, T):
                blk = A[i:i + T, j:j + T]
                m = np.abs(blk).max()
                sc = np.float32(m / 60000.0) if m > 0 else np.float32(1.0)
                out[i:i + T, j:j + T] = (blk / sc).astype(np.float16).astype(np.float64) * np.float64(sc)
        return out
    raise ValueError(how)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--s", type=int, nargs="+", default=[3])
    ap.add_argument("--quant", nargs="+", default=["fp64", "fp32", "fp16t"])
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
    for s in a.s:
        t = time.time()
        S = Schwarz64(o, cfg.q, s=s)
        L = S.coarse[0]
        Linv = sla.solve_triangular(L, np.eye(S.Nc), lower=True, check_finite=False)
        Ainv = Linv.T @ Linv
        print(f"s={s} Nc={S.Nc} setup {time.time() - t:.1f}s", flush=True)
        for q in a.quant:
            Aq = quantise(Ainv, q)
            Aq = 0.5 * (Aq + Aq.T)

            def apply(r, S=S, Aq=Aq):
                R = r[S.dm]
                Z = np.empty_like(R)
                for t_, idx in enumerate(S.groups):
                    Z[idx] = R[idx] @ S.ainv[t_]
                z = np.bincount(S.dm_flat, weights=Z.ravel(), minlength=o.N)
                return z + S.P @ (Aq @ (S.PT @ r))
            S.apply = apply
            t = time.time()
            try:
                u, it, rr = S.solve(b, tol=1e-12, max_it=400)
                print(f"  {q}: {it} iterations relres {rr:.2e} ({time.time() - t:.1f}s)", flush=True)
            except orcpy.OracleCGError as e:
                print(f"  {q}: status {e.status} after {e.iterations} relres {e.relres:.2e}", flush=True)


if __name__ == "__main__":
    main()
