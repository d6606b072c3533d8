#!/usr/bin/env python3
"""Per-kernel HBM table of the PCG iteration kernels from an ncu capture.

    python tools/ncu_hbm_table.py REPORT.ncu-rep [--config 3] [--hbm 6551.7] > table.csv

For each captured launch: ncu duration, dram__bytes_read/write, the
ALGORITHMIC bytes of the kernel (the unique bytes its job must move, from
the array shape; the model is spelled out per kernel below) and the
fractions of the HBM roofline both give. Algorithmic bytes well above
DRAM bytes mean L2 reuse (e.g. panels written by one kernel and read by the
next); DRAM well below the roofline at low occupancy means latency.
"""
from __future__ import annotations

import argparse
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def algorithmic_bytes(cfg, N_dofs, nc, ntypes, local_rows):
    """Unique bytes per launch at a config (8 B doubles, 4 B TF32/FP32)."""
    nodes = N_dofs // 3
    Bn = cfg.B * cfg.n
    vec = 8 * N_dofs          # one N-vector
    slots = 16 * nodes        # int4 slot record per node
    cmask = N_dofs            # u8
    lat = 8 * nodes           # short4
    panel64 = 8 * Bn          # block-major FP64 panel (X / Y)
    panel32 = 4 * Bn          # TF32 local panel (XL32 / ZL32)
    kp = -(-cfg.n // 32) * 32
    ainv32 = ntypes * kp * kp * 4
    nt = -(-nc // 64)
    tiles = nt * (nt + 1) // 2 * 64 * 64 * 4
    part = nt * nt * 64 * 8
    return {
        # Y panel (each block copy once) + p (dot) + slots + cmask -> Ap
        "cg_gather_kernel": panel64 + vec + slots + cmask + vec,
        # x, r read+write (8 B), xlo read+write (4 B); p, Ap read; slots2, cmask; XL32 panel written
        "as_update_kernel": 5 * vec + 2 * vec + slots + cmask + panel32,
        # irrep K1: X panel in, Y panel out (the K'' fragment streams stay in L2)
        "sym_k1_fused_kernel": 2 * panel64,
        # r, cmask, lat -> 24 partials per coarse cell
        "as_restrict_kernel": vec + cmask + lat,
        "as_restrict_warp_kernel": vec + cmask + lat,
        "as_coarse_rhs_kernel": 8 * nc * 4 + 8 * nc,
        # packed FP32 lower triangle of A_c^-1 + partials written
        "as_coarse_symv_kernel": tiles + part,
        "as_coarse_symv_reduce_kernel": part + 16 * nc,
        # XL32 read + the TF32 local inverses + ZL32 written
        "tc_local_pair_kernel": 2 * panel32 + ainv32,
        # slots2, r, cmask, ZL32 panel -> z
        "as_zl_kernel": slots + vec + cmask + panel32 + vec,
        # node_cell, lat, slots, z, cmask, p read+write, X panel written
        "as_scatter_kernel": 4 * nodes + lat + slots + vec + cmask + 2 * vec + panel64,
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("--config", default="3")
    ap.add_argument("--hbm", type=float, default=None)
    ap.add_argument("--bench-json", default=None, help="bench line (for N, Nc, types)")
    a = ap.parse_args()
    from paper_2411_12690_b200 import configs
    cfg = configs.get(int(a.config))
    hbm = a.hbm or float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
    N, nc, ntypes, lrows = cfg.lattice_dofs(), 7350, 9, None
    if a.bench_json:
        d = json.loads(open(a.bench_json).read().strip().splitlines()[-1])
        N = d["config"]["global_dofs"]
        nc = d["precond"]["coarse_dofs"]
        ntypes = d["precond"]["ntypes"]
    model = algorithmic_bytes(cfg, N, nc, ntypes, lrows)
    raw = subprocess.run(["ncu", "-i", a.report, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units = rows[0], rows[1]

    def col(r, name):
        return r[h.index(name)]

    def scale(name):  # to bytes / seconds
        u = units[h.index(name)]
        return {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "us": 1e-6, "ns": 1e-9, "ms": 1e-3,
                "usecond": 1e-6, "nsecond": 1e-9, "msecond": 1e-3}.get(u, 1)
    w = csv.writer(sys.stdout)
    w.writerow(["kernel", "time_us", "dram_read_MB", "dram_write_MB", "dram_GBps", "dram_frac",
                "algorithmic_MB", "algorithmic_GBps", "algorithmic_frac", "grid", "regs", "warps_active_pct",
                "dmma_TFLOPs"])
    k1_flop = 2.0 * cfg.n ** 2 * cfg.B
    for r in rows[2:]:
        name = col(r, "Kernel Name").split("(")[0].split("<")[0].replace("void ", "").split("::")[-1].strip()
        t = float(col(r, "gpu__time_duration.sum")) * scale("gpu__time_duration.sum")
        rd = float(col(r, "dram__bytes_read.sum")) * scale("dram__bytes_read.sum")
        wr = float(col(r, "dram__bytes_write.sum")) * scale("dram__bytes_write.sum")
        alg = model.get(name)
        w.writerow([name, f"{t * 1e6:.1f}", f"{rd / 1e6:.1f}", f"{wr / 1e6:.1f}", f"{(rd + wr) / t / 1e9:.0f}",
                    f"{(rd + wr) / t / 1e9 / hbm:.3f}", f"{alg / 1e6:.1f}" if alg else "",
                    f"{alg / t / 1e9:.0f}" if alg else "", f"{alg / t / 1e9 / hbm:.3f}" if alg else "",
                    col(r, "launch__grid_size"), col(r, "launch__registers_per_thread"),
                    col(r, "sm__warps_active.avg.pct_of_peak_sustained_active"),
                    f"{k1_flop / t / 1e12:.1f}" if name == "gemm_nt_f64" else
                    (f"{k1_flop / 7.97 / t / 1e12:.1f}" if name == "sym_k1_fused_kernel" and cfg.n == 654 else "")])


if __name__ == "__main__":
    main()
