#!/usr/bin/env python3
"""Online-stage benchmark: TSV blocks/s of (reduced solve + stress recovery).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 3] [--impl ours|reference]

One step = one pass of the hot path over the whole array: the reduced
global solve (matrix-free FP64 Jacobi-PCG from x0 = 0 to relative residual
1e-12, reference control flow linalg.cpp:292-362) followed by 2x2x2
Gauss-point (or centroid) stress + von Mises recovery of every block.

  value  blocks/s with ROMs/layout resident in HBM, device time (CUDA events
         on the context stream) of K steps, max over ranks, summed over ranks
         (replicas: weak scaling)
  e2e    the same through the public C ABI with host buffers every step:
         layout + dT upload (index/lifting on the host), solve with the
         solution read back, and the full stress field read back into pinned
         host memory
The ROM (local stage) is built once on the GPU by the product's own
tsv_build_rom and timed separately. --impl reference times the reference's
own CPU implementation (oracle/_ref: the unmodified tsvstress sources) on
the host cores for the same metric/config.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "TSV blocks/s (reduced solve + stress recovery); % of FP64/HBM roofline"
TOL = 1e-12
BC = "bottom_pin_321"
ITER_RECORD = os.path.join(ROOT, "profiles", "iterations.json")
# Jacobi-CG iterations to 1e-12 (3-2-1 BC) when no GPU run has recorded them yet
DEFAULT_ITERS = {"cfg0_3x3": 374, "cfg1_10x10": 778}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="3")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-sample", type=int, default=10, help="side of the CPU sample sub-array")
    ap.add_argument("--precond", default="schwarz2", choices=["schwarz2", "diagonal", "block_diagonal", "none"],
                    help="GPU preconditioner (the reference arm always runs its default Jacobi)")
    ap.add_argument("--no-relayout-leg", action="store_true",
                    help="skip the one e2e step through the full re-layout path")
    ap.add_argument("--no-jacobi-leg", action="store_true",
                    help="skip the one-step Jacobi-PCG comparison leg reported beside a schwarz2 headline")
    return ap.parse_args()


def dist_info():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("LOCAL_RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device, self.rows, self.proc = device, [], None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.device}", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except (OSError, FileNotFoundError):
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([v.strip() for v in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            self.proc.wait(timeout=5)

    def summary(self):
        sm = [float(r[1]) for r in self.rows if len(r) >= 9 and r[1].replace(".", "").isdigit()]
        smax = [float(r[2]) for r in self.rows if len(r) >= 9 and r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows if len(r) >= 9 for i in range(4) if r[5 + i] == "Active"})
        loaded = [v for v in sm if v > 0.5 * max(sm)] if sm else []
        return {"sm_mhz": statistics.median(loaded) if loaded else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": reasons, "samples": len(self.rows)}


# ------------------------------------------------------------------ inputs
def build_inputs(cfg, device):
    from paper_2411_12690_b200.api import build_config_rom
    t = time.perf_counter()
    rom_tsv = build_config_rom(cfg, 0, device)
    rom_dum = build_config_rom(cfg, 1, device) if cfg.dummy_seed is not None else None
    return rom_tsv, rom_dum, time.perf_counter() - t


def make_stage(cfg, rom_tsv, rom_dum, device):
    from paper_2411_12690_b200.api import ArrayLayout, GpuGlobalStage
    g = GpuGlobalStage(device)
    g.set_roms(rom_tsv, rom_dum)
    layout = ArrayLayout(cfg.rows, cfg.cols, cfg.kinds(), cfg.delta_t(), cfg.p, cfg.h)
    g.set_layout(layout)
    g.set_bc(BC)
    return g, layout


# ------------------------------------------------------- CPU (reference)
def cpu_sample(cfg, rom_tsv, rom_dum, iters, side, threads):
    """Bounded sample of the reference's CPU path (oracle/_ref, unmodified
    tsvstress sources) on a side x side sub-array of the same config and ROM:
    index + assemble (CSR) + lifting, 30 Jacobi-CG iterations, recovery of
    min(B_s, 50) blocks. Extrapolated per block to the full array with the
    solve's iteration count (same CG, parity-tested)."""
    from oracle import refpy
    from paper_2411_12690_b200.api import save_rom
    tmp = tempfile.mkdtemp(prefix="tsvbench_")

    def as_ref(rom, name):
        if rom is None or isinstance(rom, refpy.RefRom):
            return rom
        path = os.path.join(tmp, name)
        save_rom(rom, path)  # byte-identical MRST file, read by the reference's load_rom
        return refpy.load_rom(path)
    r0, r1 = as_ref(rom_tsv, "tsv.rom"), as_ref(rom_dum, "dummy.rom")
    Bs = side * side
    kinds = cfg.kinds()
    kinds_s = None if kinds is None else kinds.reshape(cfg.rows, cfg.cols)[:side, :side].ravel().copy()
    dt = cfg.delta_t()
    dt_s = dt if dt.size == 1 else dt.reshape(cfg.rows, cfg.cols)[:side, :side].ravel().copy()
    t_wall = time.perf_counter()
    t0 = time.perf_counter()
    s = refpy.RefSession(r0, r1 if (kinds_s is not None and kinds_s.any()) else None, side, side,
                         kinds=kinds_s, delta_t=dt_s, bc_mode=1)
    t_setup = time.perf_counter() - t0
    n_it = 30
    t0 = time.perf_counter()
    try:
        s.iterate(1e-300, n_it, 1, threads)
    except refpy.RefNoConvergence:
        pass
    t_solve = time.perf_counter() - t0
    nrec = min(Bs, 50)
    u = np.zeros(s.N)
    t0 = time.perf_counter()
    s.recover(u, cfg.points, 0, nrec, threads)
    t_rec = time.perf_counter() - t0
    per_block = t_setup / Bs + iters * (t_solve / n_it) / Bs + t_rec / nrec
    total = per_block * cfg.B
    for f in os.listdir(tmp):
        os.remove(os.path.join(tmp, f))
    os.rmdir(tmp)
    return {"value": cfg.B / total, "unit": "blocks/s", "cores": threads, "kind": "reference", "cpu": cpu_model_name(),
            "sample": (f"tsvstress CSR path (oracle/_ref) on a {side}x{side} sub-array of {cfg.name} with the same ROM: "
                       f"index+assemble+lift {t_setup:.2f}s, {n_it} Jacobi-CG iterations {t_solve:.2f}s, recovery of "
                       f"{nrec} blocks {t_rec:.2f}s; extrapolated per block to B={cfg.B} at {iters} iterations"),
            "seconds_per_array": total, "wall_s": time.perf_counter() - t_wall}


MODEL_CHECK = os.path.join(ROOT, "profiles", "r2", "cpu_model_check_cfg2.json")


def cpu_model_name():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def model_check():
    """How the sample extrapolation compares with a FULL run of the
    reference's CSR pipeline at config 2 (tools/cpu_model_check.py, run on
    the GPU box host and committed): the validation the reference arm quotes."""
    try:
        d = json.load(open(MODEL_CHECK))
    except (OSError, ValueError):
        return None
    f = d["full_run"]
    return {"validated_at": d["config"], "cpu": d.get("cpu"), "cores": d.get("cores"),
            "full_run_s": f["total_s"], "full_run_iterations": f["iterations"],
            "sample_model_predicted_s": d["sample_model"]["predicted_total_s"],
            "model_error": d["model_error"], "source": os.path.relpath(MODEL_CHECK, ROOT)}


def jacobi_iterations(cfg):
    """Jacobi-PCG iteration count of the config (what the reference's CG runs),
    recorded by a GPU run in profiles/iterations.json."""
    it = json.load(open(ITER_RECORD)).get(cfg.name) if os.path.exists(ITER_RECORD) else None
    return it or DEFAULT_ITERS.get(cfg.name, 1)


def host_threads():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def run_reference(args, cfg, rank, world):
    if rank != 0:
        return 0
    from oracle import refpy
    iters = jacobi_iterations(cfg)
    threads = host_threads()
    # the reference's own local stage (rom::build_rom) produces its input ROM
    rom_tsv = refpy.build_rom(cfg.d, cfg.h, cfg.t, cfg.p, cfg.m_xy, cfg.m_z, cfg.q, 0, cfg.liner_e, threads)
    rom_dum = (refpy.build_rom(cfg.d, cfg.h, cfg.t, cfg.p, cfg.m_xy, cfg.m_z, cfg.q, 1, cfg.liner_e, threads)
               if cfg.dummy_seed is not None else None)
    vals = []
    for i in range(args.warmup + args.steps):
        r = cpu_sample(cfg, rom_tsv, rom_dum, iters, args.cpu_sample, threads)
        if i >= args.warmup:
            vals.append(r)
    v = statistics.median(x["value"] for x in vals)
    line = {"metric": METRIC, "value": v, "unit": "blocks/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * cfg.B / v, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": cfg.name, "blocks": cfg.B, "iterations": iters, "tol": TOL, "precond": "diagonal",
                       "bc": BC, "points": cfg.points},
            "impl": "reference",
            "cpu_baseline": {"value": v, "unit": "blocks/s", "cores": threads, "kind": "reference",
                             "cpu": cpu_model_name(), "sample": vals[-1]["sample"]},
            "modelled": {"what": ("ms_per_step and value are the per-block extrapolation of the measured bounded "
                                  "sample to the full array at the Jacobi iteration count; each step measured "
                                  "only the sample"),
                         "measured_wall_s_per_step": statistics.median(x["wall_s"] for x in vals),
                         "model_check": model_check()},
            "e2e": {"value": v, "unit": "blocks/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# -------------------------------------------------------------- our arm
def run_ours(args, cfg, rank, local_rank, world):
    from paper_2411_12690_b200 import native
    from paper_2411_12690_b200.api import ArrayLayout, IterOptions
    from paper_2411_12690_b200.replicas import Ranks, aggregate_throughput
    L = native.load()
    dev = local_rank
    ranks = Ranks(device=dev)  # NCCL barrier / max over ranks for N replicas
    barrier, max_over_ranks = ranks.barrier, ranks.max

    rom_tsv, rom_dum, t_rom = build_inputs(cfg, dev)
    g, layout = make_stage(cfg, rom_tsv, rom_dum, dev)
    opts = IterOptions(TOL, 100000, args.precond)
    ix = g.index()
    # preconditioner set-up: once per layout (kinds + BCs; a new dT field
    # keeps it). Cold = first build in this process; warm = a rebuild of the
    # same layout (host tables + device factorisation again).
    pinfo = g.precond_setup(args.precond)
    setup_cold = pinfo["setup_ms"]
    g.set_layout(ArrayLayout(cfg.rows, cfg.cols, cfg.kinds(), cfg.delta_t(), cfg.p, cfg.h))
    g.set_bc(BC)
    pinfo = g.precond_setup(args.precond)
    pinfo["setup_ms_cold"] = setup_cold
    pinfo["setup_ms_warm"] = pinfo.pop("setup_ms")

    def step():
        sol = g.solve_global(opts, copy_out=False)
        g.recover_resident(cfg.points)
        return sol, g.timing()

    for _ in range(max(1, args.warmup)):
        sol, _ = step()
    iters = sol.iterations
    launches0 = g.timing().kernel_launches
    barrier()
    dev_ms = []
    with ClockSampler(dev) as clk:
        t0 = time.perf_counter()
        for _ in range(args.steps):
            sol, tm = step()
            dev_ms.append(tm.solve_ms + tm.recover_ms)
            iters = sol.iterations
        wall = time.perf_counter() - t0
    barrier()
    launches = g.timing().kernel_launches - launches0
    ms_step = max_over_ranks(sum(dev_ms) / len(dev_ms))
    value = aggregate_throughput(cfg.B, world, ms_step)
    solve_ms, recover_ms = tm.solve_ms, tm.recover_ms
    k7_ms, k7_launches = tm.stress_ms, tm.stress_launches  # CUDA events around every K7 launch of the last step

    # dominant kernel (K1 operator apply) on its own stream, CUDA events
    k1_ms = g.profile_apply(50)
    dmma_peak = ctypes_peak(L, dev)
    # Mirror-symmetric ROMs: K1 / K6 run as 8 irrep products (sum n_r^2 instead of
    # n^2 multiply-adds per block). `k1_flops` is the work the kernel executes;
    # the dense figure 2 n^2 B of north_star's contraction is reported beside it.
    sym = g.symmetry()
    k1_dense_flops = 2.0 * cfg.n ** 2 * cfg.B
    irrep = [d for d in sym["irrep_dofs"] if d] if sym["operator"] else []
    k1_flops = 2.0 * sum(d * d for d in irrep) * cfg.B if irrep else k1_dense_flops
    k6_dense_flops = 2.0 * cfg.n_fine * cfg.n * cfg.B
    # irrep K6: the dense basis rows split over the irreps like the reduced DoFs (1/8 to rounding)
    k6_flops = k6_dense_flops * (k1_flops / k1_dense_flops) if sym["recovery"] else k6_dense_flops

    # the same step with the reference's own Jacobi-PCG (one timed step): the
    # per-iteration kernel path the reference's preconditioner implies
    jacobi = None
    if args.precond != "diagonal" and not args.no_jacobi_leg and world == 1:
        jopts = IterOptions(TOL, 100000, "diagonal")
        g.solve_global(jopts, copy_out=False)
        sj = g.solve_global(jopts, copy_out=False)
        g.recover_resident(cfg.points)
        tj = g.timing()
        jacobi = {"iterations": sj.iterations, "ms_per_step": tj.solve_ms + tj.recover_ms,
                  "value": cfg.B / ((tj.solve_ms + tj.recover_ms) * 1e-3),
                  "ms_per_iteration": tj.solve_ms / max(1, sj.iterations)}
        rec_j = sj.iterations
    else:
        rec_j = iters if args.precond == "diagonal" else None

    # end to end through the C ABI with host buffers
    e2e = run_e2e(args, cfg, g, layout, opts, L, world, max_over_ranks, barrier) if args.e2e_steps > 0 else None

    cpu = None
    if rank == 0 and not args.no_cpu_baseline and world == 1:
        try:
            cpu = cpu_sample(cfg, rom_tsv, rom_dum, rec_j or jacobi_iterations(cfg), args.cpu_sample, host_threads())
            cpu.pop("seconds_per_array", None)
            cpu.pop("wall_s", None)
            cpu["model_check"] = model_check()
        except Exception as e:  # oracle not built: report, do not fail the bench
            cpu = {"value": None, "unit": "blocks/s", "cores": host_threads(), "kind": "reference",
                   "sample": f"unavailable: {e}"}
    if rank == 0:
        os.makedirs(os.path.dirname(ITER_RECORD), exist_ok=True)
        rec = json.load(open(ITER_RECORD)) if os.path.exists(ITER_RECORD) else {}
        rec = {k: v for k, v in rec.items() if not k.startswith("_")} | {k: v for k, v in rec.items() if k.startswith("_")}
        if rec_j:
            rec[cfg.name] = rec_j
        rec[f"{cfg.name}/{args.precond}"] = iters
        json.dump(rec, open(ITER_RECORD, "w"), indent=1, sort_keys=True)

    schwarz = args.precond == "schwarz2"
    nc = pinfo["coarse_dofs"]
    # FP64 contractions only (K1 per iteration + K6 once): the TF32 local solves
    # of the Schwarz preconditioner are HBM-bound and charged as bytes below
    flops_step = iters * k1_flops + k6_flops
    flops_step_dense = iters * k1_dense_flops + k6_dense_flops
    out_bytes = cfg.B * cfg.elements * cfg.points * 7 * 8
    hbm_peak = measured_hbm()
    if schwarz:
        # vectors (17 N-vector touches) + TF32 local panels (XL32 written, read;
        # ZL32 written, read: 16 B per block DoF) + the packed lower triangle of
        # the FP32 coarse inverse (2 Nc^2 B)
        vec_bytes = 136.0 * ix.dof_count + 16.0 * cfg.n * cfg.B + 2.0 * nc * nc
    else:
        vec_bytes = 104.0 * ix.dof_count
    # Executed-work model: K1 at the DMMA peak on the FLOPs it executes (or its X-in / Y-out panel
    # stream, whichever is longer), the vector / panel / coarse bytes at the HBM peak, recovery as K6
    # beside the stress stream. The dense model charges north_star's 2 n^2 B and 2 n_fine n B instead.
    panel_bytes = 16.0 * cfg.n * cfg.B
    t_roof_ms = 1e3 * (iters * (max(k1_flops / (dmma_peak * 1e12), panel_bytes / (hbm_peak * 1e9)) + vec_bytes / (hbm_peak * 1e9))
                       + max(k6_flops / (dmma_peak * 1e12), out_bytes / (hbm_peak * 1e9)))
    t_roof_dense_ms = 1e3 * (iters * (k1_dense_flops / (dmma_peak * 1e12) + vec_bytes / (hbm_peak * 1e9))
                             + max(k6_dense_flops / (dmma_peak * 1e12), out_bytes / (hbm_peak * 1e9)))
    k1_roof = {"bound": "tensor", "achieved": k1_flops / (k1_ms * 1e-3) / 1e12, "peak": dmma_peak,
               "unit": "TFLOP/s", "frac": k1_flops / (k1_ms * 1e-3) / 1e12 / dmma_peak,
               "traffic": k1_traffic(cfg, bool(irrep)),
               "kernel": ("sym_k1_fused_kernel (K1 operator apply on the 8 irrep blocks of a mirror-symmetric K_r: "
                          "2 sum n_r^2 B FLOP per launch)" if irrep else
                          "gemm_nt_f64 (K1 operator apply, 2n^2 B FLOP per launch)"),
               "irrep_dofs": irrep or None,
               "ms_per_launch": k1_ms, "launches_per_step": iters, "ms_per_step": iters * k1_ms,
               "dense_equivalent": {"tflops": k1_dense_flops / (k1_ms * 1e-3) / 1e12,
                                    "frac": k1_dense_flops / (k1_ms * 1e-3) / 1e12 / dmma_peak,
                                    "what": "the same launch charged with north_star's dense 2 n^2 B FLOP"},
               "peak_source": "measured live: register-only DMMA.8x8x4 loop (tsv_fp64_peak); MEASURED_PEAKS.json has no FP64 entry"}
    k7_roof = None
    if k7_launches > 0 and k7_ms > 0:
        k7_roof = {"bound": "hbm", "achieved": out_bytes / (k7_ms * 1e-3) / 1e9, "peak": hbm_peak, "unit": "GB/s",
                   "frac": out_bytes / (k7_ms * 1e-3) / 1e9 / hbm_peak,
                   "traffic": k1_traffic(cfg, False, "/k7"),
                   "kernel": "stress_kernel (K7: Gauss-point / centroid stress + von Mises; 56 B written per point, "
                             f"{out_bytes / k7_launches / 1e9:.2f} GB per launch on average)",
                   "ms_per_launch": k7_ms / k7_launches, "launches_per_step": k7_launches, "ms_per_step": k7_ms,
                   "peak_source": "MEASURED_PEAKS.json hbm_gbs (copy bandwidth, read + write)"
                                  if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else "fallback 6650 GB/s"}
    # `roofline` is the kernel with the largest share of the step; the other one is kept beside it
    k7_dominant = k7_roof is not None and k7_roof["ms_per_step"] >= k1_roof["ms_per_step"]
    line = {
        "metric": METRIC, "value": value, "unit": "blocks/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": cfg.name, "blocks": cfg.B, "array": f"{cfg.rows}x{cfg.cols}", "reduced_dofs_per_block": cfg.n,
                   "global_dofs": ix.dof_count, "fine_dofs_per_block": cfg.n_fine, "points_per_element": cfg.points,
                   "iterations": iters, "restarts": sol.restarts, "tol": TOL, "precond": args.precond, "bc": BC,
                   "coarse_dofs": nc if schwarz else None,
                   "parallelism": f"replicas x{world}" if world > 1 else "single GPU",
                   "l2": f"inputs larger than L2: {out_bytes / 1e9:.1f} GB stress output + {ix.dof_count * 8 * 6 / 1e6:.0f} MB vectors per step"},
        "roofline": k7_roof if k7_dominant else k1_roof,
        "roofline_other": k1_roof if k7_dominant else k7_roof,
        "end_to_end_roofline": {"t_roof_ms": t_roof_ms, "frac": t_roof_ms / ms_step,
                                "model": ("iters*(max(K1 FLOP/P64, 16nB/BW) + (136N + 16nB + 2Nc^2)/BW) + max(K6 FLOP/P64, 56 B/point/BW)"
                                          if schwarz else "iters*(max(K1 FLOP/P64, 16nB/BW) + 104N/BW) + max(K6 FLOP/P64, 56 B/point/BW)"),
                                "flop_model": "executed (irrep blocks)" if irrep else "dense",
                                "dense_model": {"t_roof_ms": t_roof_dense_ms, "frac": t_roof_dense_ms / ms_step,
                                                "what": "K1 = 2 n^2 B and K6 = 2 n_fine n B FLOP at the DMMA peak (round-1/2 model)"},
                                "hbm_gbs": hbm_peak},
        "value_with_setup": {"value": aggregate_throughput(cfg.B, world, ms_step + pinfo["setup_ms_warm"]),
                             "ms_per_step": ms_step + pinfo["setup_ms_warm"],
                             "what": "one solve + recovery per layout: the warm preconditioner set-up added to the step"},
        "gflops": flops_step / (ms_step * 1e-3) / 1e9,
        "gflops_dense_equivalent": flops_step_dense / (ms_step * 1e-3) / 1e9,
        "symmetry": {k: sym[k] for k in ("recovery", "operator", "fused", "defect_k", "defect_phi")},
        "phase_ms": {"solve": solve_ms, "recover": recover_ms, "k1_per_launch": k1_ms,
                     "per_iteration": solve_ms / max(1, iters)},
        "rom_build_s": t_rom,
        "precond": pinfo,
        "jacobi_leg": jacobi,
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": launches,
        "clocks": clk.summary(),
        "wall_s_per_step": wall / args.steps,
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    g.close()
    ranks.close()
    return 0


def k1_traffic(cfg, irrep=False, suffix=None):
    """DRAM bytes per launch of K1 (or, suffix "/k7", of the stress kernel) from the committed ncu capture
    (profiles/k1_traffic.json), or None."""
    try:
        t = json.load(open(os.path.join(ROOT, "profiles", "k1_traffic.json")))[cfg.name + (suffix or ("/irrep" if irrep else ""))]
        return t["dram_read_bytes"] + t["dram_write_bytes"]
    except (OSError, KeyError, ValueError):
        return None


def ctypes_peak(L, dev):
    import ctypes as C
    a, b = C.c_double(), C.c_double()
    if L.tsv_fp64_peak(dev, C.byref(a), C.byref(b)) != 0:
        return 37.16
    return a.value


def measured_hbm():
    try:
        return float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
    except Exception:
        return 6650.0


def step_delta_t(cfg, k):
    """The e2e step's input: a fresh temperature field per step. Per-block
    configs (3) draw i.i.d. U[-270, -230) K from a per-step seed; uniform
    configs keep their single dT (the upload still happens every step)."""
    dt = cfg.delta_t()
    if dt.size == 1:
        return dt.copy()
    return -270.0 + 40.0 * np.random.default_rng(2411_000 + k).random(dt.size)


def run_e2e(args, cfg, g, layout, opts, L, world, max_over_ranks, barrier):
    """Public API with host buffers, the reference's online stage per step:
    a new dT field H2D (tsv_set_delta_t; index, BCs and preconditioner stay),
    solve with u read back, recover every block into pinned host memory.
    One more step through the full re-layout path (tsv_set_layout + set_bc,
    preconditioner rebuilt) is reported beside it."""
    import ctypes as C
    from paper_2411_12690_b200.api import ArrayLayout
    from paper_2411_12690_b200.api import PinnedArray
    pinned = PinnedArray((cfg.B, cfg.elements, cfg.points, 7))  # page-locked result buffer (tsv_host_alloc)
    out = pinned.array
    kinds = cfg.kinds()
    h2d = 8 * (cfg.B if cfg.delta_t().size > 1 else 1)
    d2h = out.nbytes + 8 * g.index().dof_count
    relayout = None
    try:
        def e2e_step(k):
            g.set_delta_t(step_delta_t(cfg, k))
            g.solve_global(opts, copy_out=True)
            L.tsv_recover(g._h, cfg.points, 0, cfg.B, out.ctypes.data_as(C.c_void_p))
        e2e_step(0)  # warm-up
        barrier()
        t0 = time.perf_counter()
        for k in range(args.e2e_steps):
            e2e_step(k + 1)
        dt_s = max_over_ranks((time.perf_counter() - t0) / args.e2e_steps)
        assert np.isfinite(out[:, :, :, 6]).all()
        if not args.no_relayout_leg:
            barrier()
            t0 = time.perf_counter()
            g.set_layout(ArrayLayout(cfg.rows, cfg.cols, kinds, step_delta_t(cfg, 99), cfg.p, cfg.h))
            g.set_bc(BC)
            g.solve_global(opts, copy_out=True)
            L.tsv_recover(g._h, cfg.points, 0, cfg.B, out.ctypes.data_as(C.c_void_p))
            t_re = max_over_ranks(time.perf_counter() - t0)
            relayout = {"value": world * cfg.B / t_re, "seconds_per_step": t_re,
                        "path": "tsv_set_layout + tsv_set_bc + preconditioner set-up + tsv_solve(u -> host) + "
                                "tsv_recover(all cells -> pinned host)"}
    finally:
        out = None
        pinned.close()
    return {"value": world * cfg.B / dt_s, "unit": "blocks/s", "h2d_bytes_per_step": int(h2d),
            "d2h_bytes_per_step": int(d2h), "seconds_per_step": dt_s,
            "path": "tsv_set_delta_t(fresh dT field) + tsv_solve(u -> host) + tsv_recover(all cells -> pinned host, "
                    "tsv_host_alloc)",
            "new_layout_step": relayout}


def main():
    args = parse()
    rank, local_rank, world = dist_info()
    from paper_2411_12690_b200 import configs
    cfg = configs.get(int(args.config) if args.config.isdigit() else args.config)
    if args.impl == "reference":
        return run_reference(args, cfg, rank, world)
    return run_ours(args, cfg, rank, local_rank, world)


if __name__ == "__main__":
    sys.exit(main())
