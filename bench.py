#!/usr/bin/env python
"""Benchmark of the B200 Parareal hot path (BASELINE.json metric:
"Parareal speedup vs serial fine at 1/2/4/8 B200; RHS stencil HBM GB/s vs peak").

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg3s] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...

One bench STEP = one complete Parareal solve (pr_parareal: nu tables, coarse
initial guess, K iterations of fine/coarse/correction with the fused defect,
NCCL hand-off) of the workload, inputs already resident in HBM.  The workload
(default cfg3s) is BASELINE configs[2] (256^3, paper-shaped, 1/2/4/8 GPUs)
shortened 16x in T with the same dt and Dt, N_p = number of GPUs,
K = min(3, N_p).  `value` is the serial-equivalent fine throughput
n^3 * N_t / C_p (fine grid-point steps of the serial solution delivered per
second), so value(N)/value_serial is the Parareal speedup S_measured; the
serial fine solve is timed in the same run for S_measured and tau_f, and the
coarse propagator for tau_c (Eq.(speedup)).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from synthetic import CONFIGS  # noqa: E402

METRIC = "Parareal speedup vs serial fine at 1/2/4/8 B200; RHS stencil HBM GB/s vs peak"
UNIT = "fine point-steps/s (serial-equivalent)"
COARSE_BYTES_PER_PT = 16  # one Euler step (the fine step's bytes come from pr_grid_info)


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy burst)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def ncu_traffic(n, path):
    """dram bytes per RK4 step (sum over its launches) from the committed
    ncu --set full summary (profiles/ncu_summary.json), if one exists."""
    p = os.path.join(ROOT, "profiles", "ncu_summary.json")
    if not os.path.exists(p):
        return None
    try:
        d = json.load(open(p))
        v = d.get("fine_step_dram_bytes", {}).get(path, {}).get(str(n))
        return float(v) if v is not None else None
    except Exception:
        return None


def time_fine_steps(pr, torch, problem, device, steps=64, four_stage=False):
    """Device time per RK4 step of pr_fine on a fresh grid (CUDA events on the
    launching stream, after a warm-up); four_stage=True forces the four-pass path."""
    old = os.environ.get("PR_F2")
    if four_stage:
        os.environ["PR_F2"] = "0"
    try:
        g = pr.Grid(problem, device)
    finally:
        if four_stage:
            if old is None:
                os.environ.pop("PR_F2", None)
            else:
                os.environ["PR_F2"] = old
    n = problem.n
    u = torch.empty((n, n, n), dtype=torch.float64, device=torch.device("cuda", device))
    pr.pr_fill_sine(g, u)
    v = torch.empty_like(u)
    dt = problem.T / 2 ** 13
    pr.pr_fine(g, u, v, 0, 16, dt)
    st = torch.cuda.current_stream(u.device)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(u.device)
    e0.record(st)
    pr.pr_fine(g, u, v, 0, steps, dt)
    e1.record(st)
    torch.cuda.synchronize(u.device)
    info = pr.pr_grid_info(g)
    g.destroy()
    return e0.elapsed_time(e1) / steps, info


class Energy:
    """GPU energy counter (NVML nvmlDeviceGetTotalEnergyConsumption, mJ) of one device."""

    def __init__(self, index):
        self.h = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
        except Exception:
            self.h = None

    def read_j(self):
        if self.h is None:
            return None
        try:
            return self.nv.nvmlDeviceGetTotalEnergyConsumption(self.h) / 1e3
        except Exception:
            return None


class ClockSampler:
    FIELDS = ["index", "clocks.sm", "clocks.max.sm", "clocks_event_reasons.active",
              "clocks_event_reasons.hw_slowdown", "clocks_event_reasons.hw_thermal_slowdown",
              "clocks_event_reasons.sw_thermal_slowdown", "clocks_event_reasons.sw_power_cap",
              "power.draw"]

    def __init__(self, gpus):
        self.gpus = gpus
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", ",".join(str(g) for g in self.gpus),
                 "--query-gpu=" + ",".join(self.FIELDS), "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except Exception:
            self.proc.kill()
            out = ""
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 8:
                continue
            try:
                sm.append(float(f[1]))
                smax.append(float(f[2]))
            except ValueError:
                continue
            for nm, v in zip(names, f[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def cpu_baseline_sample(cfg, target_s=12.0):
    """The oracle (plain C, as it stands) on the host cores: serial fine RK4
    steps of the same grid, the serial-equivalent throughput in `UNIT`."""
    import oracle
    oracle.build()
    n = cfg.n
    p = oracle.Problem(n, c=cfg.c, nu0=cfg.nu0, omega=cfg.omega, T=cfg.T, nu_mode=cfg.nu_mode)
    u = oracle.initial(n)
    dt = cfg.T / cfg.Nt
    t0 = time.perf_counter()
    u = oracle.fine(p, u, 0, 1, dt)
    t1 = time.perf_counter() - t0
    steps = max(1, min(64, int(target_s / max(t1, 1e-3))))
    t0 = time.perf_counter()
    oracle.fine(p, u, 1, steps, dt)
    el = time.perf_counter() - t0
    return {"value": n ** 3 * steps / el, "unit": UNIT, "cores": oracle.threads(), "kind": "oracle",
            "sample": f"{steps} serial fine RK4 steps of the {cfg.name} grid ({n}^3) by oracle/oracle.c "
                      f"({oracle.threads()} OpenMP threads), {el:.2f} s"}


def workload_config(cfg, world, Np, K, args):
    """The `config` dict of the JSON line (identical in both arms)."""
    n = cfg.n
    return {"workload": f"{cfg.name}: {n}^3 periodic advection-diffusion, T={cfg.T:g}, "
                        f"N_t={cfg.Nt}, N_C={cfg.NC}, N_p={Np}, K={K}",
            "n": n, "T": cfg.T, "N_t": cfg.Nt, "N_C": cfg.NC, "N_p": Np, "K": K,
            "omega": cfg.omega, "nu_mode": ["stage", "step_start"][cfg.nu_mode],
            "c": list(cfg.c), "parallelism": f"time-parallel Parareal, {world} GPU(s), "
                                             f"{Np // world} slice(s)/GPU",
            "handoff": args.handoff if world > 1 else "none",
            "g_mesh": args.g_mesh,
            "l2": "inputs larger than L2 (128 MiB fields at 256^3)" if n >= 256 else
                  "fields L2-resident"}


def run_reference(args, cfg, out):
    """--impl reference: the oracle (oracle/oracle.c, as it stands) timed on the host
    cores, rank 0 only.  Each bench step is ONE multi-step orc_fine call: a bounded
    sample of the workload's serial fine solve, sized so the run ends in minutes."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    import oracle
    oracle.build()
    n = cfg.n
    Np = args.slices or world
    K = args.K if args.K is not None else min(3, Np)
    p = oracle.Problem(n, c=cfg.c, nu0=cfg.nu0, omega=cfg.omega, T=cfg.T, nu_mode=cfg.nu_mode)
    u = oracle.initial(n)
    dt = cfg.T / cfg.Nt
    t0 = time.perf_counter()
    u = oracle.fine(p, u, 0, 1, dt)  # size the sample: ~1.5 s of oracle work per step
    t1 = time.perf_counter() - t0
    S = max(1, min(64, int(round(1.5 / max(t1, 1e-3)))))
    j, times = 1, []
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        u = oracle.fine(p, u, j, S, dt)
        el = time.perf_counter() - t0
        j += S
        if i >= args.warmup:
            times.append(el)
    ms = 1e3 * statistics.mean(times)
    value = n ** 3 * S / (ms / 1e3)
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": workload_config(cfg, world, Np, K, args),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": oracle.threads(), "kind": "oracle",
                             "sample": f"each step = one orc_fine call of {S} serial fine RK4 steps of "
                                       f"the {cfg.name} grid ({n}^3), {oracle.threads()} OpenMP threads"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    emit(out, line)
    return 0


def modal_parity(cfg, Np, K, uT, defects, flags_g_mesh):
    """Self-check of the timed solve against the exact discrete modal recurrence
    (tests/modal_ref.py: independent of the oracle and of the CUDA path): the sine
    initial value has 8 Fourier modes, every operator is diagonal on them, so d^k
    and u_T of Alg.1 follow from scalar recurrences."""
    if flags_g_mesh != "full":
        return {"note": "modal pin covers G on the fine mesh only"}
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import modal_ref as M
    n = cfg.n
    th, coef = M.sine_modes(n)
    ms = M.ModalSolver(n, cfg.c, cfg.nu0, cfg.omega, cfg.nu_mode, th)
    nf, nc = cfg.Nt // Np, cfg.NC // Np
    zf = ms.fine(coef, 0, cfg.Nt, cfg.T / cfg.Nt)
    zT, hist = ms.parareal(coef, Np, nc, nf, K, cfg.T)
    dev = uT.device

    def synth(amps):  # the real field of 8 mode amplitudes, on the GPU (a check, not the path)
        return M.synthesize_torch(n, th, amps, dev)
    uf_m = synth(zf)
    M_ = float(uf_m.abs().max())
    d_m = [float((synth(h) - uf_m).abs().max()) / M_ for h in hist]
    uT_m = synth(zT)
    err = float((uT - uT_m).abs().max() / uT_m.abs().max())
    dk = [abs(a - b) for a, b in zip(defects, d_m)] if defects else None
    return {"defects_modal": d_m, "max_abs_dk_vs_modal": max(dk) if dk else None,
            "u_T_rel_err_vs_modal": err, "tol_dk": 1e-10, "tol_u_T": 1e-12,
            "ok": bool(dk is not None and max(dk) <= 1e-10 and err <= 1e-12),
            "reference": "exact discrete Fourier-mode recurrence of the same Alg.1 run (tests/modal_ref.py)"}


def claim_stdout():
    """Keep the process's stdout for the one JSON line: from here on fd 1 points at stderr,
    so banners printed by libraries (NCCL's version line under torchrun, ...) cannot precede
    or interleave with it.  Returns a writer on the original stdout."""
    sys.stdout.flush()
    saved = os.dup(1)
    os.dup2(2, 1)
    return os.fdopen(saved, "w")


def emit(out, line):
    out.write(json.dumps(line) + "\n")
    out.flush()


def main():
    out = claim_stdout()
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="cfg3s")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--K", type=int, default=None, help="override K (default min(3, N_p))")
    ap.add_argument("--slices", type=int, default=None, help="override N_p (default = world size)")
    ap.add_argument("--handoff", default="peer", choices=["nccl", "peer"],
                    help="hand-off of u^{k+1} between ranks: ncclSend/Recv or peer stores "
                         "from the correction kernel (PR_FLAG_PEER_HANDOFF)")
    ap.add_argument("--g-mesh", default="full", choices=["full", "half"],
                    help="G on the fine mesh (Alg.2, the paper's) or on the n/2 mesh with "
                         "restriction / prolongation (NEXT-4, PR_FLAG_G_HALF_MESH)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-parity", action="store_true", help="skip the modal self-check of u_T, d^k")
    ap.add_argument("--nu-mode", type=int, default=None)
    ap.add_argument("--Nt", type=int, default=None, help="override N_t (ratio sweeps, BASELINE configs[4])")
    ap.add_argument("--NC", type=int, default=None, help="override N_C")
    ap.add_argument("--tol", type=float, default=0.0,
                    help="convergence-controlled stopping tolerance (DESIGN.md C23); 0 = fixed K")
    args = ap.parse_args()

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    cfg = CONFIGS[args.config]
    if args.nu_mode is not None:
        cfg = cfg.with_(nu_mode=args.nu_mode)
    if args.Nt is not None or args.NC is not None:
        cfg = cfg.with_(Nt=args.Nt or cfg.Nt, NC=args.NC or cfg.NC,
                        name=f"{cfg.name}[Nt={args.Nt or cfg.Nt},NC={args.NC or cfg.NC}]")
    if args.impl == "reference":
        return run_reference(args, cfg, out)

    import torch
    import torch.distributed as dist
    import paper_1409_8563_b200 as pr

    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    n = cfg.n
    Np = args.slices or world
    K = args.K if args.K is not None else min(3, Np)
    nf, nc = cfg.Nt // Np, cfg.NC // Np
    assert nf * Np == cfg.Nt and nc * Np == cfg.NC, "N_t and N_C must split into N_p slices"
    problem = pr.Problem(n, c=cfg.c, nu0=cfg.nu0, omega=cfg.omega, T=cfg.T, nu_mode=cfg.nu_mode)
    grid = pr.Grid(problem, local)
    if world > 1:
        pr.comm_init_torch(grid)
    last = rank == world - 1
    dev = torch.device("cuda", local)
    stream = torch.cuda.current_stream(dev)

    def barrier():
        if world > 1:
            dist.barrier(device_ids=[local])
        torch.cuda.synchronize(dev)

    def max_over_ranks(x):
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def sum_over_ranks(x):
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.SUM)
        return float(t.item())

    u0 = torch.empty((n, n, n), dtype=torch.float64, device=dev)
    pr.pr_fill_sine(grid, u0)
    uT = torch.empty_like(u0)

    # --- serial fine reference (speedup denominator, u_fine for d^k) and tau_c, on the last rank
    dt, Dt = cfg.T / cfg.Nt, cfg.T / cfg.NC
    uref = torch.empty_like(u0) if last else None
    C_f_ms = tau_f = tau_c = 0.0
    phys = int(os.environ.get("CUDA_VISIBLE_DEVICES", str(local)).split(",")[local]) \
        if os.environ.get("CUDA_VISIBLE_DEVICES") else local
    energy = Energy(phys)
    Q_s = None
    if last:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        pr.pr_fine(grid, u0, uref, 0, 64, dt)  # warm the graphs and tables
        pr.pr_coarse(grid, u0, uT, 0, 64, Dt)
        torch.cuda.synchronize(dev)
        j0 = energy.read_j()
        e0.record(stream)
        pr.pr_fine(grid, u0, uref, 0, cfg.Nt, dt)
        e1.record(stream)
        torch.cuda.synchronize(dev)
        j1 = energy.read_j()
        Q_s = (j1 - j0) if (j0 is not None and j1 is not None) else None
        C_f_ms = e0.elapsed_time(e1)
        tau_f = C_f_ms / cfg.Nt
        if args.g_mesh == "half":  # per-slice G_c calls (restriction + prolongation each)
            pr.pr_coarse_mesh(grid, u0, uT, 0, 8, Dt)
            torch.cuda.synchronize(dev)
            e0.record(stream)
            for m in range(Np):
                pr.pr_coarse_mesh(grid, u0, uT, m * nc, nc, Dt)
            e1.record(stream)
        else:
            e0.record(stream)
            pr.pr_coarse(grid, u0, uT, 0, cfg.NC, Dt)
            e1.record(stream)
        torch.cuda.synchronize(dev)
        tau_c = e0.elapsed_time(e1) / cfg.NC
    tf_all = max_over_ranks(tau_f)
    tc_all = max_over_ranks(tau_c)
    C_f_ms = max_over_ranks(C_f_ms)

    pcfg = pr.PararealCfg(Np, nc, nf, K, tol=args.tol,
                          flags=(pr.PR_FLAG_PEER_HANDOFF if args.handoff == "peer" else 0)
                          | (pr.PR_FLAG_G_HALF_MESH if args.g_mesh == "half" else 0))
    for _ in range(args.warmup):
        pr.pr_parareal(grid, pcfg, u0, uT if last else None, uref)
    barrier()

    sampler = ClockSampler(list(range(world))) if rank == 0 else None
    if sampler:
        sampler.start()
    l0 = pr.pr_kernel_launches()
    times, fine_ms, fine_steps = [], 0.0, 0
    defects = None
    barrier()
    q0 = energy.read_j()
    for _ in range(args.steps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        d = pr.pr_parareal(grid, pcfg, u0, uT if last else None, uref)
        e1.record(stream)
        torch.cuda.synchronize(dev)
        times.append(e0.elapsed_time(e1))
        tl = pr.pr_last_timings(grid)
        fine_ms += tl["fine_ms"]
        fine_steps += pr.pr_last_monitors(grid)[1] * (Np // world) * nf
        if d is not None:
            defects = d
    barrier()
    q1 = energy.read_j()
    tl_all = [None] * world
    if world > 1:
        dist.all_gather_object(tl_all, pr.pr_last_timings(grid))
    else:
        tl_all = [pr.pr_last_timings(grid)]
    Q_p_rank = (q1 - q0) / args.steps if (q0 is not None and q1 is not None) else float("nan")
    Q_p = sum_over_ranks(Q_p_rank)
    Q_s = max_over_ranks(Q_s if Q_s is not None else float("nan"))
    launches = sum_over_ranks(pr.pr_kernel_launches() - l0)
    clocks = sampler.stop() if sampler else None
    ms_per_step = max_over_ranks(sum(times) / len(times))
    value = n ** 3 * cfg.Nt / (ms_per_step / 1e3)

    # roofline of the dominant kernel pair (one RK4 step of F), measured in the timed
    # region.  Bytes = what the two fused kernels must move per grid point (56 B: read
    # u, write acc and Yb; read Yb, u, acc, write u_new), i.e. the
    # HBM fraction of the kernels as built.  SURVEY 8(d)'s 128 B/pt unit figure (the
    # four-pass design's 16 field passes) is reported separately as an effective rate.
    info = pr.pr_grid_info(grid)
    fused = info["fine_kernels_per_step"] == 2
    impl_bytes = info["fine_bytes_per_point"]
    t_fine_step_ms = max_over_ranks(fine_ms / max(fine_steps, 1))
    achieved = impl_bytes * n ** 3 / (t_fine_step_ms / 1e3) / 1e9
    effective_128 = 128 * n ** 3 / (t_fine_step_ms / 1e3) / 1e9
    peak, peak_src = load_peaks()
    traffic = ncu_traffic(n, "fused" if fused else "four_stage")
    # the four-pass kernels measured in the same run, for comparison
    alt = None
    if rank == 0 and fused:
        t4, _ = time_fine_steps(pr, torch, problem, local, 64, four_stage=True)
        a4 = 128 * n ** 3 / (t4 / 1e3) / 1e9
        alt = {"bound": "hbm", "achieved": a4, "peak": peak, "unit": "GB/s", "frac": a4 / peak,
               "traffic": ncu_traffic(n, "four_stage"),
               "kernel": "stencil_kernel<1..4>: one fused pass per RK4 stage (4 launches, 128 B/pt)",
               "algorithmic_bytes_per_launch": 128 * n ** 3, "launch_ms": t4,
               "note": "alternative F path (PR_F2=0), timed on a separate grid after the timed region"}

    # G's own roofline: 16 B per point per Euler step at the measured tau_c
    roof_g = None
    if tc_all > 0 and args.g_mesh == "full":
        ag = 16 * n ** 3 / (tc_all / 1e3) / 1e9
        roof_g = {"bound": "hbm", "achieved": ag, "peak": peak, "unit": "GB/s", "frac": ag / peak,
                  "kernel": "coarse_persist_kernel: one Euler step of G (TMA-fed, persistent)",
                  "algorithmic_bytes_per_launch": 16 * n ** 3, "launch_ms": tc_all,
                  "note": "tau_c of the serial G run on the last rank (outside the timed region)"}

    # e2e: the same solve through the public API with host buffers (pinned), copies timed
    e2e = None
    if not args.no_e2e:
        h_u0 = u0.cpu().pin_memory()
        h_uT = torch.empty(u0.shape, dtype=torch.float64).pin_memory() if last else None
        pr.pr_parareal(grid, pcfg, h_u0, h_uT, uref)
        barrier()
        et = []
        for _ in range(max(1, args.steps)):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            pr.pr_parareal(grid, pcfg, h_u0, h_uT, uref)
            e1.record(stream)
            torch.cuda.synchronize(dev)
            et.append(e0.elapsed_time(e1))
        barrier()
        e2e_ms = max_over_ranks(sum(et) / len(et))
        e2e = {"value": n ** 3 * cfg.Nt / (e2e_ms / 1e3), "unit": UNIT,
               "h2d_bytes_per_step": world * 8 * n ** 3,
               "d2h_bytes_per_step": 8 * n ** 3 + 8 * (K + 1), "ms_per_step": e2e_ms}

    from paper_1409_8563_b200 import perfmodel as pm
    r = tc_all / tf_all
    S_meas = C_f_ms / ms_per_step
    # Eq.(speedup) with the number of time-parallel processors = GPUs: with s = N_p/W
    # slices per GPU the same pipelined model gives N_p -> W
    S_bound = pm.speedup_bound(world, K, nc, nf, tc_all, tf_all)
    S_ns = pm.speedup_bound_northstar(world, K, nc, nf, tc_all, tf_all)
    dlist = None
    if world > 1:
        obj = [defects]
        dist.broadcast_object_list(obj, src=world - 1)
        dlist = obj[0]
    else:
        dlist = defects

    # self-check of the timed solve against the exact modal recurrence (last rank has u_T)
    parity = None
    if last and not args.no_parity and args.tol <= 0:
        try:
            parity = modal_parity(cfg, Np, K, uT, defects, args.g_mesh)
        except Exception as e:  # report, never hide
            parity = {"error": repr(e), "ok": False}
    if world > 1:
        obj = [parity]
        dist.broadcast_object_list(obj, src=world - 1)
        parity = obj[0]

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline_sample(cfg)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": workload_config(cfg, world, Np, K, args),
            "speedup": {"S_measured": S_meas, "S_bound_eq_speedup_P229": S_bound,
                        "frac_of_bound": S_meas / S_bound, "S_bound_northstar_form": S_ns,
                        "E_measured": S_meas / world, "E_bound": S_bound / world,
                        "C_f_ms": C_f_ms, "C_p_ms": ms_per_step, "tau_f_ms": tf_all,
                        "tau_c_ms": tc_all, "tau_c_over_tau_f": r, "N_c_over_N_f": nc / nf,
                        "defects": dlist, "tol": args.tol,
                        "rank_timings_ms": tl_all,
                        "iterations_run": pr.pr_last_monitors(grid)[1],
                        "iterate_change_monitor": pr.pr_last_monitors(grid)[0]},
            "energy": {"Q_serial_J": Q_s, "Q_parareal_J": Q_p,
                       "gamma_measured": (Q_p / Q_s) if Q_s and Q_s == Q_s else None,
                       "gamma_ideal": world / S_meas, "gamma_bound": world / S_bound,
                       "note": "NVML total-energy counters of the GPUs only (Sec. 2.2.2 Eq.(gamma_expected), "
                               "P:257-285); Q_parareal summed over ranks per solve, Q_serial = serial fine on one GPU"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "kernel": ("fused_persist_kernel<K_A>+<K_B>: one RK4 step = 2 launches "
                                    "(stages 1+2, 3+4), design PR_FTILE=%d (%s)"
                                    % (info["fine_variant"],
                                       "per-point stage hand-off through tensor memory"
                                       if info["fine_variant"] == 23 else
                                       "per-point stage hand-off through shared memory"
                                       if info["fine_variant"] == 14 else "alternative design"))
                                   if fused else "stencil_kernel<1..4>: one RK4 step = 4 launches",
                         "launch": "one RK4 step of F (all its kernels), CUDA events on the launching "
                                   "stream around the fine phase of every timed solve",
                         "algorithmic_bytes_per_launch": impl_bytes * n ** 3,
                         "algorithmic_bytes_basis": f"{impl_bytes} B per grid point per RK4 step: the "
                                                    "fields the kernels of this F path must read and write",
                         "traffic_basis": "ncu dram__bytes_read.sum + dram__bytes_write.sum per RK4 step "
                                          "(profiles/ncu_summary.json)",
                         "traffic_frac": (traffic / (t_fine_step_ms / 1e3) / 1e9 / peak) if traffic else None,
                         "effective_gbs_four_pass_units": effective_128,
                         "effective_basis": "SURVEY 8(d) unit figure: 128 B/pt per RK4 step (four-pass design)",
                         "within_peak": bool(achieved <= 1.02 * peak),
                         "launch_ms": t_fine_step_ms, "peak_source": peak_src,
                         "point_steps_per_s": n ** 3 / (t_fine_step_ms / 1e3)},
            "roofline_four_stage": alt,
            "roofline_coarse": roof_g,
            "gpu_launches": int(launches),
            "clocks": clocks,
        }
        if parity is not None:
            line["parity"] = parity
        if e2e:
            line["e2e"] = e2e
        if cpu:
            line["cpu_baseline"] = cpu
        emit(out, line)
    grid.destroy()
    if world > 1:
        dist.barrier(device_ids=[local])
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
