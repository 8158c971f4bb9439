#!/usr/bin/env python
"""Benchmark of the wBFBT hot path on B200 (BASELINE.json metric).

A step = one pass of every SURVEY.md Sec. 8(a) row over one synthetic batch:
wb_hotpath = set_viscosity (rows a3, a4) + A u + B u + B^T p + wBFBT(p)
(rows a5-a10; row a1 is inline in every kernel) on the BASELINE.json config
C5 (64^3 Q2 x P1disc, 100 PCG iterations per Poisson inverse).

value   = whole-job steps/s (= wBFBT applies/s of full hot-path steps) with
          inputs resident in HBM, device time (CUDA events), max over ranks;
          the L2 is flushed (256 MiB memset) before every timed step, outside
          the events.
e2e     = the same step through wb_hotpath_host: host->device copies of
          mu, u, p from pinned memory and device->host copies of the four
          results inside the timed region.
Multi-GPU (torchrun): independent replicas, one problem per rank ("weak").
--impl reference: the CPU oracle as it stands on a bounded sample (rank 0).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "GDOF/s of fp64 A(mu)u apply; wBFBT applies/s; % of B200 HBM roofline"
FALLBACK_HBM = 6650.0      # B200_PROFILING.md fallback (GB/s)
FP64_PEAK_TFLOPS = 37.2    # 148 SM x 64 DFMA/clk x 2 x 1.965 GHz (microbench: 34.2 DFMA, 37.1 DMMA)


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return FALLBACK_HBM, "fallback"


# DFMA-pipe instructions per element of the k = 2 sum-factorised A using the exact zero
# centre rows ("zero-row" count; FMA = 1), and the measured DFMA
# rate of this B200 (profiles/r01_microbench_peaks.jsonl: 34.2 TFLOP/s = 17.1 T DFMA/s).
A_DFMA_PER_ELEMENT = 2538
DFMA_PEAK_INSTR_PER_S = 34.195e12 / 2


def ncu_traffic(kernel):
    """DRAM bytes per launch of `kernel` from the committed ncu capture summary
    (profiles/ncu_traffic.json, written by tools/ncu_summary.py), else None."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            return float(json.load(f)[kernel]["dram_bytes_per_launch"])
    except Exception:
        return None


class Clocks:
    """Sample nvidia-smi clocks / throttle reasons during the timed region."""

    def __init__(self, index=0):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index),
                 "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
                 "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
                 "clocks_event_reasons.sw_power_cap", "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 6:
                continue
            try:
                sm.append(float(f[0]))
                mx = float(f[1])
            except ValueError:
                continue
            for n, v in zip(names, f[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def dist_init(n_gpus):
    import torch
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)
    return rank, world, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(x, world):
    """Max of a per-rank scalar (device time) over all ranks (NCCL on GPUs, gloo on CPU)."""
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([x], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def replica_seed(rank):
    """Replicas only: rank r solves its own problem, seed r."""
    return rank


def job_throughput(world, steps, max_ms):
    """Whole-job steps/s: all ranks' steps over the slowest rank's device time."""
    return world * steps / (max_ms * 1e-3)


# ---------------------------------------------------------------------- reference arm (CPU oracle)
def oracle_sample(cfg_name="C5", seed=0, pcg_probe=(1, 3)):
    """Time the oracle as it stands on a bounded sample of the step: setup, A, B,
    B^T once at full size, and wBFBT at two small PCG counts; the full-size step
    time is extrapolated linearly in the PCG count."""
    import synth
    from oracle import Oracle
    cfg = synth.CONFIGS[cfg_name]
    inp = synth.make_inputs(cfg, seed)
    o = Oracle(cfg.N, cfg.k)
    t = {}
    t0 = time.perf_counter(); o.setup(inp["mu_q"]); t["setup"] = time.perf_counter() - t0
    t0 = time.perf_counter(); o.apply_A(inp["mu_q"], inp["u"]); t["A"] = time.perf_counter() - t0
    t0 = time.perf_counter(); o.apply_B(inp["u"]); t["B"] = time.perf_counter() - t0
    t0 = time.perf_counter(); o.apply_BT(inp["p"]); t["BT"] = time.perf_counter() - t0
    w = []
    for it in pcg_probe:
        t0 = time.perf_counter(); o.wbfbt(inp["p"], it); w.append(time.perf_counter() - t0)
    per_it = (w[1] - w[0]) / (pcg_probe[1] - pcg_probe[0])
    t_wbfbt = w[0] + per_it * (cfg.iters - pcg_probe[0])
    step = t["setup"] + t["A"] + t["B"] + t["BT"] + t_wbfbt
    n_v = 3 * (cfg.k * cfg.N + 1) ** 3
    return dict(step_s=step, t=t, wbfbt_s=t_wbfbt, per_pcg_iter_s=per_it, A_gdofs=n_v / t["A"] / 1e9,
                threads=Oracle.num_threads(), sample_s=sum(t.values()) + sum(w),
                sample=f"{cfg_name} full size: setup+A+B+B^T once; wBFBT at PCG iters {pcg_probe}, "
                       f"extrapolated linearly to {cfg.iters}")


def unit_of(cfg) -> str:
    """The `unit` string of both arms (identical, so the driver can form their ratio)."""
    return (f"hot-path steps/s (1 step = setup + A + B + B^T + wBFBT with 2x{cfg.iters} PCG iters, "
            f"{cfg.name})")


def workload_of(cfg) -> str:
    idx = {"C1": 0, "C2": 1, "C3": 2, "C4": 3, "C5": 4}.get(cfg.name)
    return (f"{cfg.name} = BASELINE.json configs[{idx}]: {cfg.N}^3 Q{cfg.k}xP{cfg.k - 1}disc, {cfg.n_sinkers} "
            f"sinkers, DR {cfg.dr:.0e}, {cfg.iters} PCG iters")


def oracle_full_step(cfg_name="C5", seed=0):
    """One complete hot-path step of the oracle as it stands, timed on the host cores:
    setup (C_w, D_w, Jacobi diagonals) + A u + B u + B^T p + wBFBT(p) with the config's
    PCG count -- the same work as one `wb_hotpath` call."""
    import synth
    from oracle import Oracle
    cfg = synth.CONFIGS[cfg_name]
    inp = synth.make_inputs(cfg, seed)
    o = Oracle(cfg.N, cfg.k)
    t = {}
    t0 = time.perf_counter(); o.setup(inp["mu_q"]); t["setup"] = time.perf_counter() - t0
    t0 = time.perf_counter(); o.apply_A(inp["mu_q"], inp["u"]); t["A"] = time.perf_counter() - t0
    t0 = time.perf_counter(); o.apply_B(inp["u"]); t["B"] = time.perf_counter() - t0
    t0 = time.perf_counter(); o.apply_BT(inp["p"]); t["BT"] = time.perf_counter() - t0
    t0 = time.perf_counter(); o.wbfbt(inp["p"], cfg.iters); t["wbfbt"] = time.perf_counter() - t0
    n_v = 3 * (cfg.k * cfg.N + 1) ** 3
    return dict(step_s=sum(t.values()), t=t, A_gdofs=n_v / t["A"] / 1e9, threads=Oracle.num_threads())


def run_reference(args):
    """The tier's reference arm: the CPU oracle (no reference implementation exists).  One
    full step is ~1 min at C5 on the box's host cores, so exactly ONE step is timed, with no
    warm-up (the oracle is deterministic host code); `steps` / `warmup` report what ran."""
    import synth
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    cfg = synth.CONFIGS[args.config]
    r = oracle_full_step(args.config)
    v = 1.0 / r["step_s"]
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": unit_of(cfg), "n_gpus": args.gpus,
            "steps": 1, "warmup": 0, "ms_per_step": r["step_s"] * 1e3,
            "steps_requested": args.steps, "warmup_requested": args.warmup,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": {"workload": workload_of(cfg), "N": cfg.N, "k": cfg.k},
            "cpu_baseline": {"value": v, "unit": unit_of(cfg), "cores": r["threads"], "kind": "oracle",
                             "sample": f"one complete {cfg.name} hot-path step (setup + A + B + B^T + wBFBT "
                                       f"with 2x{cfg.iters} PCG iterations), timed once"},
            "e2e": {"value": v, "unit": unit_of(cfg), "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "components": {"A_gdofs": r["A_gdofs"], "wbfbt_applies_per_s": 1.0 / r["t"]["wbfbt"],
                           "oracle_times_s": r["t"]}}
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------- our arm
def run_ours(args):
    import numpy as np
    import torch

    import synth
    from paper_1607_03936_b200 import Context

    rank, world, local = dist_init(args.gpus)
    cfg = synth.CONFIGS[args.config]
    inp = synth.make_inputs(cfg, seed=replica_seed(rank))
    stream = torch.cuda.current_stream()
    ctx = Context(cfg.N, cfg.k, stream=stream.cuda_stream)
    d = lambda a: torch.as_tensor(a, dtype=torch.float64, device="cuda")  # noqa: E731
    mu, u, p = d(inp["mu_q"]), d(inp["u"]), d(inp["p"])
    f64 = dict(dtype=torch.float64, device="cuda")
    yA, pB, yBT, z = (torch.empty(n, **f64) for n in (ctx.n_v, ctx.n_p, ctx.n_v, ctx.n_p))
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    iters = cfg.iters

    def step():
        ctx.hotpath(mu, u, p, iters, yA, pB, yBT, z)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    l0 = ctx.query("kernel_launches")
    barrier(world)
    torch.cuda.synchronize()
    with Clocks(local) as clk:
        for i in range(args.steps):
            flush.zero_()
            ev[i][0].record(stream)
            step()
            ev[i][1].record(stream)
        torch.cuda.synchronize()
    barrier(world)
    launches = int(ctx.query("kernel_launches") - l0)
    t_ms = sum(a.elapsed_time(b) for a, b in ev)
    t_ms = max_over_ranks(t_ms, world)
    ms_per_step = t_ms / args.steps
    value = job_throughput(world, args.steps, t_ms)

    # ---- component timings (same context, L2 flushed before each rep)
    def timed(fn, reps=args.comp_reps, cold=True):
        ts = []
        for _ in range(reps):
            if cold:
                flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream); fn(); b.record(stream)
            b.synchronize()
            ts.append(a.elapsed_time(b))
        return statistics.median(ts)

    ctx.set_viscosity(mu)
    qv = torch.empty(ctx.n_p, **f64)
    tA = timed(lambda: ctx.apply_A(u, yA))
    tAw = timed(lambda: ctx.apply_A(u, yA), cold=False)
    tB = timed(lambda: ctx.apply_B(u, pB))
    tBT = timed(lambda: ctx.apply_BT(p, yBT))
    tK = timed(lambda: ctx.apply_K(1, p, qv))
    tW = timed(lambda: ctx.apply_wbfbt(p, z, iters), reps=max(3, args.comp_reps // 4))
    tS = timed(lambda: ctx.set_viscosity(mu), reps=max(3, args.comp_reps // 4))
    # ---- setup with the viscosity-gradient weights (R17)
    ctx.set_option("weights", 1)
    tSg = timed(lambda: ctx.set_viscosity(mu), reps=max(3, args.comp_reps // 4))
    ctx.set_option("weights", 0)
    ctx.set_viscosity(mu)
    # ---- Chebyshev-accelerated Jacobi as the inner solve (side r), on the
    # interval [0.1, 1.1] x a 20-step power-iteration estimate (R16); per-iteration time
    # from graph replays, (t(50) - t(10)) / 40, warm
    v0 = torch.as_tensor(np.random.default_rng(7).standard_normal(ctx.n_p), **f64)
    lam = ctx.poisson_eigmax(1, v0, 20)
    t_eig = timed(lambda: ctx.poisson_eigmax(1, v0, 20), reps=3)
    t_cheb = {it: timed(lambda: ctx.poisson_cheb(1, p, qv, it, 0.1 * lam, 1.1 * lam), reps=5, cold=False)
              for it in (10, 50, iters)}
    cheb_iter_us = (t_cheb[50] - t_cheb[10]) / 40 * 1e3
    # wBFBT with Chebyshev-Jacobi inner solves (both sides, iters steps each)
    lam_l = ctx.poisson_eigmax(0, v0, 20)
    ctx.set_inner_cheb(0.1 * lam_l, 1.1 * lam_l, 0.1 * lam, 1.1 * lam)
    tW_cheb = timed(lambda: ctx.apply_wbfbt(p, z, iters), reps=max(3, args.comp_reps // 4))
    ctx.set_inner_cheb()
    # ---- R18: diag(A) and the Chebyshev-Jacobi smoother on A (SURVEY 8(f) #1's approximate A^-1)
    yd = torch.empty(ctx.n_v, **f64)
    t_diagA = timed(lambda: ctx.get_diagA(yd), reps=5)
    vv0 = torch.as_tensor(np.random.default_rng(8).standard_normal(ctx.n_v), **f64)
    lam_a = ctx.velocity_eigmax(vv0, 10)
    t_vs = {it: timed(lambda: ctx.velocity_cheb(u, yd, it, 0.1 * lam_a, 1.1 * lam_a), reps=3, cold=False)
            for it in (2, 6)}
    vsmooth_iter_us = (t_vs[6] - t_vs[2]) / 4 * 1e3
    # ---- R19: the FGMRES Stokes solve: per outer iteration = one wBFBT
    # (iters PCG per inner solve) + a 6-step smoother on A + one Stokes operator apply
    gz = torch.zeros(ctx.n_p, **f64)
    us, ps = torch.empty(ctx.n_v, **f64), torch.empty(ctx.n_p, **f64)
    t_st, rr_st = {}, {}
    for it_o in (2, 6):
        a_ev, b_ev = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a_ev.record(stream)
        _, _, _, rr_st[it_o] = ctx.stokes_fgmres(u, gz, us, ps, 10, it_o, 0.0, iters, 6, 0.1 * lam_a, 1.1 * lam_a)
        b_ev.record(stream)
        b_ev.synchronize()
        t_st[it_o] = a_ev.elapsed_time(b_ev)
    stokes_iter_ms = (t_st[6] - t_st[2]) / 4
    # ---- SURVEY 8(f) #2b / R20, R22: the multigrids, and the full Stokes solve with the
    # multi-sinker forcing to the paper's 1e-6 reduction
    # for the three Schur approximations (Sec. 3.2, Tables 1-2)
    mg = {}
    if cfg.k == 2:
        def ev_ms(fn):
            a_ev, b_ev = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a_ev.record(stream); fn(); b_ev.record(stream)
            b_ev.synchronize()
            return a_ev.elapsed_time(b_ev)
        t_setup_mg = ev_ms(lambda: ctx.setup_mg(3, mu))
        n_levels = int(ctx.query("mg_levels"))
        pb = torch.as_tensor(inp["p"], **f64)
        ev_ms(lambda: ctx.mg_vcycle(1, pb, qv))
        t_vc = statistics.median(ev_ms(lambda: ctx.mg_vcycle(1, pb, qv)) for _ in range(5))
        t_mg = {it: statistics.median(ev_ms(lambda: ctx.poisson_mgcg(1, pb, qv, it)) for _ in range(3)) for it in (2, 10)}
        ub = torch.as_tensor(inp["u"], **f64)
        ev_ms(lambda: ctx.velocity_vcycle(ub, yd))
        t_vvc = statistics.median(ev_ms(lambda: ctx.velocity_vcycle(ub, yd)) for _ in range(5))
        fq = torch.as_tensor(synth.forcing_at_quadrature(cfg.N, cfg.k, inp["centers"], cfg.delta, cfg.omega), **f64)
        fl = ctx.load_vector(fq, torch.empty(ctx.n_v, **f64))
        solves = {}
        for name, kind in (("wBFBT", 0), ("M_p(1/mu)", 2), ("diag(A)-BFBT", 1)):
            ctx.set_schur(kind)
            ctx.set_viscosity(mu)
            ctx.setup_mg(3, mu)
            ctx.set_velocity_mg(2)
            ctx.set_inner_mg(8 if kind == 0 else 0)
            max_it = 300
            ms = ev_ms(lambda: solves.__setitem__(name, ctx.stokes_fgmres(fl, gz, us, ps, 200, max_it, 1e-6, 20, 6, 1.0,
                                                                          2.0)[2:]))
            it_s, rr_s = solves[name]
            solves[name] = {"fgmres_iterations": it_s, "relres": rr_s, "solve_ms": ms,
                            "converged_1e-6": rr_s <= 1e-6}
        ctx.set_schur(0)
        ctx.set_viscosity(mu)
        mg = {"setup_mg_ms": t_setup_mg, "levels": n_levels, "pressure_vcycle_ms": t_vc,
              "mgcg_iter_ms": (t_mg[10] - t_mg[2]) / 8, "velocity_vcycle_ms": t_vvc,
              "stokes_solve": solves,
              "note": "SURVEY 8(f) #2b (R20, R22) and #1, #3 (not in the step): FGMRES(200) on [A B^T; B 0] with "
                      "f = the multi-sinker load vector, g = 0, rtol 1e-6, max 300 iterations; At^-1 = 2 velocity "
                      "V-cycles; wBFBT inner solves MG-PCG(8); diag(A)-BFBT inner PCG(20)"}
    # ---- dominant kernel: the fused Poisson operator inside the PCG loops (2 x iters
    # launches per step).  Profiled pass: the same hot-path step with a CUDA-event
    # pair around every such launch (library option "profile": plain launches on
    # the context stream), so its duration and share of the step are measured live.
    prof_steps = max(2, min(args.steps, 5))
    ctx.set_option("profile", 1)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for _ in range(prof_steps):
        step()
    b.record(stream)
    b.synchronize()
    prof_step_ms = a.elapsed_time(b) / prof_steps
    k_ms, k_n = ctx.query("prof_k_ms"), int(ctx.query("prof_k_count"))
    ctx.set_option("profile", 0)
    k_avg = k_ms / max(k_n, 1)

    n_el, n_nodes, n_v, n_p, n_q = ctx.n_el, ctx.n_nodes, ctx.n_v, ctx.n_p, ctx.n_q
    hbm, peak_kind = peaks()
    bytes_A = 8 * (n_el * n_q + 2 * n_v)          # mu~ + u in + y out
    # fused K kernel per launch: p_old and z = Minv r (stored by the PCG
    # update; with option kz = 0: r and Minv) in, mode-major n_p each; X^-1 (nodal) in;
    # p_new, q out
    zbox = bool(ctx.query("kz"))
    bytes_K = 8 * ((4 if zbox else 5) * n_p + n_nodes)
    kname = "k_K2_tma" if ctx.query("k_tma") else "k_K2_fused"
    roof = {"bound": "hbm", "kernel": f"{kname} (PCG: p-update + B^T + X^-1 + B + <p,q>)",
            "achieved": bytes_K / (k_avg * 1e-3) / 1e9, "peak": hbm, "unit": "GB/s",
            "frac": bytes_K / (k_avg * 1e-3) / 1e9 / hbm, "traffic": ncu_traffic(kname),
            "traffic_source": "profiles/ncu_traffic.json (dram__bytes_read.sum + dram__bytes_write.sum, "
                              "one ncu --set full capture)", "peak_kind": peak_kind,
            "algorithmic_bytes_per_launch": bytes_K,
            "algorithmic_bytes_def": ("8*(4*n_p + n_nodes): p_old, z in; p_new, q out; X in" if zbox else
                                      "8*(5*n_p + n_nodes): p_old, r, Minv in; p_new, q out; X in"), "launch_ms": k_avg, "launches_per_step": k_n / prof_steps,
            "share_of_step": k_ms / prof_steps / ms_per_step, "profiled_step_ms": prof_step_ms,
            "timing": "CUDA-event record nodes around every launch inside the captured PCG-loop graphs "
                      "(graph launch gaps as in the timed step)"}
    tKw = k_avg

    # ---- the high-order configuration C4 (Q4 x P3disc, BASELINE.json configs[3]), not in the
    # step: A / B / B^T GDOF/s, wBFBT applies/s at its 2 x 50 PCG iterations, and the fused
    # k = 4 Poisson kernel (k_K4_fused, k4_fused.cuh) launch time inside the PCG graphs
    c4 = None
    if args.config != "C4" and not args.no_c4:
        cfg4 = synth.CONFIGS["C4"]
        inp4 = synth.make_inputs(cfg4, seed=replica_seed(rank))
        ctx4 = Context(cfg4.N, cfg4.k, stream=stream.cuda_stream)
        mu4, u4, p4 = d(inp4["mu_q"]), d(inp4["u"]), d(inp4["p"])
        ctx4.set_viscosity(mu4)
        y4, q4, z4 = torch.empty(ctx4.n_v, **f64), torch.empty(ctx4.n_p, **f64), torch.empty(ctx4.n_p, **f64)
        tA4 = timed(lambda: ctx4.apply_A(u4, y4))
        tB4 = timed(lambda: ctx4.apply_B(u4, q4))
        tBT4 = timed(lambda: ctx4.apply_BT(p4, y4))
        tW4 = timed(lambda: ctx4.apply_wbfbt(p4, z4, cfg4.iters), reps=max(3, args.comp_reps // 4))
        ctx4.set_option("profile", 1)
        ctx4.apply_wbfbt(p4, z4, cfg4.iters)
        torch.cuda.synchronize()
        k4_ms, k4_n = ctx4.query("prof_k_ms"), int(ctx4.query("prof_k_count"))
        ctx4.set_option("profile", 0)
        n4 = ctx4.n_v
        c4 = {"workload": workload_of(cfg4), "A_gdofs": n4 / (tA4 * 1e-3) / 1e9, "A_ms": tA4,
              "B_gdofs": n4 / (tB4 * 1e-3) / 1e9, "BT_gdofs": n4 / (tBT4 * 1e-3) / 1e9,
              "wbfbt_ms": tW4, "wbfbt_applies_per_s": 1e3 / tW4,
              "k4_fused_launch_us": 1e3 * k4_ms / max(k4_n, 1), "k4_fused_launches_per_apply": k4_n,
              "note": "C4 (not in the step): L2 flushed before each rep; k_K4_fused timed by CUDA-event record "
                      "nodes around every launch of one wBFBT apply's captured PCG loops"}
        ctx4.close()
        del mu4, u4, p4, y4, q4, z4

    # ---- the slab code path on this one GPU (one rank, no communication): the
    # cost of its unfused K_w (B^T, plane sum, B) and launch-by-launch PCG against the fused path
    from paper_1607_03936_b200 import SlabContext, ThreadComm
    sctx = SlabContext(cfg.N, cfg.k, ThreadComm.group(1, SlabContext.plane_cap(cfg.N, cfg.k), "cuda")[0],
                       stream=stream.cuda_stream)
    sctx.set_viscosity(mu)
    tWs = timed(lambda: sctx.apply_wbfbt(p, z, iters), reps=3)
    tKs = timed(lambda: sctx.apply_K(1, p, qv), reps=10)
    slab = {"wbfbt_ms": tWs, "wbfbt_applies_per_s": 1e3 / tWs, "K_ms_cold": tKs, "ranks": 1,
            "note": "z-slab decomposition code path with one rank (not in the step): unfused K_w and a "
                    "launch-by-launch device-scalar PCG; multi-rank runs: bench.py --slab under torchrun"}
    sctx.close()

    # ---- end to end through the host entry (pinned buffers)
    pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()  # noqa: E731
    hmu, hu, hp = pin(inp["mu_q"]), pin(inp["u"]), pin(inp["p"])
    outs = [torch.empty(n, dtype=torch.float64).pin_memory() for n in (n_v, n_p, n_v, n_p)]
    ctx.hotpath_host(hmu, hu, hp, iters, *outs)
    te = []
    barrier(world)
    for _ in range(args.steps):
        flush.zero_()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        ctx.hotpath_host(hmu, hu, hp, iters, *outs)
        te.append(time.perf_counter() - t0)
    te_tot = max_over_ranks(sum(te), world)
    e2e = world * args.steps / te_tot
    h2d = 8 * (n_el * n_q + n_v + n_p)
    d2h = 8 * (2 * n_v + 2 * n_p)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        r = oracle_sample(args.config)
        cpu = {"value": 1.0 / r["step_s"], "unit": unit_of(cfg), "cores": r["threads"], "kind": "oracle",
               "sample": r["sample"], "A_gdofs": r["A_gdofs"], "sample_wall_s": r["sample_s"]}

    if rank == 0:
        line = {"metric": METRIC, "value": value,
                "unit": unit_of(cfg),
                "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic",
                "config": {"workload": workload_of(cfg), "N": cfg.N, "k": cfg.k,
                           "l2": "flushed (256 MiB memset) before every timed step",
                           "parallelism": f"replicas{world}"},
                "components": {
                    "A_gdofs": n_v / (tA * 1e-3) / 1e9, "A_ms": tA, "A_bytes": bytes_A,
                    "A_hbm_frac": bytes_A / (tA * 1e-3) / 1e9 / hbm,
                    "A_fp64_frac": A_DFMA_PER_ELEMENT * n_el / (tA * 1e-3) / DFMA_PEAK_INSTR_PER_S,
                    "A_ms_warm": tAw, "A_gdofs_warm": n_v / (tAw * 1e-3) / 1e9,
                    "B_gdofs": n_v / (tB * 1e-3) / 1e9, "BT_gdofs": n_v / (tBT * 1e-3) / 1e9,
                    "B_ms": tB, "BT_ms": tBT,
                    "B_hbm_frac": 8 * (n_v + n_p) / (tB * 1e-3) / 1e9 / hbm,
                    "BT_hbm_frac": 8 * (n_v + n_p) / (tBT * 1e-3) / 1e9 / hbm,
                    "K_ms_cold": tK, "K_ms_warm": tKw, "wbfbt_ms": tW, "wbfbt_applies_per_s": 1e3 / tW,
                    "setup_ms": tS, "setup_grad_weights_ms": tSg,
                    "cheb": {"iter_us": cheb_iter_us, "solve_ms": t_cheb[iters], "iters": iters,
                             "wbfbt_cheb_inner_ms": tW_cheb, "wbfbt_cheb_inner_applies_per_s": 1e3 / tW_cheb,
                             "interval": [0.1 * lam, 1.1 * lam], "eigmax_20_ms": t_eig,
                             "k_cheb_bytes_per_launch": 64 * n_p,
                             "note": "SURVEY 8(f) #2 (not in the step): x = P Cheb(K_r, P b), R16"},
                    "velocity_smoother": {"diagA_ms": t_diagA, "iter_us": vsmooth_iter_us,
                                          "note": "R18 (not in the step): x = Cheb(M A M, M b), Jacobi mask/diag(A)"},
                    "multigrid": mg,
                    "stokes_fgmres": {"iter_ms": stokes_iter_ms, "relres_after": {str(k): v for k, v in rr_st.items()},
                                      "note": "R19 (not in the step): FGMRES on [A B^T; B 0], f = u, g = 0; per "
                                              "iteration wBFBT (2 x iters PCG) + 6 smoother steps"},
                    "C4": c4, "slab": slab},
                "roofline": roof,
                "e2e": {"value": e2e, "unit": unit_of(cfg), "h2d_bytes_per_step": h2d,
                        "d2h_bytes_per_step": d2h},
                "gpu_launches": launches,
                "clocks": clk.summary(),
                "cpu_baseline": cpu}
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()
    return 0

# ---------------------------------------------------------------------- slab decomposition (opt-in)
def run_slab(args):
    """--slab: ONE global problem on the box N x N x (R N), R = world size, rank r owning the
    r-th cube.  The step is the same hot-path call on a
    slab context; its shared-plane sums and scalar all-reduces go through torch.distributed
    (NCCL).  Strong coupling per PCG iteration, so this is the communication-bound mode the
    survey predicts; the default (replicas) stays the headline."""
    import torch

    import synth
    from paper_1607_03936_b200 import DistComm, SlabContext, ThreadComm

    rank, world, local = dist_init(args.gpus)
    cfg = synth.CONFIGS[args.config]
    inp = synth.make_inputs(cfg, seed=replica_seed(rank))  # rank r's cube of the global viscosity
    stream = torch.cuda.current_stream()
    cap = SlabContext.plane_cap(cfg.N, cfg.k)
    comm = DistComm(cap, "cuda") if world > 1 else ThreadComm.group(1, cap, "cuda")[0]
    ctx = SlabContext(cfg.N, cfg.k, comm, stream=stream.cuda_stream)
    d = lambda a: torch.as_tensor(a, dtype=torch.float64, device="cuda")  # noqa: E731
    mu, u, p = d(inp["mu_q"]), d(inp["u"]), d(inp["p"])
    f64 = dict(dtype=torch.float64, device="cuda")
    yA, pB, yBT, z = (torch.empty(n, **f64) for n in (ctx.n_v, ctx.n_p, ctx.n_v, ctx.n_p))
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    iters = cfg.iters
    for _ in range(args.warmup):
        ctx.hotpath(mu, u, p, iters, yA, pB, yBT, z)
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    l0, x0, a0 = ctx.query("kernel_launches"), comm.n_exchange, comm.n_allreduce
    barrier(world)
    torch.cuda.synchronize()
    with Clocks(local) as clk:
        for i in range(args.steps):
            flush.zero_()
            ev[i][0].record(stream)
            ctx.hotpath(mu, u, p, iters, yA, pB, yBT, z)
            ev[i][1].record(stream)
        torch.cuda.synchronize()
    barrier(world)
    t_ms = max_over_ranks(sum(a.elapsed_time(b) for a, b in ev), world)
    if rank == 0:
        n_v_glob = 3 * (cfg.k * cfg.N + 1) ** 2 * (cfg.k * cfg.N * world + 1)
        line = {"metric": METRIC, "value": args.steps / (t_ms * 1e-3),
                "unit": f"global hot-path steps/s on the {cfg.N}x{cfg.N}x{cfg.N * world} box "
                        f"(setup + A + B + B^T + wBFBT 2x{iters} PCG), slab-decomposed",
                "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_ms / args.steps,
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic",
                "config": {"workload": workload_of(cfg) + f", z-stacked x{world}", "N": cfg.N, "k": cfg.k,
                           "l2": "flushed (256 MiB memset) before every timed step",
                           "parallelism": f"slab{world}", "n_v_global": n_v_glob},
                "gpu_launches": int(ctx.query("kernel_launches") - l0),
                "comm": {"plane_exchanges_per_step": (comm.n_exchange - x0) / args.steps,
                         "allreduces_per_step": (comm.n_allreduce - a0) / args.steps,
                         "plane_bytes": 8 * cap, "backend": "nccl" if world > 1 else "none"},
                "clocks": clk.summary()}
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C5")
    ap.add_argument("--comp-reps", type=int, default=30)  # median of >= 30 reps
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-c4", action="store_true")  # skip the high-order C4 component block
    ap.add_argument("--slab", action="store_true")  # one global z-slab-decomposed problem instead of replicas
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    if args.slab:
        return run_slab(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
