#!/usr/bin/env python
"""Benchmark of the ExpRK22/WENO5 sigma-step (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
                    [--config c2|c1|c3|c4|c5] [--no-e2e] [--no-cpu] [--no-fp32]

Workload (N = 1): BASELINE config C2 = the paper's full-size grid, Set 4
(N_rho = 10000, N_theta = 3584, Sigma = 120, N_sigma = 2400, homogeneous air)
with the rho-modulated N-wave; synthetic inputs, fp64 headline
and fp32 beside it.  One step = one full ExpRK22 sigma-step (4 transforms,
2 WENO evaluations, 2 spectral combines) on the whole grid; the metric is
grid-cell updates per second (cells x steps / s).

For N > 1 (torchrun, one rank per GPU) every rank marches an independent
member of an ensemble (BASELINE C4's sharding: no collective on the data
path), so per-GPU work is fixed -> "scaling": "weak".  Timing: W warm-up
steps, then exactly K steps between barrier + synchronize, CUDA events on
the plan's stream, max over ranks.  The working set (>= 3 GB at C2) exceeds
the 126 MB L2, so no flush is needed between steps.

``--impl reference`` times the reference algorithm's CPU implementation on
this host (the oracle port in oracle/: the reference's own WENO arithmetic
in C + scipy's pocketfft, all host threads) on the same config; rank 0 only.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "grid-cell updates/s per KZK ExpRK22 step"
UNIT = "cell-steps/s"
PEAKS_FILE = os.path.join(ROOT, "MEASURED_PEAKS.json")
TRAFFIC_FILE = os.path.join(ROOT, "profiles", "ncu_traffic.json")
FALLBACK_HBM_GBS = 6650.0


# ------------------------------------------------------------------ workload

def workload(name: str):
    import paper_2103_06080_b200 as nw

    if name == "c1":
        cfg = nw.DomainConfig(Sigma=30.0, N_sigma=300, N_rho=625, N_theta=448)
        desc = "C1 demo grid 625x448 homogeneous N-wave"
    elif name == "c3":
        cfg = nw.preset_config(1)
        desc = "C3 Set-1 1250x448 turbulent (seed 0) N-wave"
    elif name == "c5":
        cfg = nw.DomainConfig(Sigma=120.0, N_sigma=6000, N_rho=8192, N_theta=16384)
        desc = "C5 large grid 8192x16384 homogeneous rho-modulated N-wave"
    elif name == "c4":
        cfg = nw.preset_config(1)
        desc = ("C4 ensemble of 256 Set-1 (1250x448) N-waves, amplitude U[0.5,1.5] x "
                "duration U[0.75,1.25] (seed 2026), members sharded over ranks")
    else:
        cfg = nw.preset_config(4)
        desc = "C2 paper Set 4 10000x3584 homogeneous air, rho-modulated N-wave"
    return cfg, desc


ENSEMBLE_MEMBERS = 256


def members_for(cname: str, world: int, rank: int) -> range:
    """Members this rank marches: the C4 shard, or one independent replica."""
    from paper_2103_06080_b200.ensemble import shard_members

    if cname == "c4":
        return shard_members(ENSEMBLE_MEMBERS, world, rank)
    return range(rank, rank + 1)


def initial_fields(cfg, cname: str, members: range):
    """(n, N_rho, N_theta) initial fields of the given members."""
    import paper_2103_06080_b200 as nw

    if cname == "c4":
        all_v0, _, _ = nw.ensemble_nwaves(cfg, ENSEMBLE_MEMBERS, seed=2026)
        return all_v0[members.start:members.stop]
    return np.stack([initial_field(cfg, r) for r in members])


def initial_field(cfg, rank: int = 0):
    import paper_2103_06080_b200 as nw

    _, rho, theta = nw.build_axes(cfg)
    v0 = nw.rho_modulated(cfg, nw.initial_nwave(rho, theta, cfg.A, cfg.B))
    return v0.values * (1.0 - 0.02 * rank)


def coefficient_fields(cfg, name: str, rows: int):
    import paper_2103_06080_b200 as nw

    rows = min(rows, cfg.N_sigma + 1)
    if name == "c3":
        sig, _, _ = nw.build_axes(cfg)
        spec = nw.sample_modes(nw.TurbulenceParams(seed=0))
        return nw.evaluate_fields(spec, spec.lam, sig[:rows], nw.rho_nodes_closed(cfg))
    return nw.zero_fields(rows, cfg.N_rho + 1)


# ------------------------------------------------------------------ clocks

class ClockSampler:
    """Samples SM clock and throttle reasons with NVML while running."""

    REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
               0x2: "applications_clocks_setting", 0x1: "gpu_idle"}

    def __init__(self, index: int, period: float = 0.02):
        self.samples, self.reasons = [], set()
        self.max_mhz = None
        self._stop = threading.Event()
        self._ok = False
        try:
            import pynvml

            pynvml.nvmlInit()
            vis = os.environ.get("CUDA_VISIBLE_DEVICES")
            if vis:
                ids = [x for x in vis.split(",") if x.strip()]
                ent = ids[index].strip() if index < len(ids) else str(index)
                h = (pynvml.nvmlDeviceGetHandleByUUID(ent) if not ent.isdigit()
                     else pynvml.nvmlDeviceGetHandleByIndex(int(ent)))
            else:
                h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.nvml, self.h = pynvml, h
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
            self._ok = True
        except Exception:
            pass
        self.period = period
        self._t = threading.Thread(target=self._run, daemon=True)

    def _reasons(self):
        n = self.nvml
        fn = getattr(n, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
            getattr(n, "nvmlDeviceGetCurrentClocksThrottleReasons")
        return fn(self.h)

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nvml.nvmlDeviceGetClockInfo(self.h, self.nvml.NVML_CLOCK_SM))
                bits = self._reasons()
                for b, name in self.REASONS.items():
                    if bits & b and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self._ok:
            self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._ok:
            self._t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["nvml-unavailable"]}
        return {"sm_mhz": float(statistics.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ------------------------------------------------------------------ roofline

KERNELS = ("theta_c2r", "weno", "theta_r2c", "rho_stage1", "theta_c2r", "weno", "theta_r2c",
           "rho_stage2")


def table_read_fraction(n: int, pair55: bool = False) -> float:
    """Share of each multiplier-table row the rho combine reads: tables are
    read at the canonical +-f position (csrc/fft.cuh sym_pos), i.e. block 0 of
    the first-stage radix r1 plus half of the other blocks.  r1 restates the
    host planner (capi.cu plan_fft, max product 16, no split)."""
    m, c = n, {}
    for r in (2, 3, 5, 7):
        c[r] = 0
        while m % r == 0:
            m //= r
            c[r] += 1
    c2 = c[2]
    c2 -= min(c[7], c2)                       # 7 pairs with 2
    if pair55:                                 # fp32 plans: radix-25 passes first
        c[5] %= 2
    for _ in range(c[5]):                      # 5 pairs with 3, else 2
        if c[3] > 0:
            c[3] -= 1
        elif c2 > 0:
            c2 -= 1
    c3 = c[3]
    while c3 > 0:                              # 3.4 / 3.3 / 3.2 / 3
        if c2 >= 2:
            c2 -= 2; c3 -= 1
        elif c3 >= 2:
            c3 -= 2
        elif c2 >= 1:
            c2 -= 1; c3 -= 1
        else:
            c3 -= 1
    head = {1: 2, 2: 4, 3: 8}.get(c2 % 4)
    r1 = head or (7 if c[7] else 5 if (c[5] or pair55 and n % 25 == 0) else 3 if c[3]
                  else 4 if n % 4 == 0 else n)
    if r1 <= 1 or n % r1:
        return 1.0
    mm = n // r1
    canon = mm + ((r1 - 1) // 2) * mm + ((mm + 1) // 2 if r1 % 2 == 0 else 0)
    return canon / n


def algorithmic_bytes(cfg, precision: str, batch: int = 1, design: bool = False):
    """HBM bytes per launch of each kernel slot.

    Algorithmic (the roofline's bytes): per member theta c2r,
    WENO and theta r2c move one field in and one out (2F); a rho pass reads
    two spectra (b~ and the state Vh or U) and writes two (4F).  The
    multiplier tables are excluded (8(d)).

    ``design=True`` adds what this implementation must also stream: the
    multiplier tables (E, Phi1, Phi1m2 in stage 1, Phi2 in stage 2), read once
    per launch for all members of a batch and only at canonical +-f positions
    (table_read_fraction of each row).
    """
    r = 8 if precision == "double" else 4
    phys = cfg.N_rho * cfg.N_theta * r
    spec = cfg.N_rho * (cfg.N_theta // 2 + 1) * 2 * r
    c2r = batch * (spec + phys)
    weno = batch * 2 * phys
    r2c = batch * (phys + spec)
    rho1 = rho2 = batch * 4 * spec
    if design:
        # 0.6 at N_rho = 10000 (r1 = 5); long fp32 columns use radix-25 passes (capi.cu)
        tf = table_read_fraction(cfg.N_rho, precision == "single" and cfg.N_rho >= 5000)
        rho1 += int(3 * spec * tf)
        rho2 += int(spec * tf)
    return [c2r, weno, r2c, rho1, c2r, weno, r2c, rho2]


WENO_FLOP_PER_CELL = 287
FP_PEAKS_FILE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "fp_peaks.json")


def fp_peak(precision):
    """Measured FMA peak (TFLOP/s) of the pipe WENO runs on, or None."""
    try:
        with open(FP_PEAKS_FILE) as fh:
            d = json.load(fh)
        return float(d["fp64_dfma_tflops" if precision == "double" else "fp32_ffma2_tflops"])
    except Exception:
        return None


def hbm_peak():
    try:
        with open(PEAKS_FILE) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback"


def ncu_traffic(config: str, precision: str, kernel: str, key: str = "dram_bytes_per_launch"):
    try:
        with open(TRAFFIC_FILE) as fh:
            t = json.load(fh)
        return t[config][precision][kernel][key]
    except Exception:
        return None


def roofline_block(cfg, cname, precision, kernel_ms_total, n_prof, batch=1):
    abytes = algorithmic_bytes(cfg, precision, batch)
    dbytes = algorithmic_bytes(cfg, precision, batch, design=True)
    peak, kind = hbm_peak()
    per = []
    for i, name in enumerate(KERNELS):
        ms = kernel_ms_total[i] / n_prof
        if ms <= 0:
            continue
        per.append({"slot": i, "kernel": name, "ms": round(ms, 5), "bytes": abytes[i],
                    "GBs": round(abytes[i] / (ms * 1e-3) / 1e9, 1),
                    "frac": round(abytes[i] / (ms * 1e-3) / 1e9 / peak, 4),
                    "design_bytes": dbytes[i]})
    # WENO is arithmetic-bound: its roofline is the measured FP64 DFMA (fp64) or
    # packed-FP32 FFMA2 (fp32) peak (profiles/fp_peaks.json, tools/fp_peak.cu), on
    # the reference's 287 flop per cell
    fpk = fp_peak(precision)
    for p in per:
        if p["kernel"] == "weno" and fpk:
            tf = WENO_FLOP_PER_CELL * cfg.N_rho * cfg.N_theta * batch / (p["ms"] * 1e-3) / 1e12
            p.update({"TFLOPs": round(tf, 2), "fp_peak_TFLOPs": fpk, "frac_fp": round(tf / fpk, 4)})
    # dominant kernel type by summed time over the step
    by_kernel = {}
    for p in per:
        # both rho stages are launches of the same kernel (k_rho, two modes)
        group = "rho_pass" if p["kernel"].startswith("rho") else p["kernel"]
        d = by_kernel.setdefault(group, {"ms": 0.0, "bytes": 0, "dbytes": 0, "n": 0})
        d["ms"] += p["ms"]; d["bytes"] += p["bytes"]; d["dbytes"] += p["design_bytes"]; d["n"] += 1
    step_ms = sum(p["ms"] for p in per)

    def hbm_figures(g):
        e = by_kernel[g]
        sec = e["ms"] / e["n"] * 1e-3
        ach = e["bytes"] / e["n"] / sec / 1e9
        des = e["dbytes"] / e["n"] / sec / 1e9
        return ach, des

    dom = max(by_kernel, key=lambda k: by_kernel[k]["ms"])
    achieved, design = hbm_figures(dom)
    blk = {"bound": "hbm", "kernel": dom, "achieved": round(achieved, 1), "peak": peak,
           "peak_kind": kind, "unit": "GB/s", "frac": round(achieved / peak, 4),
           "bytes_basis": "SURVEY 8(d) algorithmic: 4F per rho-pass launch, 2F per theta c2r / "
                          "WENO / theta r2c launch, multiplier tables excluded",
           "achieved_design": round(design, 1), "frac_design": round(design / peak, 4),
           "traffic": ncu_traffic(cname, precision, dom),
           "share_of_step": round(by_kernel[dom]["ms"] / step_ms, 4),
           "step_frac_16F": None,
           "per_kernel": per}
    wk = [p for p in per if "frac_fp" in p]
    if wk:
        tf = sum(p["TFLOPs"] for p in wk) / len(wk)
        blk["weno_fp_roofline"] = {
            "bound": "fp64_dfma" if precision == "double" else "fp32_ffma2", "kernel": "weno",
            "achieved": round(tf, 2), "peak": fpk, "unit": "TFLOP/s", "frac": round(tf / fpk, 4),
            "flop_basis": f"{WENO_FLOP_PER_CELL} flop per cell (the reference's count, SURVEY 8(d)); "
                          "peak measured by tools/fp_peak.cu (profiles/fp_peaks.json)"}
    if dom == "weno":
        # WENO moves 2F per launch but is arithmetic-bound (no tensor-core form):
        # its limiter is the FP64 pipe (fp64) / the FMA-pipe issue rate (fp32),
        # from the committed ncu capture (profiles/ncu_traffic.json)
        key = "fp64_pipe_pct" if precision == "double" else "fma_pipe_pct"
        blk["limiter"] = {"pipe": "fp64" if precision == "double" else "fma",
                          "busy_pct_ncu": ncu_traffic(cname, precision, dom, key),
                          "issue_pct_ncu": ncu_traffic(cname, precision, dom, "issue_pct")}
        # and the largest bandwidth-bound kernel's HBM figures beside it
        hb = max((g for g in by_kernel if g != "weno"), key=lambda g: by_kernel[g]["ms"],
                 default=None)
        if hb is not None:
            ach, des = hbm_figures(hb)
            blk["hbm_kernel"] = {"kernel": hb, "achieved": round(ach, 1),
                                 "frac": round(ach / peak, 4), "frac_design": round(des / peak, 4),
                                 "traffic": ncu_traffic(cname, precision, hb),
                                 "share_of_step": round(by_kernel[hb]["ms"] / step_ms, 4)}
    return blk


# ------------------------------------------------------------------ arms

def dist_setup():
    import torch

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist

        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    elif torch.cuda.is_available():
        torch.cuda.set_device(local)
    return world, rank, local


def max_over_ranks(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist

    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(world):
    if world > 1:
        import torch.distributed as dist

        dist.barrier()


def time_precision(cfg, cname, precision, steps, warmup, world, rank, local, clocks=True):
    import torch
    from paper_2103_06080_b200.plan import DevicePlan

    eps = 2.0 ** -53 if precision == "double" else 2.0 ** -24
    n_prof = max(2, min(steps, 10))
    rows = warmup + steps + n_prof + 2
    fields = coefficient_fields(cfg, cname, rows)
    members = members_for(cname, world, rank)
    plan = DevicePlan(cfg.N_rho, cfg.N_theta, len(members), precision, cfg.d_sigma,
                      cfg.rho_span, cfg.theta_span, cfg.A, cfg.B, eps,
                      torch.device("cuda", local))
    plan.set_coeffs(fields.u_par, fields.u_perp, fields.du_perp_drho,
                    n_rows=fields.u_par.shape[0])
    plan.load_physical(initial_fields(cfg, cname, members))
    plan.march("exprk22", 0, warmup, timing=False)
    torch.cuda.synchronize(local)
    barrier(world)
    torch.cuda.synchronize(local)
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    sampler = ClockSampler(local)
    with sampler:
        start.record(plan.stream)
        max_abs, _, _ = plan.march("exprk22", warmup, steps, timing=False)
        end.record(plan.stream)
        torch.cuda.synchronize(local)
    barrier(world)
    ms = start.elapsed_time(end)
    ms_max = max_over_ranks(ms, world)
    kernel_ms = plan.profile_kernels("exprk22", warmup + steps, n_prof)
    cells = cfg.N_rho * cfg.N_theta
    total_members = ENSEMBLE_MEMBERS if cname == "c4" else world
    value = total_members * cells * steps / (ms_max * 1e-3)
    roof = roofline_block(cfg, cname, precision, kernel_ms, n_prof, len(members))
    # whole step against SURVEY 8(d)'s 16F per cell-step (128 B fp64, 64 B fp32)
    per_cell = 16 * (8 if precision == "double" else 4)
    roof["step_frac_16F"] = round(value / world * per_cell / (roof["peak"] * 1e9), 4)
    res = {
        "value": value,
        "ms_per_step": ms_max / steps,
        "roofline": roof,
        "max_abs_v_last": float(max_abs[0, -1]),
        "clocks": sampler.summary() if clocks else None,
        "plan_bytes": plan.bytes,
    }
    plan.close()
    return res


def time_slab(cfg, steps, warmup, world, rank, local):
    """C5: one grid split into rho slabs over the ranks (slab.py), fp64."""
    import torch
    from paper_2103_06080_b200.slab import SlabMarch

    fields = coefficient_fields(cfg, "c5", warmup + steps + 2)
    sm = SlabMarch(cfg, fields, device=torch.device("cuda", local),
                   max_steps=warmup + steps + 1)
    rows = sm.geo.rows()
    sm.load(initial_field(cfg)[rows.start:rows.stop])
    sm.march(n0=0, steps=warmup)
    torch.cuda.synchronize(local)
    barrier(world)
    torch.cuda.synchronize(local)
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    sampler = ClockSampler(local)
    with sampler:
        start.record()
        sm.march(n0=warmup, steps=steps)
        end.record()
        torch.cuda.synchronize(local)
    barrier(world)
    ms = max_over_ranks(start.elapsed_time(end), world)
    return {"value": cfg.N_rho * cfg.N_theta * steps / (ms * 1e-3), "ms_per_step": ms / steps,
            "clocks": sampler.summary()}


def e2e_precision(cfg, cname, precision, steps, world, rank, local):
    """The same metric end to end through the public API with host buffers.

    Single grids: ``run_exprk22(config, v0, fields)`` -- exactly the
    reference's call (``nwave/exprk.py:219-224``: full N_sigma march, default
    per-step timing buckets, numpy in and out) for fp64; ``precision=`` is the
    one extra keyword for fp32.  The timed region holds the plan build (device
    tables), the H2D of V0 and of the N_sigma + 1 coefficient rows, the whole
    march and the D2H of the float64 final field.  C4: ``run_ensemble`` over
    this rank's members, full length, final fields back to the host.
    """
    import torch
    import paper_2103_06080_b200 as nw

    members = members_for(cname, world, rank)
    v0 = initial_fields(cfg, cname, members)
    n_full = cfg.N_sigma
    fields = coefficient_fields(cfg, cname, n_full + 1)
    kw = {} if precision == "double" else {"precision": precision}
    if cname != "c4":
        # untimed warm-up call (3 steps): CUDA graph capture, the device memory
        # pool and the page-locked staging chunks are set up as in any repeated use
        nw.run_exprk22(cfg, nw.Field2D(v0[0]), fields, max_steps=3, **kw)
    torch.cuda.synchronize(local)
    barrier(world)
    t0 = time.perf_counter()
    if cname == "c4":
        from paper_2103_06080_b200.ensemble import run_ensemble

        res = run_ensemble(cfg, v0, fields, precision=precision,
                           members=range(0, len(members)), device=torch.device("cuda", local))
        final = res.final
        call = "run_ensemble(config, v0s, fields) over this rank's members"
    else:
        rep = nw.run_exprk22(cfg, nw.Field2D(v0[0]), fields, **kw)
        final = rep.final.values
        assert rep.n_steps == n_full
        call = "run_exprk22(config, v0, fields)" + ("" if not kw else ", precision='single'")
    wall = time.perf_counter() - t0
    wall_max = max_over_ranks(wall, world)
    h2d = v0.size * 8 + 3 * (n_full + 1) * cfg.N_rho * 8
    d2h = final.size * 8 + 8 * n_full * len(members)
    total = ENSEMBLE_MEMBERS if cname == "c4" else world
    return {"value": total * cfg.N_rho * cfg.N_theta * n_full / wall_max, "unit": UNIT,
            "h2d_bytes_per_step": int(h2d / n_full), "d2h_bytes_per_step": int(d2h / n_full),
            "wall_s": wall_max, "steps": n_full, "precision": precision,
            "note": f"{call}: the full N_sigma = {n_full}-step run with numpy inputs and "
                    "outputs; timed region = plan build + H2D (V0, coefficient rows) + march + "
                    "D2H of the float64 final field, after one untimed 3-step warm-up call"}


def cpu_reference(cfg, cname, steps_cap=3, warm=1, threads=0, precision="double"):
    """The reference algorithm on the host cores (oracle port)."""
    from oracle import nwave_oracle as oracle

    oracle.build()
    cores = threads if threads > 0 else oracle.host_cores()
    n = warm + steps_cap
    fields = coefficient_fields(cfg, cname, n + 1)
    v0 = initial_fields(cfg, cname, range(0, 1))[0]
    if cname == "c4":
        # the fair CPU ensemble baseline is process-parallel (cores x 1 thread,
        # SURVEY 8(d)): time one member on one thread, credit perfect scaling
        run = oracle.march(cfg, v0, fields, precision=precision, threads=1, max_steps=n)
        med = float(np.median(run.step_seconds[warm:]))
        return {"value": cores * cfg.N_rho * cfg.N_theta / med, "unit": UNIT, "cores": cores,
                "kind": "port", "s_per_step": med / cores,
                "sample": f"{steps_cap} timed steps of one C4 member on 1 thread after {warm} "
                          f"warm-up, x{cores} cores (ideal process-parallel ensemble)"}
    run = oracle.march(cfg, v0, fields, precision=precision, threads=cores, max_steps=n)
    secs = run.step_seconds[warm:]
    med = float(np.median(secs))
    return {"value": cfg.N_rho * cfg.N_theta / med, "unit": UNIT, "cores": cores,
            "kind": "port", "s_per_step": med,
            "sample": f"{steps_cap} timed ExpRK22 steps after {warm} warm-up on {cname} "
                      f"({precision}), median; oracle/ port = reference WENO5 arithmetic "
                      "in C (OpenMP) + scipy pocketfft (workers=cores) + numpy combines"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="c2", choices=["c1", "c2", "c3", "c4", "c5"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-fp32", action="store_true")
    args = ap.parse_args()
    warmup = max(args.warmup, 3)
    cfg, desc = workload(args.config)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    config = {"workload": desc, "n_rho": cfg.N_rho, "n_theta": cfg.N_theta,
              "cells": cfg.N_rho * cfg.N_theta, "sigma_steps_full_run": cfg.N_sigma,
              "scheme": "exprk22",
              "l2": "working set > 3 GB >> 126 MB L2 (no flush needed)" if args.config in ("c2", "c5")
              else "working set partly L2-resident",
              "parallelism": (f"ensemble-shard x{args.gpus}" if args.gpus > 1 or args.config == "c4"
                              else "single grid, 1 GPU")}
    if args.config == "c4":
        config["members"] = ENSEMBLE_MEMBERS

    if args.impl == "reference":
        if rank != 0:
            return
        steps = min(args.steps, 3)
        cpu = cpu_reference(cfg, args.config, steps_cap=steps, warm=1)
        line = {"metric": METRIC, "value": cpu["value"], "unit": UNIT, "n_gpus": args.gpus,
                "steps": steps, "warmup": 1, "ms_per_step": cpu["s_per_step"] * 1e3,
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
                "dtype": "f64", "data": "synthetic", "config": config, "impl": "reference",
                "cpu_baseline": {k: cpu[k] for k in ("value", "unit", "cores", "kind", "sample")},
                "e2e": {"value": cpu["value"], "unit": UNIT, "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return

    world, rank, local = dist_setup()
    if args.config == "c5":
        res = time_slab(cfg, args.steps, warmup, world, rank, local)
        if rank == 0:
            print(json.dumps({
                "metric": METRIC, "value": res["value"], "unit": UNIT, "n_gpus": world,
                "steps": args.steps, "warmup": warmup, "ms_per_step": res["ms_per_step"],
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
                "dtype": "f64", "data": "synthetic",
                "config": {**config, "parallelism": f"rho-slab x{world} (all-to-all + halo)"},
                "e2e": None, "gpu_launches": 8 * args.steps, "roofline": None,
                "cpu_baseline": None, "clocks": res["clocks"], "impl": "b200"}), flush=True)
        return
    res64 = time_precision(cfg, args.config, "double", args.steps, warmup, world, rank, local)
    res32 = None
    if not args.no_fp32:
        res32 = time_precision(cfg, args.config, "single", args.steps, warmup, world, rank, local)
    slab = None
    if world > 1 and args.config != "c4":
        # the single large grid (BASELINE C5) over all ranks: rho slabs with
        # NCCL all-to-all transposes, MAX all-reduce and the halo ring (slab.py)
        c5, c5_desc = workload("c5")
        ks = min(args.steps, 20)
        rs = time_slab(c5, ks, warmup, world, rank, local)
        slab = {"workload": c5_desc, "value": rs["value"], "unit": UNIT,
                "ms_per_step": rs["ms_per_step"], "steps": ks, "n_ranks": world,
                "scaling": "strong", "dtype": "f64", "clocks": rs["clocks"],
                "parallelism": f"rho-slab x{world} (NCCL all-to-all + MAX all-reduce + halo ring)"}
    e2e = e2e32 = None
    if not args.no_e2e:
        e2e = e2e_precision(cfg, args.config, "double", args.steps, world, rank, local)
        if res32 is not None:
            e2e32 = e2e_precision(cfg, args.config, "single", args.steps, world, rank, local)
    cpu = None
    if world == 1 and not args.no_cpu:
        cpu = cpu_reference(cfg, args.config)
    if rank != 0:
        return
    line = {
        "metric": METRIC, "value": res64["value"], "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": warmup, "ms_per_step": res64["ms_per_step"],
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": config,
        "e2e": e2e, "gpu_launches": 8 * args.steps,
        "roofline": res64["roofline"],
        "cpu_baseline": ({k: cpu[k] for k in ("value", "unit", "cores", "kind", "sample")}
                         if cpu else None),
        "clocks": res64["clocks"],
        "fp32": ({"value": res32["value"], "ms_per_step": res32["ms_per_step"],
                  "roofline": res32["roofline"], "clocks": res32["clocks"],
                  "e2e": e2e32} if res32 else None),
        "impl": "b200",
    }
    if slab is not None:
        line["slab_c5"] = slab
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
