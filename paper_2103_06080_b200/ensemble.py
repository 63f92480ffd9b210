"""Ensembles of independent marches: batched on one device, sharded over
devices (BASELINE config C4).

Members share the grid, the multiplier tables and the coefficient fields;
each has its own initial field, so one ``DevicePlan`` with ``batch =
members`` runs them all: every kernel carries the member index in its grid,
reductions (alpha_theta, max|V|) are per member, and the tables are read once
per theta mode for all members (L2 reuse).  There is no exchange step
between members: over several GPUs the members are partitioned into
contiguous shards, one process per GPU, and nothing crosses the NVLink data
path -- only the small per-member summaries are gathered at the end
(``torch.distributed`` over NCCL on GPUs, gloo in the CPU tests).
"""

from __future__ import annotations

import time
from dataclasses import dataclass

import numpy as np

from .analysis import ground_metrics_device
from .errors import InstabilityError
from .exprk import EPS_DOUBLE, EPS_SINGLE
from .grid import DomainConfig
from .plan import DevicePlan


def shard_members(n_members: int, world: int, rank: int) -> range:
    """Contiguous, balanced shard of member indices for ``rank`` (sizes differ by <= 1)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of world {world}")
    base, extra = divmod(n_members, world)
    start = rank * base + min(rank, extra)
    return range(start, start + base + (1 if rank < extra else 0))


@dataclass
class EnsembleResult:
    members: range
    final: np.ndarray | None      # (n, N_rho, N_theta) float64, when keep_fields
    max_abs_v: np.ndarray         # per member, over all steps and the final field
    peak: np.ndarray              # per member max_theta V over the roi of the ground trace row
    device_seconds: float
    n_steps: int
    rise_theta: np.ndarray | None = None  # per member 10-90 % rise (theta units) at the trace row


def run_ensemble(config: DomainConfig, v0s, fields, scheme: str = "exprk22",
                 precision: str = "double", guard: float = 10.0, max_steps: int | None = None,
                 members: range | None = None, device=None, keep_fields: bool = True,
                 trace_rho: float = 144.0) -> EnsembleResult:
    """March all ``members`` of ``v0s`` (shape (M, N_rho, N_theta)) as one batch."""
    import torch

    if scheme not in ("exprk22", "expeuler"):
        raise ValueError(f"unknown scheme {scheme!r}")
    members = members if members is not None else range(len(v0s))
    n = len(members)
    if n == 0:
        return EnsembleResult(members, None, np.zeros(0), np.zeros(0), 0.0, 0)
    n_steps = config.N_sigma if max_steps is None else min(config.N_sigma, max_steps)
    if fields.shape[0] < n_steps + 1 or fields.shape[1] < config.N_rho:
        raise ValueError("velocity fields do not cover the run grid")
    eps = EPS_DOUBLE if precision == "double" else EPS_SINGLE
    plan = DevicePlan(config.N_rho, config.N_theta, n, precision, config.d_sigma,
                      config.rho_span, config.theta_span, config.A, config.B, eps, device)
    try:
        rows = n_steps + 1
        plan.set_coeffs(fields.u_par[:rows], fields.u_perp[:rows], fields.du_perp_drho[:rows],
                        n_rows=rows)
        if isinstance(v0s, torch.Tensor):
            block = v0s[members.start:members.stop]
        else:
            block = np.asarray(v0s[members.start:members.stop], dtype=np.float64)
        plan.load_physical(block)
        t0 = time.perf_counter()
        try:
            max_abs, _, _ = plan.march(scheme, 0, n_steps, guard, timing=False)
        except InstabilityError as err:
            err.member = members.start + getattr(err, "member", 0)
            raise
        v_fin, mx = plan.store_physical()
        torch.cuda.synchronize(plan.device)
        secs = time.perf_counter() - t0
        # per-member ground metrics on the device (nwb_ground_metrics): only
        # 3 doubles per member reach the host when the fields are not kept
        gm = ground_metrics_device(config, v_fin, trace_rho, stream=plan.stream)
        peak = np.array([g.peak for g in gm])
        rise = np.array([g.rise_theta for g in gm])
        if keep_fields:  # staged through reusable page-locked chunks (hostio)
            from .hostio import to_host64

            final = to_host64(v_fin, plan.stream)
        else:
            final = None
    finally:
        plan.close()
    mabs = np.maximum(max_abs.max(axis=1) if n_steps else 0.0, mx)
    return EnsembleResult(members, final, mabs, peak, secs, n_steps, rise)


def gather_summaries(result: EnsembleResult, n_members: int, group=None):
    """All-gather per-member (max|V|, peak) into full-length arrays on every rank.

    Uses ``torch.distributed`` (the process group's backend: NCCL on GPUs,
    gloo on CPU); every rank contributes its shard, so the result is the
    whole ensemble's summary.  This is the only cross-rank traffic.
    """
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    backend = dist.get_backend(group)
    dev = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")
    local = torch.full((2, n_members), float("nan"), dtype=torch.float64, device=dev)
    idx = torch.arange(result.members.start, result.members.stop, device=dev)
    local[0, idx] = torch.as_tensor(result.max_abs_v, dtype=torch.float64, device=dev)
    local[1, idx] = torch.as_tensor(result.peak, dtype=torch.float64, device=dev)
    parts = [torch.empty_like(local) for _ in range(world)]
    dist.all_gather(parts, local, group=group)
    full = torch.stack(parts).nan_to_num(nan=-np.inf).max(dim=0).values
    return full[0].cpu().numpy(), full[1].cpu().numpy()
