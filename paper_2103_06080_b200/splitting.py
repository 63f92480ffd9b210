"""Lie-Trotter splitting baseline on the device (reference
``pkg/src/nwave/splitting.py``).

One step composes, like the reference: diffraction (Crank-Nicolson in sigma,
trapezoid in theta, sequential in the theta index), Burgers (Godunov flux),
axial convection + absorption (one theta-frequency multiplier) and transverse
convection (Lax-Wendroff), on the closed rho grid (N_rho + 1 nodes, mirrored
Neumann ghosts) x periodic theta, float64.  The arithmetic runs in
``csrc/splitting.cu`` behind ``nwb_split_*`` (include/nwb200.h); the theta
transforms of the axial stage are the march's theta kernels.  The names and
signatures are the reference's (``splitting.py:33-301``), so studies that
compare the splitting baseline with ExpRK22 (``compare_solvers``) run
entirely on the GPU.
"""

from __future__ import annotations

import ctypes
import time
import warnings
from dataclasses import dataclass

import numpy as np

from . import _lib
from .cfl import CflReport, check_cfl_splitting  # noqa: F401  (re-exported, reference names)
from .errors import BudgetExceededError, CflViolationError, InstabilityError
from .grid import DomainConfig, Field2D
from .parallel import resolve_threads
from .reports import RunReport
from .turbulence import VelocityFields

STAGE_DIFFRACTION, STAGE_BURGERS, STAGE_AXIAL, STAGE_TRANSVERSE, STAGE_LIE = range(5)


def _torch():
    import torch

    return torch


class SplitPlan:
    """One ``nwb_split`` plan: Thomas factorisation, theta FFT tables, buffers."""

    def __init__(self, n_nodes: int, n_theta: int, d_sigma: float, d_rho: float, d_theta: float,
                 theta_span: float, A: float, B: float, device=None):
        torch = _torch()
        from .plan import resolve_device

        self.lib = _lib.lib()
        self.device = resolve_device(device)
        self.n, self.nt = int(n_nodes), int(n_theta)
        self.d_sigma = float(d_sigma)
        self._h = ctypes.c_void_p()
        with torch.cuda.device(self.device):
            self.stream = torch.cuda.Stream(device=self.device)
            _lib.check(self.lib.nwb_split_create(ctypes.byref(self._h), self.n, self.nt,
                                                 float(d_sigma), float(d_rho), float(d_theta),
                                                 float(theta_span), float(A), float(B),
                                                 self.device.index), "nwb_split_create")
            _lib.check(self.lib.nwb_split_set_stream(self._h, self.stream.cuda_stream),
                       "nwb_split_set_stream")
        self.n_rows = 0

    def close(self):
        if getattr(self, "_h", None) and self._h.value:
            self.lib.nwb_split_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _dev(self, a):
        torch = _torch()
        if isinstance(a, torch.Tensor):
            return a.to(device=self.device, dtype=torch.float64).contiguous()
        return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).to(self.device)

    def _sync_in(self):
        torch = _torch()
        self.stream.wait_stream(torch.cuda.current_stream(self.device))

    def _sync_out(self):
        torch = _torch()
        torch.cuda.current_stream(self.device).wait_stream(self.stream)

    def set_coeffs(self, u_par, u_perp, du_ds, du_dr, n_rows: int):
        arrs = [None if a is None else self._dev(a[:n_rows]) for a in (u_par, u_perp, du_ds, du_dr)]
        ref = next(a for a in arrs if a is not None)
        ld = ref.shape[1] if ref.dim() == 2 else ref.shape[0]
        self._sync_in()
        _lib.check(self.lib.nwb_split_set_coeffs(
            self._h, *[None if a is None else a.data_ptr() for a in arrs], int(n_rows), int(ld), 1),
            "nwb_split_set_coeffs")
        self._keep = arrs
        self.n_rows = n_rows

    def stage(self, stage: int, v, row: int = 0):
        torch = _torch()
        x = self._dev(v).reshape(self.n, self.nt)
        out = torch.empty_like(x)
        self._sync_in()
        _lib.check(self.lib.nwb_split_stage(self._h, int(stage), int(row), x.data_ptr(),
                                            out.data_ptr()), "nwb_split_stage")
        self._sync_out()
        return out

    def load(self, v):
        x = self._dev(v).reshape(self.n, self.nt)
        self._sync_in()
        _lib.check(self.lib.nwb_split_load(self._h, x.data_ptr()), "nwb_split_load")
        self.stream.synchronize()

    def store(self):
        torch = _torch()
        out = torch.empty((self.n, self.nt), dtype=torch.float64, device=self.device)
        _lib.check(self.lib.nwb_split_store(self._h, out.data_ptr()), "nwb_split_store")
        self._sync_out()
        return out

    def march(self, n0: int, n_steps: int, guard: float, max_seconds: float | None,
              total_steps: int):
        mabs = np.zeros(max(n_steps, 0))
        fs, fv = ctypes.c_int(-1), ctypes.c_double(0.0)
        rc = self.lib.nwb_split_march(self._h, int(n0), int(n_steps), float(guard),
                                      float(max_seconds) if max_seconds is not None else -1.0,
                                      mabs.ctypes.data_as(ctypes.c_void_p), ctypes.byref(fs),
                                      ctypes.byref(fv))
        if rc == _lib.NWB_EINSTABILITY:
            m = fv.value
            # lie_step flags a non-finite field at sigma_n (splitting.py:229-230),
            # the march's guard at sigma_{n+1} (:287-289)
            n = fs.value if not np.isfinite(m) else fs.value + 1
            raise InstabilityError(n * self.d_sigma, m)
        if rc == _lib.NWB_EBUDGET:
            raise BudgetExceededError(f"exceeded {max_seconds:.0f} s at step {fs.value}/{total_steps}")
        _lib.check(rc, "nwb_split_march", d_sigma=self.d_sigma)
        return mabs


def _plan_for(v_shape, d_sigma, d_rho, d_theta, theta_span, A=0.0, B=0.0) -> SplitPlan:
    return SplitPlan(v_shape[0], v_shape[1], d_sigma, d_rho, d_theta, theta_span, A, B)


def _out(x, like):
    torch = _torch()
    if isinstance(like, torch.Tensor):
        return x
    return x.cpu().numpy()


def step_diffraction_cn(v, d_sigma: float, d_rho: float, d_theta: float):
    """Diffraction stage on a closed (Neumann) rho axis (reference ``splitting.py:138-145``)."""
    p = _plan_for(tuple(v.shape), d_sigma, d_rho, d_theta, 1.0)
    try:
        return _out(p.stage(STAGE_DIFFRACTION, v), v)
    finally:
        p.close()


def godunov_flux(u_l, u_r, B: float):
    """Exact Riemann flux of g(u) = -(B/2) u^2 (reference ``splitting.py:148-157``)."""
    torch = _torch()
    from .plan import resolve_device

    lib = _lib.lib()
    dev = resolve_device(None)
    ul = np.asarray(u_l, dtype=np.float64)
    ur = np.asarray(u_r, dtype=np.float64)
    ul, ur = np.broadcast_arrays(ul, ur)
    a = torch.from_numpy(np.ascontiguousarray(ul)).to(dev)
    b = torch.from_numpy(np.ascontiguousarray(ur)).to(dev)
    out = torch.empty_like(a)
    _lib.check(lib.nwb_godunov_flux(a.numel(), a.data_ptr(), b.data_ptr(), float(B), out.data_ptr(),
                                    torch.cuda.current_stream(dev).cuda_stream), "godunov_flux")
    res = out.cpu().numpy()
    return float(res) if res.ndim == 0 else res


def step_burgers_godunov(v, B: float, d_sigma: float, d_theta: float):
    """Conservative Godunov update of the Burgers stage (reference ``splitting.py:160-166``)."""
    p = _plan_for(tuple(v.shape), d_sigma, 1.0, d_theta, 1.0, 0.0, B)
    try:
        return _out(p.stage(STAGE_BURGERS, v), v)
    finally:
        p.close()


def step_axial_absorption_spectral(v, u_par_col, A: float, d_sigma: float, theta_span: float,
                                   workers: int = 1):
    """Axial convection + absorption multiplier in theta-frequency space
    (reference ``splitting.py:169-185``; ``workers`` accepted, unused)."""
    p = _plan_for(tuple(v.shape), d_sigma, 1.0, 1.0, theta_span, A, 0.0)
    try:
        col = np.asarray(u_par_col, dtype=np.float64)[None, :]
        p.set_coeffs(col, None, None, None, 1)
        return _out(p.stage(STAGE_AXIAL, v, 0), v)
    finally:
        p.close()


def step_transverse_lw(v, u_perp_col, du_perp_dsigma_col, du_perp_drho_col, d_sigma: float,
                       d_rho: float):
    """Lax-Wendroff transverse convection (reference ``splitting.py:188-207``)."""
    p = _plan_for(tuple(v.shape), d_sigma, d_rho, 1.0, 1.0)
    try:
        cols = [np.asarray(c, dtype=np.float64)[None, :]
                for c in (u_perp_col, du_perp_dsigma_col, du_perp_drho_col)]
        p.set_coeffs(None, *cols, 1)
        return _out(p.stage(STAGE_TRANSVERSE, v, 0), v)
    finally:
        p.close()


@dataclass
class SplittingState:
    """Marched field on the closed rho grid plus the current step index."""

    field: Field2D
    sigma_index: int = 0


def _config_plan(config: DomainConfig, device=None) -> SplitPlan:
    return SplitPlan(config.N_rho + 1, config.N_theta, config.d_sigma, config.d_rho,
                     config.d_theta, config.theta_span, config.A, config.B, device)


def lie_step(state: SplittingState, fields: VelocityFields, config: DomainConfig,
             workers: int = 1) -> SplittingState:
    """One Lie-Trotter step (reference ``splitting.py:233-250``)."""
    n = state.sigma_index
    p = _config_plan(config)
    try:
        rows = [np.asarray(getattr(fields, k)[n:n + 1, :config.N_rho + 1], dtype=np.float64)
                for k in ("u_par", "u_perp", "du_perp_dsigma", "du_perp_drho")]
        p.set_coeffs(*rows, 1)
        v = p.stage(STAGE_LIE, state.field.values, 0).cpu().numpy()
    finally:
        p.close()
    if not np.all(np.isfinite(v)):
        raise InstabilityError(n * config.d_sigma, float(np.max(np.abs(v))))
    return SplittingState(Field2D(v), n + 1)


def run_splitting(config: DomainConfig, v0, fields: VelocityFields, snapshot_sigmas=None,
                  threads: int = 1, guard: float = 10.0, max_seconds: float | None = None,
                  cfl: str = "warn", v_max_bound: float = 5.0, max_steps: int | None = None,
                  device=None) -> RunReport:
    """March the splitting solver to sigma = Sigma on the device (reference
    ``splitting.py:253-301``).  ``v0`` lives on the closed rho grid, shape
    (N_rho + 1, N_theta); snapshots are the state after step n (n = 0: the
    initial field), copied to host memory."""
    from .exprk import _snapshot_steps
    from .hostio import to_host64

    n_nodes = config.N_rho + 1
    n_steps = config.N_sigma if max_steps is None else min(config.N_sigma, max_steps)
    values = v0.values if isinstance(v0, Field2D) else np.asarray(v0)
    if tuple(values.shape) != (n_nodes, config.N_theta):
        raise ValueError(f"initial field shape {tuple(values.shape)} does not match the closed "
                         f"grid ({n_nodes}, {config.N_theta})")
    if fields.shape[0] < n_steps + 1 or fields.shape[1] < n_nodes:
        raise ValueError("velocity fields do not cover the run grid")
    u_perp_max = float(np.max(np.abs(np.asarray(fields.u_perp))))
    report = check_cfl_splitting(config, v_max_bound, u_perp_max)
    if not report.passed:
        if cfl == "error":
            raise CflViolationError(str(report))
        warnings.warn(f"CFL check failed: {report}", stacklevel=2)
    eff_threads = resolve_threads(threads)
    plan_snaps = _snapshot_steps(config, snapshot_sigmas)
    values = np.array(values, dtype=np.float64)
    snapshots: dict[float, Field2D] = {}
    max_abs = float(np.max(np.abs(values)))
    if 0 in plan_snaps:
        snapshots[plan_snaps[0]] = Field2D(values.copy())
    p = _config_plan(config, device)
    step_ms = []
    try:
        p.set_coeffs(fields.u_par, fields.u_perp, fields.du_perp_dsigma, fields.du_perp_drho,
                     n_steps + 1 if n_steps + 1 <= fields.shape[0] else fields.shape[0])
        p.load(values)
        t_start = time.perf_counter()
        cuts = sorted(n for n in plan_snaps if 0 < n <= n_steps)
        n_cur = 0
        for stop in cuts + ([n_steps] if n_steps not in cuts else []):
            if stop > n_cur:
                budget = None
                if max_seconds is not None:
                    budget = max(max_seconds - (time.perf_counter() - t_start), 0.0)
                t0 = time.perf_counter()
                m = p.march(n_cur, stop - n_cur, guard, budget, n_steps)
                step_ms.append(np.full(stop - n_cur, (time.perf_counter() - t0) / (stop - n_cur)))
                max_abs = max(max_abs, float(np.max(m)))
                n_cur = stop
            if stop in plan_snaps:
                snapshots[plan_snaps[stop]] = Field2D(to_host64(p.store(), p.stream))
        final = Field2D(to_host64(p.store(), p.stream))
        wall = time.perf_counter() - t_start
    finally:
        p.close()
    return RunReport(
        solver="splitting", n_steps=n_steps, d_sigma=config.d_sigma, wall_seconds=wall,
        max_abs_v=max_abs, final=final, snapshots=snapshots,
        step_seconds=np.concatenate(step_ms) if step_ms else np.zeros(0),
        threads=eff_threads)
