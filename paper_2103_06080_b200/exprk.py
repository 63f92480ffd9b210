"""ExpRK22 / exponential-Euler march on B200 -- the drop-in hot path.

Same names, signatures, return types and error behaviour as
``nwave.exprk`` (reference ``pkg/src/nwave/exprk.py``):

* ``phi1`` / ``phi2``            -- ``exprk.py:42-84``  (device ``k_phi``)
* ``PhiMultipliers``             -- ``exprk.py:87-108``
* ``build_multipliers``          -- ``exprk.py:111-131`` (device ``k_tables``)
* ``SpectralTransforms``         -- ``exprk.py:134-148`` (device rfft2/irfft2)
* ``exprk22_step`` / ``exp_euler_step`` -- ``exprk.py:151-196`` (generic
  ``b_eval`` callable; combines on the device with numpy rounding)
* ``check_cfl_exprk``            -- ``exprk.py:199-205``
* ``run_exprk22``                -- ``exprk.py:219-331`` (the fused march:
  six kernels per ExpRK22 step, state resident in HBM)

There is no CPU fallback: without libnwb200.so or a CUDA device every entry
point raises ``BackendError``.
"""

from __future__ import annotations

import time
import warnings
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from ._lib import check, ptr
from .cfl import check_cfl_exprk  # noqa: F401  (re-exported like the reference)
from .errors import CflViolationError, InstabilityError
from .grid import TWO_PI, DomainConfig, Field2D
from .parallel import resolve_threads
from .plan import DevicePlan, cached_plan, resolve_device
from .reports import RunReport

EPS_DOUBLE = 2.0 ** -53
EPS_SINGLE = 2.0 ** -24


def _torch():
    import torch

    return torch


# ---------------------------------------------------------------------- phi

def _phi(z, shift: int, device=None):
    torch = _torch()
    lib = _lib.lib()
    arr = np.asarray(z, dtype=np.complex128)
    flat = np.ascontiguousarray(np.atleast_1d(arr).ravel())
    dev = resolve_device(device)
    with torch.cuda.device(dev):
        zt = torch.from_numpy(flat).to(dev)
        out = torch.empty_like(zt)
        check(lib.nwb_phi(ptr(zt), flat.size, shift, ptr(out),
                          torch.cuda.current_stream(dev).cuda_stream), "nwb_phi")
        res = out.cpu().numpy()
    return res[0] if arr.ndim == 0 else res.reshape(arr.shape)


def phi1(z):
    """phi1(z) = (e^z - 1)/z; 18-term series below |z| = 0.5."""
    return _phi(z, 1)


def phi2(z):
    """phi2(z) = (e^z - 1 - z)/z^2; 18-term series below |z| = 0.5."""
    return _phi(z, 2)


# ---------------------------------------------------------------------- tables

@dataclass
class PhiMultipliers:
    """Multiplier tables on the rfft2 half-spectrum, shape (n_rho, n_theta//2+1).

    Row j is the signed rho mode of ``np.fft.fftfreq``, column k the theta
    mode.  Host copies (numpy) as in the reference; device copies used by
    the step functions are cached in ``_device``.
    """

    E: np.ndarray
    Phi1: np.ndarray
    Phi2: np.ndarray
    z: np.ndarray
    xi: np.ndarray
    omega: np.ndarray
    d_sigma: float
    eps: float
    Phi1m2: np.ndarray = None
    _device: dict = field(default_factory=dict, repr=False, compare=False)

    def __post_init__(self):
        if self.Phi1m2 is None:
            self.Phi1m2 = self.Phi1 - self.Phi2

    def device_tables(self, device, cdt):
        torch = _torch()
        key = (str(device), cdt)
        if key not in self._device:
            self._device[key] = tuple(
                torch.from_numpy(np.ascontiguousarray(a)).to(device=device, dtype=cdt)
                for a in (self.E, self.Phi1, self.Phi1m2, self.Phi2))
        return self._device[key]


def build_multipliers(config: DomainConfig, machine_eps: float = EPS_DOUBLE,
                      dtype=np.complex128, device=None) -> PhiMultipliers:
    """E, Phi1, Phi2 (cast to ``dtype``) and z (complex128), built on the device."""
    torch = _torch()
    lib = _lib.lib()
    single = np.dtype(dtype) == np.complex64
    cdt = torch.complex64 if single else torch.complex128
    nr, kk = config.N_rho, config.N_theta // 2 + 1
    dev = resolve_device(device)
    with torch.cuda.device(dev):
        tabs = [torch.empty((nr, kk), dtype=cdt, device=dev) for _ in range(4)]
        z = torch.empty((nr, kk), dtype=torch.complex128, device=dev)
        check(lib.nwb_tables(_lib.F32 if single else _lib.F64, nr, config.N_theta,
                             config.rho_span, config.theta_span, config.d_sigma, config.A,
                             float(machine_eps), ptr(tabs[0]), ptr(tabs[1]), ptr(tabs[2]),
                             ptr(tabs[3]), ptr(z), torch.cuda.current_stream(dev).cuda_stream),
              "nwb_tables")
        E, P1, P2, P12, zz = (t.cpu().numpy() for t in (*tabs, z))
    j = np.fft.fftfreq(nr) * nr
    k = np.arange(kk, dtype=np.float64)
    mult = PhiMultipliers(E=E, Phi1=P1, Phi2=P2, z=zz, xi=TWO_PI * j / config.rho_span,
                          omega=TWO_PI * k / config.theta_span, d_sigma=config.d_sigma,
                          eps=machine_eps, Phi1m2=P12)
    mult._device[(str(dev), cdt)] = (tabs[0], tabs[1], tabs[3], tabs[2])
    return mult


# ---------------------------------------------------------------------- transforms

def _precision_of(x) -> str:
    torch = _torch()
    dt = x.dtype
    if isinstance(x, torch.Tensor):
        return "single" if dt in (torch.float32, torch.complex64) else "double"
    return "single" if np.dtype(dt) in (np.float32, np.complex64) else "double"


class SpectralTransforms:
    """Counted rfft2/irfft2 pair on the device (scipy.fft conventions).

    numpy in -> numpy out; CUDA tensor in -> CUDA tensor out.  ``workers``
    is accepted for API compatibility and ignored.
    """

    def __init__(self, n_rho: int, n_theta: int, workers: int = 1, device=None):
        self.shape = (n_rho, n_theta)
        self.workers = workers
        self.count = 0
        self.device = device

    def _plan(self, x) -> DevicePlan:
        return cached_plan(self.shape[0], self.shape[1], 1, _precision_of(x), self.device)

    def forward(self, real2d):
        torch = _torch()
        self.count += 1
        plan = self._plan(real2d)
        is_t = isinstance(real2d, torch.Tensor)
        x = plan.to_device(real2d, plan.rdt).reshape(1, *self.shape)
        out = plan.rfft2(x)[0]
        return out if is_t else out.cpu().numpy()

    def inverse(self, half):
        torch = _torch()
        self.count += 1
        plan = self._plan(half)
        is_t = isinstance(half, torch.Tensor)
        x = plan.to_device(half, plan.cdt).reshape(1, self.shape[0], self.shape[1] // 2 + 1)
        out = plan.irfft2(x)[0]
        return out if is_t else out.cpu().numpy()


# ---------------------------------------------------------------------- step API

_NUMPY_FMA: dict = {}


def numpy_cmul_is_fused(dtype=np.complex128) -> bool:
    """Does this host's numpy round complex products with a fused multiply-add?

    numpy's SIMD loops (AVX2 / AVX-512) compute re = fma(ar, br, -(ai bi)),
    im = fma(ar, bi, ai br); its scalar loop rounds every product.  The
    generic step API reproduces whichever this host's numpy does, so results
    handed back to numpy callers match ``E * vhat`` bitwise (reference test
    ``tests/test_exprk.py:131-138``).  Decided once per dtype from exact
    rational arithmetic on a fixed sample.
    """
    key = np.dtype(dtype).name
    if key not in _NUMPY_FMA:
        from fractions import Fraction

        rng = np.random.default_rng(12345)
        a = (rng.standard_normal(64) + 1j * rng.standard_normal(64)).astype(dtype)
        b = (rng.standard_normal(64) + 1j * rng.standard_normal(64)).astype(dtype)
        c = a * b
        real_t = a.real.dtype.type
        fused = [real_t(float(Fraction(float(x.real)) * Fraction(float(y.real))
                              + Fraction(float(-(x.imag * y.imag)))))
                 for x, y in zip(a, b)]
        _NUMPY_FMA[key] = bool(np.array_equal(c.real, np.array(fused, dtype=real_t)))
    return _NUMPY_FMA[key]


def _combine(mode, d_sigma, tables, vh, b1=None, b2=None):
    torch = _torch()
    lib = _lib.lib()
    E, P1, P12, P2 = tables
    out = torch.empty_like(vh)
    prec = _lib.F64 if vh.dtype == torch.complex128 else _lib.F32
    if numpy_cmul_is_fused(np.complex128 if prec == _lib.F64 else np.complex64):
        mode |= 8
    check(lib.nwb_combine(prec, vh.numel(), mode, float(d_sigma), ptr(E), ptr(P1), ptr(P12),
                          ptr(P2), ptr(vh), ptr(b1), ptr(b2), ptr(out),
                          torch.cuda.current_stream(vh.device).cuda_stream), "nwb_combine")
    return out


def _dev_spec(x, like):
    torch = _torch()
    if isinstance(x, torch.Tensor):
        return x.to(device=like.device, dtype=like.dtype).contiguous()
    return torch.from_numpy(np.ascontiguousarray(x)).to(device=like.device,
                                                          dtype=like.dtype).contiguous()


def _step_setup(vhat, mult, transforms):
    torch = _torch()
    as_np = not isinstance(vhat, torch.Tensor)
    dev = vhat.device if not as_np else resolve_device(getattr(transforms, "device", None))
    cdt = torch.complex64 if _precision_of(vhat) == "single" else torch.complex128
    vh = _dev_spec(vhat, torch.empty(0, dtype=cdt, device=dev))
    return as_np, vh, mult.device_tables(dev, cdt)


def _out(x, as_np):
    return x.cpu().numpy() if as_np else x


def exprk22_step(vhat, mult: PhiMultipliers, b_eval, d_sigma, transforms,
                 timings: dict | None = None):
    """One two-stage ExpRK22 step; returns (vhat_next, v_n) (reference ``:151-178``)."""
    torch = _torch()
    as_np, vh, tabs = _step_setup(vhat, mult, transforms)
    sync = lambda: torch.cuda.synchronize(vh.device)
    t0 = time.perf_counter()
    v = transforms.inverse(vhat)
    t1 = time.perf_counter()
    b1 = b_eval(0, v)
    t2 = time.perf_counter()
    bh1 = _dev_spec(transforms.forward(b1), vh)
    ev = _combine(0, d_sigma, tabs, vh)
    vstar = _combine(1, d_sigma, tabs, ev, bh1)
    v_star = transforms.inverse(_out(vstar, as_np))
    sync()
    t3 = time.perf_counter()
    b2 = b_eval(1, v_star)
    t4 = time.perf_counter()
    bh2 = _dev_spec(transforms.forward(b2), vh)
    vnext = _combine(2, d_sigma, tabs, ev, bh1, bh2)
    res = _out(vnext, as_np)
    sync()
    t5 = time.perf_counter()
    if timings is not None:
        timings["nonlinear"] = (t2 - t1) + (t4 - t3)
        timings["linear"] = (t1 - t0) + (t3 - t2) + (t5 - t4)
    return res, v


def exp_euler_step(vhat, mult: PhiMultipliers, b_eval, d_sigma, transforms,
                   timings: dict | None = None):
    """Exponential Euler; bitwise ExpRK22's stage value (reference ``:181-196``)."""
    torch = _torch()
    as_np, vh, tabs = _step_setup(vhat, mult, transforms)
    t0 = time.perf_counter()
    v = transforms.inverse(vhat)
    t1 = time.perf_counter()
    b1 = b_eval(0, v)
    t2 = time.perf_counter()
    bh1 = _dev_spec(transforms.forward(b1), vh)
    res = _out(_combine(3, d_sigma, tabs, vh, bh1), as_np)
    torch.cuda.synchronize(vh.device)
    t3 = time.perf_counter()
    if timings is not None:
        timings["nonlinear"] = t2 - t1
        timings["linear"] = (t1 - t0) + (t3 - t2)
    return res, v


# ---------------------------------------------------------------------- march

def _snapshot_steps(config: DomainConfig, snapshot_sigmas) -> dict[int, float]:
    plan = {}
    for s in (snapshot_sigmas or ()):
        n = int(round(s / config.d_sigma))
        if 0 <= n <= config.N_sigma:
            plan[n] = float(s)
    return plan


def _to_host64(t) -> np.ndarray:
    """Device tensor -> fresh float64 numpy array in ordinary host memory,
    through reusable page-locked staging chunks (``hostio.to_host64``)."""
    from .hostio import to_host64

    return to_host64(t)


def _as_host_field(x) -> np.ndarray:
    torch = _torch()
    if isinstance(x, torch.Tensor):
        return x.detach().to("cpu", torch.float64).numpy()
    return np.asarray(x.values if isinstance(x, Field2D) else x)


def run_exprk22(config: DomainConfig, v0, fields, snapshot_sigmas=None,
                scheme: str = "exprk22", precision: str = "double", threads: int = 1,
                guard: float = 10.0, max_seconds: float | None = None, cfl: str = "warn",
                v_max_bound: float = 5.0, max_steps: int | None = None, device=None,
                timing: bool = True) -> RunReport:
    """March to sigma = Sigma on the device (reference ``exprk.py:219-331``).

    Extra keywords: ``device`` (CUDA device; default current), ``timing``
    (default: per-step buckets from device time stamps the march kernels
    write -- nonlinear = WENO, linear = the rest, as ``exprk.py:176-177`` --
    read back once after the march; ``False`` skips the read-back and
    reports the average step time in every slot).  Both replay the same
    CUDA graph.
    """
    if scheme not in ("exprk22", "expeuler"):
        raise ValueError(f"unknown scheme {scheme!r}")
    if precision not in ("double", "single"):
        raise ValueError(f"unknown precision {precision!r}")
    torch = _torch()
    nr, nt = config.N_rho, config.N_theta
    n_steps = config.N_sigma if max_steps is None else min(config.N_sigma, max_steps)
    values = v0.values if isinstance(v0, Field2D) else v0
    if tuple(values.shape) != (nr, nt):
        raise ValueError(f"initial field shape {tuple(values.shape)} does not match grid "
                         f"({nr}, {nt})")
    if fields.shape[0] < n_steps + 1 or fields.shape[1] < nr:
        raise ValueError("velocity fields do not cover the run grid")
    report = check_cfl_exprk(config, fields, v_max_bound)
    if not report.passed:
        if cfl == "error":
            raise CflViolationError(str(report))
        warnings.warn(f"CFL check failed: {report}", stacklevel=2)
    threads_eff = resolve_threads(threads)
    eps = EPS_DOUBLE if precision == "double" else EPS_SINGLE

    plan = DevicePlan(nr, nt, 1, precision, config.d_sigma, config.rho_span,
                      config.theta_span, config.A, config.B, eps, device)
    try:
        rows = n_steps + 1
        plan.set_coeffs(fields.u_par[:rows], fields.u_perp[:rows], fields.du_perp_drho[:rows],
                        n_rows=rows)
        if not isinstance(values, torch.Tensor):
            values = np.asarray(values, dtype=np.float64)
        plan.load_physical(values)
        snap_plan = _snapshot_steps(config, snapshot_sigmas)
        t_start = time.perf_counter()
        # march in segments between snapshot steps; each snapshot (v_n at the
        # start of step n) is a c2r of the state into a two-buffer device ring,
        # streamed to host memory while the next segment runs
        from .hostio import SnapshotStreamer

        streamer = SnapshotStreamer(plan) if any(n < n_steps for n in snap_plan) else None
        cuts = sorted(n for n in snap_plan if n < n_steps)
        parts_abs, parts_ms, n_cur = [], [], 0
        for stop in cuts + [n_steps]:
            if stop > n_cur:
                budget = None
                if max_seconds is not None:
                    budget = max(max_seconds - (time.perf_counter() - t_start), 0.0)
                mabs, sms, _ = plan.march(scheme, n_cur, stop - n_cur, guard, budget,
                                          timing=timing, total_steps=n_steps)
                parts_abs.append(mabs)
                if sms is not None:
                    parts_ms.append(sms)
                n_cur = stop
            if stop < n_steps:
                streamer.capture(snap_plan[stop])
        max_abs = np.concatenate(parts_abs, axis=1) if parts_abs else np.zeros((1, 0))
        step_ms = np.concatenate(parts_ms, axis=0) if parts_ms else None
        v_fin, mx = plan.store_physical()
        m = float(mx[0])
        if not np.isfinite(m) or m > guard:
            raise InstabilityError(n_steps * config.d_sigma, m)
        max_abs_v = max(float(np.max(max_abs)) if n_steps else 0.0, m)
        final = Field2D(_to_host64(v_fin[0]))
        snapshots = {}
        if streamer is not None:
            got = streamer.finish()
            snapshots = {sig: Field2D(got[sig][0]) for sig in sorted(got, key=float)}
        if n_steps in snap_plan:
            snapshots[snap_plan[n_steps]] = final.copy()
        wall = time.perf_counter() - t_start
    finally:
        plan.close()
    if step_ms is not None:
        nonlin = step_ms[:, 1].astype(np.float64) / 1e3
        lin = np.maximum(step_ms[:, 0].astype(np.float64) / 1e3 - nonlin, 0.0)
        step_s = nonlin + lin
    else:
        step_s = np.full(n_steps, wall / max(n_steps, 1))
        nonlin = lin = None
    return RunReport(
        solver=scheme, n_steps=n_steps, d_sigma=config.d_sigma, wall_seconds=wall,
        max_abs_v=max_abs_v, final=final, snapshots=snapshots, step_seconds=step_s,
        step_nonlinear=nonlin, step_linear=lin,
        transforms=(4 if scheme == "exprk22" else 2) * n_steps, threads=threads_eff,
        precision=precision)
