"""Medium coefficient fields consumed by the march.

``VelocityFields`` / ``zero_fields`` are the hot path's coefficient
container (reference ``pkg/src/nwave/turbulence.py:92-111,231-235``).  The
random-mode generator (``sample_modes`` / ``evaluate_fields``, reference
``turbulence.py:123-203``) is restated here on the host so the
inhomogeneous configurations (BASELINE C3, turbulent C4/C5) can be built on
a box where the reference package does not exist.  It is input
preparation, not part of the measured step; the device port is SURVEY row
f1.

Sampling uses the same PCG64 streams (``SeedSequence(seed).spawn(2)``:
child 0 -> phases, child 1 -> angles) so the mode set is bitwise the
reference's for a given seed; the mode sum accumulates modes in ascending
order with the cos(a)cos(b) - sin(a)sin(b) split of ``turbulence.py:145-180``.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .errors import ConfigError


@dataclass
class VelocityFields:
    """Dimensionless velocity tables on the (sigma, rho) grid.

    All four arrays have shape (n_sigma_nodes, n_rho_nodes).  The march
    reads ``u_par``, ``u_perp`` and ``du_perp_drho``; ``du_perp_dsigma`` is
    carried for API compatibility (the reference solver never reads it).
    """

    u_par: np.ndarray
    u_perp: np.ndarray
    du_perp_dsigma: np.ndarray
    du_perp_drho: np.ndarray

    @property
    def shape(self):
        return self.u_par.shape

    def max_abs(self) -> float:
        if hasattr(self.u_par, "abs"):  # device tensors
            return float(max(self.u_par.abs().max(), self.u_perp.abs().max()))
        return float(max(np.max(np.abs(self.u_par)), np.max(np.abs(self.u_perp))))


def zero_fields(n_sigma_nodes: int, n_rho_nodes: int) -> VelocityFields:
    """Quiescent medium U = 0."""
    shape = (n_sigma_nodes, n_rho_nodes)
    return VelocityFields(np.zeros(shape), np.zeros(shape),
                          np.zeros(shape), np.zeros(shape))


@dataclass(frozen=True)
class TurbulenceParams:
    """Physical parameters of the random velocity field (reference ``:26-73``)."""

    n_modes: int = 500
    sigma_u: float = 3.0
    c0: float = 343.0
    T0: float = 2.0e-2
    k_min: float | None = None
    k_max: float | None = None
    seed: int = 0

    def __post_init__(self):
        if not isinstance(self.n_modes, (int, np.integer)) or self.n_modes < 1:
            raise ConfigError(f"n_modes must be a positive integer, got {self.n_modes!r}")
        for name in ("sigma_u", "c0", "T0"):
            if not getattr(self, name) > 0:
                raise ConfigError(f"{name} must be positive")
        if self.wavenumber_min >= self.wavenumber_max:
            raise ConfigError("k_min must be below k_max")

    @property
    def lam(self) -> float:
        return self.T0 * self.c0

    @property
    def L(self) -> float:
        return 4.0 * self.lam

    @property
    def wavenumber_min(self) -> float:
        return 0.1 / self.L if self.k_min is None else self.k_min

    @property
    def wavenumber_max(self) -> float:
        return 9.0 / self.L if self.k_max is None else self.k_max


@dataclass
class TurbulenceSpec:
    phases: np.ndarray
    angles: np.ndarray
    wavenumbers: np.ndarray
    amp1: np.ndarray
    amp2: np.ndarray
    lam: float
    c0: float

    @property
    def n_modes(self) -> int:
        return len(self.phases)


def energy_spectrum(k, sigma_u: float, L: float):
    """Gaussian spectrum (1/8) sigma_u^2 K^3 L^4 exp(-(K L / 2)^2)."""
    k = np.asarray(k, dtype=np.float64)
    if np.any(k < 0):
        raise ValueError("energy_spectrum: negative wavenumber")
    out = 0.125 * sigma_u ** 2 * k ** 3 * L ** 4 * np.exp(-((k * L / 2.0) ** 2))
    return out if out.ndim else float(out)


def sample_modes(params: TurbulenceParams) -> TurbulenceSpec:
    n = params.n_modes
    seq_phase, seq_angle = np.random.SeedSequence(params.seed).spawn(2)
    phases = np.random.Generator(np.random.PCG64(seq_phase)).uniform(0.0, 2.0 * np.pi, n)
    angles = np.random.Generator(np.random.PCG64(seq_angle)).uniform(0.0, 2.0 * np.pi, n)
    if n == 1:
        k = np.array([params.wavenumber_min])
    else:
        k = np.linspace(params.wavenumber_min, params.wavenumber_max, n)
    amp = np.sqrt(energy_spectrum(k, params.sigma_u, params.L) / n)
    return TurbulenceSpec(phases=phases, angles=angles, wavenumbers=k,
                          amp1=-amp * np.sin(angles), amp2=amp * np.cos(angles),
                          lam=params.lam, c0=params.c0)


def evaluate_fields(spec: TurbulenceSpec, lam: float, sigma_nodes,
                    rho_nodes) -> VelocityFields:
    """Mode sum and analytic derivatives, normalised by c0 (host, vectorised)."""
    sig = np.ascontiguousarray(sigma_nodes, dtype=np.float64)
    rho = np.ascontiguousarray(rho_nodes, dtype=np.float64)
    shape = (len(sig), len(rho))
    acc = [np.zeros(shape) for _ in range(4)]
    kx = spec.wavenumbers * np.cos(spec.angles)
    ky = spec.wavenumbers * np.sin(spec.angles)
    lam = float(lam)
    w_ds = -spec.amp2 * kx * lam
    w_dr = -spec.amp2 * ky * lam
    for n in range(len(kx)):
        arg_b = ky[n] * lam * rho + spec.phases[n]
        cb, sb = np.cos(arg_b)[None, :], np.sin(arg_b)[None, :]
        arg_a = kx[n] * lam * sig
        ca, sa = np.cos(arg_a)[:, None], np.sin(arg_a)[:, None]
        c = ca * cb - sa * sb
        s = sa * cb + ca * sb
        acc[0] += spec.amp1[n] * c
        acc[1] += spec.amp2[n] * c
        acc[2] += w_ds[n] * s
        acc[3] += w_dr[n] * s
    inv_c0 = 1.0 / spec.c0
    return VelocityFields(*(a * inv_c0 for a in acc))


def evaluate_fields_device(spec: TurbulenceSpec, lam: float, sigma_nodes, rho_nodes,
                           device=None) -> VelocityFields:
    """Device mode sum: the fields stay resident in HBM.

    Same split, mode order and scaling as the host version and the reference
    ``_mode_sum``; returns a ``VelocityFields`` of float64 CUDA tensors that
    ``run_exprk22`` / ``DevicePlan.set_coeffs`` consume without a host round
    trip (kernels ``k_mode_trig`` / ``k_mode_sum`` in csrc/tables.cu).
    """
    import torch

    from . import _lib
    from ._lib import check, ptr
    from .plan import resolve_device

    lib = _lib.lib()
    dev = resolve_device(device)
    lam = float(lam)
    kx = spec.wavenumbers * np.cos(spec.angles)
    ky = spec.wavenumbers * np.sin(spec.angles)
    params = np.stack([kx, ky, spec.phases, spec.amp1, spec.amp2,
                       -spec.amp2 * kx * lam, -spec.amp2 * ky * lam]).astype(np.float64)
    n_modes = params.shape[1]
    sig = np.ascontiguousarray(sigma_nodes, dtype=np.float64)
    rho = np.ascontiguousarray(rho_nodes, dtype=np.float64)
    with torch.cuda.device(dev):
        t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
        p_d, s_d, r_d = t(params), t(sig), t(rho)
        scratch = torch.empty(2 * (len(sig) + len(rho)) * n_modes, dtype=torch.float64, device=dev)
        outs = [torch.empty((len(sig), len(rho)), dtype=torch.float64, device=dev) for _ in range(4)]
        check(lib.nwb_turbulence_fields(n_modes, ptr(p_d), lam, 1.0 / spec.c0, ptr(s_d), len(sig),
                                        ptr(r_d), len(rho), ptr(scratch), *(ptr(o) for o in outs),
                                        torch.cuda.current_stream(dev).cuda_stream),
              "nwb_turbulence_fields")
    return VelocityFields(*outs)


def downsample_fields(fields: VelocityFields, factor_sigma: int,
                      factor_rho: int) -> VelocityFields:
    """Keep every factor-th node on each axis (reference ``:212-228``)."""
    n_sig, n_rho = fields.shape
    if factor_sigma < 1 or factor_rho < 1:
        raise ValueError("downsample factors must be >= 1")
    for n, f, name in ((n_sig, factor_sigma, "factor_sigma"), (n_rho, factor_rho, "factor_rho")):
        if (n - 1) % f and n % f:
            raise ValueError(f"{name}={f} does not divide extent {n}")
    sl = (slice(None, None, factor_sigma), slice(None, None, factor_rho))
    arrs = (fields.u_par, fields.u_perp, fields.du_perp_dsigma, fields.du_perp_drho)
    if not isinstance(fields.u_par, np.ndarray) and hasattr(fields.u_par, "is_cuda"):
        # device-resident fields (evaluate_fields_device) stay on the device
        return VelocityFields(*(a[sl].contiguous() for a in arrs))
    return VelocityFields(*(np.ascontiguousarray(a[sl]) for a in arrs))
