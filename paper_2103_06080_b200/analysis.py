"""Synthetic inputs and ground metrics around the hot path.

* ``initial_nwave`` -- the N-wave pulse (reference
  ``pkg/src/nwave/analysis.py:28-43``), rho-independent.
* ``GRID_SETS`` / ``preset_config`` -- Table-1 presets (``analysis.py:231-245``).
* ``ensemble_nwaves`` -- BASELINE config C4's amplitude/duration-varied
  members (a builder extension defined in SURVEY 8(d)): member i is
  a_i ((theta-3pi)/(2 pi d_i)) (tanh(s(theta-3pi-pi d_i)) - tanh(s(theta-3pi+pi d_i)))
  with a ~ U[0.5, 1.5], d ~ U[0.75, 1.25] from ``default_rng(seed)``.
* ``rho_modulated`` -- V0 (1 + 0.1 cos(2 pi 4 rho / rho_span)), the C2/C5
  variant that exercises the rho transforms.
* ``ground_metrics`` -- peak and interpolated 10-90 % rise time of the
  trace at the ground (sigma = Sigma); not in the reference,
  computed by the same function on both sides of a parity test.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from .grid import DomainConfig, Field2D, _index_range, build_axes

GRID_SETS = {
    1: dict(N_sigma=300, N_rho=1250, N_theta=7 * 64),
    2: dict(N_sigma=600, N_rho=2500, N_theta=7 * 128),
    3: dict(N_sigma=1200, N_rho=5000, N_theta=7 * 256),
    4: dict(N_sigma=2400, N_rho=10000, N_theta=7 * 512),
}

#: pulse period in seconds (reference ``turbulence.py:36``, T0)
T0_SECONDS = 2.0e-2


def preset_config(set_id: int, **overrides) -> DomainConfig:
    if set_id not in GRID_SETS:
        raise ValueError(f"unknown grid set {set_id}; choose from 1..4")
    params = dict(GRID_SETS[set_id])
    params.update(overrides)
    return DomainConfig(**params)


def _nwave_row(theta: np.ndarray, steep: float, amp: float = 1.0,
               dur: float | None = None) -> np.ndarray:
    if dur is None:
        return ((theta - 3.0 * np.pi) / (2.0 * np.pi)
                * (np.tanh(steep * (theta - 4.0 * np.pi))
                   - np.tanh(steep * (theta - 2.0 * np.pi))))
    centre = theta - 3.0 * np.pi
    return amp * (centre / (2.0 * np.pi * dur)) * (
        np.tanh(steep * (centre - np.pi * dur)) - np.tanh(steep * (centre + np.pi * dur)))


def initial_nwave(rho_nodes, theta_nodes, A: float, B: float = 0.05) -> Field2D:
    """V0(theta) = ((theta-3pi)/2pi)(tanh(s(theta-4pi)) - tanh(s(theta-2pi))), s = B/4A."""
    if A == 0:
        raise ValueError("initial_nwave: A must be nonzero (pulse width is B/4A)")
    row = _nwave_row(np.asarray(theta_nodes, dtype=np.float64), B / (4.0 * A))
    return Field2D(np.tile(row, (len(rho_nodes), 1)))


def ensemble_nwaves(config: DomainConfig, members: int, seed: int = 2026):
    """(members, N_rho, N_theta) float64 initial fields plus (amp, dur) draws."""
    rng = np.random.default_rng(seed)
    amp = rng.uniform(0.5, 1.5, members)
    dur = rng.uniform(0.75, 1.25, members)
    _, rho, theta = build_axes(config)
    steep = config.B / (4.0 * config.A)
    out = np.empty((members, len(rho), len(theta)))
    for i in range(members):
        out[i] = _nwave_row(theta, steep, amp[i], dur[i])[None, :]
    return out, amp, dur


def rho_modulated(config: DomainConfig, v0: Field2D, depth: float = 0.1,
                  mode: int = 4) -> Field2D:
    _, rho, _ = build_axes(config)
    mod = 1.0 + depth * np.cos(2.0 * np.pi * mode * (rho - config.rho_min) / config.rho_span)
    return Field2D(v0.values * mod[:, None])


@dataclass
class GroundMetrics:
    rho: float
    peak: float
    rise_theta: float
    rise_seconds: float


def _upward_crossing(y: np.ndarray, x: np.ndarray, level: float, start: int) -> float:
    for i in range(max(start, 1), len(y)):
        if y[i - 1] < level <= y[i]:
            t = (level - y[i - 1]) / (y[i] - y[i - 1])
            return float(x[i - 1] + t * (x[i] - x[i - 1]))
    return float("nan")


def ground_metrics(config: DomainConfig, field: Field2D, trace_rho: float = 144.0,
                   ) -> GroundMetrics:
    """Peak and 10-90 % rise time of the theta trace at ``trace_rho``.

    theta_10 is the first upward crossing of 0.1 P scanning from the roi
    start; theta_90 the next upward crossing of 0.9 P; both linearly
    interpolated between nodes (node-index crossings are quantised to
    d_theta).  Seconds = rise_theta * T0 / (2 pi).
    """
    _, rho, theta = build_axes(config)
    j = int(round((trace_rho - config.rho_min) / config.d_rho))
    k0, k1 = _index_range(theta, *config.roi_theta)
    y = field.values[j, k0:k1 + 1]
    x = theta[k0:k1 + 1]
    peak = float(np.max(y))
    t10 = _upward_crossing(y, x, 0.1 * peak, 0)
    i10 = int(np.searchsorted(x, t10)) if np.isfinite(t10) else len(y)
    t90 = _upward_crossing(y, x, 0.9 * peak, i10)
    rise = t90 - t10
    return GroundMetrics(float(rho[j]), peak, rise, rise * T0_SECONDS / (2.0 * np.pi))


def ground_metrics_device(config: DomainConfig, v, trace_rho: float = 144.0,
                          stream=None) -> list[GroundMetrics]:
    """``ground_metrics`` of every member of a device field in one kernel
    (``nwb_ground_metrics``): ``v`` is a CUDA tensor (batch, N_rho, N_theta) or
    (N_rho, N_theta) in float64 or float32; only 3 doubles per member cross
    to the host.  Bitwise the host definition above (same node values, same
    rounded interpolation)."""
    import torch

    from . import _lib

    if not (isinstance(v, torch.Tensor) and v.is_cuda):
        raise TypeError("ground_metrics_device needs a CUDA tensor")
    v = v.contiguous()
    vb = v.reshape(-1, config.N_rho, config.N_theta)
    prec = {torch.float64: _lib.F64, torch.float32: _lib.F32}.get(vb.dtype)
    if prec is None:
        raise TypeError(f"unsupported dtype {vb.dtype}")
    _, rho, theta = build_axes(config)
    j = int(round((trace_rho - config.rho_min) / config.d_rho))
    k0, k1 = _index_range(theta, *config.roi_theta)
    x = torch.as_tensor(theta[k0:k1 + 1], dtype=torch.float64, device=vb.device)
    out = torch.empty((vb.shape[0], 3), dtype=torch.float64, device=vb.device)
    lib = _lib.load_library()
    s = stream if stream is not None else torch.cuda.current_stream(vb.device)
    _lib.check(lib.nwb_ground_metrics(prec, vb.shape[0], config.N_rho, config.N_theta,
                                      _lib.ptr(vb), j, k0, k1, _lib.ptr(x), _lib.ptr(out),
                                      ctypes.c_void_p(s.cuda_stream)), "ground_metrics")
    res = out.cpu().numpy()
    return [GroundMetrics(float(rho[j]), float(pk), float(t90 - t10),
                          float((t90 - t10) * T0_SECONDS / (2.0 * np.pi)))
            for pk, t10, t90 in res]
