"""TEST INFRASTRUCTURE ONLY -- CPU oracle for the ExpRK22/WENO5 step.

This module is the checker: only ``tests/``, ``__graft_entry__.smoke()``
and ``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import
it.  The product package (``paper_2103_06080_b200``) never does.

It restates the reference's hot path (arXiv 2103.06080 ``nwave`` package,
``/root/reference/pkg/src/nwave``) on the CPU:

* phi functions        -- ``exprk.py:42-84``  (0.5 cutoff, 18-term Horner)
* multiplier tables    -- ``exprk.py:87-131`` (``build_multipliers``)
* transforms           -- ``exprk.py:134-148`` (scipy.fft rfft2/irfft2; the
                          reference's third-party FFT is scipy's pocketfft,
                          unpinned ``scipy>=1.12``; 1.18.1 in this image)
* WENO5 b(sigma, V)    -- ``weno.py:25-124`` via ``weno_oracle.c`` (ctypes),
                          with a numpy restatement as a second opinion
* step functions       -- ``exprk.py:151-196``
* march                -- ``exprk.py:219-331``

Pinned against golden vectors produced by importing the reference itself
(``tests/golden/make_golden.py``); ``tests/test_oracle.py`` checks it.
"""

from __future__ import annotations

import ctypes
import math
import os
import subprocess
import time
from dataclasses import dataclass

import numpy as np
import scipy.fft as sfft

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_build", "liboracle_weno.so")

EPS_DOUBLE = 2.0 ** -53
EPS_SINGLE = 2.0 ** -24
TWO_PI = 2.0 * math.pi
SERIES_CUTOFF = 0.5
SERIES_TERMS = 18


# ------------------------------------------------------------------ build

def build(force: bool = False) -> str:
    """Compile weno_oracle.c with gcc into oracle/_build (checker build)."""
    src = os.path.join(HERE, "weno_oracle.c")
    if (not force and os.path.exists(LIB_PATH)
            and os.path.getmtime(LIB_PATH) >= os.path.getmtime(src)):
        return LIB_PATH
    os.makedirs(os.path.dirname(LIB_PATH), exist_ok=True)
    cmd = ["gcc", "-O3", "-fopenmp", "-ffp-contract=off", "-fPIC", "-shared",
           "-o", LIB_PATH, src, "-lm"]
    subprocess.run(cmd, check=True)
    return LIB_PATH


_lib = None


def _clib():
    global _lib
    if _lib is None:
        lib = ctypes.CDLL(build())
        dp, fp = ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_float)
        lib.oracle_weno5_b_f64.argtypes = [dp, ctypes.c_int, ctypes.c_int, dp, dp, dp,
                                           ctypes.c_double, ctypes.c_double,
                                           ctypes.c_double, dp, ctypes.c_int]
        lib.oracle_weno5_b_f32.argtypes = [fp, ctypes.c_int, ctypes.c_int, fp, fp, fp,
                                           ctypes.c_float, ctypes.c_double,
                                           ctypes.c_double, fp, ctypes.c_int]
        _lib = lib
    return _lib


def host_cores() -> int:
    return len(os.sched_getaffinity(0))


# ------------------------------------------------------------------ phi

def _phi_series(z, shift):
    acc = np.full_like(z, 1.0 / math.factorial(SERIES_TERMS - 1 + shift))
    for m in range(SERIES_TERMS - 2, -1, -1):
        acc = acc * z + 1.0 / math.factorial(m + shift)
    return acc


def phi(z, shift):
    arr = np.atleast_1d(np.asarray(z, dtype=np.complex128))
    out = np.empty_like(arr)
    small = np.abs(arr) < SERIES_CUTOFF
    if small.any():
        out[small] = _phi_series(arr[small], shift)
    if (~small).any():
        zb = arr[~small]
        ez = np.exp(zb)
        out[~small] = (ez - 1.0) / zb if shift == 1 else (ez - 1.0 - zb) / (zb * zb)
    return out[0] if np.ndim(z) == 0 else out


@dataclass
class Tables:
    E: np.ndarray
    Phi1: np.ndarray
    Phi2: np.ndarray
    Phi1m2: np.ndarray
    z: np.ndarray


def build_tables(n_rho, n_theta, rho_span, theta_span, d_sigma, A, eps,
                 dtype=np.complex128) -> Tables:
    j = np.fft.fftfreq(n_rho) * n_rho
    k = np.arange(n_theta // 2 + 1, dtype=np.float64)
    xi = TWO_PI * j / rho_span
    om = TWO_PI * k / theta_span
    den = 1j * om[None, :] + eps / (4.0 * np.pi)
    z = d_sigma * (-(xi[:, None] ** 2) / (4.0 * np.pi * den) - A * om[None, :] ** 2)
    E = np.exp(z).astype(dtype)
    P1 = phi(z, 1).astype(dtype)
    P2 = phi(z, 2).astype(dtype)
    return Tables(E, P1, P2, P1 - P2, z)


# ------------------------------------------------------------------ WENO

def weno5_b(v, u_par, u_perp, du, b_coef, d_rho, d_theta, threads=0):
    """b(sigma, V) through the C restatement (dtype of ``v`` selects fp64/fp32)."""
    lib = _clib()
    v = np.ascontiguousarray(v)
    nr, nt = v.shape
    if v.dtype == np.float64:
        cast = lambda a: np.ascontiguousarray(a, dtype=np.float64)
        ptr = lambda a: a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
        fn, b = lib.oracle_weno5_b_f64, float(b_coef)
    elif v.dtype == np.float32:
        cast = lambda a: np.ascontiguousarray(a, dtype=np.float32)
        ptr = lambda a: a.ctypes.data_as(ctypes.POINTER(ctypes.c_float))
        fn, b = lib.oracle_weno5_b_f32, float(np.float32(b_coef))
    else:
        raise TypeError(f"unsupported dtype {v.dtype}")
    up, uq, dd = cast(u_par), cast(u_perp), cast(du)
    out = np.empty_like(v)
    rc = fn(ptr(v), nr, nt, ptr(up), ptr(uq), ptr(dd), b, float(d_rho), float(d_theta),
            ptr(out), int(threads))
    if rc != 0:
        raise MemoryError("oracle_weno5_b allocation failed")
    return out


def _face_np(a0, a1, a2, a3, a4):
    s0 = 13.0 / 12.0 * ((a0 - 2.0 * a1) + a2) ** 2 + 0.25 * ((a0 - 4.0 * a1) + 3.0 * a2) ** 2
    s1 = 13.0 / 12.0 * ((a1 - 2.0 * a2) + a3) ** 2 + 0.25 * (a1 - a3) ** 2
    s2 = 13.0 / 12.0 * ((a2 - 2.0 * a3) + a4) ** 2 + 0.25 * ((3.0 * a2 - 4.0 * a3) + a4) ** 2
    w0 = 0.1 / (1e-6 + s0) ** 2
    w1 = 0.6 / (1e-6 + s1) ** 2
    w2 = 0.3 / (1e-6 + s2) ** 2
    q0 = (2.0 * a0 - 7.0 * a1) + 11.0 * a2
    q1 = (-a1 + 5.0 * a2) + 2.0 * a3
    q2 = (2.0 * a2 + 5.0 * a3) - a4
    return ((w0 * q0 + w1 * q1) + w2 * q2) / (6.0 * ((w0 + w1) + w2))


def _div_np(fp, fm, axis, inv_dx):
    r = lambda a, s: np.roll(a, -s, axis=axis)      # r(a, s)[i] = a[i+s]
    fhat = (_face_np(r(fp, -2), r(fp, -1), fp, r(fp, 1), r(fp, 2))
            + _face_np(r(fm, 3), r(fm, 2), r(fm, 1), fm, r(fm, -1)))
    return (fhat - np.roll(fhat, 1, axis=axis)) * inv_dx


def weno5_b_numpy(v, u_par, u_perp, du, b_coef, d_rho, d_theta):
    """Vectorised fp64 restatement (second opinion for the C oracle)."""
    v = np.asarray(v, dtype=np.float64)
    c = TWO_PI * np.asarray(u_par, dtype=np.float64)[:, None]
    a_th = float(np.max(np.abs(c + b_coef * v))) if v.size else 0.0
    a_rh = float(np.max(np.abs(u_perp))) if len(u_perp) else 0.0
    g = -c * v - 0.5 * b_coef * v * v
    dth = _div_np(0.5 * (g + a_th * v), 0.5 * (g - a_th * v), 1, 1.0 / d_theta)
    h = np.asarray(u_perp, dtype=np.float64)[:, None] * v
    drh = _div_np(0.5 * (h + a_rh * v), 0.5 * (h - a_rh * v), 0, 1.0 / d_rho)
    return (np.asarray(du, dtype=np.float64)[:, None] * v - dth) - drh


# ------------------------------------------------------------------ transforms

class Transforms:
    def __init__(self, shape, workers=1):
        self.shape = tuple(shape)
        self.workers = workers
        self.count = 0

    def forward(self, v):
        self.count += 1
        return sfft.rfft2(v, workers=self.workers)

    def inverse(self, vh):
        self.count += 1
        return sfft.irfft2(vh, s=self.shape, workers=self.workers)


def step_exprk22(vhat, tabs, b_eval, d_sigma, tr):
    v = tr.inverse(vhat)
    bh1 = tr.forward(b_eval(0, v))
    ev = tabs.E * vhat
    v_star = tr.inverse(ev + d_sigma * tabs.Phi1 * bh1)
    bh2 = tr.forward(b_eval(1, v_star))
    return ev + d_sigma * (tabs.Phi1m2 * bh1 + tabs.Phi2 * bh2), v


def step_expeuler(vhat, tabs, b_eval, d_sigma, tr):
    v = tr.inverse(vhat)
    bh1 = tr.forward(b_eval(0, v))
    return tabs.E * vhat + d_sigma * tabs.Phi1 * bh1, v


@dataclass
class OracleRun:
    final: np.ndarray
    max_abs_v: float
    snapshots: dict
    step_seconds: np.ndarray
    transforms: int
    failed_sigma: float | None = None


def march(config, v0, fields, scheme="exprk22", precision="double", threads=0,
          max_steps=None, snapshot_sigmas=None, guard=10.0) -> OracleRun:
    """CPU march with the reference's semantics (``exprk.py:219-331``).

    ``config`` is any object with the DomainConfig attributes; ``fields``
    any object with ``u_par``/``u_perp``/``du_perp_drho`` arrays.  On a guard
    violation the run stops and ``failed_sigma`` is set (instead of raising)
    so tests can compare the failure point.
    """
    workers = threads if threads > 0 else host_cores()
    nr, nt = config.N_rho, config.N_theta
    n_steps = config.N_sigma if max_steps is None else min(config.N_sigma, max_steps)
    rdt = np.float64 if precision == "double" else np.float32
    cdt = np.complex128 if precision == "double" else np.complex64
    eps = EPS_DOUBLE if precision == "double" else EPS_SINGLE
    tabs = build_tables(nr, nt, config.rho_span, config.theta_span, config.d_sigma,
                        config.A, eps, cdt)
    rows = [np.ascontiguousarray(getattr(fields, name)[:, :nr], dtype=rdt)
            for name in ("u_par", "u_perp", "du_perp_drho")]
    d_sigma, b_coef = rdt(config.d_sigma), rdt(config.B)
    tr = Transforms((nr, nt), workers)
    vhat = tr.forward(np.ascontiguousarray(v0, dtype=rdt))
    tr.count = 0
    plan = {}
    for s in (snapshot_sigmas or []):
        n = int(round(s / config.d_sigma))
        if 0 <= n <= config.N_sigma:
            plan[n] = float(s)
    step = step_exprk22 if scheme == "exprk22" else step_expeuler
    snaps, secs, max_abs = {}, np.zeros(n_steps), 0.0
    for n in range(n_steps):
        def b_eval(stage, v, _row=n):
            r = _row + stage
            return weno5_b(v, rows[0][r], rows[1][r], rows[2][r], b_coef,
                           config.d_rho, config.d_theta, workers)
        t0 = time.perf_counter()
        vhat, v_n = step(vhat, tabs, b_eval, d_sigma, tr)
        secs[n] = time.perf_counter() - t0
        m = float(np.max(np.abs(v_n)))
        if not np.isfinite(m) or m > guard:
            return OracleRun(np.asarray(v_n, np.float64), m, snaps, secs[:n + 1],
                             tr.count, failed_sigma=n * config.d_sigma)
        max_abs = max(max_abs, m)
        if n in plan:
            snaps[plan[n]] = np.asarray(v_n, dtype=np.float64).copy()
    v_fin = tr.inverse(vhat)
    m = float(np.max(np.abs(v_fin)))
    failed = None if (np.isfinite(m) and m <= guard) else n_steps * config.d_sigma
    max_abs = max(max_abs, m)
    final = np.asarray(v_fin, dtype=np.float64).copy()
    if n_steps in plan:
        snaps[plan[n_steps]] = final.copy()
    return OracleRun(final, max_abs, snaps, secs, tr.count - 1, failed)


@dataclass
class OracleBatchRun:
    final: np.ndarray          # (M, N_rho, N_theta) float64
    max_abs_v: np.ndarray      # per member
    transforms: int


def march_batch(config, v0s, fields, scheme="exprk22", precision="double", threads=0,
                max_steps=None) -> OracleBatchRun:
    """``march`` for M independent members sharing grid, tables and coefficients
    (BASELINE C4).  Per member the arithmetic is the reference's
    (``exprk.py:151-178,219-331``): scipy's rfft2/irfft2 over the last two axes
    transform every member on its own, WENO runs member by member, the combines
    are the same elementwise numpy expressions.  The tables are built once.
    """
    workers = threads if threads > 0 else host_cores()
    nr, nt = config.N_rho, config.N_theta
    n_steps = config.N_sigma if max_steps is None else min(config.N_sigma, max_steps)
    rdt = np.float64 if precision == "double" else np.float32
    cdt = np.complex128 if precision == "double" else np.complex64
    eps = EPS_DOUBLE if precision == "double" else EPS_SINGLE
    tabs = build_tables(nr, nt, config.rho_span, config.theta_span, config.d_sigma,
                        config.A, eps, cdt)
    rows = [np.ascontiguousarray(getattr(fields, name)[:, :nr], dtype=rdt)
            for name in ("u_par", "u_perp", "du_perp_drho")]
    d_sigma, b_coef = rdt(config.d_sigma), rdt(config.B)
    v0s = np.ascontiguousarray(v0s, dtype=rdt)
    tr = Transforms((nr, nt), workers)
    vhat = tr.forward(v0s)
    tr.count = 0
    step = step_exprk22 if scheme == "exprk22" else step_expeuler
    max_abs = np.zeros(len(v0s))
    for n in range(n_steps):
        def b_eval(stage, v, _row=n):
            r = _row + stage
            return np.stack([weno5_b(v[i], rows[0][r], rows[1][r], rows[2][r], b_coef,
                                     config.d_rho, config.d_theta, workers)
                             for i in range(len(v))])
        vhat, v_n = step(vhat, tabs, b_eval, d_sigma, tr)
        max_abs = np.maximum(max_abs, np.max(np.abs(v_n), axis=(1, 2)))
    v_fin = tr.inverse(vhat)
    max_abs = np.maximum(max_abs, np.max(np.abs(v_fin), axis=(1, 2)))
    return OracleBatchRun(np.asarray(v_fin, np.float64), max_abs.astype(np.float64),
                          tr.count - 1)
