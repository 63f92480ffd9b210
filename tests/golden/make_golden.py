"""Generate the golden fixtures of this directory from the REFERENCE itself.

Run in the build container (where /root/reference exists), never on the GPU
box:

    python tests/golden/make_golden.py [--ref /root/reference/pkg]

It copies the reference package to a scratch directory (numba needs a
writable cache), imports ``nwave`` from there and records inputs and
outputs of the hot-path functions: weno5_b, phi1/phi2, build_multipliers,
rfft2/irfft2 (scipy, as the reference calls it), one exprk22_step and
exp_euler_step, short marches (fp64/fp32, radix 2/3/5/7 grids) and the full
BASELINE C1 and C3 marches.  The fixtures pin the CPU oracle
(tests/test_oracle.py) and, through it, the GPU path.
"""

from __future__ import annotations

import argparse
import json
import os
import shutil
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))


def _import_reference(ref_pkg: str):
    scratch = tempfile.mkdtemp(prefix="nwave_ref_")
    shutil.copytree(ref_pkg, os.path.join(scratch, "pkg"))
    os.environ.setdefault("NUMBA_CACHE_DIR", os.path.join(scratch, "numba_cache"))
    sys.path.insert(0, os.path.join(scratch, "pkg", "src"))
    import nwave  # noqa: F401

    return nwave


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ref", default="/root/reference/pkg")
    args = ap.parse_args()
    nwave = _import_reference(args.ref)
    from nwave.analysis import initial_nwave, preset_config
    from nwave.exprk import (EPS_DOUBLE, EPS_SINGLE, SpectralTransforms, build_multipliers,
                             exp_euler_step, exprk22_step, phi1, phi2, run_exprk22)
    from nwave.grid import DomainConfig, Field2D, build_axes, l2_norm, rho_nodes_closed
    from nwave.turbulence import (TurbulenceParams, evaluate_fields, sample_modes,
                                  zero_fields)
    from nwave.weno import weno5_b

    rng = np.random.default_rng(20240917)
    out = {}

    # --- WENO: random data, N-wave with turbulent coefficients, fp32
    spec1 = sample_modes(TurbulenceParams(seed=1))
    cases = {}
    v = rng.standard_normal((40, 56))
    up, uq, du = (0.03 * rng.standard_normal(40) for _ in range(3))
    cases["rand"] = (v, up, uq, du, 0.05, 0.31, 0.23)
    cfg = DomainConfig(N_rho=64, N_theta=56, N_sigma=8, Sigma=3.2)
    _, rho, theta = build_axes(cfg)
    f = evaluate_fields(spec1, spec1.lam, np.array([0.0, 0.4]), rho)
    vn = initial_nwave(rho, theta, cfg.A, cfg.B).values
    vn = vn * (1.0 + 0.1 * np.cos(2 * np.pi * 3 * rho / cfg.rho_span))[:, None]
    cases["nwave_turb"] = (vn, f.u_par[1], f.u_perp[1], f.du_perp_drho[1], cfg.B,
                           cfg.d_rho, cfg.d_theta)
    cases["small_odd"] = (rng.standard_normal((7, 9)), *(0.02 * rng.standard_normal(7)
                                                          for _ in range(3)), 0.05, 0.5, 0.7)
    for name, (v, up, uq, du, b, dr, dt) in cases.items():
        out[f"weno_{name}_v"] = v
        out[f"weno_{name}_coef"] = np.stack([up, uq, du])
        out[f"weno_{name}_par"] = np.array([b, dr, dt])
        out[f"weno_{name}_out"] = weno5_b(v, up, uq, du, np.float64(b), dr, dt)
        v32 = v.astype(np.float32)
        c32 = [c.astype(np.float32) for c in (up, uq, du)]
        out[f"weno_{name}_out32"] = weno5_b(v32, *c32, np.float32(b), dr, dt)

    # --- phi
    zs = []
    for m in (1e-8, 1e-5, 1e-4, 1e-3, 0.05, 0.4999, 0.5001, 1.0, 3.0, 20.0):
        for a in (0.0, 0.5, np.pi / 2, 2.2, np.pi):
            zs.append(m * np.exp(1j * a))
    zs += [0.0, -1e18, -1e18 + 5j, -2.0, 1.0]
    zs = np.array(zs, dtype=np.complex128)
    out["phi_z"] = zs
    out["phi1"] = phi1(zs)
    out["phi2"] = phi2(zs)

    # --- multiplier tables (radix-3 rho, radix-7 theta) and single precision
    cfg_t = DomainConfig(N_rho=48, N_theta=42, N_sigma=77)
    m = build_multipliers(cfg_t, EPS_DOUBLE)
    for k in ("E", "Phi1", "Phi2", "z"):
        out[f"tab48_{k}"] = getattr(m, k)
    ms = build_multipliers(DomainConfig(N_rho=16, N_theta=14), EPS_SINGLE, dtype=np.complex64)
    for k in ("E", "Phi1", "Phi2", "Phi1m2"):
        out[f"tab16s_{k}"] = getattr(ms, k)

    # --- transforms exactly as the reference calls them
    tr = SpectralTransforms(48, 42)
    x = rng.standard_normal((48, 42))
    out["fft_x"] = x
    out["fft_rfft2"] = tr.forward(x)
    h = rng.standard_normal((48, 22)) + 1j * rng.standard_normal((48, 22))
    out["fft_half"] = h
    out["fft_irfft2"] = tr.inverse(h)

    # --- one step with the WENO right-hand side
    cfg_s = DomainConfig(N_rho=32, N_theta=28, N_sigma=50, Sigma=20.0)
    _, rho_s, theta_s = build_axes(cfg_s)
    fs = evaluate_fields(spec1, spec1.lam, np.array([0.0, cfg_s.d_sigma]), rho_s)
    ms_ = build_multipliers(cfg_s, EPS_DOUBLE)
    v0 = initial_nwave(rho_s, theta_s, cfg_s.A, cfg_s.B).values * (
        1 + 0.2 * np.sin(2 * np.pi * rho_s / cfg_s.rho_span))[:, None]
    tr_s = SpectralTransforms(32, 28)
    vh0 = tr_s.forward(v0)

    def b_eval(stage, v):
        return weno5_b(v, fs.u_par[stage], fs.u_perp[stage], fs.du_perp_drho[stage],
                       np.float64(cfg_s.B), cfg_s.d_rho, cfg_s.d_theta)

    out["step_vh0"] = vh0
    out["step_coef"] = np.stack([fs.u_par, fs.u_perp, fs.du_perp_drho])
    out["step_exprk22"] = exprk22_step(vh0, ms_, b_eval, cfg_s.d_sigma, tr_s)[0]
    out["step_euler"] = exp_euler_step(vh0, ms_, b_eval, cfg_s.d_sigma, tr_s)[0]

    # --- short marches: (name, config, turbulent?, rho-modulated?)
    runs = {
        "m64x56": (DomainConfig(N_rho=64, N_theta=56, N_sigma=12, Sigma=4.8), 1),
        "m48x42": (DomainConfig(N_rho=48, N_theta=42, N_sigma=10, Sigma=4.0), 2),
        "m50x40": (DomainConfig(N_rho=50, N_theta=40, N_sigma=10, Sigma=4.0), 3),
    }
    sig_meta = {}
    for name, (c, seed) in runs.items():
        sigma, rho_c, theta_c = build_axes(c)
        spec = sample_modes(TurbulenceParams(seed=seed))
        fl = evaluate_fields(spec, spec.lam, sigma, rho_nodes_closed(c))
        v0 = initial_nwave(rho_c, theta_c, c.A, c.B).values * (
            1 + 0.1 * np.cos(2 * np.pi * 2 * rho_c / c.rho_span))[:, None]
        out[f"{name}_v0"] = v0
        out[f"{name}_coef"] = np.stack([fl.u_par, fl.u_perp, fl.du_perp_dsigma, fl.du_perp_drho])
        for prec in ("double", "single"):
            for scheme in ("exprk22", "expeuler"):
                rep = run_exprk22(c, Field2D(v0), fl, precision=prec, scheme=scheme,
                                  snapshot_sigmas=[c.d_sigma * 3, c.Sigma])
                key = f"{name}_{prec}_{scheme}"
                out[f"{key}_final"] = rep.final.values
                out[f"{key}_snap3"] = rep.snapshots[c.d_sigma * 3].values
                sig_meta[key] = {"max_abs_v": rep.max_abs_v}
        sig_meta[name] = {"config": {k: getattr(c, k) for k in
                                     ("Sigma", "N_sigma", "N_rho", "N_theta")}}

    # --- BASELINE C1 (demo grid, homogeneous) and C3 (Set 1, turbulent seed 0)
    c1 = DomainConfig(Sigma=30.0, N_sigma=300, N_rho=625, N_theta=448)
    _, rho1, theta1 = build_axes(c1)
    v01 = initial_nwave(rho1, theta1, c1.A, c1.B)
    for prec in ("double", "single"):
        rep = run_exprk22(c1, v01, zero_fields(301, 626), precision=prec, threads=0)
        key = f"c1_{prec}"
        out[f"{key}_final"] = rep.final.values.astype(np.float64 if prec == "double" else np.float32)
        sig_meta[key] = {"max_abs_v": rep.max_abs_v,
                         "l2": l2_norm(rep.final, c1.d_rho, c1.d_theta),
                         "max": float(rep.final.values.max()),
                         "min": float(rep.final.values.min())}
    c3 = preset_config(1)
    sig3, rho3, theta3 = build_axes(c3)
    spec0 = sample_modes(TurbulenceParams(seed=0))
    f3 = evaluate_fields(spec0, spec0.lam, sig3, rho_nodes_closed(c3))
    v03 = initial_nwave(rho3, theta3, c3.A, c3.B)
    for prec in ("double", "single"):
        rep = run_exprk22(c3, v03, f3, precision=prec, threads=0, snapshot_sigmas=[60.0])
        key = f"c3_{prec}"
        out[f"{key}_final_sub"] = rep.final.values[::8].copy()
        out[f"{key}_snap60_sub"] = rep.snapshots[60.0].values[::8].copy()
        out[f"{key}_row144"] = rep.final.values[int(round(144 / c3.d_rho))].copy()
        sig_meta[key] = {"max_abs_v": rep.max_abs_v,
                         "l2": l2_norm(rep.final, c3.d_rho, c3.d_theta),
                         "max": float(rep.final.values.max()),
                         "min": float(rep.final.values.min())}
    # the turbulence generator itself at a small size (host restatement check)
    fsmall = evaluate_fields(spec0, spec0.lam, sig3[:5], rho_nodes_closed(c3)[:33])
    out["turb_small"] = np.stack([fsmall.u_par, fsmall.u_perp, fsmall.du_perp_dsigma,
                                  fsmall.du_perp_drho])

    np.savez_compressed(os.path.join(HERE, "golden.npz"), **out)
    with open(os.path.join(HERE, "golden_meta.json"), "w") as fh:
        json.dump({"reference": "arxiv/paper_2103_06080 nwave 0.1.0 (pkg/src/nwave)",
                   "numpy": np.__version__, "scipy": __import__("scipy").__version__,
                   "numba": __import__("numba").__version__, "runs": sig_meta},
                  fh, indent=1, sort_keys=True)
    print("wrote", os.path.join(HERE, "golden.npz"))


if __name__ == "__main__":
    main()
