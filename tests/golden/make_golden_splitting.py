"""Golden fixtures of the splitting baseline from the REFERENCE.

Run in the build container (where /root/reference exists), never on the GPU box:

    python tests/golden/make_golden_splitting.py [--ref /root/reference/pkg]

Imports ``nwave`` from a scratch copy (numba needs a writable cache) and
records inputs and outputs of ``nwave/splitting.py``: each Lie-Trotter stage
(``step_diffraction_cn``, ``step_burgers_godunov``, ``godunov_flux``,
``step_axial_absorption_spectral``, ``step_transverse_lw``), one ``lie_step``,
two ``run_splitting`` marches (turbulent medium, snapshots) and one
``compare_solvers`` report with the reference's default (splitting, exprk22)
pair.  Output: golden_splitting.npz + golden_splitting.json.
"""

from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

from make_golden import _import_reference  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ref", default="/root/reference/pkg")
    args = ap.parse_args()
    _import_reference(args.ref)
    from nwave.analysis import compare_solvers, initial_nwave
    from nwave.grid import DomainConfig, build_axes, rho_nodes_closed
    from nwave.splitting import (SplittingState, godunov_flux, lie_step, run_splitting,
                                 step_axial_absorption_spectral, step_burgers_godunov,
                                 step_diffraction_cn, step_transverse_lw)
    from nwave.grid import Field2D
    from nwave.turbulence import TurbulenceParams, evaluate_fields, sample_modes

    out, meta = {}, {"runs": {}}
    rng = np.random.default_rng(7)

    # --- stages on a small closed grid (41 x 48) with turbulent coefficients
    c = DomainConfig(N_rho=40, N_theta=48, N_sigma=10, Sigma=4.0)
    sig, _, theta = build_axes(c)
    rho_c = rho_nodes_closed(c)
    spec = sample_modes(TurbulenceParams(seed=3))
    f = evaluate_fields(spec, spec.lam, sig, rho_c)
    v = initial_nwave(rho_c, theta, c.A, c.B).values * (1.0 + 0.2 * np.cos(rho_c / 37.0))[:, None]
    v = v + 0.05 * rng.standard_normal(v.shape)
    out["st_v"] = v
    out["st_coef"] = np.stack([f.u_par[2], f.u_perp[2], f.du_perp_dsigma[2], f.du_perp_drho[2]])
    out["st_diffraction"] = step_diffraction_cn(v, c.d_sigma, c.d_rho, c.d_theta)
    out["st_godunov"] = step_burgers_godunov(v, c.B, c.d_sigma, c.d_theta)
    ul, ur = rng.standard_normal(64), rng.standard_normal(64)
    out["st_flux_in"] = np.stack([ul, ur])
    out["st_flux"] = godunov_flux(ul, ur, c.B)
    out["st_axial"] = step_axial_absorption_spectral(v, f.u_par[2], c.A, c.d_sigma, c.theta_span)
    out["st_transverse"] = step_transverse_lw(v, f.u_perp[2], f.du_perp_dsigma[2],
                                              f.du_perp_drho[2], c.d_sigma, c.d_rho)
    st = lie_step(SplittingState(Field2D(v), 2), f, c)
    out["st_lie"] = st.field.values
    meta["stage_config"] = dict(N_rho=c.N_rho, N_theta=c.N_theta, N_sigma=c.N_sigma, Sigma=c.Sigma)

    # --- marches: the small grid (10 steps) and a 250 x 112 grid (40 steps)
    for name, cfg, seed, nstep in (("s41x48", c, 3, None),
                                   ("s251x112", DomainConfig(N_rho=250, N_theta=112, N_sigma=40,
                                                             Sigma=16.0), 5, None)):
        sig, _, theta = build_axes(cfg)
        rho_c = rho_nodes_closed(cfg)
        spec = sample_modes(TurbulenceParams(seed=seed))
        fl = evaluate_fields(spec, spec.lam, sig, rho_c)
        v0 = initial_nwave(rho_c, theta, cfg.A, cfg.B)
        snaps = [cfg.d_sigma * 3, cfg.Sigma]
        rep = run_splitting(cfg, v0, fl, snapshot_sigmas=snaps, threads=1)
        out[f"{name}_coef"] = np.stack([fl.u_par, fl.u_perp, fl.du_perp_dsigma, fl.du_perp_drho])
        out[f"{name}_v0"] = v0.values
        out[f"{name}_final"] = rep.final.values
        out[f"{name}_snap3"] = rep.snapshots[snaps[0]].values
        meta["runs"][name] = dict(config=dict(N_rho=cfg.N_rho, N_theta=cfg.N_theta,
                                              N_sigma=cfg.N_sigma, Sigma=cfg.Sigma),
                                  seed=seed, max_abs_v=rep.max_abs_v, n_steps=rep.n_steps,
                                  snapshots=snaps)

    # --- compare_solvers with the reference's default pair (splitting, exprk22)
    cfg = DomainConfig(N_rho=250, N_theta=112, N_sigma=40, Sigma=16.0)
    sig, _, _ = build_axes(cfg)
    spec = sample_modes(TurbulenceParams(seed=5))
    fl = evaluate_fields(spec, spec.lam, sig, rho_nodes_closed(cfg))
    rep = compare_solvers(cfg, fl, [8.0, 16.0], trace_sigma=16.0, trace_rho=144.0)
    meta["compare"] = dict(checkpoints=[[cp.sigma, cp.rel_l2_roi, cp.amplitude_ratio]
                                        for cp in rep.checkpoints],
                           overshoot_splitting=rep.overshoot_splitting,
                           overshoot_exprk22=rep.overshoot_exprk22)

    np.savez_compressed(os.path.join(HERE, "golden_splitting.npz"), **out)
    with open(os.path.join(HERE, "golden_splitting.json"), "w") as fh:
        json.dump(meta, fh, indent=1)
    print("wrote", len(out), "arrays")


if __name__ == "__main__":
    main()
