"""Golden fixtures for the study orchestration and the
snapshot output path (f2), generated from the REFERENCE itself.

Run in the build container (where /root/reference exists), never on the
GPU box:

    python tests/golden/make_golden_studies.py [--ref /root/reference/pkg]

Records, with the reference ``nwave`` package: a convergence study of both
exponential solvers on a small turbulent grid (with and without the roi), a
solver comparison (ExpEuler vs ExpRK22) with the overshoot trace,
``max_overshoot`` on fixed traces, and the bytes of the NWAV binary and CSV
writers for a fixed field.  Output: golden_studies.json next to this file.
"""

from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

from make_golden import _import_reference  # noqa: E402

# the study grid (shared with tests/test_studies*.py)
GRID = dict(N_rho=64, N_theta=56, N_sigma=32, Sigma=2.4)
N_REF, N_LIST = 32, [4, 8, 16]
SEED = 1


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ref", default="/root/reference/pkg")
    args = ap.parse_args()
    _import_reference(args.ref)
    from nwave import fieldio
    from nwave.analysis import compare_solvers, convergence_study, max_overshoot
    from nwave.grid import DomainConfig, Field2D, build_axes, rho_nodes_closed
    from nwave.turbulence import TurbulenceParams, evaluate_fields, sample_modes

    out = {"grid": GRID, "n_ref": N_REF, "n_list": N_LIST, "seed": SEED}
    cfg = DomainConfig(**GRID)
    spec = sample_modes(TurbulenceParams(seed=SEED))
    sig_ref = np.arange(N_REF + 1) * (cfg.Sigma / N_REF)
    master = evaluate_fields(spec, spec.lam, sig_ref, rho_nodes_closed(cfg))
    conv = {}
    for solver in ("exprk22", "expeuler"):
        for roi in (False, True):
            rows = convergence_study(cfg, N_LIST, N_REF, solver=solver, fields_master=master,
                                     use_roi=roi)
            conv[f"{solver}_roi{int(roi)}"] = [[r.n_sigma, r.err, r.beta, r.unstable] for r in rows]
    out["convergence"] = conv

    fields = evaluate_fields(spec, spec.lam, np.arange(cfg.N_sigma + 1) * cfg.d_sigma,
                             rho_nodes_closed(cfg))
    rep = compare_solvers(cfg, fields, [0.6, 1.2, 2.4], trace_sigma=2.4, trace_rho=144.0,
                          solver_pair=("expeuler", "exprk22"))
    out["compare"] = {
        "checkpoints": [[c.sigma, c.rel_l2_roi, c.amplitude_ratio] for c in rep.checkpoints],
        "overshoot_a": rep.overshoot_splitting, "overshoot_b": rep.overshoot_exprk22,
    }

    rng = np.random.default_rng(20240917)
    traces = {"random": rng.standard_normal(40), "ramp": np.linspace(0, 1, 17),
              "ripple": np.sin(np.linspace(0, 3 * np.pi, 50)) + 0.05 * rng.standard_normal(50)}
    out["overshoot_traces"] = {k: v.tolist() for k, v in traces.items()}
    out["overshoot"] = {k: max_overshoot(v) for k, v in traces.items()}

    field = Field2D(rng.standard_normal((5, 7)))
    _, rho, theta = build_axes(DomainConfig(N_rho=5, N_theta=7, N_sigma=4, Sigma=1.0))
    with tempfile.TemporaryDirectory() as tmp:
        fb, fc = os.path.join(tmp, "f.bin"), os.path.join(tmp, "f.csv")
        fieldio.write_field_binary(fb, field, 0.25, 0.5, 1.75)
        fieldio.write_field_csv(fc, field, rho, theta)
        out["fieldio"] = {
            "values": field.values.tolist(),
            "bin_sha256": hashlib.sha256(open(fb, "rb").read()).hexdigest(),
            "csv_sha256": hashlib.sha256(open(fc, "rb").read()).hexdigest(),
        }
    with open(os.path.join(HERE, "golden_studies.json"), "w") as fh:
        json.dump(out, fh, indent=1, sort_keys=True)
    print("wrote golden_studies.json")


if __name__ == "__main__":
    main()
