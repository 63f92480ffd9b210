"""Developer diagnostic: time the C2 march kernels under rho-pass knob settings
(NWB_RHO_* env variables are read at plan creation).  Debug bits skip work,
so those rows are timing decompositions, not valid results."""

import os
import re
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2103_06080_b200 as P  # noqa: E402
from paper_2103_06080_b200.plan import DevicePlan  # noqa: E402

KNOBS = ("NWB_RHO_HALF", "NWB_PAIR55", "NWB_RHO_BULK", "NWB_THETA_BULK", "NWB_RHO_STAGGER", "NWB_RHO_DEBUG", "NWB_RHO_PREFETCH", "NWB_RHO_NEXTPF", "NWB_RHO_ROLL", "NWB_RHO_WS", "NWB_RHO_WS_DEBUG", "NWB_RHO_SYM", "NWB_RHO_THREADS", "NWB_RHO_SPLIT", "NWB_RHO_PERSIST",
         "NWB_MAXPROD_R", "NWB_MAXPROD_H", "NWB_THETA_ROWS", "NWB_THETA_ROWS_C2R", "NWB_THETA_THREADS", "NWB_THETA_STREAM", "NWB_THETA_DEBUG", "NWB_PAD", "NWB_PAD_N")


def run(prec, env, preset=4):
    for k in KNOBS:
        os.environ.pop(k, None)
    os.environ.update(env)
    c = P.preset_config(preset)
    _, rho, theta = P.build_axes(c)
    v0 = P.rho_modulated(c, P.initial_nwave(rho, theta, c.A, c.B)).values
    plan = DevicePlan(c.N_rho, c.N_theta, 1, prec, c.d_sigma, c.rho_span, c.theta_span, c.A, c.B,
                      2.0**-53 if prec == "double" else 2.0**-24)
    plan.set_coeffs(None, None, None, n_rows=64)
    plan.load_physical(v0)
    try:  # debug knobs skip work, so the state may blow up: time it anyway
        plan.march("exprk22", 0, 4, timing=False)
    except P.InstabilityError:
        pass
    km = plan.profile_kernels("exprk22", 4, 8) / 8
    plan.close()
    return [round(float(x), 4) for x in km]


if __name__ == "__main__":
    prec = sys.argv[1] if len(sys.argv) > 1 else "double"
    combos = [dict(a.split("=", 1) for a in re.split(r",(?=NWB_)", spec)) if spec else {}
              for spec in (sys.argv[2:] or [""])]
    for env in combos:
        try:
            km = run(prec, env)
        except Exception as e:  # keep probing the other settings
            print(prec, env, "FAILED:", e, flush=True)
            continue
        print(prec, env, "c2r weno r2c rho x2:", km, "rho sum", round(km[3] + km[7], 4), flush=True)
