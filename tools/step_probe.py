"""Developer diagnostic: C2 step time (untimed graph march, host clock around a
synchronised march of 40 steps) under plan-creation env knobs, each setting alternated over several rounds
on one box.  usage: python tools/step_probe.py double|single "" "NWB_X=1,NWB_Y=2" ..."""
import os
import re
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2103_06080_b200 as P  # noqa: E402
from paper_2103_06080_b200.plan import DevicePlan  # noqa: E402

sys.path.insert(0, os.path.join(ROOT, "tools"))
from rho_probe import KNOBS  # noqa: E402

EXTRA = ("NWB_OVERLAP", "NWB_RHO_HALF", "NWB_RHO_R1")


def step_ms(prec, env, preset=4, steps=40):
    for k in KNOBS + EXTRA:
        os.environ.pop(k, None)
    os.environ.update(env)
    c = P.preset_config(preset)
    _, rho, theta = P.build_axes(c)
    v0 = P.rho_modulated(c, P.initial_nwave(rho, theta, c.A, c.B)).values
    plan = DevicePlan(c.N_rho, c.N_theta, 1, prec, c.d_sigma, c.rho_span, c.theta_span, c.A, c.B,
                      2.0**-53 if prec == "double" else 2.0**-24)
    plan.set_coeffs(None, None, None, n_rows=steps + 8)
    plan.load_physical(v0)
    plan.march("exprk22", 0, 4, timing=False)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    plan.march("exprk22", 4, steps, timing=False)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    plan.close()
    return dt * 1e3 / steps


if __name__ == "__main__":
    prec = sys.argv[1] if len(sys.argv) > 1 else "double"
    combos = [dict(a.split("=", 1) for a in re.split(r",(?=NWB_)", spec)) if spec else {}
              for spec in (sys.argv[2:] or [""])]
    res = {i: [] for i in range(len(combos))}
    for _ in range(3):
        for i, env in enumerate(combos):
            try:
                res[i].append(step_ms(prec, env))
            except Exception as e:  # keep probing the other settings
                print(prec, env, "FAILED:", e, flush=True)
    for i, env in enumerate(combos):
        print(prec, env, "ms/step", [round(x, 4) for x in res[i]], flush=True)
