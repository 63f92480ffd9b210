"""Developer check: the TMEM half-column rho kernel (NWB_RHO_HALF=1) against
the default rho kernel on C2 fp64, K steps (the two differ only in FFT
factorisation order, so the fields agree to rounding)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2103_06080_b200 as P  # noqa: E402
from paper_2103_06080_b200.grid import max_relative  # noqa: E402

K = int(sys.argv[1]) if len(sys.argv) > 1 else 20
c2 = P.preset_config(4)
sig, rho, theta = P.build_axes(c2)
spec = P.sample_modes(P.TurbulenceParams(seed=0))
fd = P.turbulence.evaluate_fields_device(spec, spec.lam, sig[:K + 1], P.rho_nodes_closed(c2))
f = P.VelocityFields(*(t.cpu().numpy() for t in (fd.u_par, fd.u_perp, fd.du_perp_dsigma,
                                                 fd.du_perp_drho)))
v0 = P.rho_modulated(c2, P.initial_nwave(rho, theta, c2.A, c2.B))
out = {}
for half in ("0", "1"):
    os.environ["NWB_RHO_HALF"] = half
    out[half] = P.run_exprk22(c2, v0, f, max_steps=K)
a, b = out["0"], out["1"]
print("half vs default max-rel", max_relative(a.final.values, b.final.values),
      "maxabs", a.max_abs_v, b.max_abs_v)
