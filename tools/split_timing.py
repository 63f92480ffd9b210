"""Per-step time of the device splitting baseline on the
paper's grid sets, seed-0 turbulence (the reference's cost study setup,
analysis.py:274-306: step 0 dropped as warm-up)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2103_06080_b200 as nw  # noqa: E402

for sid in (1, 2, 3):
    c = nw.preset_config(sid)
    sig, _, theta = nw.build_axes(c)
    spec = nw.sample_modes(nw.TurbulenceParams(seed=0))
    f = nw.evaluate_fields(spec, spec.lam, sig[:12], nw.rho_nodes_closed(c))
    v0 = nw.initial_nwave(nw.rho_nodes_closed(c), theta, c.A, c.B)
    rep = nw.run_splitting(c, v0, f, max_steps=10)
    rep = nw.run_splitting(c, v0, f, max_steps=10)
    print(f"set {sid} closed grid {c.N_rho + 1}x{c.N_theta}: splitting {rep.wall_seconds / 10 * 1e3:.3f} ms/step "
          f"(device, 10 steps)", flush=True)
