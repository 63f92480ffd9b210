"""Developer diagnostic: where the end-to-end run_exprk22 time goes at C2
(full 2400-step march, host arrays), by timing the DevicePlan calls the
public entry point makes (each wrapped with a device synchronise)."""
import functools
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2103_06080_b200 as nw  # noqa: E402
from paper_2103_06080_b200 import exprk  # noqa: E402
from paper_2103_06080_b200.plan import DevicePlan  # noqa: E402

prec = sys.argv[1] if len(sys.argv) > 1 else "double"
T = {}


def timed(name, fn):
    @functools.wraps(fn)
    def w(*a, **k):
        torch.cuda.synchronize()
        t = time.perf_counter()
        r = fn(*a, **k)
        torch.cuda.synchronize()
        T[name] = T.get(name, 0.0) + time.perf_counter() - t
        return r
    return w


for n in ("__init__", "set_coeffs", "load_physical", "march", "store_physical", "close"):
    setattr(DevicePlan, n, timed(n, getattr(DevicePlan, n)))
exprk._to_host64 = timed("to_host64", exprk._to_host64)

cfg = nw.preset_config(4)
sig, rho, theta = nw.build_axes(cfg)
v0 = nw.rho_modulated(cfg, nw.initial_nwave(rho, theta, cfg.A, cfg.B))
f = nw.zero_fields(cfg.N_sigma + 1, cfg.N_rho + 1)
nw.run_exprk22(cfg, v0, f, max_steps=3, precision=prec)
T.clear()
t = time.perf_counter()
rep = nw.run_exprk22(cfg, v0, f, precision=prec)
wall = time.perf_counter() - t
print(prec, "wall s", round(wall, 4), {k: round(v, 4) for k, v in T.items()},
      "unaccounted", round(wall - sum(T.values()), 4), "steps", rep.n_steps)
