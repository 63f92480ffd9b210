"""Developer check: warp-specialised rho pass (NWB_RHO_WS) vs the default pass, bitwise."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2103_06080_b200 as nw
from paper_2103_06080_b200.plan import DevicePlan

def run(nr, nt, batch, prec, scheme, ws):
    os.environ.pop("NWB_RHO_WS", None)
    if ws:
        os.environ["NWB_RHO_WS"] = ws
    cfg = nw.DomainConfig(N_rho=nr, N_theta=nt, N_sigma=4, Sigma=1.6)
    _, rho, theta = nw.build_axes(cfg)
    v0 = nw.rho_modulated(cfg, nw.initial_nwave(rho, theta, cfg.A, cfg.B)).values
    v0 = np.stack([v0 * (1 + 0.1 * i) for i in range(batch)]) if batch > 1 else v0
    plan = DevicePlan(nr, nt, batch, prec, cfg.d_sigma, cfg.rho_span, cfg.theta_span, cfg.A, cfg.B,
                      nw.EPS_DOUBLE if prec == "double" else nw.EPS_SINGLE)
    plan.set_coeffs(None, None, None, n_rows=8)
    plan.load_physical(v0)
    plan.march(scheme, 0, 4)
    out, _ = plan.store_physical()
    plan.close()
    return out.cpu().numpy()

ok = True
for nr, nt, batch, prec, scheme in [(64, 56, 1, "double", "exprk22"), (625, 448, 1, "double", "exprk22"),
                                    (10000, 64, 1, "double", "exprk22"), (50, 56, 4, "double", "exprk22"),
                                    (105, 70, 1, "double", "expeuler"), (1000, 448, 1, "single", "exprk22"),
                                    (10000, 3584, 1, "double", "exprk22")]:
    a = run(nr, nt, batch, prec, scheme, None)
    for ws in ("256", "256,256", "384,128"):
        b = run(nr, nt, batch, prec, scheme, ws)
        eq = np.array_equal(a, b)
        ok &= eq
        print(nr, nt, batch, prec, scheme, ws, "bitwise" if eq else f"DIFF max {np.max(np.abs(a - b)):.3e}", flush=True)
print("ALL OK" if ok else "MISMATCH")
