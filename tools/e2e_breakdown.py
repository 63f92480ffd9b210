"""Where does run_exprk22's end-to-end time go at C2?  (developer tool)"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2103_06080_b200 as nw
from paper_2103_06080_b200.plan import DevicePlan

cfg = nw.preset_config(4)
_, rho, theta = nw.build_axes(cfg)
v0 = nw.rho_modulated(cfg, nw.initial_nwave(rho, theta, cfg.A, cfg.B)).values
f = nw.zero_fields(201, cfg.N_rho + 1)
torch.zeros(1, device="cuda")
for rep in range(2):
    T = {}
    t = time.perf_counter(); s = t
    plan = DevicePlan(cfg.N_rho, cfg.N_theta, 1, "double", cfg.d_sigma, cfg.rho_span, cfg.theta_span, cfg.A, cfg.B, 2.0**-53)
    torch.cuda.synchronize(); T["plan"] = time.perf_counter() - t; t = time.perf_counter()
    plan.set_coeffs(f.u_par, f.u_perp, f.du_perp_drho, n_rows=201)
    torch.cuda.synchronize(); T["coeffs"] = time.perf_counter() - t; t = time.perf_counter()
    plan.load_physical(v0)
    torch.cuda.synchronize(); T["load"] = time.perf_counter() - t; t = time.perf_counter()
    plan.march("exprk22", 0, 200, timing=False)
    torch.cuda.synchronize(); T["march"] = time.perf_counter() - t; t = time.perf_counter()
    out, mx = plan.store_physical()
    torch.cuda.synchronize(); T["store"] = time.perf_counter() - t; t = time.perf_counter()
    host = out[0].to("cpu", torch.float64).numpy()
    T["d2h"] = time.perf_counter() - t; t = time.perf_counter()
    plan.close()
    T["close"] = time.perf_counter() - t
    T["total"] = time.perf_counter() - s
    print({k: round(v * 1e3, 1) for k, v in T.items()})
t = time.perf_counter()
rep = nw.run_exprk22(cfg, v0, f, max_steps=200, timing=False)
print("run_exprk22 wall ms", round((time.perf_counter() - t) * 1e3, 1))
