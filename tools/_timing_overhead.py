"""scratch: wall time of run_exprk22 with the default per-step timing buckets
(timed graph replays) vs timing=False (plain graph replays), small and large grids."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2103_06080_b200 as nw
for name, cfg in (("c1", nw.DomainConfig(Sigma=30.0, N_sigma=300, N_rho=625, N_theta=448)),
                  ("set1", nw.preset_config(1)), ("set3", nw.preset_config(3))):
    _, rho, theta = nw.build_axes(cfg)
    v0 = nw.initial_nwave(rho, theta, cfg.A, cfg.B)
    f = nw.zero_fields(cfg.N_sigma + 1, cfg.N_rho + 1)
    steps = min(cfg.N_sigma, 300)
    for timing in (True, False, True, False):
        t0 = time.perf_counter()
        rep = nw.run_exprk22(cfg, v0, f, max_steps=steps, timing=timing)
        t = time.perf_counter() - t0
        print(name, "timing" if timing else "graph", f"{t / steps * 1e3:.4f} ms/step wall,",
              f"device step median {np.median(rep.step_seconds) * 1e3:.4f} ms", flush=True)
