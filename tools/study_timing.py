"""Wall time of convergence studies with sequential vs concurrent marches
(SURVEY row f3): the paper's criterion-1 study at full scale (5000 x 1792,
N_sigma 200..1200 vs 2400) and a Set-1 study (1250 x 448, 75..300 vs 600)."""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2103_06080_b200 as nw  # noqa: E402


def study(cfg, n_list, n_ref, conc):
    spec = nw.sample_modes(nw.TurbulenceParams(seed=0))
    sigma = np.arange(n_ref + 1) * (cfg.Sigma / n_ref)
    master = nw.turbulence.evaluate_fields_device(spec, spec.lam, sigma, nw.rho_nodes_closed(cfg))
    import torch
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    rows = nw.convergence_study(cfg, n_list, n_ref, fields_master=master, timing=False,
                                concurrency=conc)
    torch.cuda.synchronize()
    return time.perf_counter() - t0, [(r.n_sigma, r.err, r.beta) for r in rows]


full = nw.DomainConfig(Sigma=30.0, N_sigma=2400, N_rho=5000, N_theta=7 * 256)
set1 = nw.DomainConfig(Sigma=120.0, N_sigma=600, N_rho=1250, N_theta=448)
out = {}
for name, cfg, nl, nref in (("criterion1_full", full, [200, 300, 400, 600, 800, 1200], 2400),
                            ("set1", set1, [75, 100, 150, 200, 300], 600)):
    study(cfg, nl[:1], nl[0] * 2, 1)  # warm-up
    res = {}
    for conc in (1, 2, 4):
        t, betas = study(cfg, nl, nref, conc)
        res[f"conc{conc}_s"] = round(t, 3)
        res[f"conc{conc}_rows"] = [[n, e, b] for n, e, b in betas]
    out[name] = res
    print(name, json.dumps(res), flush=True)
