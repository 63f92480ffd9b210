"""scratch: small runs of every kernel family for compute-sanitizer."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2103_06080_b200 as nw
c = nw.DomainConfig(N_rho=64, N_theta=56, N_sigma=4, Sigma=1.6)
sig, rho, theta = nw.build_axes(c)
spec = nw.sample_modes(nw.TurbulenceParams(seed=1))
f = nw.evaluate_fields(spec, spec.lam, sig, nw.rho_nodes_closed(c))
v0 = nw.rho_modulated(c, nw.initial_nwave(rho, theta, c.A, c.B), depth=0.3)
for prec in ("double", "single"):
    r = nw.run_exprk22(c, v0, f, precision=prec, snapshot_sigmas=[0.4, 1.6])
    print(prec, r.max_abs_v)
r = nw.run_exprk22(c, v0, f, scheme="expeuler", timing=False)
print("euler", r.max_abs_v)
# long fp64 column (bulk loads, stagger, prefetch) on a small theta extent
c2 = nw.DomainConfig(N_rho=10000, N_theta=14, N_sigma=2, Sigma=1.0)
_, rho2, theta2 = nw.build_axes(c2)
v2 = nw.rho_modulated(c2, nw.initial_nwave(rho2, theta2, c2.A, c2.B))
print("long", nw.run_exprk22(c2, v2, nw.zero_fields(3, 10001)).max_abs_v)
print("long32", nw.run_exprk22(c2, v2, nw.zero_fields(3, 10001), precision="single").max_abs_v)
tr = nw.SpectralTransforms(48, 42)
x = np.random.default_rng(0).standard_normal((48, 42))
print("fft", float(np.abs(tr.inverse(tr.forward(x)) - x).max()))
print("weno", float(np.abs(nw.weno5_b(v0.values, f.u_par[0, :64], f.u_perp[0, :64], f.du_perp_drho[0, :64], c.B, c.d_rho, c.d_theta)).max()))
vc = nw.initial_nwave(nw.rho_nodes_closed(c), theta, c.A, c.B)
print("split", nw.run_splitting(c, vc, f).max_abs_v)
from paper_2103_06080_b200.slab import SlabMarch
sm = SlabMarch(c, f)
sm.load(v0.values)
sm.march()
print("slab", sm.final_rows()[1])
from paper_2103_06080_b200.ensemble import run_ensemble
v0s, _, _ = nw.ensemble_nwaves(c, 3, seed=2026)
print("ens", run_ensemble(c, v0s, f).max_abs_v)
print("ok")
