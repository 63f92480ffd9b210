"""Developer diagnostic: run every parity probe on the GPU and print the
errors (no early stop).  Uses the oracle as the checker."""

import os
import sys
import time
import traceback

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import nwave_oracle as O  # noqa: E402
import paper_2103_06080_b200 as P  # noqa: E402
from paper_2103_06080_b200 import _build  # noqa: E402

G = dict(np.load(os.path.join(ROOT, "tests", "golden", "golden.npz")))


def mrel(a, b):
    a = np.asarray(a); b = np.asarray(b)
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300))


def probe(name, fn):
    t = time.time()
    try:
        r = fn()
        print(f"[{name}] {r}  ({time.time()-t:.2f}s)", flush=True)
    except Exception:
        print(f"[{name}] EXC", flush=True)
        traceback.print_exc()


def weno():
    out = []
    for name in ("rand", "nwave_turb", "small_odd"):
        v = G[f"weno_{name}_v"]; up, uq, du = G[f"weno_{name}_coef"]; b, dr, dt = G[f"weno_{name}_par"]
        g = P.weno5_b(v, up, uq, du, b, dr, dt)
        out.append((name, mrel(g, G[f"weno_{name}_out"])))
        g32 = P.weno5_b(v.astype(np.float32), up.astype(np.float32), uq.astype(np.float32),
                        du.astype(np.float32), b, dr, dt)
        out.append((name + "32", mrel(g32, G[f"weno_{name}_out32"])))
    return out


def fft():
    tr = P.SpectralTransforms(48, 42)
    a = mrel(tr.forward(G["fft_x"]), G["fft_rfft2"])
    b = mrel(tr.inverse(G["fft_half"]), G["fft_irfft2"])
    res = [("48x42 fwd", a), ("48x42 inv", b)]
    import scipy.fft as sf
    rng = np.random.default_rng(0)
    for (nr, nt) in [(625, 448), (1250, 448), (10000, 3584), (8192, 16384), (64, 56), (50, 40), (7, 14)]:
        x = rng.standard_normal((nr, nt))
        tr = P.SpectralTransforms(nr, nt)
        X = tr.forward(x)
        ref = sf.rfft2(x, workers=8)
        h = ref + 0.0
        h[:, 0] += 1j * rng.standard_normal(nr) * 0.1
        y = tr.inverse(h)
        res.append((f"{nr}x{nt}", mrel(X, ref), mrel(y, sf.irfft2(h, s=(nr, nt), workers=8))))
        x32 = x.astype(np.float32)
        X32 = tr.forward(x32)
        res.append((f"{nr}x{nt} f32", mrel(X32, ref)))
    return res


def phi():
    z = G["phi_z"]
    return [mrel(P.phi1(z), G["phi1"]), mrel(P.phi2(z), G["phi2"])]


def tables():
    cfg = P.DomainConfig(N_rho=48, N_theta=42, N_sigma=77)
    m = P.build_multipliers(cfg)
    return [(k, mrel(getattr(m, k), G[f"tab48_{k}"])) for k in ("E", "Phi1", "Phi2", "z")]


def steps():
    cfg = P.DomainConfig(N_rho=32, N_theta=28, N_sigma=50, Sigma=20.0)
    m = P.build_multipliers(cfg)
    coef = G["step_coef"]

    def b_eval(stage, v):
        return P.weno5_b(v, coef[0][stage], coef[1][stage], coef[2][stage], cfg.B, cfg.d_rho, cfg.d_theta)
    tr = P.SpectralTransforms(32, 28)
    a = P.exprk22_step(G["step_vh0"], m, b_eval, cfg.d_sigma, tr)[0]
    b = P.exp_euler_step(G["step_vh0"], m, b_eval, cfg.d_sigma, tr)[0]
    return [mrel(a, G["step_exprk22"]), mrel(b, G["step_euler"])]


def marches():
    import json
    meta = json.load(open(os.path.join(ROOT, "tests", "golden", "golden_meta.json")))
    res = []
    for name in ("m64x56", "m48x42", "m50x40"):
        c = P.DomainConfig(**meta["runs"][name]["config"])
        f = P.VelocityFields(*G[f"{name}_coef"])
        for prec in ("double", "single"):
            for scheme in ("exprk22", "expeuler"):
                rep = P.run_exprk22(c, G[f"{name}_v0"], f, precision=prec, scheme=scheme,
                                    snapshot_sigmas=[c.d_sigma * 3, c.Sigma])
                key = f"{name}_{prec}_{scheme}"
                res.append((key, mrel(rep.final.values, G[f"{key}_final"]),
                            mrel(rep.snapshots[c.d_sigma * 3].values, G[f"{key}_snap3"]),
                            rep.max_abs_v - meta["runs"][key]["max_abs_v"]))
    return res


def c1():
    c1 = P.DomainConfig(Sigma=30.0, N_sigma=300, N_rho=625, N_theta=448)
    _, rho, theta = P.build_axes(c1)
    v0 = P.initial_nwave(rho, theta, c1.A, c1.B)
    out = []
    for prec in ("double", "single"):
        t = time.time()
        rep = P.run_exprk22(c1, v0, P.zero_fields(301, 626), precision=prec)
        out.append((prec, mrel(rep.final.values, G[f"c1_{prec}_final"]),
                    P.relative_error(P.Field2D(G[f"c1_{prec}_final"]), rep.final, c1.d_rho, c1.d_theta),
                    time.time() - t, float(np.median(rep.step_seconds))))
    return out


def c3():
    c3 = P.preset_config(1)
    sig, rho, theta = P.build_axes(c3)
    spec = P.sample_modes(P.TurbulenceParams(seed=0))
    f = P.evaluate_fields(spec, spec.lam, sig, P.rho_nodes_closed(c3))
    v0 = P.initial_nwave(rho, theta, c3.A, c3.B)
    out = []
    for prec in ("double", "single"):
        rep = P.run_exprk22(c3, v0, f, precision=prec, snapshot_sigmas=[60.0])
        out.append((prec, mrel(rep.final.values[::8], G[f"c3_{prec}_final_sub"]),
                    mrel(rep.snapshots[60.0].values[::8], G[f"c3_{prec}_snap60_sub"]),
                    rep.max_abs_v, float(np.median(rep.step_seconds))))
    return out


def big():
    import torch
    from paper_2103_06080_b200.plan import DevicePlan
    out = []
    for prec in ("double", "single"):
        c = P.preset_config(4)
        _, rho, theta = P.build_axes(c)
        v0 = P.rho_modulated(c, P.initial_nwave(rho, theta, c.A, c.B)).values
        plan = DevicePlan(c.N_rho, c.N_theta, 1, prec, c.d_sigma, c.rho_span, c.theta_span, c.A, c.B,
                          2.0**-53 if prec == "double" else 2.0**-24)
        plan.set_coeffs(None, None, None, n_rows=64)
        plan.load_physical(v0)
        plan.march("exprk22", 0, 4, timing=False)
        torch.cuda.synchronize()
        t = time.time()
        ma, sm, _ = plan.march("exprk22", 4, 40, timing=True)
        torch.cuda.synchronize()
        dt = time.time() - t
        out.append((prec, "ms/step events", float(np.median(sm[:, 0])), "wall/step", dt / 40 * 1e3))
        t = time.time()
        plan.march("exprk22", 44, 16, timing=False)
        torch.cuda.synchronize()
        out.append(("graph ms/step", (time.time() - t) / 16 * 1e3))
        km = plan.profile_kernels("exprk22", 50, 8) / 8
        out.append(("kernels ms [c2r weno r2c rho] x2", [round(float(x), 4) for x in km]))
        plan.close()
    return out


if __name__ == "__main__":
    _build.build()
    which = sys.argv[1:] or ["weno", "fft", "phi", "tables", "steps", "marches", "c1", "c3", "big"]
    for w in which:
        probe(w, globals()[w])
