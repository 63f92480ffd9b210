"""GPU parity on exactly the configurations ``bench.py`` reports (BASELINE.json
configs C2, C4, C5), against the CPU oracle on the same inputs.

Tolerances are the north star's: fp64 max-relative <= 1e-10 on the field,
fp32 relative L2 <= 1e-4 against the reference's ``precision="single"`` path.
The oracle restates ``run_exprk22`` (``nwave/exprk.py:219-331``) and is pinned
bitwise to reference goldens (tests/test_oracle.py).

* C2 (Set 4, 10000 x 3584): K = 20 steps, fp64 on the rho-modulated N-wave
  (the bench's input) and on seed-0 turbulence, fp32 on the bench's input.
* C4: the full 256-member ensemble on the Set-1 grid (the bench's batch size),
  K = 10, every member's max|V|, full field and ground metrics (peak, rise).
* C5 (8192 x 16384) in fp32 through the rho-slab kernels, K = 3.
"""

import numpy as np
import pytest

import paper_2103_06080_b200 as nw
from paper_2103_06080_b200.grid import max_relative

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

FP64_FIELD = 1e-10
FP32_RELL2 = 1e-4
K_C2 = 20


def rel_l2(ref, num):
    ref = np.asarray(ref, np.float64)
    num = np.asarray(num, np.float64)
    return float(np.linalg.norm(ref - num) / np.linalg.norm(ref))


def c2_inputs():
    c2 = nw.preset_config(4)
    _, rho, theta = nw.build_axes(c2)
    v0 = nw.rho_modulated(c2, nw.initial_nwave(rho, theta, c2.A, c2.B))
    return c2, v0


def test_c2_fp64_k20_rho_modulated(cuda, oracle):
    """The bench headline input (C2 fp64), K = 20 steps."""
    c2, v0 = c2_inputs()
    f = nw.zero_fields(K_C2 + 1, c2.N_rho + 1)
    rep = nw.run_exprk22(c2, v0, f, max_steps=K_C2)
    ref = oracle.march(c2, v0.values, f, max_steps=K_C2)
    err = max_relative(ref.final, rep.final.values)
    assert err <= FP64_FIELD, err
    assert abs(rep.max_abs_v - ref.max_abs_v) <= 1e-12
    assert rep.transforms == 4 * K_C2


def test_c2_fp64_k20_turbulent(cuda, oracle):
    """C2 grid with seed-0 turbulence (every rho path active), K = 20."""
    c2 = nw.preset_config(4)
    sig, rho, theta = nw.build_axes(c2)
    spec = nw.sample_modes(nw.TurbulenceParams(seed=0))
    fd = nw.turbulence.evaluate_fields_device(spec, spec.lam, sig[:K_C2 + 1],
                                              nw.rho_nodes_closed(c2))
    f = nw.VelocityFields(*(t.cpu().numpy() for t in (fd.u_par, fd.u_perp, fd.du_perp_dsigma,
                                                      fd.du_perp_drho)))
    v0 = nw.initial_nwave(rho, theta, c2.A, c2.B)
    rep = nw.run_exprk22(c2, v0, f, max_steps=K_C2)
    ref = oracle.march(c2, v0.values, f, max_steps=K_C2)
    err = max_relative(ref.final, rep.final.values)
    assert err <= FP64_FIELD, err
    assert abs(rep.max_abs_v - ref.max_abs_v) <= 1e-12
    # the medium acted along rho: the field is no longer rho-independent
    assert np.ptp(rep.final.values[:, c2.N_theta // 2 + 50]) > 0


def test_c2_fp32_k20(cuda, oracle):
    """The bench's fp32 figure (C2, rho-modulated), K = 20, vs the reference's
    single-precision arithmetic."""
    c2, v0 = c2_inputs()
    f = nw.zero_fields(K_C2 + 1, c2.N_rho + 1)
    rep = nw.run_exprk22(c2, v0, f, max_steps=K_C2, precision="single")
    ref = oracle.march(c2, v0.values, f, max_steps=K_C2, precision="single")
    assert rep.final.values.dtype == np.float64
    err = rel_l2(ref.final, rep.final.values)
    assert err <= FP32_RELL2, err
    assert rep.max_abs_v == pytest.approx(ref.max_abs_v, rel=1e-5)


def test_c4_full_ensemble_256_members(cuda, oracle):
    """BASELINE C4 at the bench's batch size: 256 Set-1 members in one batched
    plan, seed-0 turbulence (so the rho transforms act), K = 10."""
    from paper_2103_06080_b200.ensemble import run_ensemble

    K = 10
    c1 = nw.preset_config(1)
    sig, _, _ = nw.build_axes(c1)
    spec = nw.sample_modes(nw.TurbulenceParams(seed=0))
    f = nw.evaluate_fields(spec, spec.lam, sig[:K + 1], nw.rho_nodes_closed(c1))
    v0s, _, _ = nw.ensemble_nwaves(c1, 256, seed=2026)
    res = run_ensemble(c1, v0s, f, max_steps=K)
    ref = oracle.march_batch(c1, v0s, f, max_steps=K)
    assert res.final.shape == (256, c1.N_rho, c1.N_theta)
    # every member's guard maximum
    assert np.max(np.abs(res.max_abs_v - ref.max_abs_v)) <= 1e-12
    # every member's full field
    errs = [max_relative(ref.final[i], res.final[i]) for i in range(256)]
    assert max(errs) <= FP64_FIELD, max(errs)
    # the ground metrics of every member (device kernel) vs the host definition
    # on the oracle's field: N-wave peak and interpolated 10-90 % rise at rho = 144
    for i in range(256):
        g = nw.ground_metrics(c1, nw.Field2D(ref.final[i]))
        assert abs(res.peak[i] - g.peak) <= 1e-10 * abs(g.peak)
        assert abs(res.rise_theta[i] - g.rise_theta) <= 1e-8 * abs(g.rise_theta)


def test_c5_fp32_slab_k3(cuda, oracle):
    """BASELINE C5 grid (8192 x 16384) in fp32 through the rho-slab kernels."""
    from paper_2103_06080_b200.slab import SlabMarch

    K = 3
    cfg = nw.DomainConfig(Sigma=120.0, N_sigma=6000, N_rho=8192, N_theta=16384)
    _, rho, theta = nw.build_axes(cfg)
    v0 = nw.rho_modulated(cfg, nw.initial_nwave(rho, theta, cfg.A, cfg.B)).values
    f = nw.zero_fields(K + 2, cfg.N_rho + 1)
    sm = SlabMarch(cfg, f, precision="single", max_steps=K)
    sm.load(v0)
    sm.march()
    rows, vmax = sm.final_rows()
    ref = oracle.march(cfg, v0, f, max_steps=K, precision="single")
    err = rel_l2(ref.final, rows.cpu().numpy())
    assert err <= FP32_RELL2, err
    assert max(max(sm.max_abs), vmax) == pytest.approx(ref.max_abs_v, rel=1e-5)
