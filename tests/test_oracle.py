"""CPU: pin the oracle (test infrastructure) to golden vectors produced by the
reference itself (tests/golden/make_golden.py)."""

import numpy as np
import pytest

from paper_2103_06080_b200.grid import DomainConfig, Field2D, build_axes, l2_norm
from paper_2103_06080_b200.turbulence import VelocityFields, zero_fields

WENO_CASES = ("rand", "nwave_turb", "small_odd")


@pytest.mark.parametrize("name", WENO_CASES)
def test_weno_fp64_bitwise(golden, oracle, name):
    v = golden[f"weno_{name}_v"]
    up, uq, du = golden[f"weno_{name}_coef"]
    b, dr, dt = golden[f"weno_{name}_par"]
    got = oracle.weno5_b(v, up, uq, du, b, dr, dt)
    assert np.array_equal(got, golden[f"weno_{name}_out"])
    got_np = oracle.weno5_b_numpy(v, up, uq, du, b, dr, dt)
    assert np.array_equal(got_np, golden[f"weno_{name}_out"])


@pytest.mark.parametrize("name", WENO_CASES)
def test_weno_fp32_bitwise(golden, oracle, name):
    v = golden[f"weno_{name}_v"].astype(np.float32)
    up, uq, du = (c.astype(np.float32) for c in golden[f"weno_{name}_coef"])
    b, dr, dt = golden[f"weno_{name}_par"]
    got = oracle.weno5_b(v, up, uq, du, np.float32(b), dr, dt)
    assert got.dtype == np.float32
    assert np.array_equal(got, golden[f"weno_{name}_out32"])


def test_weno_thread_count_invariant(golden, oracle):
    v = golden["weno_rand_v"]
    up, uq, du = golden["weno_rand_coef"]
    a = oracle.weno5_b(v, up, uq, du, 0.05, 0.3, 0.2, threads=1)
    b = oracle.weno5_b(v, up, uq, du, 0.05, 0.3, 0.2, threads=4)
    assert np.array_equal(a, b)


def test_phi(golden, oracle):
    z = golden["phi_z"]
    assert np.array_equal(oracle.phi(z, 1), golden["phi1"])
    assert np.array_equal(oracle.phi(z, 2), golden["phi2"])


def test_tables(golden, oracle):
    cfg = DomainConfig(N_rho=48, N_theta=42, N_sigma=77)
    t = oracle.build_tables(48, 42, cfg.rho_span, cfg.theta_span, cfg.d_sigma, cfg.A,
                            oracle.EPS_DOUBLE)
    for k, a in (("E", t.E), ("Phi1", t.Phi1), ("Phi2", t.Phi2), ("z", t.z)):
        assert np.array_equal(a, golden[f"tab48_{k}"]), k
    cs = DomainConfig(N_rho=16, N_theta=14)
    ts = oracle.build_tables(16, 14, cs.rho_span, cs.theta_span, cs.d_sigma, cs.A,
                             oracle.EPS_SINGLE, np.complex64)
    for k, a in (("E", ts.E), ("Phi1", ts.Phi1), ("Phi2", ts.Phi2), ("Phi1m2", ts.Phi1m2)):
        assert a.dtype == np.complex64
        assert np.array_equal(a, golden[f"tab16s_{k}"]), k


def test_transforms(golden, oracle):
    tr = oracle.Transforms((48, 42))
    assert np.array_equal(tr.forward(golden["fft_x"]), golden["fft_rfft2"])
    assert np.array_equal(tr.inverse(golden["fft_half"]), golden["fft_irfft2"])
    assert tr.count == 2


def test_step_functions(golden, oracle):
    cfg = DomainConfig(N_rho=32, N_theta=28, N_sigma=50, Sigma=20.0)
    tabs = oracle.build_tables(32, 28, cfg.rho_span, cfg.theta_span, cfg.d_sigma, cfg.A,
                               oracle.EPS_DOUBLE)
    coef = golden["step_coef"]

    def b_eval(stage, v):
        return oracle.weno5_b(v, coef[0][stage], coef[1][stage], coef[2][stage], cfg.B,
                              cfg.d_rho, cfg.d_theta)

    tr = oracle.Transforms((32, 28))
    got = oracle.step_exprk22(golden["step_vh0"], tabs, b_eval, cfg.d_sigma, tr)[0]
    assert np.array_equal(got, golden["step_exprk22"])
    got = oracle.step_expeuler(golden["step_vh0"], tabs, b_eval, cfg.d_sigma, tr)[0]
    assert np.array_equal(got, golden["step_euler"])


def _fields(coef):
    return VelocityFields(*coef)


@pytest.mark.parametrize("name", ["m64x56", "m48x42", "m50x40"])
@pytest.mark.parametrize("prec", ["double", "single"])
@pytest.mark.parametrize("scheme", ["exprk22", "expeuler"])
def test_short_marches(golden, golden_meta, oracle, name, prec, scheme):
    c = DomainConfig(**golden_meta["runs"][name]["config"])
    run = oracle.march(c, golden[f"{name}_v0"], _fields(golden[f"{name}_coef"]), scheme=scheme,
                       precision=prec, snapshot_sigmas=[c.d_sigma * 3, c.Sigma])
    key = f"{name}_{prec}_{scheme}"
    assert np.array_equal(run.final, golden[f"{key}_final"])
    assert np.array_equal(run.snapshots[c.d_sigma * 3], golden[f"{key}_snap3"])
    assert run.max_abs_v == golden_meta["runs"][key]["max_abs_v"]
    assert run.transforms == (4 if scheme == "exprk22" else 2) * c.N_sigma


def test_c1_march_fp64(golden, golden_meta, oracle):
    """BASELINE config C1 (demo grid, homogeneous), full 300 steps."""
    from paper_2103_06080_b200.analysis import initial_nwave

    c1 = DomainConfig(Sigma=30.0, N_sigma=300, N_rho=625, N_theta=448)
    _, rho, theta = build_axes(c1)
    run = oracle.march(c1, initial_nwave(rho, theta, c1.A, c1.B).values, zero_fields(301, 626))
    assert np.array_equal(run.final, golden["c1_double_final"])
    sig = golden_meta["runs"]["c1_double"]
    assert run.max_abs_v == sig["max_abs_v"]
    assert l2_norm(Field2D(run.final), c1.d_rho, c1.d_theta) == pytest.approx(sig["l2"], rel=1e-14)


def test_turbulence_host_restatement(golden):
    from paper_2103_06080_b200.analysis import preset_config
    from paper_2103_06080_b200.grid import rho_nodes_closed
    from paper_2103_06080_b200.turbulence import (TurbulenceParams, evaluate_fields,
                                                  sample_modes)

    c3 = preset_config(1)
    sig, _, _ = build_axes(c3)
    spec = sample_modes(TurbulenceParams(seed=0))
    f = evaluate_fields(spec, spec.lam, sig[:5], rho_nodes_closed(c3)[:33])
    got = np.stack([f.u_par, f.u_perp, f.du_perp_dsigma, f.du_perp_drho])
    ref = golden["turb_small"]
    assert np.max(np.abs(got - ref)) <= 1e-15 * np.max(np.abs(ref))


@pytest.mark.parametrize("precision", ["double", "single"])
def test_march_batch_equals_member_marches(oracle, precision):
    """The batched oracle march (used to check the 256-member C4 GPU run) is the
    per-member march, bitwise: every member is transformed and WENO'd on its own."""
    from paper_2103_06080_b200.analysis import ensemble_nwaves
    from paper_2103_06080_b200.grid import rho_nodes_closed
    from paper_2103_06080_b200.turbulence import (TurbulenceParams, evaluate_fields,
                                                  sample_modes)

    c = DomainConfig(N_rho=40, N_theta=56, N_sigma=5, Sigma=2.0)
    sig, _, _ = build_axes(c)
    spec = sample_modes(TurbulenceParams(seed=0))
    f = evaluate_fields(spec, spec.lam, sig, rho_nodes_closed(c))
    v0s, _, _ = ensemble_nwaves(c, 3, seed=2026)
    run = oracle.march_batch(c, v0s, f, precision=precision)
    assert run.transforms == 4 * c.N_sigma
    for i in range(3):
        one = oracle.march(c, v0s[i], f, precision=precision)
        assert np.array_equal(run.final[i], one.final)
        assert run.max_abs_v[i] == one.max_abs_v
