"""GPU parity: the sm_100a path (through the C ABI / public API) against the
CPU oracle and the reference goldens.  Tolerances (BASELINE.json north star):
fp64 max-relative <= 1e-10 on fields, fp32 relative L2 <= 1e-4; kernel-level
fp64 checks are held much tighter (<= 1e-13) to catch regressions early."""

import json

import numpy as np
import pytest

import paper_2103_06080_b200 as nw
from paper_2103_06080_b200.grid import max_relative

pytestmark = pytest.mark.gpu

FP64_FIELD = 1e-10
FP64_KERNEL = 1e-13
FP32_RELL2 = 1e-4


def rel_l2(ref, num):
    ref = np.asarray(ref, np.float64)
    num = np.asarray(num, np.float64)
    return float(np.linalg.norm(ref - num) / np.linalg.norm(ref))


# ------------------------------------------------------------------ WENO

@pytest.mark.parametrize("name", ["rand", "nwave_turb", "small_odd"])
def test_weno_vs_golden(cuda, golden, name):
    v = golden[f"weno_{name}_v"]
    up, uq, du = golden[f"weno_{name}_coef"]
    b, dr, dt = golden[f"weno_{name}_par"]
    got = nw.weno5_b(v, up, uq, du, b, dr, dt)
    assert got.dtype == np.float64
    assert max_relative(golden[f"weno_{name}_out"], got) <= FP64_KERNEL
    got32 = nw.weno5_b(*(a.astype(np.float32) for a in (v, up, uq, du)), np.float32(b), dr, dt)
    assert got32.dtype == np.float32
    assert rel_l2(golden[f"weno_{name}_out32"], got32) <= 1e-6


@pytest.mark.parametrize("shape", [(1250, 448), (257, 130), (3, 5), (16, 2048), (130, 70),
                                   (33, 96)])
def test_weno_fp32_packed_vs_oracle(cuda, oracle, shape):
    """fp32 WENO runs k_weno_x2 (two columns per lane on the packed FFMA2 pipe):
    partial 64-column tiles, periodic wrap, extents below one tile."""
    rng = np.random.default_rng(7 + sum(shape))
    v = rng.standard_normal(shape).astype(np.float32)
    up, uq, du = (np.float32(0.03) * rng.standard_normal(shape[0]).astype(np.float32)
                  for _ in range(3))
    ref = oracle.weno5_b(v, up, uq, du, 0.05, 0.32, 0.21)
    got = nw.weno5_b(v, up, uq, du, np.float32(0.05), 0.32, 0.21)
    assert got.dtype == np.float32 and got.shape == shape
    assert rel_l2(ref, got) <= 1e-6


@pytest.mark.parametrize("shape", [(1250, 448), (257, 130), (3, 5), (16, 2048)])
def test_weno_vs_oracle_random_shapes(cuda, oracle, shape):
    rng = np.random.default_rng(sum(shape))
    v = rng.standard_normal(shape)
    up, uq, du = (0.03 * rng.standard_normal(shape[0]) for _ in range(3))
    ref = oracle.weno5_b(v, up, uq, du, 0.05, 0.32, 0.21)
    got = nw.weno5_b(v, up, uq, du, 0.05, 0.32, 0.21)
    assert max_relative(ref, got) <= FP64_KERNEL


def test_weno_batched_and_device_tensors(cuda, oracle):
    import torch

    rng = np.random.default_rng(5)
    v = rng.standard_normal((3, 40, 56))
    up, uq, du = (0.02 * rng.standard_normal(40) for _ in range(3))
    out = nw.weno5_b(torch.from_numpy(v).to(cuda), *(torch.from_numpy(c).to(cuda) for c in (up, uq, du)),
                     0.05, 0.3, 0.2)
    assert out.is_cuda and out.shape == (3, 40, 56)
    for i in range(3):
        # alpha_theta is per member (each member is an independent field)
        ref = oracle.weno5_b(v[i], up, uq, du, 0.05, 0.3, 0.2)
        assert max_relative(ref, out[i].cpu().numpy()) <= FP64_KERNEL


# ------------------------------------------------------------------ transforms

@pytest.mark.parametrize("shape", [(48, 42), (625, 448), (1250, 448), (10000, 3584),
                                   (8192, 16384), (7, 14), (50, 40), (2, 2)])
def test_rfft2_irfft2_vs_scipy(cuda, shape):
    import scipy.fft as sfft

    rng = np.random.default_rng(shape[0])
    x = rng.standard_normal(shape)
    tr = nw.SpectralTransforms(*shape)
    X = tr.forward(x)
    ref = sfft.rfft2(x, workers=8)
    assert max_relative(ref, X) <= 1e-14
    h = ref.copy()
    h[:, 0] += 0.3j * rng.standard_normal(shape[0])     # imaginary DC / Nyquist garbage
    h[:, -1] += 0.3j * rng.standard_normal(shape[0])    # must be dropped like pocketfft
    y = tr.inverse(h)
    assert max_relative(sfft.irfft2(h, s=shape, workers=8), y) <= 1e-14
    assert tr.count == 2
    x32 = x.astype(np.float32)
    assert rel_l2(ref, tr.forward(x32)) <= 1e-6


def test_transforms_golden(cuda, golden):
    tr = nw.SpectralTransforms(48, 42)
    assert max_relative(golden["fft_rfft2"], tr.forward(golden["fft_x"])) <= 1e-14
    assert max_relative(golden["fft_irfft2"], tr.inverse(golden["fft_half"])) <= 1e-14


def test_unsupported_sizes_fail_loudly(cuda):
    with pytest.raises(nw.UnsupportedSizeError):
        nw.SpectralTransforms(11, 14).forward(np.zeros((11, 14)))
    with pytest.raises(nw.UnsupportedSizeError):
        nw.SpectralTransforms(16, 15).forward(np.zeros((16, 15)))


# ------------------------------------------------------------------ tables / phi

def test_phi_vs_golden(cuda, golden):
    z = golden["phi_z"]
    for fn, key in ((nw.phi1, "phi1"), (nw.phi2, "phi2")):
        ref = golden[key]
        got = fn(z)
        assert np.all(np.abs(got - ref) <= 1e-14 * np.maximum(np.abs(ref), 1e-300))


def test_tables_vs_golden(cuda, golden):
    m = nw.build_multipliers(nw.DomainConfig(N_rho=48, N_theta=42, N_sigma=77))
    for k in ("E", "Phi1", "Phi2", "z"):
        ref = golden[f"tab48_{k}"]
        assert np.max(np.abs(getattr(m, k) - ref)) <= 1e-15 * max(np.max(np.abs(ref)), 1.0), k
    ms = nw.build_multipliers(nw.DomainConfig(N_rho=16, N_theta=14), nw.EPS_SINGLE,
                              dtype=np.complex64)
    for k in ("E", "Phi1", "Phi2", "Phi1m2"):
        assert getattr(ms, k).dtype == np.complex64
        assert np.max(np.abs(getattr(ms, k) - golden[f"tab16s_{k}"])) <= 1e-7, k


def test_tables_set4_vs_oracle_sample(cuda, oracle):
    """Set-4 tables on the device vs the oracle on a row sample (j symmetric)."""
    cfg = nw.preset_config(4)
    m = nw.build_multipliers(cfg)
    rows = np.r_[0:5, 4998:5003, 9995:10000]
    j = (np.fft.fftfreq(cfg.N_rho) * cfg.N_rho)[rows]
    k = np.arange(cfg.N_theta // 2 + 1, dtype=np.float64)
    xi = 2.0 * np.pi * j / cfg.rho_span
    om = 2.0 * np.pi * k / cfg.theta_span
    den = 1j * om[None, :] + oracle.EPS_DOUBLE / (4.0 * np.pi)
    z = cfg.d_sigma * (-(xi[:, None] ** 2) / (4.0 * np.pi * den) - cfg.A * om[None, :] ** 2)
    for got, ref in ((m.E[rows], np.exp(z)), (m.Phi1[rows], oracle.phi(z, 1)),
                     (m.Phi2[rows], oracle.phi(z, 2))):
        err = np.abs(got - ref) / np.maximum(np.abs(ref), 1e-300)
        assert np.max(err[np.abs(ref) > 1e-280]) <= 2e-15, np.max(err)
    # bitwise symmetry j <-> -j
    assert np.array_equal(m.E[1:5], m.E[-1:-5:-1])


# ------------------------------------------------------------------ step API

def test_step_functions_vs_golden(cuda, golden):
    cfg = nw.DomainConfig(N_rho=32, N_theta=28, N_sigma=50, Sigma=20.0)
    m = nw.build_multipliers(cfg)
    coef = golden["step_coef"]

    def b_eval(stage, v):
        return nw.weno5_b(v, coef[0][stage], coef[1][stage], coef[2][stage], cfg.B,
                          cfg.d_rho, cfg.d_theta)

    tr = nw.SpectralTransforms(32, 28)
    a, v = nw.exprk22_step(golden["step_vh0"], m, b_eval, cfg.d_sigma, tr)
    assert max_relative(golden["step_exprk22"], a) <= FP64_KERNEL
    b, _ = nw.exp_euler_step(golden["step_vh0"], m, b_eval, cfg.d_sigma, tr)
    assert max_relative(golden["step_euler"], b) <= FP64_KERNEL
    assert tr.count == 6


# ------------------------------------------------------------------ marches

@pytest.mark.parametrize("name", ["m64x56", "m48x42", "m50x40"])
@pytest.mark.parametrize("scheme", ["exprk22", "expeuler"])
def test_short_marches_vs_golden(cuda, golden, golden_meta, name, scheme):
    c = nw.DomainConfig(**golden_meta["runs"][name]["config"])
    f = nw.VelocityFields(*golden[f"{name}_coef"])
    for prec in ("double", "single"):
        rep = nw.run_exprk22(c, golden[f"{name}_v0"], f, precision=prec, scheme=scheme,
                             snapshot_sigmas=[c.d_sigma * 3, c.Sigma])
        key = f"{name}_{prec}_{scheme}"
        ref_max = golden_meta["runs"][key]["max_abs_v"]
        assert rep.precision == prec and rep.solver == scheme
        assert rep.transforms == (4 if scheme == "exprk22" else 2) * c.N_sigma
        assert set(rep.snapshots) == {c.d_sigma * 3, c.Sigma}
        if prec == "double":
            assert max_relative(golden[f"{key}_final"], rep.final.values) <= FP64_FIELD
            assert max_relative(golden[f"{key}_snap3"], rep.snapshots[c.d_sigma * 3].values) <= FP64_FIELD
            assert abs(rep.max_abs_v - ref_max) <= 1e-12
        else:
            assert rel_l2(golden[f"{key}_final"], rep.final.values) <= FP32_RELL2
            assert abs(rep.max_abs_v - ref_max) <= 1e-5
        assert rep.final.values.dtype == np.float64


def test_c1_full_march(cuda, golden, golden_meta):
    """BASELINE C1: demo grid, homogeneous, 300 steps, fp64 and fp32."""
    c1 = nw.DomainConfig(Sigma=30.0, N_sigma=300, N_rho=625, N_theta=448)
    _, rho, theta = nw.build_axes(c1)
    v0 = nw.initial_nwave(rho, theta, c1.A, c1.B)
    rep = nw.run_exprk22(c1, v0, nw.zero_fields(301, 626))
    sig = golden_meta["runs"]["c1_double"]
    assert max_relative(golden["c1_double_final"], rep.final.values) <= FP64_FIELD
    assert abs(rep.max_abs_v - sig["max_abs_v"]) <= 1e-12
    assert nw.l2_norm(rep.final, c1.d_rho, c1.d_theta) == pytest.approx(sig["l2"], rel=1e-12)
    rs = nw.run_exprk22(c1, v0, nw.zero_fields(301, 626), precision="single")
    assert rel_l2(golden["c1_single_final"], rs.final.values) <= FP32_RELL2
    # ground metrics agree (computed by one function on both fields)
    g_ref = nw.ground_metrics(c1, nw.Field2D(golden["c1_double_final"]))
    g_got = nw.ground_metrics(c1, rep.final)
    assert g_got.peak == pytest.approx(g_ref.peak, rel=1e-10)
    assert g_got.rise_theta == pytest.approx(g_ref.rise_theta, rel=1e-8)


def test_c3_turbulent_march(cuda, golden, golden_meta):
    """BASELINE C3: Set 1, turbulent medium (seed 0), 300 steps to the ground."""
    c3 = nw.preset_config(1)
    sig, rho, theta = nw.build_axes(c3)
    spec = nw.sample_modes(nw.TurbulenceParams(seed=0))
    f = nw.evaluate_fields(spec, spec.lam, sig, nw.rho_nodes_closed(c3))
    v0 = nw.initial_nwave(rho, theta, c3.A, c3.B)
    rep = nw.run_exprk22(c3, v0, f, snapshot_sigmas=[60.0])
    meta = golden_meta["runs"]["c3_double"]
    assert max_relative(golden["c3_double_final_sub"], rep.final.values[::8]) <= FP64_FIELD
    assert max_relative(golden["c3_double_snap60_sub"], rep.snapshots[60.0].values[::8]) <= FP64_FIELD
    assert abs(rep.max_abs_v - meta["max_abs_v"]) <= 1e-12
    assert rep.max_abs_v <= 5.0  # acceptance criterion 10
    row = rep.final.values[int(round(144 / c3.d_rho))]
    assert max_relative(golden["c3_double_row144"], row) <= FP64_FIELD
    rs = nw.run_exprk22(c3, v0, f, precision="single")
    assert rel_l2(golden["c3_single_final_sub"], rs.final.values[::8]) <= FP32_RELL2


def test_c2_truncated_vs_oracle(cuda, oracle):
    """BASELINE C2 (Set 4, 10000 x 3584), rho-modulated N-wave, K = 3 steps."""
    c2 = nw.preset_config(4)
    _, rho, theta = nw.build_axes(c2)
    v0 = nw.rho_modulated(c2, nw.initial_nwave(rho, theta, c2.A, c2.B))
    f = nw.zero_fields(5, c2.N_rho + 1)
    rep = nw.run_exprk22(c2, v0, f, max_steps=3)
    ref = oracle.march(c2, v0.values, f, max_steps=3)
    assert max_relative(ref.final, rep.final.values) <= FP64_FIELD
    assert abs(rep.max_abs_v - ref.max_abs_v) <= 1e-12


def test_determinism_bitwise(cuda, golden, golden_meta):
    c = nw.DomainConfig(**golden_meta["runs"]["m64x56"]["config"])
    f = nw.VelocityFields(*golden["m64x56_coef"])
    a = nw.run_exprk22(c, golden["m64x56_v0"], f)
    b = nw.run_exprk22(c, golden["m64x56_v0"], f, timing=False)
    assert np.array_equal(a.final.values, b.final.values)


def test_instability_guard_first_step(cuda, oracle):
    cfg = nw.DomainConfig(N_rho=32, N_theta=28, N_sigma=40, Sigma=40.0, A=1e-4, B=4.0)
    _, rho, theta = nw.build_axes(cfg)
    v0 = 3.0 * np.cos(2 * np.pi * (theta - cfg.theta_min) / cfg.theta_span)[None, :] * np.ones((32, 1))
    f = nw.zero_fields(41, 33)
    ref = oracle.march(cfg, v0, f, guard=4.0)
    assert ref.failed_sigma is not None
    with pytest.warns(UserWarning):
        with pytest.raises(nw.InstabilityError) as ei:
            nw.run_exprk22(cfg, v0, f, guard=4.0)
    assert ei.value.sigma == pytest.approx(ref.failed_sigma)


def test_zero_field_stays_zero(cuda):
    cfg = nw.DomainConfig(N_rho=32, N_theta=28, N_sigma=5, Sigma=1.0)
    rep = nw.run_exprk22(cfg, nw.Field2D(np.zeros((32, 28))), nw.zero_fields(6, 33))
    assert rep.max_abs_v == 0.0
    assert np.all(rep.final.values == 0.0)


def test_validation_errors(cuda):
    cfg = nw.DomainConfig(N_rho=32, N_theta=28, N_sigma=5, Sigma=1.0)
    f = nw.zero_fields(6, 33)
    with pytest.raises(ValueError):
        nw.run_exprk22(cfg, np.zeros((32, 28)), f, scheme="rk4")
    with pytest.raises(ValueError):
        nw.run_exprk22(cfg, np.zeros((32, 28)), f, precision="half")
    with pytest.raises(ValueError):
        nw.run_exprk22(cfg, np.zeros((31, 28)), f)
    with pytest.raises(ValueError):
        nw.run_exprk22(cfg, np.zeros((32, 28)), nw.zero_fields(3, 33))
    hot = nw.DomainConfig(N_rho=32, N_theta=28, N_sigma=2, Sigma=100.0)
    with pytest.raises(nw.CflViolationError):
        nw.run_exprk22(hot, np.zeros((32, 28)), nw.zero_fields(3, 33), cfl="error")


def test_budget_exceeded(cuda):
    cfg = nw.DomainConfig(N_rho=64, N_theta=56, N_sigma=4000, Sigma=40.0)
    _, rho, theta = nw.build_axes(cfg)
    with pytest.raises(nw.BudgetExceededError):
        nw.run_exprk22(cfg, nw.initial_nwave(rho, theta, cfg.A, cfg.B),
                       nw.zero_fields(4001, 65), max_seconds=1e-4)


def test_device_plan_batch_members_independent(cuda, oracle):
    """Ensemble plan: every member equals its own single run (C4 building block)."""
    import torch
    from paper_2103_06080_b200.plan import DevicePlan

    cfg = nw.DomainConfig(N_rho=50, N_theta=56, N_sigma=6, Sigma=2.4)
    v0s, _, _ = nw.ensemble_nwaves(cfg, 4, seed=2026)
    f = nw.zero_fields(7, 51)
    plan = DevicePlan(50, 56, 4, "double", cfg.d_sigma, cfg.rho_span, cfg.theta_span, cfg.A,
                      cfg.B, nw.EPS_DOUBLE)
    plan.set_coeffs(f.u_par, f.u_perp, f.du_perp_drho)
    plan.load_physical(v0s)
    max_abs, _, _ = plan.march("exprk22", 0, 6)
    out, mx = plan.store_physical()
    out = out.cpu().numpy()
    for i in range(4):
        ref = oracle.march(cfg, v0s[i], f)
        assert max_relative(ref.final, out[i]) <= FP64_FIELD
        assert max(max_abs[i].max(), mx[i]) == pytest.approx(ref.max_abs_v, abs=1e-12)
    plan.close()


def test_spectrum_roundtrip_through_plan(cuda):
    import torch
    from paper_2103_06080_b200.plan import DevicePlan

    rng = np.random.default_rng(3)
    x = rng.standard_normal((2, 40, 56))
    plan = DevicePlan(40, 56, 2, "double")
    plan.load_physical(x)
    vh = plan.store_spectrum().cpu().numpy()
    import scipy.fft as sfft

    assert max_relative(sfft.rfft2(x, axes=(1, 2)), vh) <= 1e-14
    plan.load_spectrum(vh)
    back, mx = plan.store_physical()
    assert max_relative(x, back.cpu().numpy()) <= 1e-14
    assert mx == pytest.approx(np.abs(x).max(axis=(1, 2)), rel=1e-14)
    plan.close()


def test_run_ensemble_members_match_single_runs(cuda, oracle):
    """BASELINE C4 building block: batched ensemble == per-member oracle runs."""
    from paper_2103_06080_b200.ensemble import run_ensemble, shard_members

    cfg = nw.DomainConfig(N_rho=50, N_theta=56, N_sigma=8, Sigma=3.2)
    v0s, _, _ = nw.ensemble_nwaves(cfg, 6, seed=2026)
    f = nw.zero_fields(9, 51)
    res = run_ensemble(cfg, v0s, f, members=shard_members(6, 2, 1))
    assert list(res.members) == [3, 4, 5]
    for i, m in enumerate(res.members):
        ref = oracle.march(cfg, v0s[m], f)
        assert max_relative(ref.final, res.final[i]) <= FP64_FIELD
        assert res.max_abs_v[i] == pytest.approx(ref.max_abs_v, abs=1e-12)


def test_device_turbulence_generator_vs_reference(cuda, golden):
    """device mode sum == reference evaluate_fields (golden)."""
    c3 = nw.preset_config(1)
    sig, _, _ = nw.build_axes(c3)
    spec = nw.sample_modes(nw.TurbulenceParams(seed=0))
    f = nw.turbulence.evaluate_fields_device(spec, spec.lam, sig[:5], nw.rho_nodes_closed(c3)[:33])
    got = np.stack([t.cpu().numpy() for t in (f.u_par, f.u_perp, f.du_perp_dsigma, f.du_perp_drho)])
    ref = golden["turb_small"]
    assert np.max(np.abs(got - ref)) <= 1e-14 * np.max(np.abs(ref))


def test_c3_with_device_medium(cuda, golden, golden_meta):
    """C3 marched with coefficients generated and kept on the device."""
    c3 = nw.preset_config(1)
    sig, rho, theta = nw.build_axes(c3)
    spec = nw.sample_modes(nw.TurbulenceParams(seed=0))
    f = nw.turbulence.evaluate_fields_device(spec, spec.lam, sig, nw.rho_nodes_closed(c3))
    rep = nw.run_exprk22(c3, nw.initial_nwave(rho, theta, c3.A, c3.B), f)
    assert max_relative(golden["c3_double_final_sub"], rep.final.values[::8]) <= FP64_FIELD
    assert abs(rep.max_abs_v - golden_meta["runs"]["c3_double"]["max_abs_v"]) <= 1e-12


@pytest.mark.parametrize("n_rho,n_theta,precision,scheme", [
    (64, 56, "double", "exprk22"), (45, 56, "double", "exprk22"), (105, 70, "double", "expeuler"),
    (98, 48, "single", "exprk22"), (10000, 64, "double", "exprk22")])
def test_symmetric_table_reads_bitwise(cuda, monkeypatch, n_rho, n_theta, precision, scheme):
    """The rho combine reads the phi tables at the canonical +-f position
    (fft.cuh sym_pos); the tables are bitwise j <-> -j symmetric, so the march
    must be bitwise identical to full-row reads (NWB_RHO_SYM=0)."""
    from paper_2103_06080_b200.plan import DevicePlan

    cfg = nw.DomainConfig(N_rho=n_rho, N_theta=n_theta, N_sigma=4, Sigma=1.6)
    _, rho, theta = nw.build_axes(cfg)
    v0 = nw.rho_modulated(cfg, nw.initial_nwave(rho, theta, cfg.A, cfg.B)).values
    eps = nw.EPS_DOUBLE if precision == "double" else nw.EPS_SINGLE
    outs = []
    for sym in ("0", "1"):
        monkeypatch.setenv("NWB_RHO_SYM", sym)
        plan = DevicePlan(n_rho, n_theta, 1, precision, cfg.d_sigma, cfg.rho_span,
                          cfg.theta_span, cfg.A, cfg.B, eps)
        plan.set_coeffs(None, None, None, n_rows=8)
        plan.load_physical(v0)
        plan.march(scheme, 0, 4)
        out, _ = plan.store_physical()
        outs.append(out.cpu().numpy())
        plan.close()
    assert np.array_equal(outs[0], outs[1])


@pytest.mark.parametrize("knobs", [{"NWB_RHO_WS": "256"}, {"NWB_RHO_ROLL": "2"},
                                   {"NWB_RHO_PREFETCH": "100", "NWB_RHO_NEXTPF": "148"}])
@pytest.mark.parametrize("n_rho,n_theta,batch,precision", [
    (625, 448, 1, "double"), (10000, 64, 1, "double"), (50, 56, 3, "double"),
    (1000, 448, 1, "single")])
def test_rho_pass_variants_bitwise(cuda, monkeypatch, knobs, n_rho, n_theta, batch, precision):
    """Scheduling variants of the rho pass (warp-specialised k_rho_ws, rolling
    and entry L2 prefetches) only move data earlier or elsewhere: the march is
    bitwise identical to the default pass."""
    from paper_2103_06080_b200.plan import DevicePlan

    cfg = nw.DomainConfig(N_rho=n_rho, N_theta=n_theta, N_sigma=4, Sigma=1.6)
    _, rho, theta = nw.build_axes(cfg)
    v0 = nw.rho_modulated(cfg, nw.initial_nwave(rho, theta, cfg.A, cfg.B)).values
    if batch > 1:
        v0 = np.stack([v0 * (1.0 + 0.1 * i) for i in range(batch)])
    eps = nw.EPS_DOUBLE if precision == "double" else nw.EPS_SINGLE
    outs = []
    for env in ({}, knobs):
        for k in ("NWB_RHO_WS", "NWB_RHO_ROLL", "NWB_RHO_PREFETCH", "NWB_RHO_NEXTPF"):
            monkeypatch.delenv(k, raising=False)
        for k, v in env.items():
            monkeypatch.setenv(k, v)
        plan = DevicePlan(n_rho, n_theta, batch, precision, cfg.d_sigma, cfg.rho_span,
                          cfg.theta_span, cfg.A, cfg.B, eps)
        plan.set_coeffs(None, None, None, n_rows=8)
        plan.load_physical(v0)
        plan.march("exprk22", 0, 4)
        out, _ = plan.store_physical()
        outs.append(out.cpu().numpy())
        plan.close()
    assert np.array_equal(outs[0], outs[1])


@pytest.mark.parametrize("n_rho,n_theta,batch,precision", [
    (2048, 1024, 1, "double"), (2025, 1050, 1, "double"), (1000, 448, 5, "double"),
    (2025, 1050, 1, "single"), (2048, 1024, 1, "single"), (1000, 448, 5, "single")])
def test_weno_theta_walk_bitwise(cuda, monkeypatch, n_rho, n_theta, batch, precision):
    """The row-walk theta faces of k_weno / k_weno_x2 (32-row tiles;
    NWB_WENO_WALK=0 selects the row-by-row version) evaluate the same operands in
    the same order: the march, and the WENO operator alone, are bitwise identical."""
    from paper_2103_06080_b200.plan import DevicePlan

    cfg = nw.DomainConfig(N_rho=n_rho, N_theta=n_theta, N_sigma=3, Sigma=1.2)
    _, rho, theta = nw.build_axes(cfg)
    v0 = nw.rho_modulated(cfg, nw.initial_nwave(rho, theta, cfg.A, cfg.B)).values
    if batch > 1:
        v0 = np.stack([v0 * (1.0 + 0.1 * i) for i in range(batch)])
    eps = nw.EPS_DOUBLE if precision == "double" else nw.EPS_SINGLE
    rng = np.random.default_rng(7)
    v = rng.standard_normal((n_rho, n_theta))
    up, uq, du = (0.03 * rng.standard_normal(n_rho) for _ in range(3))
    b_ops, outs = [], []
    for walk in ("0", "1"):
        monkeypatch.setenv("NWB_WENO_WALK", walk)
        plan = DevicePlan(n_rho, n_theta, batch, precision, cfg.d_sigma, cfg.rho_span,
                          cfg.theta_span, cfg.A, cfg.B, eps)
        plan.set_coeffs(None, None, None, n_rows=8)
        plan.load_physical(v0)
        plan.march("exprk22", 0, 3)
        out, _ = plan.store_physical()
        outs.append(out.cpu().numpy())
        plan.close()
        if batch == 1:
            dt = np.float64 if precision == "double" else np.float32
            b_ops.append(np.asarray(nw.weno5_b(v.astype(dt), up.astype(dt), uq.astype(dt),
                                               du.astype(dt), 0.05, 0.32, 0.21)))
    assert np.array_equal(outs[0], outs[1])
    if b_ops:
        assert np.array_equal(b_ops[0], b_ops[1])


@pytest.mark.parametrize("n_rho,n_theta,batch", [
    (2048, 1024, 1), (2025, 1050, 1), (1050, 2100, 1), (512, 1024, 4), (1000, 448, 5)])
def test_weno_tma_staging_bitwise(cuda, monkeypatch, n_rho, n_theta, batch):
    """fp64 walk tiles staged by one TMA tensor copy per warp (zero-filled box,
    periodic seam patched; NWB_WENO_TMA=0 selects the cp.async staging) hold the
    same operands: the march and the WENO operator alone are bitwise identical,
    including grids whose theta extent is not a multiple of the 32-column tile."""
    from paper_2103_06080_b200.plan import DevicePlan

    cfg = nw.DomainConfig(N_rho=n_rho, N_theta=n_theta, N_sigma=3, Sigma=1.2)
    _, rho, theta = nw.build_axes(cfg)
    v0 = nw.rho_modulated(cfg, nw.initial_nwave(rho, theta, cfg.A, cfg.B)).values
    if batch > 1:
        v0 = np.stack([v0 * (1.0 + 0.1 * i) for i in range(batch)])
    rng = np.random.default_rng(11)
    v = rng.standard_normal((n_rho, n_theta))
    up, uq, du = (0.03 * rng.standard_normal(n_rho) for _ in range(3))
    b_ops, outs = [], []
    for tma in ("0", "1"):
        monkeypatch.setenv("NWB_WENO_TMA", tma)
        plan = DevicePlan(n_rho, n_theta, batch, "double", cfg.d_sigma, cfg.rho_span,
                          cfg.theta_span, cfg.A, cfg.B, nw.EPS_DOUBLE)
        plan.set_coeffs(None, None, None, n_rows=8)
        plan.load_physical(v0)
        plan.march("exprk22", 0, 3)
        out, _ = plan.store_physical()
        outs.append(out.cpu().numpy())
        plan.close()
        b_ops.append(np.asarray(nw.weno5_b(v, up, uq, du, 0.05, 0.32, 0.21)))
    assert np.array_equal(outs[0], outs[1])
    assert np.array_equal(b_ops[0], b_ops[1])


@pytest.mark.parametrize("precision", ["double", "single"])
def test_large_host_load_staged_equals_device_load(cuda, precision):
    """Host arrays above 64 MB go through the page-locked staging chunks of
    plan.to_device (with the fp64 -> fp32 conversion on the host side): the
    loaded state must equal a load of the same values from a device tensor."""
    import torch

    from paper_2103_06080_b200.plan import DevicePlan

    n_rho, n_theta = 4096, 2100  # 68.8 MB in fp64: several 32 MB chunks
    rng = np.random.default_rng(11)
    v0 = rng.standard_normal((n_rho, n_theta))
    outs = []
    for src in (v0, torch.from_numpy(v0).to("cuda:0")):
        plan = DevicePlan(n_rho, n_theta, 1, precision, 0.01, 1.0, 1.0, 0.0, 0.0,
                          nw.EPS_DOUBLE if precision == "double" else nw.EPS_SINGLE)
        plan.load_physical(src)
        out, _ = plan.store_physical()
        outs.append(out.cpu().numpy())
        plan.close()
    assert np.array_equal(outs[0], outs[1])


@pytest.mark.parametrize("shape", [(10000, 3584), (1250, 448), (8192, 16384)])
def test_transforms_vs_cufft(cuda, shape):
    """Cross-check against cuFFT (torch.fft, library code used only here as a
    second opinion beside scipy): rfft2 / irfft2 of the C2, Set-1 and C5 grids."""
    import torch

    g = torch.Generator(device=cuda).manual_seed(shape[0])
    x = torch.randn(shape, dtype=torch.float64, device=cuda, generator=g)
    tr = nw.SpectralTransforms(*shape)
    ours = tr.forward(x)
    ref = torch.fft.rfft2(x)
    err = float((ours - ref).abs().max() / ref.abs().max())
    assert err <= 1e-14, err
    back = tr.inverse(ref)
    ref_back = torch.fft.irfft2(ref, s=shape)
    err = float((back - ref_back).abs().max() / ref_back.abs().max())
    assert err <= 1e-14, err


@pytest.mark.parametrize("n_rho,batch", [(2000, 1), (1250, 2)])
def test_rho_half_tmem_vs_oracle(cuda, oracle, monkeypatch, n_rho, batch):
    """The TMEM half-column rho kernel (k_rho_half, NWB_RHO_HALF=1, off by
    default): a turbulent ExpRK22 march against the oracle (north-star bar) and
    against the default rho kernel (same arithmetic, other FFT grouping)."""
    from paper_2103_06080_b200.plan import DevicePlan

    cfg = nw.DomainConfig(N_rho=n_rho, N_theta=64, N_sigma=5, Sigma=2.0)
    sig, rho, theta = nw.build_axes(cfg)
    spec = nw.sample_modes(nw.TurbulenceParams(seed=3))
    f = nw.evaluate_fields(spec, spec.lam, sig, nw.rho_nodes_closed(cfg))
    v0 = nw.rho_modulated(cfg, nw.initial_nwave(rho, theta, cfg.A, cfg.B), depth=0.3).values
    v0s = np.stack([v0 * (1.0 + 0.05 * i) for i in range(batch)])
    outs = []
    for half in ("0", "1"):
        monkeypatch.setenv("NWB_RHO_HALF", half)
        plan = DevicePlan(n_rho, cfg.N_theta, batch, "double", cfg.d_sigma, cfg.rho_span,
                          cfg.theta_span, cfg.A, cfg.B, nw.EPS_DOUBLE)
        plan.set_coeffs(f.u_par, f.u_perp, f.du_perp_drho)
        plan.load_physical(v0s if batch > 1 else v0)
        plan.march("exprk22", 0, cfg.N_sigma)
        out, _ = plan.store_physical()
        outs.append(out.cpu().numpy().reshape(batch, n_rho, cfg.N_theta))
        plan.close()
    for i in range(batch):
        assert max_relative(outs[0][i], outs[1][i]) <= FP64_KERNEL
        ref = oracle.march(cfg, v0s[i], f)
        assert max_relative(ref.final, outs[1][i]) <= FP64_FIELD
