"""GPU: the splitting baseline (reference ``nwave/splitting.py``)
through ``nwb_split_*`` against the reference goldens and the CPU oracle.

The device diffraction solve evaluates the reference's Thomas recurrences as
parallel affine scans and the trapezoid prefix as a running sum, so results
agree to rounding (not bitwise): stage outputs <= 1e-13, marched fields
<= 1e-10 max-relative (the north star's fp64 bar)."""

import json
import os

import numpy as np
import pytest

import paper_2103_06080_b200 as nw
from paper_2103_06080_b200.grid import max_relative

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
STAGE_TOL = 1e-13
FIELD_TOL = 1e-10


@pytest.fixture(scope="module")
def gs():
    return dict(np.load(os.path.join(HERE, "golden", "golden_splitting.npz")))


@pytest.fixture(scope="module")
def gmeta():
    with open(os.path.join(HERE, "golden", "golden_splitting.json")) as fh:
        return json.load(fh)


def test_stage_functions_vs_golden(cuda, gs, gmeta):
    c = nw.DomainConfig(**gmeta["stage_config"])
    v = gs["st_v"]
    up, uq, dus, dur = gs["st_coef"]
    got = nw.step_diffraction_cn(v, c.d_sigma, c.d_rho, c.d_theta)
    assert max_relative(gs["st_diffraction"], got) <= STAGE_TOL
    assert np.array_equal(nw.step_burgers_godunov(v, c.B, c.d_sigma, c.d_theta), gs["st_godunov"])
    assert np.array_equal(nw.godunov_flux(*gs["st_flux_in"], c.B), gs["st_flux"])
    got = nw.step_axial_absorption_spectral(v, up, c.A, c.d_sigma, c.theta_span)
    assert max_relative(gs["st_axial"], got) <= STAGE_TOL
    got = nw.step_transverse_lw(v, uq, dus, dur, c.d_sigma, c.d_rho)
    assert max_relative(gs["st_transverse"], got) <= STAGE_TOL
    f = nw.VelocityFields(*(np.repeat(a[None, :], 4, axis=0) for a in gs["st_coef"]))
    st = nw.lie_step(nw.SplittingState(nw.Field2D(v), 2), f, c)
    assert st.sigma_index == 3
    assert max_relative(gs["st_lie"], st.field.values) <= STAGE_TOL


@pytest.mark.parametrize("name", ["s41x48", "s251x112"])
def test_run_splitting_vs_golden(cuda, gs, gmeta, name):
    meta = gmeta["runs"][name]
    c = nw.DomainConfig(**meta["config"])
    f = nw.VelocityFields(*gs[f"{name}_coef"])
    rep = nw.run_splitting(c, gs[f"{name}_v0"], f, snapshot_sigmas=meta["snapshots"])
    assert rep.solver == "splitting" and rep.n_steps == meta["n_steps"]
    assert max_relative(gs[f"{name}_final"], rep.final.values) <= FIELD_TOL
    assert max_relative(gs[f"{name}_snap3"], rep.snapshots[meta["snapshots"][0]].values) <= FIELD_TOL
    assert np.array_equal(rep.snapshots[meta["snapshots"][1]].values, rep.final.values)
    assert abs(rep.max_abs_v - meta["max_abs_v"]) <= 1e-12
    assert rep.step_seconds.shape == (meta["n_steps"],)


def test_run_splitting_set1_vs_oracle(cuda):
    """The paper's Set-1 grid (closed rho grid 1251 x 448), seed-0 turbulence,
    K = 6 steps against the CPU oracle."""
    from oracle import splitting_oracle

    K = 6
    c = nw.preset_config(1)
    sig, _, theta = nw.build_axes(c)
    spec = nw.sample_modes(nw.TurbulenceParams(seed=0))
    f = nw.evaluate_fields(spec, spec.lam, sig[:K + 1], nw.rho_nodes_closed(c))
    v0 = nw.initial_nwave(nw.rho_nodes_closed(c), theta, c.A, c.B).values
    rep = nw.run_splitting(c, v0, f, max_steps=K)
    ref = splitting_oracle.march(c, v0, f, max_steps=K)
    assert max_relative(ref.final, rep.final.values) <= FIELD_TOL
    assert abs(rep.max_abs_v - ref.max_abs_v) <= 1e-12


def test_compare_solvers_reference_default_pair(cuda, gmeta):
    """compare_solvers with the reference's default (splitting, exprk22) pair,
    both marches on the device, against the reference's own report."""
    cfg = nw.DomainConfig(N_rho=250, N_theta=112, N_sigma=40, Sigma=16.0)
    sig, _, _ = nw.build_axes(cfg)
    spec = nw.sample_modes(nw.TurbulenceParams(seed=5))
    fl = nw.evaluate_fields(spec, spec.lam, sig, nw.rho_nodes_closed(cfg))
    rep = nw.compare_solvers(cfg, fl, [8.0, 16.0], trace_sigma=16.0, trace_rho=144.0)
    ref = gmeta["compare"]
    for c, (s, rel, amp) in zip(rep.checkpoints, ref["checkpoints"]):
        assert c.sigma == s
        assert c.rel_l2_roi == pytest.approx(rel, rel=1e-7)
        assert c.amplitude_ratio == pytest.approx(amp, rel=1e-10)
    assert rep.overshoot_splitting == pytest.approx(ref["overshoot_splitting"], rel=1e-7)
    assert rep.overshoot_exprk22 == pytest.approx(ref["overshoot_exprk22"], rel=1e-7)


def test_splitting_guard_budget_and_validation(cuda):
    c = nw.DomainConfig(N_rho=40, N_theta=48, N_sigma=10, Sigma=4.0)
    _, _, theta = nw.build_axes(c)
    rho_c = nw.rho_nodes_closed(c)
    v0 = nw.initial_nwave(rho_c, theta, c.A, c.B).values
    f = nw.zero_fields(11, 41)
    with pytest.raises(ValueError):
        nw.run_splitting(c, v0[:-1], f)
    with pytest.raises(nw.InstabilityError) as ei:
        nw.run_splitting(c, 50.0 * v0, f, guard=1.0, cfl="warn")
    assert ei.value.sigma == pytest.approx(c.d_sigma)  # after step 1 (splitting.py:287-289)
    with pytest.raises(nw.BudgetExceededError, match="at step 1/10"):
        nw.run_splitting(c, v0, f, max_seconds=0.0)


def test_cost_scaling_both_solvers(cuda):
    """The reference's default cost study (splitting + exprk22) on Sets 1-2."""
    rows = nw.cost_scaling_study([1, 2], steps=3, reps=1)
    assert [(r.solver, r.set_id) for r in rows] == [("splitting", 1), ("splitting", 2),
                                                     ("exprk22", 1), ("exprk22", 2)]
    assert all(r.per_step_seconds > 0 for r in rows)
