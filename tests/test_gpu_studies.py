"""GPU tests of SURVEY 8(f) rows f2/f3 on the sm_100a path: the reference's
studies (convergence, solver comparison, cost scaling) driving the device
march, checked against goldens from the reference itself; device ground
metrics (nwb_ground_metrics) against the host definition; the ensemble's
per-member metrics."""

import json
import os

import numpy as np
import pytest

import paper_2103_06080_b200 as nw
from paper_2103_06080_b200 import studies

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.fixture(scope="module")
def gs():
    with open(os.path.join(HERE, "golden", "golden_studies.json")) as fh:
        return json.load(fh)


def setup(gs):
    cfg = nw.DomainConfig(**gs["grid"])
    spec = nw.sample_modes(nw.TurbulenceParams(seed=gs["seed"]))
    sig = np.arange(gs["n_ref"] + 1) * (cfg.Sigma / gs["n_ref"])
    master = nw.evaluate_fields(spec, spec.lam, sig, nw.rho_nodes_closed(cfg))
    fields = nw.evaluate_fields(spec, spec.lam, np.arange(cfg.N_sigma + 1) * cfg.d_sigma,
                                nw.rho_nodes_closed(cfg))
    return cfg, master, fields


@pytest.mark.parametrize("solver", ["exprk22", "expeuler"])
@pytest.mark.parametrize("roi", [False, True])
def test_convergence_study_on_device_vs_reference(cuda, gs, solver, roi):
    cfg, master, _ = setup(gs)
    rows = nw.convergence_study(cfg, gs["n_list"], gs["n_ref"], solver=solver,
                                fields_master=master, use_roi=roi)
    for r, (n, err, beta, unstable) in zip(rows, gs["convergence"][f"{solver}_roi{int(roi)}"]):
        assert r.n_sigma == n and r.unstable == unstable
        # errors are differences of fields that agree to ~1e-15: 1e-8 relative is loose
        assert r.err == pytest.approx(err, rel=1e-8)
        assert (r.beta is None) == (beta is None)
        if beta is not None:
            assert r.beta == pytest.approx(beta, rel=1e-8)


def test_compare_solvers_on_device_vs_reference(cuda, gs):
    cfg, _, fields = setup(gs)
    rep = nw.compare_solvers(cfg, fields, [0.6, 1.2, 2.4], trace_sigma=2.4, trace_rho=144.0,
                             solver_pair=("expeuler", "exprk22"))
    for c, (s, rel, amp) in zip(rep.checkpoints, gs["compare"]["checkpoints"]):
        assert c.sigma == s
        assert c.rel_l2_roi == pytest.approx(rel, rel=1e-8)
        assert c.amplitude_ratio == pytest.approx(amp, rel=1e-12)
    assert rep.overshoot_splitting == pytest.approx(gs["compare"]["overshoot_a"], rel=1e-8)
    assert rep.overshoot_exprk22 == pytest.approx(gs["compare"]["overshoot_b"], rel=1e-8)


def test_cost_scaling_study_runs_on_device(cuda):
    rows = nw.cost_scaling_study([1, 2], solver="exprk22", steps=3, reps=2)
    assert [r.set_id for r in rows] == [1, 2]
    assert rows[0].growth_vs_previous is None and rows[1].growth_vs_previous > 0
    t = rows[1].timing
    assert t.per_step_seconds > 0 and t.total_seconds == pytest.approx(
        t.per_step_seconds * nw.GRID_SETS[2]["N_sigma"])


@pytest.mark.parametrize("dtype", ["float64", "float32"])
def test_ground_metrics_device_matches_host(cuda, golden, dtype):
    import torch

    c1 = nw.DomainConfig(Sigma=30.0, N_sigma=300, N_rho=625, N_theta=448)
    base = golden["c1_double_final"]
    rng = np.random.default_rng(5)
    fields = [base, base * 0.7 + 0.01 * rng.standard_normal(base.shape),
              np.roll(base, 37, axis=1), np.zeros_like(base)]
    fields = [f.astype(dtype).astype(np.float64) for f in fields]
    dev = torch.as_tensor(np.stack(fields).astype(dtype), device=cuda)
    got = nw.ground_metrics_device(c1, dev)
    for f, g in zip(fields, got):
        ref = nw.ground_metrics(c1, nw.Field2D(f))
        assert g.peak == ref.peak and g.rho == ref.rho
        # bitwise the host arithmetic (NaN when a crossing is absent)
        assert np.array_equal(np.array([g.rise_theta, g.rise_seconds]),
                              np.array([ref.rise_theta, ref.rise_seconds]), equal_nan=True)


def test_ensemble_ground_metrics(cuda):
    from paper_2103_06080_b200.ensemble import run_ensemble

    cfg = nw.preset_config(1, N_sigma=300)
    v0s, _, _ = nw.ensemble_nwaves(cfg, 4, seed=2026)
    res = run_ensemble(cfg, v0s, nw.zero_fields(301, cfg.N_rho + 1), max_steps=20)
    for i in range(4):
        ref = nw.ground_metrics(cfg, nw.Field2D(res.final[i]))
        assert res.peak[i] == ref.peak
        assert res.rise_theta[i] == ref.rise_theta or (np.isnan(res.rise_theta[i])
                                                        and np.isnan(ref.rise_theta))
