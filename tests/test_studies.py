"""CPU tests of the study orchestration and the snapshot
output path (f2) against goldens produced by the reference itself
(tests/golden/make_golden_studies.py).  The marches inside the studies are
run by the CPU oracle (test infrastructure), injected through the studies'
single ``_run_solver`` hook; the GPU tests run the same studies on the
device (tests/test_gpu_studies.py)."""

import hashlib
import json
import os
from types import SimpleNamespace

import numpy as np
import pytest

import paper_2103_06080_b200 as nw
from paper_2103_06080_b200 import fieldio, studies

HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.fixture(scope="module")
def gs():
    with open(os.path.join(HERE, "golden", "golden_studies.json")) as fh:
        return json.load(fh)


def study_setup(gs):
    cfg = nw.DomainConfig(**gs["grid"])
    spec = nw.sample_modes(nw.TurbulenceParams(seed=gs["seed"]))
    n_ref = gs["n_ref"]
    sig = np.arange(n_ref + 1) * (cfg.Sigma / n_ref)
    master = nw.evaluate_fields(spec, spec.lam, sig, nw.rho_nodes_closed(cfg))
    fields = nw.evaluate_fields(spec, spec.lam, np.arange(cfg.N_sigma + 1) * cfg.d_sigma,
                                nw.rho_nodes_closed(cfg))
    return cfg, master, fields


@pytest.fixture
def oracle_solver(monkeypatch, oracle):
    """studies._run_solver backed by the CPU oracle march."""

    def run(solver, config, fields, threads=1, guard=10.0, snapshot_sigmas=None, **kw):
        _, rho, theta = nw.build_axes(config)
        if solver == "splitting":
            from oracle import splitting_oracle

            v0 = nw.initial_nwave(nw.rho_nodes_closed(config), theta, config.A, config.B).values
            r = splitting_oracle.march(config, v0, fields, snapshot_sigmas=snapshot_sigmas,
                                       guard=guard)
        else:
            v0 = nw.initial_nwave(rho, theta, config.A, config.B).values
            r = oracle.march(config, v0, fields, scheme=solver, guard=guard,
                             snapshot_sigmas=snapshot_sigmas)
        if r.failed_sigma is not None:
            raise nw.InstabilityError(r.failed_sigma, r.max_abs_v)
        return SimpleNamespace(final=nw.Field2D(r.final),
                               snapshots={s: nw.Field2D(f) for s, f in r.snapshots.items()})

    monkeypatch.setattr(studies, "_run_solver", run)
    return run


def check_rows(rows, ref, rel):
    assert len(rows) == len(ref)
    for r, (n, err, beta, unstable) in zip(rows, ref):
        assert r.n_sigma == n and r.unstable == unstable
        assert r.err == pytest.approx(err, rel=rel)
        if beta is None:
            assert r.beta is None
        else:
            assert r.beta == pytest.approx(beta, rel=rel)


# ------------------------------------------------------------------ f3 studies

@pytest.mark.parametrize("solver", ["exprk22", "expeuler"])
@pytest.mark.parametrize("roi", [False, True])
def test_convergence_study_logic_vs_reference(gs, oracle_solver, solver, roi):
    cfg, master, _ = study_setup(gs)
    rows = studies.convergence_study(cfg, gs["n_list"], gs["n_ref"], solver=solver,
                                     fields_master=master, use_roi=roi)
    check_rows(rows, gs["convergence"][f"{solver}_roi{int(roi)}"], 1e-9)


def test_compare_solvers_logic_vs_reference(gs, oracle_solver):
    cfg, _, fields = study_setup(gs)
    rep = studies.compare_solvers(cfg, fields, [0.6, 1.2, 2.4], trace_sigma=2.4, trace_rho=144.0,
                                  solver_pair=("expeuler", "exprk22"))
    ref = gs["compare"]
    for c, (s, rel, amp) in zip(rep.checkpoints, ref["checkpoints"]):
        assert c.sigma == s
        assert c.rel_l2_roi == pytest.approx(rel, rel=1e-9)
        assert c.amplitude_ratio == pytest.approx(amp, rel=1e-12)
    assert rep.overshoot_splitting == pytest.approx(ref["overshoot_a"], rel=1e-9)
    assert rep.overshoot_exprk22 == pytest.approx(ref["overshoot_b"], rel=1e-9)


def test_max_overshoot_vs_reference(gs):
    for name, trace in gs["overshoot_traces"].items():
        assert studies.max_overshoot(np.array(trace)) == gs["overshoot"][name]


def test_convergence_rate_and_errors(gs):
    assert studies.convergence_rate(4e-3, 1e-3, 10, 20) == pytest.approx(2.0)
    with pytest.raises(ValueError):
        studies.convergence_rate(0.0, 1e-3, 10, 20)
    with pytest.raises(ValueError):
        studies.convergence_rate(1e-3, 1e-4, 20, 10)
    cfg, master, fields = study_setup(gs)
    with pytest.raises(ValueError, match="divide"):
        studies.convergence_study(cfg, [5], gs["n_ref"], fields_master=master)
    with pytest.raises(ValueError, match="master"):
        studies.convergence_study(cfg, [4], gs["n_ref"])
    with pytest.raises(ValueError, match="sigma rows"):
        studies.convergence_study(cfg, [4], 16, fields_master=master)
    with pytest.raises(ValueError, match="unknown solver"):
        studies.convergence_study(cfg, [4], gs["n_ref"], solver="godunov", fields_master=master)
    with pytest.raises(ValueError, match="unknown solver"):
        studies.compare_solvers(cfg, fields, [1.2], solver_pair=("rk4", "exprk22"))


def test_unstable_run_breaks_rate_chain(gs, monkeypatch):
    """An InstabilityError row is flagged and the next row gets no rate."""
    cfg, master, _ = study_setup(gs)
    ref = nw.Field2D(np.ones((cfg.N_rho, cfg.N_theta)))

    def run(solver, config, fields, **kw):
        if config.N_sigma == 8:
            raise nw.InstabilityError(0.5, 11.0)
        return SimpleNamespace(final=nw.Field2D(np.full((cfg.N_rho, cfg.N_theta),
                                                        1.0 + 1.0 / config.N_sigma)))

    monkeypatch.setattr(studies, "_run_solver", run)
    rows = studies.convergence_study(cfg, [4, 8, 16], gs["n_ref"], fields_master=master,
                                     reference=ref)
    assert [r.unstable for r in rows] == [False, True, False]
    assert rows[0].beta is None and rows[2].beta is None and np.isnan(rows[1].err)


# ------------------------------------------------------------------ f2 output

def test_nwav_and_csv_bytes_match_reference(gs, tmp_path):
    g = gs["fieldio"]
    field = nw.Field2D(np.array(g["values"]))
    _, rho, theta = nw.build_axes(nw.DomainConfig(N_rho=5, N_theta=7, N_sigma=4, Sigma=1.0))
    fb, fc = tmp_path / "f.bin", tmp_path / "f.csv"
    fieldio.write_field_binary(fb, field, 0.25, 0.5, 1.75)
    fieldio.write_field_csv(fc, field, rho, theta)
    assert hashlib.sha256(fb.read_bytes()).hexdigest() == g["bin_sha256"]
    assert hashlib.sha256(fc.read_bytes()).hexdigest() == g["csv_sha256"]
    back, dr, dt, s = fieldio.read_field_binary(fb)
    assert np.array_equal(back.values, field.values) and (dr, dt, s) == (0.25, 0.5, 1.75)


def test_nwav_errors(tmp_path):
    p = tmp_path / "bad.bin"
    fieldio.write_grid_binary(p, np.zeros((2, 3)), 1.0, 1.0)
    raw = p.read_bytes()
    p.write_bytes(b"XXXX" + raw[4:])
    with pytest.raises(IOError, match="magic"):
        fieldio.read_grid_binary(p)
    p.write_bytes(raw[:-8])
    with pytest.raises(IOError, match="payload"):
        fieldio.read_grid_binary(p)
    p.write_bytes(raw[:20])
    with pytest.raises(IOError, match="header"):
        fieldio.read_grid_binary(p)
    with pytest.raises(ValueError):
        fieldio.write_grid_binary(p, np.zeros(3), 1.0, 1.0)
    with pytest.raises(ValueError):
        fieldio.write_field_csv(p, nw.Field2D(np.zeros((2, 3))), np.zeros(3), np.zeros(3))


def test_snapshot_writer_names(tmp_path):
    cfg = nw.DomainConfig(N_rho=4, N_theta=6, N_sigma=4, Sigma=1.0)
    rep = SimpleNamespace(snapshots={0.5: nw.Field2D(np.ones((4, 6))),
                                     1.0: nw.Field2D(np.zeros((4, 6)))})
    w = fieldio.SnapshotWriter(tmp_path / "out.d", cfg)
    paths = w.write_report(rep)
    names = [os.path.basename(p) for p in paths]
    assert names == ["V_sigma0000p500.bin", "V_sigma0000p500.csv",
                     "V_sigma0001p000.bin", "V_sigma0001p000.csv"]
    vals, _, _, s = fieldio.read_grid_binary(paths[0])
    assert s == 0.5 and np.array_equal(vals, np.ones((4, 6)))


def test_compare_solvers_default_pair_splitting_vs_reference(oracle_solver):
    """The reference's default pair (splitting, exprk22) on the oracle marches
    equals the reference's own report (tests/golden/golden_splitting.json)."""
    import json
    import os

    with open(os.path.join(os.path.dirname(__file__), "golden", "golden_splitting.json")) as fh:
        ref = json.load(fh)["compare"]
    cfg = nw.DomainConfig(N_rho=250, N_theta=112, N_sigma=40, Sigma=16.0)
    sig, _, _ = nw.build_axes(cfg)
    spec = nw.sample_modes(nw.TurbulenceParams(seed=5))
    fl = nw.evaluate_fields(spec, spec.lam, sig, nw.rho_nodes_closed(cfg))
    rep = studies.compare_solvers(cfg, fl, [8.0, 16.0], trace_sigma=16.0, trace_rho=144.0)
    for c, (s, rel, amp) in zip(rep.checkpoints, ref["checkpoints"]):
        assert c.sigma == s
        assert c.rel_l2_roi == pytest.approx(rel, rel=1e-9)
        assert c.amplitude_ratio == pytest.approx(amp, rel=1e-12)
    assert rep.overshoot_splitting == pytest.approx(ref["overshoot_splitting"], rel=1e-9)
    assert rep.overshoot_exprk22 == pytest.approx(ref["overshoot_exprk22"], rel=1e-9)
