"""GPU: the drop-in march API's host-facing behaviour (reference
``nwave/exprk.py:219-331``) -- snapshots streamed to host memory through a
two-buffer device ring, the per-step timing buckets (device time stamps
written by the march kernels of the replayed step graph), the wall-clock
budget and the guard's failure sigma."""

import numpy as np
import pytest

import paper_2103_06080_b200 as nw
from paper_2103_06080_b200.plan import DevicePlan

pytestmark = pytest.mark.gpu


def _set(n):
    c = nw.preset_config(n)
    _, rho, theta = nw.build_axes(c)
    return c, nw.rho_modulated(c, nw.initial_nwave(rho, theta, c.A, c.B))


def test_streamed_snapshots_equal_device_copies(cuda):
    """Streamed snapshots (c2r of the state between graph segments) are bitwise
    the stage-1 c2r output the march copies on the device (v_n at step start)."""
    c, v0 = _set(1)
    K = 12
    f = nw.zero_fields(K + 2, c.N_rho + 1)
    steps = [0, 1, 5, 11]
    rep = nw.run_exprk22(c, v0, f, max_steps=K, snapshot_sigmas=[s * c.d_sigma for s in steps])
    plan = DevicePlan(c.N_rho, c.N_theta, 1, "double", c.d_sigma, c.rho_span, c.theta_span,
                      c.A, c.B)
    plan.set_coeffs(f.u_par, f.u_perp, f.du_perp_drho, n_rows=K + 1)
    plan.load_physical(v0.values)
    _, _, bufs = plan.march("exprk22", 0, K, snap_steps=steps)
    for s in steps:
        got = rep.snapshots[s * c.d_sigma].values
        assert np.array_equal(got, bufs[s][0].cpu().numpy()), s
    fin, _ = plan.store_physical()
    assert np.array_equal(rep.final.values, fin[0].cpu().numpy())
    plan.close()


def test_many_snapshots_do_not_grow_device_memory(cuda):
    """101 snapshots of the C2 grid (Set 4, 287 MB each, 29 GB on the host):
    device memory stays within two snapshot buffers of a snapshot-free run;
    every snapshot is returned."""
    import torch

    c, v0 = _set(4)
    K = 100
    f = nw.zero_fields(K + 2, c.N_rho + 1)
    nw.run_exprk22(c, v0, f, max_steps=2)  # warm the pool
    torch.cuda.synchronize()
    torch.cuda.reset_peak_memory_stats()
    base = nw.run_exprk22(c, v0, f, max_steps=K)
    peak_plain = torch.cuda.max_memory_allocated()
    torch.cuda.reset_peak_memory_stats()
    rep = nw.run_exprk22(c, v0, f, max_steps=K,
                         snapshot_sigmas=[n * c.d_sigma for n in range(K + 1)])
    peak_snap = torch.cuda.max_memory_allocated()
    field = c.N_rho * c.N_theta * 8
    assert peak_snap - peak_plain <= 2 * field + (16 << 20), (peak_plain, peak_snap)
    assert len(rep.snapshots) == K + 1
    assert np.array_equal(rep.snapshots[K * c.d_sigma].values, rep.final.values)
    assert np.array_equal(rep.final.values, base.final.values)
    # snapshot n is v_n: its max|V| is the guard value of step n
    for n in (0, 37, 99):
        m = float(np.max(np.abs(rep.snapshots[n * c.d_sigma].values)))
        assert m <= rep.max_abs_v


def test_default_timing_buckets_and_graph_path_agree(cuda):
    """The default call (per-step buckets from the kernels' time stamps)
    fills the reference's per-step arrays and is bitwise the untimed call."""
    c, v0 = _set(1)
    K = 20
    f = nw.zero_fields(K + 2, c.N_rho + 1)
    a = nw.run_exprk22(c, v0, f, max_steps=K)
    b = nw.run_exprk22(c, v0, f, max_steps=K, timing=False)
    assert np.array_equal(a.final.values, b.final.values)
    assert a.step_seconds.shape == (K,) and a.step_nonlinear.shape == (K,)
    assert np.all(a.step_seconds > 0) and np.all(a.step_nonlinear > 0)
    assert np.all(a.step_linear >= 0)
    np.testing.assert_allclose(a.step_nonlinear + a.step_linear, a.step_seconds, rtol=1e-6)
    # a graph step of Set 1 takes well under a millisecond
    assert np.median(a.step_seconds) < 1e-3


def test_zero_budget_stops_after_first_step(cuda):
    """max_seconds=0 raises after step 1, like the reference's per-step check."""
    c, v0 = _set(1)
    f = nw.zero_fields(c.N_sigma + 1, c.N_rho + 1)
    with pytest.raises(nw.BudgetExceededError, match=r"at step 1/300"):
        nw.run_exprk22(c, v0, f, max_seconds=0.0)


def test_instability_sigma_through_check(cuda):
    """The guard failure reaches the caller with the reference's sigma = n d_sigma."""
    cfg = nw.DomainConfig(N_rho=32, N_theta=28, N_sigma=40, Sigma=40.0, A=1e-4, B=4.0)
    _, rho, theta = nw.build_axes(cfg)
    v0 = 3.0 * np.cos(2 * np.pi * (theta - cfg.theta_min) / cfg.theta_span)[None, :] * np.ones((32, 1))
    with pytest.warns(UserWarning):
        with pytest.raises(nw.InstabilityError) as ei:
            nw.run_exprk22(cfg, v0, nw.zero_fields(41, 33), guard=4.0)
    e = ei.value
    assert np.isfinite(e.sigma) and e.sigma == pytest.approx(e.step * cfg.d_sigma)
    assert e.max_abs > 4.0
