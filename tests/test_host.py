"""CPU (no GPU): host-side logic of the drop-in API and the C-ABI library
(loads, exports every symbol include/nwb200.h declares; no compute calls)."""

import os
import re

import numpy as np
import pytest

import paper_2103_06080_b200 as nw
from paper_2103_06080_b200 import _lib
from paper_2103_06080_b200.exprk import _snapshot_steps

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_builds_and_exports_every_header_symbol():
    from paper_2103_06080_b200 import _build

    _build.build()
    lib = _lib.load_library()
    with open(os.path.join(ROOT, "include", "nwb200.h")) as fh:
        header = fh.read()
    declared = set(re.findall(r"\b(nwb_[a-z0-9_]+)\s*\(", header))
    assert declared == set(_lib.ABI_SYMBOLS)
    for name in declared:
        assert hasattr(lib, name), name
    assert lib.nwb_abi_version() == 1


def test_library_is_sm100a():
    import subprocess

    from paper_2103_06080_b200 import _build

    path = _build.build()
    out = subprocess.run(["cuobjdump", "--list-elf", path], capture_output=True, text=True)
    assert "sm_100a" in out.stdout


def test_no_cpu_fallback_without_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is visible")
    with pytest.raises(nw.BackendError):
        nw.weno5_b(np.zeros((4, 4)), np.zeros(4), np.zeros(4), np.zeros(4), 0.05, 0.1, 0.1)
    with pytest.raises(nw.BackendError):
        nw.SpectralTransforms(8, 8).forward(np.zeros((8, 8)))
    cfg = nw.DomainConfig(N_rho=8, N_theta=8, N_sigma=2)
    with pytest.raises(nw.BackendError):
        nw.run_exprk22(cfg, np.zeros((8, 8)), nw.zero_fields(3, 9))


def test_product_package_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_2103_06080_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                with open(os.path.join(dirpath, f)) as fh:
                    src = fh.read()
                assert "oracle" not in re.sub(r"#.*|//.*", "", src).replace("oracle/", ""), f


def test_error_mapping():
    assert issubclass(nw.ConfigError, ValueError)
    assert issubclass(nw.InstabilityError, RuntimeError)
    e = nw.InstabilityError(1.5, 12.0)
    assert e.sigma == 1.5 and e.max_abs == 12.0 and "1.5" in str(e)
    assert issubclass(nw.UnsupportedSizeError, ValueError)
    assert issubclass(nw.UnsupportedSizeError, nw.BackendError)


def test_instability_message_carries_sigma():
    from paper_2103_06080_b200._lib import instability_from_message

    e = instability_from_message("nwb_march: max|V| left the guard: step=7 member=3 "
                                 "max_abs=12.5", d_sigma=0.25)
    assert isinstance(e, nw.InstabilityError)
    assert e.sigma == 1.75 and e.max_abs == 12.5 and e.step == 7 and e.member == 3
    e = instability_from_message("max|V| left the guard: step=2 member=0 max_abs=nan")
    assert np.isnan(e.sigma) and np.isnan(e.max_abs) and e.step == 2


def test_variant_build_needs_explicit_output():
    from paper_2103_06080_b200 import _build

    with pytest.raises(ValueError):
        _build.build(defines=("NWB_WENO_WALK=0",))


def test_domain_config_validation_and_spacings():
    c = nw.DomainConfig()
    assert c.N_rho == 1250 and c.N_theta == 448 and c.N_sigma == 300
    assert c.d_sigma == 120.0 / 300
    assert c.d_theta == pytest.approx(28 * np.pi / 448)
    for bad in (dict(Sigma=0.0), dict(N_rho=0), dict(N_theta=2.5), dict(A=-1.0),
                dict(rho_max=-1.0), dict(roi_rho=(0.0, 500.0)), dict(B=float("nan"))):
        with pytest.raises(nw.ConfigError):
            nw.DomainConfig(**bad)


def test_field2d_and_norms():
    f = nw.Field2D(np.arange(12, dtype=np.int64).reshape(3, 4))
    assert f.values.dtype == np.float64 and f.n_rho == 3 and f.n_theta == 4
    with pytest.raises(nw.ConfigError):
        nw.Field2D(np.zeros(5))
    g = nw.Field2D(np.ones((3, 4)))
    assert nw.l2_norm(g, 0.5, 2.0) == pytest.approx(np.sqrt(12.0))
    assert nw.relative_error(g, g, 1.0, 1.0) == 0.0
    with pytest.raises(ValueError):
        nw.relative_error(nw.Field2D(np.zeros((3, 4))), g, 1.0, 1.0)
    with pytest.raises(ValueError):
        nw.l2_norm(nw.Field2D(np.full((2, 2), np.nan)), 1.0, 1.0)
    assert nw.max_relative(np.array([1.0, -2.0]), np.array([1.0, -2.5])) == 0.25


def test_axes_and_region():
    c = nw.DomainConfig(N_rho=10, N_theta=8, N_sigma=4, Sigma=2.0)
    s, r, t = nw.build_axes(c)
    assert len(s) == 5 and len(r) == 10 and len(t) == 8
    assert s[-1] == pytest.approx(2.0)
    assert len(nw.rho_nodes_closed(c)) == 11
    sub, rr, tt = nw.extract_region(nw.Field2D(np.ones((10, 8))), r, t, (40.0, 120.0),
                                    (0.0, 15 * np.pi))
    assert sub.n_rho == len(rr) and rr[0] >= 40.0 - 1e-9 and rr[-1] <= 120.0 + 1e-9


def test_snapshot_plan_rounds_like_reference():
    c = nw.DomainConfig(N_sigma=300)
    plan = _snapshot_steps(c, [0.0, 60.0, 120.0, 130.0, 0.39])
    assert plan == {0: 0.0, 150: 60.0, 300: 120.0, 1: 0.39}
    assert _snapshot_steps(c, None) == {}


def test_initial_nwave_and_ensemble_members():
    c = nw.preset_config(1)
    _, rho, theta = nw.build_axes(c)
    v0 = nw.initial_nwave(rho, theta, c.A, c.B)
    assert v0.values.shape == (1250, 448)
    assert np.max(np.abs(v0.values)) == pytest.approx(0.9375, abs=1e-3)
    with pytest.raises(ValueError):
        nw.initial_nwave(rho, theta, 0.0)
    members, amp, dur = nw.ensemble_nwaves(c, 8, seed=2026)
    assert members.shape == (8, 1250, 448)
    assert np.all((amp >= 0.5) & (amp <= 1.5)) and np.all((dur >= 0.75) & (dur <= 1.25))
    again, _, _ = nw.ensemble_nwaves(c, 8, seed=2026)
    assert np.array_equal(members, again)
    # amplitude 1, duration 1 is the reference pulse up to rounding
    row = nw.analysis._nwave_row(theta, c.B / (4 * c.A), 1.0, 1.0)
    assert np.max(np.abs(row - v0.values[0])) <= 1e-12
    # the pulse stays inside the periodic window
    nz = np.nonzero(np.abs(members[:, 0]).max(axis=0) > 1e-8)[0]
    assert theta[nz[0]] > 1.5 * np.pi and theta[nz[-1]] < 4.5 * np.pi


def test_ground_metrics_interpolate_rise():
    c = nw.DomainConfig(N_rho=10, N_theta=448)
    _, _, theta = nw.build_axes(c)
    # linear ramp of width pi starting at 2 pi (both corners on nodes, d_theta = pi/16)
    y = np.clip((theta - 2 * np.pi) / np.pi, 0.0, 1.0)
    f = nw.Field2D(np.tile(y, (10, 1)))
    g = nw.ground_metrics(c, f, trace_rho=40.0)
    assert g.peak == 1.0
    assert g.rise_theta == pytest.approx(0.8 * np.pi, rel=1e-9)
    assert g.rise_seconds == pytest.approx(g.rise_theta * 0.02 / (2 * np.pi))


def test_cfl_report():
    c = nw.preset_config(4)
    rep = nw.check_cfl_exprk(c, nw.zero_fields(2, 10), 5.0)
    assert rep.passed and rep.burgers_margin == pytest.approx(1.9635, rel=1e-4)
    assert rep.transverse_margin == np.inf
    bad = nw.check_cfl_splitting(nw.DomainConfig(N_sigma=2, Sigma=100.0))
    assert not bad.passed and "FAIL" in str(bad)


def test_downsample_fields():
    f = nw.VelocityFields(*(np.arange(25.0).reshape(5, 5) for _ in range(4)))
    d = nw.downsample_fields(f, 2, 1)
    assert d.shape == (3, 5) and np.array_equal(d.u_par[1], f.u_par[2])
    with pytest.raises(ValueError):
        nw.downsample_fields(f, 3, 1)


def test_bench_roofline_bookkeeping():
    import bench

    cfg, _ = bench.workload("c2")
    b = bench.algorithmic_bytes(cfg, "double")
    F = cfg.N_rho * cfg.N_theta * 8
    spec = cfg.N_rho * (cfg.N_theta // 2 + 1) * 16
    # tables read at canonical +-f positions: 60 % of each row at N_rho = 10000 (r1 = 5)
    assert bench.table_read_fraction(cfg.N_rho) == pytest.approx(0.6)
    # SURVEY 8(d) algorithmic bytes: 2F per theta / WENO launch, 4F per rho launch
    assert b[0] == spec + F and b[1] == 2 * F and b[2] == F + spec
    assert b[3] == 4 * spec and b[7] == 4 * spec
    d = bench.algorithmic_bytes(cfg, "double", design=True)
    assert d[3] == 4 * spec + int(1.8 * spec) and d[7] == 4 * spec + int(0.6 * spec)
    blk = bench.roofline_block(cfg, "c2", "double", [1.0, 2.0, 1.0, 3.0, 1.0, 2.0, 1.0, 2.5], 1)
    # both rho stages are one kernel (k_rho): 5.5 ms beats WENO's 4 ms
    assert blk["kernel"] == "rho_pass" and blk["unit"] == "GB/s"
    assert blk["achieved"] == pytest.approx((b[3] + b[7]) / 5.5e-3 / 1e9, rel=1e-3)
    assert blk["achieved_design"] == pytest.approx((d[3] + d[7]) / 5.5e-3 / 1e9, rel=1e-3)
    assert 0 < blk["frac"] < blk["frac_design"] < 10
    blk = bench.roofline_block(cfg, "c2", "double", [1.0, 4.0, 1.0, 1.0, 1.0, 4.0, 1.0, 1.0], 1)
    assert blk["kernel"] == "weno"
    # tables are shared by the members of a batch
    b4 = bench.algorithmic_bytes(cfg, "double", 4, design=True)
    assert b4[3] == 4 * 4 * spec + int(1.8 * spec) and b4[1] == 4 * 2 * F


def _freq_of_pos(n, stages):
    f = []
    for p in range(n):
        rem, ff, mult, L = p, 0, 1, n
        for r in stages:
            s = L // r
            q = rem // s
            rem -= q * s
            ff += q * mult
            mult *= r
            L = s
        f.append(ff)
    return f


def _sym_pos(p, r1, m):
    """Python restatement of csrc/fft.cuh sym_pos."""
    q1 = p // m
    if q1 == 0:
        return p
    rest = p - q1 * m
    q2 = r1 - q1
    if q1 < q2 or (q1 == q2 and 2 * rest <= m - 1):
        return p
    return q2 * m + (m - 1 - rest)


@pytest.mark.parametrize("stages", [[5, 2, 5, 2, 5, 2, 5, 2], [2, 5, 5, 2, 2, 2, 5, 5], [4, 4, 2],
                                    [3, 3, 5], [7, 2, 7], [8, 5, 5, 2], [5], [2, 2], [3, 5, 7]])
def test_symmetric_table_position_map(stages):
    """sym_pos maps every digit-reversed position to one holding the same |f|
    (f or n - f), is idempotent, folds every block but the first onto its
    mirror, and touches about half of each table row."""
    n = int(np.prod(stages))
    freq = _freq_of_pos(n, stages)
    pos_of = {f: p for p, f in enumerate(freq)}
    m = n // stages[0]
    canon = set()
    for p in range(n):
        c = _sym_pos(p, stages[0], m)
        assert freq[c] in (freq[p], (n - freq[p]) % n)
        assert _sym_pos(c, stages[0], m) == c
        canon.add(c)
        # outside block 0 (f = 0 mod r1, kept whole) the partner of p maps to
        # the same canonical position
        if p >= m:
            assert _sym_pos(pos_of[(n - freq[p]) % n], stages[0], m) == c
    assert len(canon) <= n // 2 + m + 1


def test_par_copyto_matches_copyto():
    """The threaded host copy used by the staged transfers: same bytes as
    np.copyto, including the fp64 -> fp32 narrowing of fp32 plans."""
    from paper_2103_06080_b200.hostio import par_copyto

    rng = np.random.default_rng(7)
    src = rng.standard_normal(1_000_003)
    for dt in (np.float64, np.float32):
        a, b = np.empty(src.size, dt), np.empty(src.size, dt)
        par_copyto(a, src)
        np.copyto(b, src, casting="unsafe")
        assert np.array_equal(a, b)


def test_cfl_u_perp_max_without_abs_temporary():
    """max(max u, -min u) reproduces max|u| bit for bit (NaN, inf, -0.0)."""
    from paper_2103_06080_b200.cfl import check_cfl_exprk

    c = nw.preset_config(1)
    for arr in ([[1.0, -3.0]], [[-3.0, -1.0]], [[np.nan, 1.0]], [[1.0, np.nan]],
                [[-np.inf, 1.0]], [[-0.0, -0.0]]):
        a = np.array(arr)
        f = nw.VelocityFields(a, a, a, a)
        assert repr(check_cfl_exprk(c, f).u_perp_max) == repr(float(np.max(np.abs(a))))
