"""GPU: the rho-slab path (nwb_slab_* kernels + slab.py orchestration) on one
rank, against the CPU oracle.  The multi-rank communication pattern is
covered on CPU (tests/test_slab_cpu.py); a single rank exercises every slab
kernel, the halo-extended WENO and the layout changes (local copies)."""

import numpy as np
import pytest

import paper_2103_06080_b200 as nw
from paper_2103_06080_b200.grid import max_relative

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("shape", [(64, 56), (50, 40)])
def test_slab_march_single_rank_vs_oracle(cuda, oracle, shape):
    from paper_2103_06080_b200.slab import SlabMarch

    cfg = nw.DomainConfig(N_rho=shape[0], N_theta=shape[1], N_sigma=6, Sigma=2.4)
    sig, rho, theta = nw.build_axes(cfg)
    spec = nw.sample_modes(nw.TurbulenceParams(seed=2))
    f = nw.evaluate_fields(spec, spec.lam, sig, nw.rho_nodes_closed(cfg))
    v0 = nw.rho_modulated(cfg, nw.initial_nwave(rho, theta, cfg.A, cfg.B), depth=0.3).values
    sm = SlabMarch(cfg, f)
    sm.load(v0)
    sm.march()
    rows, vmax = sm.final_rows()
    ref = oracle.march(cfg, v0, f)
    assert max_relative(ref.final, rows.cpu().numpy()) <= 1e-10
    assert max(max(sm.max_abs), vmax) == pytest.approx(ref.max_abs_v, abs=1e-12)


def test_slab_c5_geometry_truncated(cuda, oracle):
    """BASELINE C5 grid (8192 x 16384) through the slab kernels, K = 2 steps."""
    from paper_2103_06080_b200.slab import SlabMarch

    cfg = nw.DomainConfig(Sigma=120.0, N_sigma=6000, N_rho=8192, N_theta=16384)
    _, rho, theta = nw.build_axes(cfg)
    v0 = nw.rho_modulated(cfg, nw.initial_nwave(rho, theta, cfg.A, cfg.B)).values
    f = nw.zero_fields(4, cfg.N_rho + 1)
    sm = SlabMarch(cfg, f, max_steps=2)
    sm.load(v0)
    sm.march()
    rows, _ = sm.final_rows()
    ref = oracle.march(cfg, v0, f, max_steps=2)
    assert max_relative(ref.final, rows.cpu().numpy()) <= 1e-10
