"""CPU: the splitting-baseline oracle (oracle/splitting_oracle.py) reproduces the
reference's ``nwave/splitting.py`` goldens bitwise."""

import json
import os

import numpy as np
import pytest

from paper_2103_06080_b200.grid import DomainConfig
from paper_2103_06080_b200.turbulence import VelocityFields

HERE = os.path.dirname(os.path.abspath(__file__))
GS = os.path.join(HERE, "golden", "golden_splitting.npz")


@pytest.fixture(scope="module")
def gs():
    return dict(np.load(GS))


@pytest.fixture(scope="module")
def gmeta():
    with open(os.path.join(HERE, "golden", "golden_splitting.json")) as fh:
        return json.load(fh)


@pytest.fixture(scope="module")
def so():
    from oracle import splitting_oracle

    return splitting_oracle


def test_stages_bitwise(gs, gmeta, so):
    c = DomainConfig(**gmeta["stage_config"])
    v = gs["st_v"]
    up, uq, dus, dur = gs["st_coef"]
    assert np.array_equal(so.diffraction_cn(v, c.d_sigma, c.d_rho, c.d_theta), gs["st_diffraction"])
    assert np.array_equal(so.burgers_godunov(v, c.B, c.d_sigma, c.d_theta), gs["st_godunov"])
    assert np.array_equal(so.godunov_flux(*gs["st_flux_in"], c.B), gs["st_flux"])
    assert np.array_equal(so.axial_absorption(v, up, c.A, c.d_sigma, c.theta_span), gs["st_axial"])
    assert np.array_equal(so.transverse_lw(v, uq, dus, dur, c.d_sigma, c.d_rho),
                          gs["st_transverse"])


@pytest.mark.parametrize("name", ["s41x48", "s251x112"])
def test_march_bitwise(gs, gmeta, so, name):
    meta = gmeta["runs"][name]
    c = DomainConfig(**meta["config"])
    f = VelocityFields(*gs[f"{name}_coef"])
    run = so.march(c, gs[f"{name}_v0"], f, snapshot_sigmas=meta["snapshots"])
    assert run.failed_sigma is None
    assert np.array_equal(run.final, gs[f"{name}_final"])
    assert np.array_equal(run.snapshots[meta["snapshots"][0]], gs[f"{name}_snap3"])
    assert run.max_abs_v == meta["max_abs_v"]
