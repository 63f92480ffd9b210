"""CFL precondition of the march (host-side, unchanged).

``run_exprk22`` applies the splitting solver's inequality pair
(reference ``exprk.py:199-205`` -> ``splitting.py:38-75``):
B v_max d_sigma <= d_theta and |U_perp|max d_sigma <= d_rho.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .grid import DomainConfig


@dataclass
class CflReport:
    """Allowed step over actual step for both bounds; >= 1 passes."""

    burgers_margin: float
    transverse_margin: float
    v_max_bound: float
    u_perp_max: float
    n_theta_allowed: float
    n_rho_allowed: float

    @property
    def passed(self) -> bool:
        return self.burgers_margin >= 1.0 and self.transverse_margin >= 1.0

    def __str__(self) -> str:
        verdict = "pass" if self.passed else "FAIL"
        return (f"CFL burgers margin {self.burgers_margin:.3f} "
                f"(N_theta <= {self.n_theta_allowed:.1f}), "
                f"transverse margin {self.transverse_margin:.3f} "
                f"(N_rho <= {self.n_rho_allowed:.1f}): {verdict}")


def check_cfl_splitting(config: DomainConfig, v_max_bound: float = 5.0,
                        u_perp_max: float = 0.05) -> CflReport:
    burgers_step = config.B * v_max_bound * config.d_sigma
    transverse_step = u_perp_max * config.d_sigma
    bm = config.d_theta / burgers_step if burgers_step > 0 else np.inf
    tm = config.d_rho / transverse_step if transverse_step > 0 else np.inf
    return CflReport(bm, tm, v_max_bound, u_perp_max, config.N_theta * bm, config.N_rho * tm)


def check_cfl_exprk(config: DomainConfig, fields, v_max_bound: float = 5.0) -> CflReport:
    if fields is None:
        u_perp_max = 0.0
    elif hasattr(fields.u_perp, "abs"):      # device tensor (device-generated medium)
        u_perp_max = float(fields.u_perp.abs().max())
    else:
        # max |u| as max(max u, -min u): the same value (NaN and +-inf included)
        # without np.abs's full-size temporary (C2: 192 MB)
        u = np.asarray(fields.u_perp)
        hi, lo = float(np.max(u)), float(np.min(u))
        u_perp_max = hi if np.isnan(hi) else abs(max(hi, -lo))
    return check_cfl_splitting(config, v_max_bound, u_perp_max)
