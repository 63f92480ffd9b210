"""B200-native ExpRK22/WENO5 step for the KZK-type sonic-boom equation
(arXiv 2103.06080), a drop-in for the hot path of the reference ``nwave``
package.

The names below mirror ``nwave``'s exports for that path
(reference ``pkg/src/nwave/__init__.py:6-41``).  The arithmetic runs in
hand-written sm_100a kernels (libnwb200.so, C ABI in include/nwb200.h);
PyTorch only provides device memory and streams.  Importing this package
needs neither a GPU nor the library; calling a compute entry point without
them raises ``BackendError`` (there is no CPU fallback).
"""

__version__ = "0.1.0"

from .errors import (BackendError, BudgetExceededError, CflViolationError, ConfigError,
                     InstabilityError, UnsupportedSizeError)
from .grid import (DomainConfig, Field2D, build_axes, extract_region, l2_norm,
                   max_relative, relative_error, rho_nodes_closed, uniform_nodes)
from .turbulence import (TurbulenceParams, TurbulenceSpec, VelocityFields,
                         downsample_fields, energy_spectrum, evaluate_fields, sample_modes,
                         zero_fields)
from .reports import RunReport
from .cfl import CflReport, check_cfl_exprk, check_cfl_splitting
from .weno import weno5_b
from .exprk import (EPS_DOUBLE, EPS_SINGLE, PhiMultipliers, SpectralTransforms,
                    build_multipliers, exp_euler_step, exprk22_step, phi1, phi2,
                    run_exprk22)
from .analysis import (GRID_SETS, GroundMetrics, ensemble_nwaves, ground_metrics,
                       ground_metrics_device, initial_nwave, preset_config, rho_modulated)
from .studies import (CheckpointComparison, ComparisonReport, ConvergenceRow, ScalingRow,
                      TimingReport, compare_solvers, convergence_rate, convergence_study,
                      cost_scaling_study, max_overshoot)
from .splitting import (SplittingState, godunov_flux, lie_step, run_splitting,
                        step_axial_absorption_spectral, step_burgers_godunov,
                        step_diffraction_cn, step_transverse_lw)
from . import fieldio

__all__ = [
    "BackendError", "BudgetExceededError", "CflViolationError", "ConfigError",
    "InstabilityError", "UnsupportedSizeError", "DomainConfig", "Field2D", "build_axes",
    "extract_region", "l2_norm", "max_relative", "relative_error", "rho_nodes_closed",
    "uniform_nodes", "TurbulenceParams", "TurbulenceSpec", "VelocityFields",
    "downsample_fields", "energy_spectrum", "evaluate_fields", "sample_modes",
    "zero_fields", "RunReport", "CflReport", "check_cfl_exprk", "check_cfl_splitting",
    "weno5_b", "EPS_DOUBLE", "EPS_SINGLE", "PhiMultipliers", "SpectralTransforms",
    "build_multipliers", "exp_euler_step", "exprk22_step", "phi1", "phi2", "run_exprk22",
    "GRID_SETS", "GroundMetrics", "ensemble_nwaves", "ground_metrics", "ground_metrics_device",
    "initial_nwave", "preset_config", "rho_modulated", "CheckpointComparison",
    "ComparisonReport", "ConvergenceRow", "ScalingRow", "TimingReport", "compare_solvers",
    "convergence_rate", "convergence_study", "cost_scaling_study", "max_overshoot", "fieldio",
    "SplittingState", "godunov_flux", "lie_step", "run_splitting",
    "step_axial_absorption_spectral", "step_burgers_godunov", "step_diffraction_cn",
    "step_transverse_lw",
]
