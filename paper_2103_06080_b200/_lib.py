"""ctypes binding of libnwb200.so (the C ABI in include/nwb200.h).

There is no CPU fallback: if the library is missing or no CUDA device is
visible, every entry point raises ``BackendError``.
"""

from __future__ import annotations

import ctypes
import os
import threading

from .errors import (BackendError, BudgetExceededError, InstabilityError,
                     UnsupportedSizeError)

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("NWB_LIB") or os.path.join(HERE, "libnwb200.so")

NWB_OK = 0
NWB_EINVAL = -1
NWB_EUNSUPPORTED = -2
NWB_ECUDA = -3
NWB_ENOMEM = -4
NWB_EINSTABILITY = -5
NWB_EBUDGET = -6

F64 = 0
F32 = 1
SCHEME_EXPRK22 = 0
SCHEME_EXPEULER = 1

ABI_SYMBOLS = (
    "nwb_abi_version", "nwb_last_error", "nwb_device_count", "nwb_plan_create",
    "nwb_plan_destroy", "nwb_plan_set_stream", "nwb_plan_bytes", "nwb_plan_set_coeffs",
    "nwb_plan_load_physical", "nwb_plan_load_spectrum", "nwb_plan_store_spectrum",
    "nwb_plan_store_physical", "nwb_march", "nwb_step", "nwb_rfft2", "nwb_irfft2",
    "nwb_weno5_b", "nwb_tables", "nwb_phi", "nwb_combine", "nwb_profile_kernels",
    "nwb_turbulence_fields", "nwb_slab_create", "nwb_slab_destroy", "nwb_slab_set_stream",
    "nwb_slab_layout", "nwb_slab_set_coeffs", "nwb_slab_theta_c2r", "nwb_slab_weno",
    "nwb_slab_theta_r2c", "nwb_slab_rho", "nwb_slab_set_blocks", "nwb_slab_rho_range",
    "nwb_ground_metrics",
    "nwb_split_create",
    "nwb_split_destroy", "nwb_split_set_stream", "nwb_split_set_coeffs", "nwb_split_load",
    "nwb_split_store", "nwb_split_stage", "nwb_split_march", "nwb_godunov_flux",
)

_lock = threading.Lock()
_lib = None

c_int, c_double, c_void_p = ctypes.c_int, ctypes.c_double, ctypes.c_void_p
c_ll = ctypes.c_longlong
P = ctypes.POINTER


def _declare(lib):
    sig = {
        "nwb_abi_version": (c_int, []),
        "nwb_last_error": (ctypes.c_char_p, []),
        "nwb_device_count": (c_int, []),
        "nwb_plan_create": (c_int, [P(c_void_p), c_int, c_int, c_int, c_int, c_double,
                                    c_double, c_double, c_double, c_double, c_double, c_int]),
        "nwb_plan_destroy": (c_int, [c_void_p]),
        "nwb_plan_set_stream": (c_int, [c_void_p, c_void_p]),
        "nwb_plan_bytes": (c_ll, [c_void_p]),
        "nwb_plan_set_coeffs": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_int, c_int,
                                        c_int]),
        "nwb_plan_load_physical": (c_int, [c_void_p, c_void_p]),
        "nwb_plan_load_spectrum": (c_int, [c_void_p, c_void_p]),
        "nwb_plan_store_spectrum": (c_int, [c_void_p, c_void_p]),
        "nwb_plan_store_physical": (c_int, [c_void_p, c_void_p, c_void_p]),
        "nwb_march": (c_int, [c_void_p, c_int, c_int, c_int, c_double, c_double, c_void_p,
                              c_int, c_void_p, c_void_p, c_void_p, P(c_int), P(c_int),
                              P(c_double)]),
        "nwb_step": (c_int, [c_void_p, c_int, c_int]),
        "nwb_profile_kernels": (c_int, [c_void_p, c_int, c_int, c_int, c_void_p]),
        "nwb_rfft2": (c_int, [c_void_p, c_void_p, c_void_p]),
        "nwb_irfft2": (c_int, [c_void_p, c_void_p, c_void_p]),
        "nwb_weno5_b": (c_int, [c_int, c_int, c_int, c_int, c_void_p, c_void_p, c_void_p,
                                c_void_p, c_double, c_double, c_double, c_void_p, c_void_p,
                                c_void_p]),
        "nwb_tables": (c_int, [c_int, c_int, c_int, c_double, c_double, c_double, c_double,
                               c_double, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                               c_void_p]),
        "nwb_phi": (c_int, [c_void_p, c_ll, c_int, c_void_p, c_void_p]),
        "nwb_ground_metrics": (c_int, [c_int, c_int, c_int, c_int, c_void_p, c_int, c_int, c_int,
                                       c_void_p, c_void_p, c_void_p]),
        "nwb_slab_create": (c_int, [P(c_void_p), c_int, c_int, c_int, c_int, c_int, c_int, c_int,
                                    c_double, c_double, c_double, c_double, c_double, c_double,
                                    c_int]),
        "nwb_slab_destroy": (c_int, [c_void_p]),
        "nwb_slab_set_stream": (c_int, [c_void_p, c_void_p]),
        "nwb_slab_layout": (c_int, [c_void_p, P(c_int), P(c_int)]),
        "nwb_slab_set_blocks": (c_int, [c_void_p, c_int, c_void_p]),
        "nwb_slab_rho_range": (c_int, [c_void_p, c_int, c_int, c_int, c_void_p, c_void_p, c_void_p,
                                       c_void_p]),
        "nwb_slab_set_coeffs": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_int, c_int,
                                        c_int]),
        "nwb_slab_theta_c2r": (c_int, [c_void_p, c_void_p, c_void_p, c_int, c_void_p]),
        "nwb_slab_weno": (c_int, [c_void_p, c_void_p, c_void_p, c_int, c_void_p]),
        "nwb_slab_theta_r2c": (c_int, [c_void_p, c_void_p, c_void_p]),
        "nwb_slab_rho": (c_int, [c_void_p, c_int, c_void_p, c_void_p, c_void_p, c_void_p]),
        "nwb_turbulence_fields": (c_int, [c_int, c_void_p, c_double, c_double, c_void_p, c_int,
                                          c_void_p, c_int, c_void_p, c_void_p, c_void_p,
                                          c_void_p, c_void_p, c_void_p]),
        "nwb_combine": (c_int, [c_int, c_ll, c_int, c_double, c_void_p, c_void_p, c_void_p,
                                c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p]),
        "nwb_split_create": (c_int, [P(c_void_p), c_int, c_int, c_double, c_double, c_double,
                                     c_double, c_double, c_double, c_int]),
        "nwb_split_destroy": (c_int, [c_void_p]),
        "nwb_split_set_stream": (c_int, [c_void_p, c_void_p]),
        "nwb_split_set_coeffs": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_int,
                                         c_int, c_int]),
        "nwb_split_load": (c_int, [c_void_p, c_void_p]),
        "nwb_split_store": (c_int, [c_void_p, c_void_p]),
        "nwb_split_stage": (c_int, [c_void_p, c_int, c_int, c_void_p, c_void_p]),
        "nwb_split_march": (c_int, [c_void_p, c_int, c_int, c_double, c_double, c_void_p,
                                    P(c_int), P(c_double)]),
        "nwb_godunov_flux": (c_int, [c_ll, c_void_p, c_void_p, c_double, c_void_p, c_void_p]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args


def load_library():
    """Load libnwb200.so (no device needed); raises BackendError if absent."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise BackendError(
                    f"{LIB_PATH} is missing: build it with `python -m "
                    "paper_2103_06080_b200._build` (there is no CPU fallback)")
            try:
                lib = ctypes.CDLL(LIB_PATH)
            except OSError as exc:  # pragma: no cover - loader failure
                raise BackendError(f"cannot load {LIB_PATH}: {exc}") from exc
            _declare(lib)
            _lib = lib
    return _lib


def lib():
    """The library, after checking that a CUDA device is usable."""
    import torch

    if not torch.cuda.is_available():
        raise BackendError("no CUDA device visible: the B200 backend has no CPU fallback")
    return load_library()


def last_error() -> str:
    raw = load_library().nwb_last_error()
    return raw.decode(errors="replace") if raw else ""


def instability_from_message(msg: str, d_sigma: float | None = None) -> InstabilityError:
    """InstabilityError(sigma, max_abs) from the library's guard message
    (``step=<n> member=<i> max_abs=<v>``): sigma = n * d_sigma like the
    reference (``exprk.py:297-299``); nan when the step size is not known."""
    import re

    fields = dict(re.findall(r"(step|member|max_abs)=(\S+)", msg))
    step = int(fields["step"]) if "step" in fields else None
    value = float(fields["max_abs"]) if "max_abs" in fields else float("nan")
    sigma = step * d_sigma if (step is not None and d_sigma is not None) else float("nan")
    err = InstabilityError(sigma, value)
    err.step = step
    err.member = int(fields["member"]) if "member" in fields else None
    return err


def check(rc: int, what: str = "", d_sigma: float | None = None):
    if rc == NWB_OK:
        return
    msg = f"{what}: {last_error()}" if what else last_error()
    if rc == NWB_EINVAL:
        raise ValueError(msg)
    if rc == NWB_EUNSUPPORTED:
        raise UnsupportedSizeError(msg)
    if rc == NWB_EINSTABILITY:
        raise instability_from_message(msg, d_sigma)
    if rc == NWB_EBUDGET:
        raise BudgetExceededError(msg)
    raise BackendError(f"{msg} (code {rc})")


def ptr(t) -> int | None:
    """Device pointer of a torch tensor (or None)."""
    return None if t is None else t.data_ptr()
