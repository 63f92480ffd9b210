"""Device plan: owns one ``nwb_plan`` (tables, twiddles, workspaces) plus
the torch stream the plan's kernels run on.

PyTorch is only plumbing here: it allocates device buffers, provides the
stream and moves host arrays in and out.  All arithmetic runs in
libnwb200.so.
"""

from __future__ import annotations

import ctypes
from contextlib import contextmanager

import numpy as np

from . import _lib
from ._lib import check, ptr
from .errors import InstabilityError
from .hostio import par_copyto

_STAGE_BYTES = 32 << 20  # page-locked staging chunk for large host -> device copies


def _torch():
    import torch

    return torch


def real_dtype(precision: str):
    torch = _torch()
    return torch.float64 if precision == "double" else torch.float32


def cplx_dtype(precision: str):
    torch = _torch()
    return torch.complex128 if precision == "double" else torch.complex64


def resolve_device(device=None):
    torch = _torch()
    _lib.lib()  # raises BackendError without CUDA
    if device is None:
        return torch.device("cuda", torch.cuda.current_device())
    dev = torch.device(device)
    if dev.type != "cuda":
        raise ValueError(f"the B200 backend runs on CUDA devices only, got {dev}")
    return torch.device("cuda", dev.index if dev.index is not None else torch.cuda.current_device())


class DevicePlan:
    """One grid (n_rho x n_theta) x ``batch`` members on one device."""

    def __init__(self, n_rho: int, n_theta: int, batch: int = 1, precision: str = "double",
                 d_sigma: float = 1.0, rho_span: float = 1.0, theta_span: float = 1.0,
                 A: float = 0.0, B: float = 0.0, eps: float = 2.0 ** -53, device=None):
        torch = _torch()
        if precision not in ("double", "single"):
            raise ValueError(f"unknown precision {precision!r}")
        self.lib = _lib.lib()
        self.device = resolve_device(device)
        self.n_rho, self.n_theta, self.batch = int(n_rho), int(n_theta), int(batch)
        self.kk = self.n_theta // 2 + 1
        self.precision = precision
        self.rdt = real_dtype(precision)
        self.cdt = cplx_dtype(precision)
        self.d_sigma = float(d_sigma)
        self._h = ctypes.c_void_p()
        with torch.cuda.device(self.device):
            self.stream = torch.cuda.Stream(device=self.device)
            check(self.lib.nwb_plan_create(
                ctypes.byref(self._h), self.n_rho, self.n_theta, self.batch,
                _lib.F64 if precision == "double" else _lib.F32, float(d_sigma),
                float(rho_span), float(theta_span), float(A), float(B), float(eps),
                self.device.index), "nwb_plan_create")
            check(self.lib.nwb_plan_set_stream(self._h, self.stream.cuda_stream),
                  "nwb_plan_set_stream")
        self.n_rows = 0

    # ------------------------------------------------------------ plumbing
    @contextmanager
    def on_stream(self):
        """Run torch work on the plan's stream, ordered after the caller's."""
        torch = _torch()
        with torch.cuda.device(self.device):
            cur = torch.cuda.current_stream(self.device)
            self.stream.wait_stream(cur)
            with torch.cuda.stream(self.stream):
                yield
            cur.wait_stream(self.stream)

    def close(self):
        if getattr(self, "_h", None) and self._h.value:
            self.lib.nwb_plan_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def bytes(self) -> int:
        return int(self.lib.nwb_plan_bytes(self._h))

    def to_device(self, arr, dtype):
        torch = _torch()
        if isinstance(arr, torch.Tensor):
            return arr.to(device=self.device, dtype=dtype).contiguous()
        host_np = np.ascontiguousarray(arr)
        host = torch.from_numpy(host_np)
        if host.numel() * host.element_size() < 2 * _STAGE_BYTES:
            return host.to(device=self.device, dtype=dtype, non_blocking=False).contiguous()
        # large host arrays (a C2 field is 287 MB): through two page-locked staging
        # chunks from torch's caching host allocator, so the (multi-threaded) host
        # copy of chunk i+1 overlaps the DMA of chunk i -- a pageable copy runs at
        # ~11 GB/s
        out = torch.empty(tuple(host.shape), dtype=dtype, device=self.device)
        src, dst = host.reshape(-1), out.reshape(-1)
        src_np = host_np.reshape(-1)
        per = _STAGE_BYTES // max(src.element_size(), out.element_size())
        bufs = [torch.empty(per, dtype=dtype, pin_memory=True) for _ in range(2)]
        done = [None, None]
        stream = torch.cuda.current_stream(self.device)
        for i, s in enumerate(range(0, src.numel(), per)):
            e, k = min(src.numel(), s + per), i & 1
            if done[k] is not None:
                done[k].synchronize()
            par_copyto(bufs[k][: e - s].numpy(), src_np[s:e])
            dst[s:e].copy_(bufs[k][: e - s], non_blocking=True)
            done[k] = torch.cuda.Event()
            done[k].record(stream)
        stream.synchronize()
        return out

    # ------------------------------------------------------------ state
    def set_coeffs(self, u_par, u_perp, du_drho, n_rows: int | None = None):
        """Coefficient tables (n_sigma_rows, >= n_rho), host numpy or device fp64."""
        torch = _torch()
        arrays = []
        for a in (u_par, u_perp, du_drho):
            if a is None:
                arrays.append(None)
                continue
            if isinstance(a, torch.Tensor):
                arrays.append(a.to(device=self.device, dtype=torch.float64).contiguous())
            else:
                arrays.append(np.ascontiguousarray(a, dtype=np.float64))
        ref = next((a for a in arrays if a is not None), None)
        rows = n_rows if n_rows is not None else (ref.shape[0] if ref is not None else 1)
        ld = ref.shape[1] if ref is not None else self.n_rho
        if ref is not None and ref.shape[0] < rows:
            raise ValueError("coefficient tables have fewer rows than requested")
        if ref is not None and not isinstance(ref, torch.Tensor) and \
                sum(a[:rows].nbytes for a in arrays if a is not None) >= 2 * _STAGE_BYTES:
            # large host tables (C2: 3 x 192 MB) through the page-locked staging
            # chunks of to_device instead of a pageable copy
            with self.on_stream():
                arrays = [None if a is None else self.to_device(a[:rows], torch.float64)
                          for a in arrays]
            ref = next(a for a in arrays if a is not None)
        on_dev = int(ref is not None and isinstance(ref, torch.Tensor))

        def p(a):
            if a is None:
                return None
            return a.data_ptr() if isinstance(a, torch.Tensor) else a.ctypes.data

        with self.on_stream():
            check(self.lib.nwb_plan_set_coeffs(self._h, p(arrays[0]), p(arrays[1]),
                                               p(arrays[2]), int(rows), int(ld), on_dev),
                  "nwb_plan_set_coeffs")
        self.n_rows = rows

    def load_physical(self, v0):
        """v0: (batch, n_rho, n_theta) or (n_rho, n_theta), host or device."""
        with self.on_stream():
            v = self.to_device(v0, self.rdt).reshape(self.batch, self.n_rho, self.n_theta)
            check(self.lib.nwb_plan_load_physical(self._h, ptr(v)), "load_physical")
            self.stream.synchronize()

    def load_spectrum(self, vhat):
        with self.on_stream():
            x = self.to_device(vhat, self.cdt).reshape(self.batch, self.n_rho, self.kk)
            check(self.lib.nwb_plan_load_spectrum(self._h, ptr(x)), "load_spectrum")
            self.stream.synchronize()

    def store_spectrum(self):
        torch = _torch()
        with self.on_stream():
            out = torch.empty((self.batch, self.n_rho, self.kk), dtype=self.cdt, device=self.device)
            check(self.lib.nwb_plan_store_spectrum(self._h, ptr(out)), "store_spectrum")
        return out

    def store_physical(self):
        """(V = irfft2(Vhat) on device, max|V| per member as numpy)."""
        torch = _torch()
        mx = np.zeros(self.batch)
        with self.on_stream():
            out = torch.empty((self.batch, self.n_rho, self.n_theta), dtype=self.rdt,
                              device=self.device)
            check(self.lib.nwb_plan_store_physical(
                self._h, ptr(out), mx.ctypes.data_as(ctypes.c_void_p)), "store_physical")
        return out, mx

    # ------------------------------------------------------------ march
    def march(self, scheme: str, n0: int, n_steps: int, guard: float = 10.0,
              max_seconds: float | None = None, snap_steps=(), timing: bool = True,
              total_steps: int | None = None):
        """Advance the device state; returns (max_abs[batch, n_steps],
        step_ms[n_steps, 3] or None, {step: device snapshot}).

        Both modes replay a captured CUDA graph per step; ``timing`` adds the
        per-step bucket events (nonlinear = WENO + theta r2c, rest linear).
        ``snap_steps`` inside the range are copied to fresh device buffers
        (run_exprk22 streams its snapshots instead, see ``SnapshotStreamer``).
        Raises InstabilityError with the reference's sigma = n * d_sigma of the
        first offending step, BudgetExceededError when out of wall clock
        (``max_seconds`` counted from this call; the message numbers steps out
        of ``total_steps``, default n0 + n_steps).
        """
        torch = _torch()
        code = _lib.SCHEME_EXPRK22 if scheme == "exprk22" else _lib.SCHEME_EXPEULER
        snaps = sorted(set(int(s) for s in snap_steps if n0 <= int(s) < n0 + n_steps))
        max_abs = np.zeros((self.batch, max(n_steps, 0)))
        step_ms = np.zeros((max(n_steps, 0), 3), dtype=np.float32) if timing else None
        fail_step, fail_member, fail_value = ctypes.c_int(-1), ctypes.c_int(-1), ctypes.c_double(0)
        with self.on_stream():
            bufs = {s: torch.empty((self.batch, self.n_rho, self.n_theta), dtype=self.rdt,
                                   device=self.device) for s in snaps}
            steps_arr = (ctypes.c_int * max(len(snaps), 1))(*snaps)
            ptrs_arr = (ctypes.c_void_p * max(len(snaps), 1))(*[bufs[s].data_ptr() for s in snaps])
            rc = self.lib.nwb_march(
                self._h, code, int(n0), int(n_steps), float(guard),
                float(max_seconds) if max_seconds is not None else -1.0,
                steps_arr, len(snaps), ptrs_arr, max_abs.ctypes.data_as(ctypes.c_void_p),
                step_ms.ctypes.data_as(ctypes.c_void_p) if step_ms is not None else None,
                ctypes.byref(fail_step), ctypes.byref(fail_member), ctypes.byref(fail_value))
        if rc == _lib.NWB_EINSTABILITY:
            err = InstabilityError(fail_step.value * self.d_sigma, fail_value.value)
            err.step = fail_step.value
            err.member = fail_member.value
            raise err
        if rc == _lib.NWB_EBUDGET:
            from .errors import BudgetExceededError

            total = total_steps if total_steps is not None else n0 + n_steps
            raise BudgetExceededError(
                f"exceeded {max_seconds:.0f} s at step {fail_step.value}/{total}")
        check(rc, "nwb_march", d_sigma=self.d_sigma)
        return max_abs, step_ms, bufs

    def store_physical_into(self, out):
        """c2r of the state into ``out`` (batch, n_rho, n_theta) on the plan
        stream (same kernel as the stage-1 c2r: bitwise the step-start field)."""
        with self.on_stream():
            check(self.lib.nwb_plan_store_physical(self._h, ptr(out), None), "store_physical")

    def profile_kernels(self, scheme: str, n0: int, n_steps: int) -> np.ndarray:
        """Summed device ms per kernel slot over n_steps steps (CUDA events
        around every launch): [c2r, weno, r2c, rho] x stage 1, stage 2."""
        code = _lib.SCHEME_EXPRK22 if scheme == "exprk22" else _lib.SCHEME_EXPEULER
        out = np.zeros(8, dtype=np.float32)
        check(self.lib.nwb_profile_kernels(self._h, code, int(n0), int(n_steps),
                                           out.ctypes.data_as(ctypes.c_void_p)),
              "nwb_profile_kernels")
        return out.astype(np.float64)

    def step(self, scheme: str, n: int):
        code = _lib.SCHEME_EXPRK22 if scheme == "exprk22" else _lib.SCHEME_EXPEULER
        check(self.lib.nwb_step(self._h, code, int(n)), "nwb_step")

    # ------------------------------------------------------------ transforms
    def rfft2(self, x):
        """(batch, n_rho, n_theta) real device tensor -> natural half spectrum."""
        torch = _torch()
        with self.on_stream():
            x = x.to(device=self.device, dtype=self.rdt).contiguous()
            out = torch.empty(x.shape[:-1] + (self.kk,), dtype=self.cdt, device=self.device)
            check(self.lib.nwb_rfft2(self._h, ptr(x), ptr(out)), "nwb_rfft2")
        return out

    def irfft2(self, x):
        torch = _torch()
        with self.on_stream():
            x = x.to(device=self.device, dtype=self.cdt).contiguous()
            out = torch.empty(x.shape[:-1] + (self.n_theta,), dtype=self.rdt, device=self.device)
            check(self.lib.nwb_irfft2(self._h, ptr(x), ptr(out)), "nwb_irfft2")
        return out


_plan_cache: dict = {}


def cached_plan(n_rho, n_theta, batch=1, precision="double", device=None) -> DevicePlan:
    """Table-less-use plan (transforms only), cached per geometry and device."""
    dev = resolve_device(device)
    key = (int(n_rho), int(n_theta), int(batch), precision, dev.index)
    plan = _plan_cache.get(key)
    if plan is None:
        if len(_plan_cache) > 16:
            _plan_cache.pop(next(iter(_plan_cache))).close()
        plan = DevicePlan(n_rho, n_theta, batch, precision, device=dev)
        _plan_cache[key] = plan
    return plan
