"""``weno5_b`` -- the WENO5 nonlinear right-hand side on the device.

Drop-in for ``nwave.weno.weno5_b`` (reference ``pkg/src/nwave/weno.py:106-124``):
same arguments, same result.  Inputs may be numpy arrays (the result is a
numpy array, like the reference) or CUDA tensors (the result stays on the
device).  ``v`` may carry a leading batch axis; the coefficient vectors are
then shared by every member.  The arithmetic runs in the ``k_weno`` /
``k_alpha_theta`` kernels of libnwb200.so.
"""

from __future__ import annotations

import numpy as np

from . import _lib
from ._lib import check, ptr
from .plan import resolve_device

WENO_EPS = 1e-6


def weno5_b(v, u_par, u_perp, du_perp_drho, b_coef, d_rho, d_theta, device=None):
    import torch

    lib = _lib.lib()
    is_torch = isinstance(v, torch.Tensor)
    if is_torch and v.is_cuda:
        dev = v.device
    else:
        dev = resolve_device(device)
    np_dtype = v.dtype if not is_torch else None
    if is_torch:
        rdt = v.dtype
    else:
        rdt = torch.float32 if np.asarray(v).dtype == np.float32 else torch.float64
    if rdt not in (torch.float32, torch.float64):
        raise TypeError(f"weno5_b: unsupported dtype {rdt}")
    prec = _lib.F64 if rdt == torch.float64 else _lib.F32

    def dev_t(a, dt):
        if isinstance(a, torch.Tensor):
            return a.to(device=dev, dtype=dt).contiguous()
        return torch.from_numpy(np.ascontiguousarray(a)).to(device=dev, dtype=dt).contiguous()

    with torch.cuda.device(dev):
        x = dev_t(v, rdt)
        if x.ndim not in (2, 3):
            raise ValueError("weno5_b: v must be (n_rho, n_theta) or (batch, n_rho, n_theta)")
        batch = 1 if x.ndim == 2 else x.shape[0]
        nr, nt = x.shape[-2], x.shape[-1]
        coefs = [dev_t(c, rdt).reshape(-1) for c in (u_par, u_perp, du_perp_drho)]
        for c in coefs:
            if c.numel() != nr:
                raise ValueError("weno5_b: coefficient vectors must have one value per rho node")
        out = torch.empty_like(x)
        ws = torch.zeros(batch + 1, dtype=torch.float64, device=dev)
        stream = torch.cuda.current_stream(dev).cuda_stream
        check(lib.nwb_weno5_b(prec, batch, nr, nt, ptr(x), ptr(coefs[0]), ptr(coefs[1]),
                              ptr(coefs[2]), float(b_coef), float(d_rho), float(d_theta),
                              ptr(out), ptr(ws), stream), "nwb_weno5_b")
    if is_torch:
        return out
    return out.cpu().numpy().astype(np_dtype, copy=False)
