"""One large grid over G GPUs: rho-slab decomposition (BASELINE C5).

Rank r owns rho rows ``rows_r`` on the physical / theta side (theta c2r,
WENO, theta r2c act on whole rows) and theta modes ``modes_r`` on the rho side
(the rho passes transform whole columns).  Per ExpRK22 stage:

    rho pass (own modes)  --all-to-all-->  theta c2r (own rows)
      -> all-reduce MAX of [alpha_theta, max|V|]   (alpha must be global, weno.py:114)
      -> 3-row halo exchange with the ring neighbours (periodic rho)
      -> WENO -> theta r2c  --all-to-all-->  next rho pass

The all-to-alls move (G-1)/G of the local slab each way; on NVSwitch every
peer is at full bandwidth.  Collectives go through ``torch.distributed``
(NCCL on GPUs; gloo in the CPU tests); a single rank (``group=None``) runs the
same code path with local copies.  The per-slab compute is pluggable:
``GpuSlabOps`` calls the sm_100a kernels through ``nwb_slab_*``; the CPU
tests plug in a numpy implementation to check the decomposition logic.

The reduction values are IEEE bit patterns of non-negative doubles held in an
int64 tensor, so the MAX all-reduce is exact and order-independent (the
march stays bitwise reproducible for any G).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from .ensemble import shard_members
from .errors import InstabilityError
from .grid import DomainConfig

RHO_STAGE1, RHO_STAGE2, RHO_EULER, RHO_INIT = 0, 1, 2, 3


@dataclass
class SlabGeometry:
    n_rho: int
    n_theta: int
    world: int
    rank: int

    @property
    def kk(self) -> int:
        return self.n_theta // 2 + 1

    def rows(self, r: int | None = None) -> range:
        return shard_members(self.n_rho, self.world, self.rank if r is None else r)

    def modes(self, r: int | None = None) -> range:
        return shard_members(self.kk, self.world, self.rank if r is None else r)


def _dist():
    import torch.distributed as dist

    return dist


class _Comm:
    """Collectives of the slab march (or local copies for a single rank)."""

    def __init__(self, group, geo: SlabGeometry):
        self.group = group
        self.geo = geo

    def all_to_all(self, sends, recv_shapes, like):
        """sends[s]: tensor for rank s; returns list of tensors received from each rank."""
        import torch

        G = self.geo.world
        if G == 1:
            return [sends[0].clone()]
        real = torch.is_complex(like)
        flat_in = torch.cat([(torch.view_as_real(t) if real else t).reshape(-1) for t in sends])
        in_splits = [t.numel() * (2 if real else 1) for t in sends]
        out_splits = [int(np.prod(sh)) * (2 if real else 1) for sh in recv_shapes]
        flat_out = torch.empty(sum(out_splits), dtype=flat_in.dtype, device=flat_in.device)
        _dist().all_to_all_single(flat_out, flat_in, out_splits, in_splits, group=self.group)
        outs, o = [], 0
        for sh, n in zip(recv_shapes, out_splits):
            chunk = flat_out[o:o + n]
            o += n
            if real:
                chunk = torch.view_as_complex(chunk.reshape(*sh, 2))
            outs.append(chunk.reshape(sh))
        return outs

    def max_(self, t):
        if self.geo.world > 1:
            _dist().all_reduce(t, op=_dist().ReduceOp.MAX, group=self.group)

    def halo(self, v_ext, rows: int):
        """Fill rows 0..2 (previous rank's last rows) and rows+3..rows+5 (next rank's first)."""
        G, r = self.geo.world, self.geo.rank
        if G == 1:
            v_ext[0:3] = v_ext[rows:rows + 3]
            v_ext[rows + 3:rows + 6] = v_ext[3:6]
            return
        dist = _dist()
        prev, nxt = (r - 1) % G, (r + 1) % G
        send_up = v_ext[3:6].contiguous()            # my first rows -> prev's bottom halo
        send_dn = v_ext[rows:rows + 3].contiguous()   # my last rows -> next's top halo
        recv_top = v_ext.new_empty(send_up.shape)
        recv_bot = v_ext.new_empty(send_up.shape)
        # messages between one pair of ranks match in posting order; with two
        # ranks prev == next sends "up" (its first rows = my bottom halo) first
        recvs = [dist.P2POp(dist.irecv, recv_top, prev, self.group),
                 dist.P2POp(dist.irecv, recv_bot, nxt, self.group)]
        if prev == nxt:
            recvs.reverse()
        ops = [dist.P2POp(dist.isend, send_up, prev, self.group),
               dist.P2POp(dist.isend, send_dn, nxt, self.group)] + recvs
        for req in dist.batch_isend_irecv(ops):
            req.wait()
        v_ext[0:3] = recv_top
        v_ext[rows + 3:rows + 6] = recv_bot


class GpuSlabOps:
    """Per-slab kernels on this rank's GPU (``nwb_slab_*`` in libnwb200.so)."""

    def __init__(self, config: DomainConfig, geo: SlabGeometry, precision: str = "double",
                 device=None):
        import torch

        from . import _lib
        from ._lib import check
        from .exprk import EPS_DOUBLE, EPS_SINGLE
        from .plan import cplx_dtype, real_dtype, resolve_device

        self.lib = _lib.lib()
        self.check = check
        self.dev = resolve_device(device)
        self.geo = geo
        self.rdt, self.cdt = real_dtype(precision), cplx_dtype(precision)
        rows, modes = geo.rows(), geo.modes()
        if len(rows) < 3:
            raise ValueError("each rank needs >= 3 rho rows (WENO halo)")
        self._h = ctypes.c_void_p()
        eps = EPS_DOUBLE if precision == "double" else EPS_SINGLE
        with torch.cuda.device(self.dev):
            self.stream = torch.cuda.Stream(device=self.dev)
            check(self.lib.nwb_slab_create(
                ctypes.byref(self._h), geo.n_rho, geo.n_theta, rows.start, len(rows),
                modes.start, len(modes), _lib.F64 if precision == "double" else _lib.F32,
                config.d_sigma, config.rho_span, config.theta_span, config.A, config.B, eps,
                self.dev.index), "nwb_slab_create")
            check(self.lib.nwb_slab_set_stream(self._h, self.stream.cuda_stream), "slab stream")
            ldr, ldp = ctypes.c_int(), ctypes.c_int()
            check(self.lib.nwb_slab_layout(self._h, ctypes.byref(ldr), ctypes.byref(ldp)), "layout")
            z = lambda *shape, dt: torch.zeros(shape, dtype=dt, device=self.dev)
            self.spec_rows = z(geo.kk, ldr.value, dt=self.cdt)
            self.v_ext = z(len(rows) + 6, geo.n_theta, dt=self.rdt)
            self.b = z(len(rows), geo.n_theta, dt=self.rdt)
            self.bt_rho = z(len(modes), ldp.value, dt=self.cdt)
            self.t_rho = z(len(modes), ldp.value, dt=self.cdt)
            self.vh = z(len(modes), ldp.value, dt=self.cdt)
            self.u = z(len(modes), ldp.value, dt=self.cdt)
            self.red = z(2, dt=torch.int64)

    def close(self):
        if getattr(self, "_h", None) and self._h.value:
            self.lib.nwb_slab_destroy(self._h)
            self._h = ctypes.c_void_p()

    __del__ = close

    def _run(self, fn, *args):
        import torch

        cur = torch.cuda.current_stream(self.dev)
        self.stream.wait_stream(cur)
        self.check(fn(self._h, *args), fn.__name__)
        cur.wait_stream(self.stream)

    def set_coeffs(self, fields, rows_needed):
        import torch

        arrs = []
        for name in ("u_par", "u_perp", "du_perp_drho"):
            a = getattr(fields, name)[:rows_needed]
            arrs.append(a.to(self.dev, torch.float64).contiguous() if isinstance(a, torch.Tensor)
                        else torch.from_numpy(np.ascontiguousarray(a, np.float64)).to(self.dev))
        self._coef = arrs
        self._run(self.lib.nwb_slab_set_coeffs, *(a.data_ptr() for a in arrs), rows_needed,
                  arrs[0].shape[1], 1)

    def c2r(self, row: int, reduce: bool = True):
        self._run(self.lib.nwb_slab_theta_c2r, self.spec_rows.data_ptr(), self.v_ext.data_ptr(),
                  row, self.red.data_ptr() if reduce else None)

    def weno(self, row: int):
        self._run(self.lib.nwb_slab_weno, self.v_ext.data_ptr(), self.b.data_ptr(), row,
                  self.red.data_ptr())

    def r2c(self, src=None):
        self._run(self.lib.nwb_slab_theta_r2c, (self.b if src is None else src).data_ptr(),
                  self.spec_rows.data_ptr())

    def rho(self, mode: int):
        self._run(self.lib.nwb_slab_rho, mode, self.bt_rho.data_ptr(), self.t_rho.data_ptr(),
                  self.vh.data_ptr(), self.u.data_ptr())

    def red_values(self):
        return self.red.cpu().numpy().view(np.float64)

    def rows_field(self):
        return self.v_ext[3:3 + len(self.geo.rows())]


class SlabMarch:
    """Drives the per-slab kernels and the collectives (see module docstring)."""

    def __init__(self, config: DomainConfig, fields, precision: str = "double", group=None,
                 ops=None, device=None, max_steps: int | None = None):
        self.cfg = config
        if group is not None or _dist().is_available() and _dist().is_initialized():
            world, rank = _dist().get_world_size(group), _dist().get_rank(group)
        else:
            world, rank = 1, 0
        self.geo = SlabGeometry(config.N_rho, config.N_theta, world, rank)
        self.comm = _Comm(group, self.geo)
        self.ops = ops or GpuSlabOps(config, self.geo, precision, device)
        self.n_steps = config.N_sigma if max_steps is None else min(config.N_sigma, max_steps)
        self.ops.set_coeffs(fields, self.n_steps + 1)
        self.max_abs = []

    # -- layout changes ----------------------------------------------------
    def _rho_to_theta(self):
        g, o = self.geo, self.ops
        me_rows = g.rows()
        sends = [o.t_rho[:, g.rows(s).start:g.rows(s).stop].contiguous() for s in range(g.world)]
        shapes = [(len(g.modes(r)), len(me_rows)) for r in range(g.world)]
        recv = self.comm.all_to_all(sends, shapes, o.t_rho)
        for r, blk in enumerate(recv):
            m = g.modes(r)
            o.spec_rows[m.start:m.stop, :len(me_rows)] = blk

    def _theta_to_rho(self):
        g, o = self.geo, self.ops
        n_me = len(g.rows())
        sends = [o.spec_rows[g.modes(s).start:g.modes(s).stop, :n_me].contiguous()
                 for s in range(g.world)]
        shapes = [(len(g.modes()), len(g.rows(r))) for r in range(g.world)]
        recv = self.comm.all_to_all(sends, shapes, o.spec_rows)
        for r, blk in enumerate(recv):
            rr = g.rows(r)
            o.bt_rho[:, rr.start:rr.stop] = blk

    # -- march -------------------------------------------------------------
    def load(self, v0_rows):
        """v0_rows: this rank's rows of V0, shape (len(rows), N_theta)."""
        import torch

        o = self.ops
        src = torch.as_tensor(np.ascontiguousarray(v0_rows)).to(o.b.device, o.b.dtype) \
            if not isinstance(v0_rows, torch.Tensor) else v0_rows.to(o.b.device, o.b.dtype)
        o.r2c(src)
        self._theta_to_rho()
        o.rho(RHO_INIT)

    def _stage(self, row: int, mode: int, guard_slot: bool):
        o = self.ops
        self._rho_to_theta()
        o.red.zero_()
        o.c2r(row, reduce=True)
        self.comm.max_(o.red)
        if guard_slot:
            self.max_abs.append(float(o.red_values()[1]))
        self.comm.halo(o.v_ext, len(self.geo.rows()))
        o.weno(row)
        o.r2c()
        self._theta_to_rho()
        o.rho(mode)

    def march(self, scheme: str = "exprk22", guard: float = 10.0, n0: int = 0,
              steps: int | None = None):
        """March ``steps`` steps from absolute step ``n0`` (default: the whole run)."""
        stop = self.n_steps if steps is None else min(self.n_steps, n0 + steps)
        for n in range(n0, stop):
            if scheme == "exprk22":
                self._stage(n, RHO_STAGE1, True)
                self._stage(n + 1, RHO_STAGE2, False)
            else:
                self._stage(n, RHO_EULER, True)
            m = self.max_abs[-1]
            if not np.isfinite(m) or m > guard:
                raise InstabilityError(n * self.cfg.d_sigma, m)
        return self

    def final_rows(self):
        """This rank's rows of V at the end of the march, and the global max|V|."""
        o = self.ops
        self._rho_to_theta()
        o.red.zero_()
        o.c2r(self.n_steps, reduce=True)
        self.comm.max_(o.red)
        return o.rows_field(), float(o.red_values()[1])
