"""One large grid over G GPUs: rho-slab decomposition (BASELINE C5).

Rank r owns rho rows ``rows_r`` on the physical / theta side (theta c2r,
WENO, theta r2c act on whole rows) and theta modes ``modes_r`` on the rho side
(the rho passes transform whole columns).  Per ExpRK22 stage:

    rho pass (own modes, in chunks)  --point-to-point per chunk-->  theta c2r (own rows)
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

Transit layouts are chosen so the all-to-alls move the arrays in place:
the theta-side spectrum ``spec_rows`` is (kk, rows) unpadded, so the block
exchanged with rank r (its modes x my rows) is one contiguous segment; the
rho-side ``bt_rho`` / ``t_rho`` are block-major -- the block of rank b's rows
(my modes x rows_b) is contiguous at modes * row_start_b (``nwb_slab_set_blocks``;
the rho kernels read and write that layout).  Both sides are then exactly
``all_to_all_single``'s rank-ordered segments: no packing or unpacking
copies.  The rho pass runs in mode chunks (``chunks``, 4 by default on
several ranks): each chunk's blocks leave by point-to-point sends right after
its transforms (on the process group's stream) while the next chunk
transforms, so that transpose overlaps compute; the theta -> rho transpose
is one in-place all_to_all_single (a row chunk of the theta-side spectrum is
not contiguous).  The divergence guard is kept on the device (a per-step
history of the all-reduced max|V|) and checked on the host every
``GUARD_EVERY`` steps.
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


def rank_row_starts(n_rho: int, world: int) -> list[int]:
    """Row partition of the rho axis over ``world`` ranks (shard_members)."""
    return [shard_members(n_rho, world, r).start for r in range(world)] + [n_rho]


def blocks_to_natural(flat, modes: int, starts):
    """Block-major rho-side layout -> (modes, n_rho) natural layout."""
    nat = flat.new_empty((modes, starts[-1]))
    for b in range(len(starts) - 1):
        a, e = starts[b], starts[b + 1]
        nat[:, a:e] = flat[modes * a:modes * e].reshape(modes, e - a)
    return nat


def natural_to_blocks(nat, flat, starts):
    """(modes, n_rho) natural layout -> block-major rho-side layout (in place)."""
    modes = nat.shape[0]
    for b in range(len(starts) - 1):
        a, e = starts[b], starts[b + 1]
        flat[modes * a:modes * e] = nat[:, a:e].reshape(-1)


class _Comm:
    """Collectives of the slab march (or local copies for a single rank)."""

    def __init__(self, group, geo: SlabGeometry):
        self.group = group
        self.geo = geo

    def exchange(self, out_flat, in_flat, out_splits, in_splits):
        """all_to_all_single on flat complex buffers whose rank-ordered
        segments are the blocks (in place, no packing)."""
        import torch

        if self.geo.world == 1:
            out_flat.copy_(in_flat)
            return
        real = torch.is_complex(in_flat)
        o = torch.view_as_real(out_flat).reshape(-1) if real else out_flat
        i = torch.view_as_real(in_flat).reshape(-1) if real else in_flat
        f = 2 if real else 1
        _dist().all_to_all_single(o, i, [f * n for n in out_splits], [f * n for n in in_splits],
                                  group=self.group)

    def sendrecv_async(self, sends, recvs):
        """Point-to-point sends [(dst, tensor)] and receives [(src, tensor)],
        issued after the work queued on the current stream; returns handles
        for ``wait``.  The NCCL kernels run on the process group's stream, so
        kernels queued on other streams afterwards overlap them."""
        import torch

        dist = _dist()
        ops = []
        for dst, t in sends:
            ops.append(dist.P2POp(dist.isend, torch.view_as_real(t) if torch.is_complex(t) else t,
                                  dst, self.group))
        for src, t in recvs:
            ops.append(dist.P2POp(dist.irecv, torch.view_as_real(t) if torch.is_complex(t) else t,
                                  src, self.group))
        return dist.batch_isend_irecv(ops) if ops else []

    def wait(self, handles):
        for h in handles:
            h.wait()

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
            assert ldr.value == len(rows)  # unpadded theta-side spectrum
            starts = rank_row_starts(geo.n_rho, geo.world)
            sarr = (ctypes.c_int * len(starts))(*starts)
            check(self.lib.nwb_slab_set_blocks(self._h, geo.world, sarr), "slab blocks")
            self.spec_rows = z(geo.kk, len(rows), dt=self.cdt)
            self.v_ext = z(len(rows) + 6, geo.n_theta, dt=self.rdt)
            self.b = z(len(rows), geo.n_theta, dt=self.rdt)
            self.bt_rho = z(len(modes) * geo.n_rho, dt=self.cdt)  # block-major transit
            self.t_rho = z(len(modes) * geo.n_rho, dt=self.cdt)
            self.vh = z(len(modes), ldp.value, dt=self.cdt)
            self.u = z(len(modes), ldp.value, dt=self.cdt)
            self.red = z(2, dt=torch.int64)

    def close(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            self.lib.nwb_slab_destroy(h)
            h.value = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # interpreter shutdown: modules may already be gone
            pass

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

    def rho(self, mode: int, k0: int = 0, k1: int | None = None, out=None):
        """rho pass over local modes [k0, k1) into ``out`` (default t_rho)."""
        k1 = len(self.geo.modes()) if k1 is None else k1
        dst = self.t_rho if out is None else out
        self._run(self.lib.nwb_slab_rho_range, mode, k0, k1, self.bt_rho.data_ptr(),
                  dst.data_ptr(), self.vh.data_ptr(), self.u.data_ptr())

    def red_values(self):
        return self.red.cpu().numpy().view(np.float64)

    def rows_field(self):
        return self.v_ext[3:3 + len(self.geo.rows())]


class SlabMarch:
    """Drives the per-slab kernels and the collectives (see module docstring)."""

    GUARD_EVERY = 16

    def __init__(self, config: DomainConfig, fields, precision: str = "double", group=None,
                 ops=None, device=None, max_steps: int | None = None, comm=None,
                 chunks: int | None = None):
        """``comm``: an object with ``geo`` (SlabGeometry) and the ``exchange`` /
        ``max_`` / ``halo`` collectives, replacing torch.distributed (the GPU tests
        drive several virtual ranks in one process through host barriers)."""
        import torch

        self.cfg = config
        if comm is not None:
            world, rank = comm.geo.world, comm.geo.rank
        elif group is not None or _dist().is_available() and _dist().is_initialized():
            world, rank = _dist().get_world_size(group), _dist().get_rank(group)
        else:
            world, rank = 1, 0
        self.geo = SlabGeometry(config.N_rho, config.N_theta, world, rank)
        self.comm = comm if comm is not None else _Comm(group, self.geo)
        self.ops = ops or GpuSlabOps(config, self.geo, precision, device)
        self.n_steps = config.N_sigma if max_steps is None else min(config.N_sigma, max_steps)
        self.ops.set_coeffs(fields, self.n_steps + 1)
        self.max_abs = []
        # per-step all-reduced max|V| (IEEE bits), on the ops' device
        self.hist = torch.zeros(max(self.n_steps, 1), dtype=torch.int64, device=self.ops.red.device)
        self._checked = 0
        g = self.geo
        rows_me, modes_me = len(g.rows()), len(g.modes())
        # all-to-all segment sizes (complex elements), rank order
        self._t2r_in = [len(g.modes(s)) * rows_me for s in range(g.world)]
        self._t2r_out = [modes_me * len(g.rows(r)) for r in range(g.world)]
        # the rho pass runs in mode chunks; chunk c's rho -> theta exchange
        # (point-to-point, in place) overlaps chunk c+1's transforms
        self.chunks = max(1, chunks if chunks is not None else (4 if g.world > 1 else 1))
        self._starts = rank_row_starts(g.n_rho, g.world)

    @staticmethod
    def _chunk(n: int, chunks: int, c: int):
        return (n * c) // chunks, (n * (c + 1)) // chunks

    # -- layout changes (in place: see the module docstring) ----------------
    def _rho_exchange(self, mode: int):
        """rho pass + rho -> theta exchange.  One rank: the rho pass writes
        the theta-side spectrum directly (the layouts coincide).  Several: mode
        chunks, each chunk's blocks sent point to point right after its
        transforms while the next chunk transforms."""
        g, o = self.geo, self.ops
        if g.world == 1:
            o.rho(mode, out=o.spec_rows.reshape(-1))
            return
        me, rows_me, modes_me = g.rank, len(g.rows()), len(g.modes())
        t_flat, s_rows = o.t_rho.reshape(-1), o.spec_rows
        pending = []
        for c in range(self.chunks):
            a, b = self._chunk(modes_me, self.chunks, c)
            if b > a:
                o.rho(mode, a, b)
            sends, recvs = [], []
            for r in range(g.world):
                st, ln = self._starts[r], self._starts[r + 1] - self._starts[r]
                if b > a and ln > 0:  # my chunk of rank r's row block
                    seg = t_flat[modes_me * st + a * ln:modes_me * st + b * ln]
                    if r == me:
                        s_rows[g.modes().start + a:g.modes().start + b].reshape(-1).copy_(seg)
                    else:
                        sends.append((r, seg))
                mr = g.modes(r)
                ar, br = self._chunk(len(mr), self.chunks, c)
                if r != me and br > ar and rows_me > 0:
                    recvs.append((r, s_rows[mr.start + ar:mr.start + br].reshape(-1)))
            pending.append(self.comm.sendrecv_async(sends, recvs))
        for h in pending:
            self.comm.wait(h)

    def _theta_to_rho(self):
        o = self.ops
        self.comm.exchange(o.bt_rho.reshape(-1), o.spec_rows.reshape(-1), self._t2r_out, self._t2r_in)

    # -- march -------------------------------------------------------------
    def load(self, v0_rows):
        """v0_rows: this rank's rows of V0, shape (len(rows), N_theta)."""
        import torch

        o = self.ops
        src = torch.as_tensor(np.ascontiguousarray(v0_rows)).to(o.b.device, o.b.dtype) \
            if not isinstance(v0_rows, torch.Tensor) else v0_rows.to(o.b.device, o.b.dtype)
        o.r2c(src)
        self._theta_to_rho()
        self._rho_exchange(RHO_INIT)

    def _stage(self, row: int, mode: int, guard_step: int | None):
        o = self.ops
        o.red.zero_()
        o.c2r(row, reduce=True)
        self.comm.max_(o.red)
        if guard_step is not None:
            self.hist[guard_step] = o.red[1]  # device copy: no host sync per step
        self.comm.halo(o.v_ext, len(self.geo.rows()))
        o.weno(row)
        o.r2c()
        self._theta_to_rho()
        self._rho_exchange(mode)

    def _check_guard(self, upto: int, guard: float):
        """Host check of the guard history for steps [checked, upto)."""
        if upto <= self._checked:
            return
        vals = self.hist[self._checked:upto].cpu().numpy().view(np.float64)
        for i, m in enumerate(vals):
            m = float(m)
            self.max_abs.append(m)
            if not np.isfinite(m) or m > guard:
                raise InstabilityError((self._checked + i) * self.cfg.d_sigma, m)
        self._checked = upto

    def march(self, scheme: str = "exprk22", guard: float = 10.0, n0: int = 0,
              steps: int | None = None):
        """March ``steps`` steps from absolute step ``n0`` (default: the whole run)."""
        stop = self.n_steps if steps is None else min(self.n_steps, n0 + steps)
        if n0 != self._checked:
            self._checked = n0
        for n in range(n0, stop):
            if scheme == "exprk22":
                self._stage(n, RHO_STAGE1, n)
                self._stage(n + 1, RHO_STAGE2, None)
            else:
                self._stage(n, RHO_EULER, n)
            if (n + 1 - n0) % self.GUARD_EVERY == 0:
                self._check_guard(n + 1, guard)
        self._check_guard(stop, guard)
        return self

    def final_rows(self):
        """This rank's rows of V at the end of the march, and the global max|V|."""
        o = self.ops
        o.red.zero_()
        o.c2r(self.n_steps, reduce=True)
        self.comm.max_(o.red)
        return o.rows_field(), float(o.red_values()[1])
