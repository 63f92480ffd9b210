"""TEST INFRASTRUCTURE: numpy per-slab ops with the GpuSlabOps interface, so the
rho-slab decomposition (paper_2103_06080_b200/slab.py) can be checked on CPU
ranks over gloo.  Conventions (those of the GPU slab): spec_rows = rfft_theta
of the owned rows (transposed, (kk, rows)); bt_rho / t_rho in the block-major
transit layout of slab.py (block of rank b's rows contiguous at modes *
row_start_b), holding rfft_theta of b / ifft_rho of the state spectrum; the
arithmetic restates exprk.py:151-178 and weno.py."""

import numpy as np
import torch

from oracle import nwave_oracle as O
from paper_2103_06080_b200.slab import blocks_to_natural, natural_to_blocks, rank_row_starts

TWO_PI = 2.0 * np.pi


class NumpySlabOps:
    def __init__(self, config, geo):
        self.cfg, self.geo = config, geo
        rows, modes = geo.rows(), geo.modes()
        tabs = O.build_tables(config.N_rho, config.N_theta, config.rho_span, config.theta_span,
                              config.d_sigma, config.A, O.EPS_DOUBLE)
        sl = slice(modes.start, modes.stop)
        self.E, self.P1, self.P12, self.P2 = (t[:, sl].T.copy() for t in
                                              (tabs.E, tabs.Phi1, tabs.Phi1m2, tabs.Phi2))
        z = lambda *s, dt: torch.zeros(s, dtype=dt)
        c, r = torch.complex128, torch.float64
        self.spec_rows = z(geo.kk, len(rows), dt=c)
        self.v_ext = z(len(rows) + 6, config.N_theta, dt=r)
        self.b = z(len(rows), config.N_theta, dt=r)
        self.bt_rho = z(len(modes) * config.N_rho, dt=c)
        self.t_rho = z(len(modes) * config.N_rho, dt=c)
        self.starts = rank_row_starts(config.N_rho, geo.world)
        self.vh = z(len(modes), config.N_rho, dt=c)
        self.u = z(len(modes), config.N_rho, dt=c)
        self.red = z(2, dt=torch.int64)

    def set_coeffs(self, fields, rows_needed):
        nr = self.cfg.N_rho
        self.up, self.uq, self.du = (np.asarray(getattr(fields, n)[:rows_needed, :nr], np.float64)
                                     for n in ("u_par", "u_perp", "du_perp_drho"))

    def _rows(self):
        return self.geo.rows()

    def c2r(self, row, reduce=True):
        rows = self._rows()
        v = np.fft.irfft(self.spec_rows.numpy().T, n=self.cfg.N_theta, axis=1)
        self.v_ext[3:3 + len(rows)] = torch.from_numpy(v)
        if reduce:
            c = TWO_PI * self.up[row, rows.start:rows.stop][:, None]
            vals = np.array([np.max(np.abs(c + self.cfg.B * v)), np.max(np.abs(v))])
            self.red.copy_(torch.from_numpy(vals.view(np.int64)))

    def weno(self, row):
        cfg, rows = self.cfg, self._rows()
        ve = self.v_ext.numpy()
        a_th = float(self.red.numpy().view(np.float64)[0])
        a_rh = float(np.max(np.abs(self.uq[row])))
        gidx = (np.arange(rows.start - 3, rows.stop + 3)) % cfg.N_rho
        c = TWO_PI * self.up[row, gidx][:, None]
        g = -c * ve - 0.5 * cfg.B * ve * ve
        dth = O._div_np(0.5 * (g + a_th * ve), 0.5 * (g - a_th * ve), 1, 1.0 / cfg.d_theta)
        h = self.uq[row, gidx][:, None] * ve
        drh = O._div_np(0.5 * (h + a_rh * ve), 0.5 * (h - a_rh * ve), 0, 1.0 / cfg.d_rho)
        du = self.du[row, gidx][:, None]
        out = (du * ve - dth) - drh
        self.b.copy_(torch.from_numpy(out[3:3 + len(rows)]))

    def r2c(self, src=None):
        x = (self.b if src is None else src).numpy()
        self.spec_rows.copy_(torch.from_numpy(np.fft.rfft(x, axis=1).T.copy()))

    def rho(self, mode, k0=0, k1=None, out=None):
        """Modes [k0, k1) of the rho pass into ``out`` (default t_rho), both in
        the block-major transit layout (one block = natural (modes, n_rho))."""
        nmodes = len(self.geo.modes())
        k1 = nmodes if k1 is None else k1
        sl = slice(k0, k1)
        bt = blocks_to_natural(self.bt_rho, nmodes, self.starts).numpy()[sl]
        bh = np.fft.fft(bt, axis=1)
        ds = self.cfg.d_sigma
        vh, u = self.vh.numpy()[sl], self.u.numpy()[sl]
        E, P1, P12, P2 = self.E[sl], self.P1[sl], self.P12[sl], self.P2[sl]
        if mode == 3:
            new = bh
        elif mode == 0:
            ev = E * vh
            u[:] = ev + ds * P12 * bh
            new = None
            res = np.fft.ifft(ev + ds * P1 * bh, axis=1)
        elif mode == 1:
            new = u + ds * P2 * bh
        else:
            new = E * vh + ds * P1 * bh
        if new is not None:
            vh[:] = new
            res = np.fft.ifft(new, axis=1)
        dst = self.t_rho if out is None else out
        chunk = torch.from_numpy(np.ascontiguousarray(res))
        for b in range(len(self.starts) - 1):
            a, e = self.starts[b], self.starts[b + 1]
            dst[nmodes * a + k0 * (e - a):nmodes * a + k1 * (e - a)] = chunk[:, a:e].reshape(-1)

    def red_values(self):
        return self.red.numpy().view(np.float64)

    def rows_field(self):
        return self.v_ext[3:3 + len(self._rows())]
