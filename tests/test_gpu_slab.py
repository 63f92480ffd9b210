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


def test_slab_tma_staging_bitwise(cuda, monkeypatch):
    """The halo-extended slab WENO stages its fp64 tiles by TMA (rows + 6 halo
    rows in the tensor map); NWB_WENO_TMA=0 selects cp.async: bitwise equal."""
    from paper_2103_06080_b200.slab import SlabMarch

    cfg = nw.DomainConfig(Sigma=2.4, N_sigma=6, N_rho=1050, N_theta=2100)
    _, rho, theta = nw.build_axes(cfg)
    v0 = nw.rho_modulated(cfg, nw.initial_nwave(rho, theta, cfg.A, cfg.B)).values
    f = nw.zero_fields(4, cfg.N_rho + 1)
    outs = []
    for tma in ("0", "1"):
        monkeypatch.setenv("NWB_WENO_TMA", tma)
        sm = SlabMarch(cfg, f, max_steps=2)
        sm.load(v0)
        sm.march()
        rows, _ = sm.final_rows()
        outs.append(rows.cpu().numpy())
    assert np.array_equal(outs[0], outs[1])


class _ThreadComm:
    """Collectives between virtual ranks that are host threads of one process
    (each with its own slab plan and stream on the one GPU).  Data moves by
    device copies after host barriers -- no kernel ever waits on another
    rank's kernel, so nothing relies on concurrent residency."""

    def __init__(self, geo, shared, barrier):
        self.geo, self.shared, self.barrier = geo, shared, barrier

    def _sync(self):
        import torch

        torch.cuda.synchronize()
        self.barrier.wait()

    def exchange(self, out_flat, in_flat, out_splits, in_splits):
        r, G = self.geo.rank, self.geo.world
        self._sync()
        self.shared[r] = (in_flat, [sum(in_splits[:s]) for s in range(G)], in_splits)
        self._sync()
        o = 0
        for src in range(G):
            buf, offs, sizes = self.shared[src]
            n = out_splits[src]
            assert sizes[r] == n
            out_flat[o:o + n].copy_(buf[offs[r]:offs[r] + n])
            o += n
        self._sync()

    def sendrecv_async(self, sends, recvs):
        r = self.geo.rank
        self._sync()
        for dst, t in sends:
            self.shared[(r, dst)] = t
        self._sync()
        for src, t in recvs:
            t.copy_(self.shared[(src, r)])
        self._sync()
        return []

    def wait(self, handles):
        pass

    def max_(self, t):
        import torch

        r, G = self.geo.rank, self.geo.world
        self._sync()
        self.shared[r] = t.clone()
        self._sync()
        t.copy_(torch.stack([self.shared[s] for s in range(G)]).max(dim=0).values)
        self._sync()

    def halo(self, v_ext, rows):
        r, G = self.geo.rank, self.geo.world
        self._sync()
        self.shared[r] = (v_ext[3:6].clone(), v_ext[rows:rows + 3].clone())
        self._sync()
        v_ext[0:3] = self.shared[(r - 1) % G][1]
        v_ext[rows + 3:rows + 6] = self.shared[(r + 1) % G][0]
        self._sync()


@pytest.mark.parametrize("world", [2, 3])
def test_slab_virtual_ranks_vs_oracle(cuda, oracle, world):
    """G ranks of the rho-slab march as threads on one GPU: the block-major
    transit layout of the rho kernels (several blocks), the in-place
    all-to-all segments, the MAX all-reduce and the halo ring, against the
    single-process oracle."""
    import threading

    import torch

    from paper_2103_06080_b200.slab import SlabGeometry, SlabMarch

    cfg = nw.DomainConfig(N_rho=48, N_theta=56, N_sigma=5, Sigma=2.0)
    sig, rho, theta = nw.build_axes(cfg)
    spec = nw.sample_modes(nw.TurbulenceParams(seed=4))
    f = nw.evaluate_fields(spec, spec.lam, sig, nw.rho_nodes_closed(cfg))
    v0 = nw.rho_modulated(cfg, nw.initial_nwave(rho, theta, cfg.A, cfg.B), depth=0.3).values
    shared, barrier = {}, threading.Barrier(world)
    out, errors = {}, []

    def rank_main(r):
        try:
            torch.cuda.set_device(0)
            geo = SlabGeometry(cfg.N_rho, cfg.N_theta, world, r)
            sm = SlabMarch(cfg, f, comm=_ThreadComm(geo, shared, barrier))
            rows = geo.rows()
            sm.load(v0[rows.start:rows.stop])
            sm.march()
            mine, vmax = sm.final_rows()
            out[r] = (rows, mine.cpu().numpy(), vmax, list(sm.max_abs))
        except BaseException as exc:  # surfaced below
            errors.append(exc)
            barrier.abort()

    ths = [threading.Thread(target=rank_main, args=(r,)) for r in range(world)]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    if errors:
        raise errors[0]
    full = np.zeros((cfg.N_rho, cfg.N_theta))
    for rows, mine, _, _ in out.values():
        full[rows.start:rows.stop] = mine
    ref = oracle.march(cfg, v0, f)
    assert max_relative(ref.final, full) <= 1e-10
    for _, _, vmax, max_abs in out.values():
        assert max(max(max_abs), vmax) == pytest.approx(ref.max_abs_v, abs=1e-12)
