"""CPU: the rho-slab decomposition of one grid over G ranks.

G = 1 (local copies) and G = 2 / 3 over gloo, with numpy per-slab ops
(tests/slab_numpy_ops.py) standing in for the GPU kernels: the gathered
field must equal the single-process oracle march to roundoff.  This checks
the layout changes (all-to-all), the MAX all-reduce of alpha_theta / max|V|
and the periodic 3-row halo ring.
"""

import os
import socket
import sys

import numpy as np
import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _case():
    import paper_2103_06080_b200 as nw

    cfg = nw.DomainConfig(N_rho=24, N_theta=28, N_sigma=4, Sigma=1.6)
    sig, rho, theta = nw.build_axes(cfg)
    spec = nw.sample_modes(nw.TurbulenceParams(seed=3))
    fields = nw.evaluate_fields(spec, spec.lam, sig, nw.rho_nodes_closed(cfg))
    v0 = nw.rho_modulated(cfg, nw.initial_nwave(rho, theta, cfg.A, cfg.B), depth=0.3).values
    return cfg, fields, v0


def _run_rank(rank, world, port, out_path, group_backend="gloo"):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import torch.distributed as dist
    from slab_numpy_ops import NumpySlabOps

    from paper_2103_06080_b200.slab import SlabGeometry, SlabMarch

    if world > 1:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group(group_backend, rank=rank, world_size=world)
    try:
        cfg, fields, v0 = _case()
        geo = SlabGeometry(cfg.N_rho, cfg.N_theta, world, rank)
        sm = SlabMarch(cfg, fields, ops=NumpySlabOps(cfg, geo))
        rows = geo.rows()
        sm.load(v0[rows.start:rows.stop])
        sm.march()
        mine, vmax = sm.final_rows()
        np.savez(f"{out_path}.{rank}.npz", rows=np.array([rows.start, rows.stop]),
                 v=mine.numpy(), vmax=vmax, max_abs=np.array(sm.max_abs))
    finally:
        if world > 1:
            dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world", [1, 2, 3])
def test_slab_march_matches_single_process_oracle(tmp_path, world):
    from oracle import nwave_oracle

    out = str(tmp_path / "slab")
    if world == 1:
        _run_rank(0, 1, 0, out)
    else:
        mp.spawn(_run_rank, args=(world, _free_port(), out), nprocs=world, join=True)
    cfg, fields, v0 = _case()
    field = np.zeros((cfg.N_rho, cfg.N_theta))
    for r in range(world):
        d = np.load(f"{out}.{r}.npz")
        a, b = d["rows"]
        field[a:b] = d["v"]
        vmax, max_abs = float(d["vmax"]), d["max_abs"]
    ref = nwave_oracle.march(cfg, v0, fields)
    assert np.max(np.abs(field - ref.final)) <= 1e-13 * np.max(np.abs(ref.final))
    assert max(max_abs.max(), vmax) == pytest.approx(ref.max_abs_v, rel=1e-13)


def test_block_major_transit_layout_roundtrip():
    """The rho-side transit layout (slab.py): rank b's rows form one contiguous
    (modes x rows_b) block at modes * start_b, i.e. exactly all_to_all_single's
    rank-ordered segments; natural <-> block-major is a bijection."""
    import torch

    from paper_2103_06080_b200.slab import (SlabGeometry, blocks_to_natural, natural_to_blocks,
                                            rank_row_starts)

    for n_rho, world in ((24, 1), (24, 3), (10, 4), (7, 2)):
        starts = rank_row_starts(n_rho, world)
        assert starts[0] == 0 and starts[-1] == n_rho and all(a <= b for a, b in zip(starts, starts[1:]))
        modes = 5
        nat = torch.arange(modes * n_rho, dtype=torch.float64).reshape(modes, n_rho)
        flat = torch.empty(modes * n_rho, dtype=torch.float64)
        natural_to_blocks(nat, flat, starts)
        for b in range(world):
            a, e = starts[b], starts[b + 1]
            assert torch.equal(flat[modes * a:modes * e].reshape(modes, e - a), nat[:, a:e])
        assert torch.equal(blocks_to_natural(flat, modes, starts), nat)
        geo = SlabGeometry(n_rho, 16, world, 0)
        assert starts[:-1] == [geo.rows(r).start for r in range(world)]
