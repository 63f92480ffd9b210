"""CPU, world_size 2 over gloo: the ensemble sharding layer.

Members are partitioned with ``shard_members``; each rank marches its shard
(here with the CPU oracle standing in for the device march, since the test
host has no GPU) and ``gather_summaries`` all-gathers the per-member
summaries.  The gathered result must equal the single-process ensemble.
"""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2103_06080_b200.ensemble import EnsembleResult, gather_summaries, shard_members


def test_shards_cover_members_exactly_once():
    for n in (0, 1, 7, 256, 257):
        for world in (1, 2, 3, 4, 8):
            got = [i for r in range(world) for i in shard_members(n, world, r)]
            assert got == list(range(n))
            sizes = [len(shard_members(n, world, r)) for r in range(world)]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard_members(4, 2, 2)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _small_case():
    import paper_2103_06080_b200 as nw

    cfg = nw.DomainConfig(N_rho=20, N_theta=28, N_sigma=4, Sigma=1.6)
    v0s, _, _ = nw.ensemble_nwaves(cfg, 5, seed=2026)
    return cfg, v0s, nw.zero_fields(5, 21)


def _oracle_shard(cfg, v0s, fields, members):
    from oracle import nwave_oracle

    nwave_oracle.build()
    j = int(round((144.0 - cfg.rho_min) / cfg.d_rho)) % cfg.N_rho
    mabs, peak = [], []
    for i in members:
        run = nwave_oracle.march(cfg, v0s[i], fields, threads=1)
        mabs.append(run.max_abs_v)
        peak.append(run.final[j].max())
    return EnsembleResult(members, None, np.array(mabs), np.array(peak), 0.0, cfg.N_sigma)


def _worker(rank, world, port, out_path):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cfg, v0s, fields = _small_case()
        res = _oracle_shard(cfg, v0s, fields, shard_members(len(v0s), world, rank))
        mabs, peak = gather_summaries(res, len(v0s))
        if rank == 0:
            np.savez(out_path, mabs=mabs, peak=peak)
    finally:
        dist.destroy_process_group()


def test_two_rank_ensemble_equals_single_process(tmp_path):
    out = str(tmp_path / "gathered.npz")
    mp.spawn(_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    got = np.load(out)
    cfg, v0s, fields = _small_case()
    ref = _oracle_shard(cfg, v0s, fields, range(len(v0s)))
    assert np.array_equal(got["mabs"], ref.max_abs_v)
    assert np.array_equal(got["peak"], ref.peak)
