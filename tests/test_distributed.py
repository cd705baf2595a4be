"""Multi-rank optimize (shots sharded, positions all-gathered, scalars reduced in rank
order) on the gloo backend with the CPU oracle ops: world_size 2 must reproduce the
single-rank run, for even and uneven shot splits."""

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_2108_02991_b200 as spk


def _cfg(n_c, n_decim=1):
    return spk.OptimizerConfig(n_c=n_c, n_s=32, dims=2, n_decim=n_decim, n_git=4, n_pit=60,
                               grad_mode="exact", grid_n=8, seed=4, perturbation=0.25)


def _hw():
    return spk.HardwareSpec(g_max=0.04, s_max=180.0, gamma=42.576e6, raster_dt=1e-5,
                            dwell_dt=1e-5, fov=0.192, matrix=16, dims=2)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, n_c, out_path, n_decim=1):
    from cpu_ops import OracleOps

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        res = spk.optimize(_cfg(n_c, n_decim), _hw(), ops=OracleOps())
        if rank == 0:
            np.savez(out_path, coords=res.pattern.coords, costs=res.trace.costs(),
                     steps=np.array([r.step for r in res.trace.records]),
                     feas=np.array([r.feas_residual for r in res.trace.records]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n_c", [6, 5])
def test_two_ranks_match_one(tmp_path, n_c):
    from cpu_ops import OracleOps

    single = spk.optimize(_cfg(n_c), _hw(), ops=OracleOps())
    out = str(tmp_path / "r.npz")
    mp.spawn(_worker, args=(2, _free_port(), n_c, out), nprocs=2, join=True)
    got = np.load(out)
    assert got["coords"].shape == single.pattern.coords.shape
    # sharding changes only the summation order of the cost / BB scalars
    assert np.allclose(got["costs"], single.trace.costs(), rtol=1e-12, atol=0)
    assert np.allclose(got["steps"], [r.step for r in single.trace.records], rtol=1e-9)
    assert np.abs(got["coords"] - single.pattern.coords).max() <= 1e-9
    assert np.array_equal(got["feas"] <= 1e-6, np.ones_like(got["feas"], dtype=bool))


@pytest.mark.parametrize("world,n_c", [(3, 7), (2, 4)])
def test_multilevel_ranks_match_one(tmp_path, world, n_c):
    """Multi-resolution schedule (two levels, upsample between them; reference
    src/optimizer.py:276-291) with more ranks than an even split allows: every level
    re-shards the same shot ranges, so the sharded run must track the single-rank one."""
    from cpu_ops import OracleOps

    single = spk.optimize(_cfg(n_c, 2), _hw(), ops=OracleOps())
    out = str(tmp_path / "r.npz")
    mp.spawn(_worker, args=(world, _free_port(), n_c, out, 2), nprocs=world, join=True)
    got = np.load(out)
    assert got["coords"].shape == single.pattern.coords.shape
    assert len(got["costs"]) == len(single.trace.records)
    assert np.allclose(got["costs"], single.trace.costs(), rtol=1e-12, atol=0)
    assert np.allclose(got["steps"], [r.step for r in single.trace.records], rtol=1e-9)
    assert np.abs(got["coords"] - single.pattern.coords).max() <= 1e-9
