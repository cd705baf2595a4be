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


def _worker_too_few(rank, world, port, out_dir):
    from cpu_ops import OracleOps

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        try:
            spk.optimize(_cfg(2, 0), _hw(), ops=OracleOps())
            msg = "no error"
        except ValueError as exc:
            msg = str(exc)
        with open(os.path.join(out_dir, f"r{rank}.txt"), "w") as fh:
            fh.write(msg)
    finally:
        dist.destroy_process_group()


def test_fewer_shots_than_ranks_raises_everywhere(tmp_path):
    """2 shots over 3 ranks: every rank raises ValueError before any collective (no rank
    waits in an all-gather for a rank that has no targets)."""
    mp.spawn(_worker_too_few, args=(3, _free_port(), str(tmp_path)), nprocs=3, join=True)
    for r in range(3):
        msg = (tmp_path / f"r{r}.txt").read_text()
        assert "cannot be sharded over 3 ranks" in msg, (r, msg)


def _patched_attraction(k, fld, grad_mode="consistent"):
    """A host evaluator in the reference's shape (what tests monkeypatch into
    optimizer.eval_attraction, reference tests/test_optimizer.py:224): the fp64 exact sum."""
    from oracle import oracle as orc

    cost, grad = orc.attraction_exact(k.points(), fld.density.grid, fld.kernel_eps)
    return spk.AttractionResult(cost=cost, grad=grad, n_clamped=0)


def _patched_repulsion(k, cfg):
    from oracle import oracle as orc

    return orc.repulsion(k.points(), cfg.kernel_eps)


def _worker_patched(rank, world, port, n_c, out_path):
    from cpu_ops import OracleOps
    import paper_2108_02991_b200.optimizer as om

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    om.eval_attraction = _patched_attraction
    om.eval_repulsion = _patched_repulsion
    try:
        res = spk.optimize(_cfg(n_c), _hw(), ops=OracleOps())
        if rank == 0:
            np.savez(out_path, coords=res.pattern.coords, costs=res.trace.costs())
    finally:
        dist.destroy_process_group()


def test_patched_evaluator_two_ranks_match_one(tmp_path, monkeypatch):
    """The patched-evaluator path (host gradient of the whole pattern) sharded over two
    ranks keeps each rank's rows and reproduces the single-rank run."""
    from cpu_ops import OracleOps
    import paper_2108_02991_b200.optimizer as om

    monkeypatch.setattr(om, "eval_attraction", _patched_attraction)
    monkeypatch.setattr(om, "eval_repulsion", _patched_repulsion)
    single = spk.optimize(_cfg(5), _hw(), ops=OracleOps())
    monkeypatch.undo()
    out = str(tmp_path / "p.npz")
    mp.spawn(_worker_patched, args=(2, _free_port(), 5, out), nprocs=2, join=True)
    got = np.load(out)
    assert np.allclose(got["costs"], single.trace.costs(), rtol=1e-12, atol=0)
    assert np.abs(got["coords"] - single.pattern.coords).max() <= 1e-9


def _worker_overlap(rank, world, port, n_c, out_path):
    from cpu_ops import OverlapOracleOps

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    os.environ["SPK_OVERLAP"] = "1"
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ops = OverlapOracleOps()
        res = spk.optimize(_cfg(n_c), _hw(), ops=ops)
        if rank == 0:
            np.savez(out_path, coords=res.pattern.coords, costs=res.trace.costs(),
                     calls=np.int64(ops.overlap_calls))
    finally:
        dist.destroy_process_group()


def test_overlap_schedule_two_ranks_matches_plain(tmp_path, monkeypatch):
    """The K2-under-polish schedule (per-rank K2 rows computed with the projection, K1
    alone in the next evaluation, polish groups ordered by the previous sweeps) on two
    gloo ranks reproduces the plain single-rank loop: the oracle's lattice sums are
    row-wise fp64, so the results must match to the rank-order reduction of the scalars."""
    from cpu_ops import OracleOps

    monkeypatch.setenv("SPK_OVERLAP", "0")
    single = spk.optimize(_cfg(5), _hw(), ops=OracleOps())
    out = str(tmp_path / "o.npz")
    mp.spawn(_worker_overlap, args=(2, _free_port(), 5, out), nprocs=2, join=True)
    got = np.load(out)
    assert int(got["calls"]) > 0
    assert np.allclose(got["costs"], single.trace.costs(), rtol=1e-12, atol=0)
    assert np.abs(got["coords"] - single.pattern.coords).max() <= 1e-9


def _worker_k1_pipe(rank, world, port, n_c, out_path):
    from cpu_ops import OverlapOracleOps

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    os.environ["SPK_OVERLAP"] = "1"
    os.environ["SPK_K1_PIPE"] = "1"
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ops = OverlapOracleOps()
        calls = []
        orig = ops.repulsion_sums

        def counted(t4, s4, cfg):
            calls.append((t4.shape[0], s4.shape[0]))
            return orig(t4, s4, cfg)

        ops.repulsion_sums = counted
        res = spk.optimize(_cfg(n_c), _hw(), ops=ops)
        if rank == 0:
            np.savez(out_path, coords=res.pattern.coords, costs=res.trace.costs(),
                     blocks=np.array(calls, dtype=np.int64))
    finally:
        dist.destroy_process_group()


def test_k1_pipeline_two_ranks_matches_plain(tmp_path, monkeypatch):
    """K1 under the polish (ShardedRun._k1_pipelined, opt-in SPK_K1_PIPE=1, even shards):
    each polish group's positions are all-gathered as the group finishes and
    the (target group, source group) blocks of K1 run as soon as both are final.  On two
    gloo ranks (6 shots each, 3 groups of 2) the iteration equals the plain single-rank
    loop to fp64 summation order, and the K1 work really ran as blocks."""
    from cpu_ops import OracleOps

    monkeypatch.setenv("SPK_OVERLAP", "0")
    single = spk.optimize(_cfg(12), _hw(), ops=OracleOps())
    out = str(tmp_path / "k.npz")
    mp.spawn(_worker_k1_pipe, args=(2, _free_port(), 12, out), nprocs=2, join=True)
    got = np.load(out)
    n_s = single.pattern.coords.shape[1]
    blocks = got["blocks"]
    # group-sized target blocks against 1, 2, 3 gathered groups (2 ranks x 2 shots each)
    assert (blocks[:, 0] == 2 * n_s).any() and (blocks[:, 1] == 3 * 4 * n_s).any()
    assert np.allclose(got["costs"], single.trace.costs(), rtol=1e-12, atol=0)
    assert np.abs(got["coords"] - single.pattern.coords).max() <= 1e-9


def _worker_spatial(rank, world, port, n_c, out_path):
    from cpu_ops import OracleOps

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    os.environ["SPK_SPATIAL"] = "1"
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        res = spk.optimize(_cfg(n_c, 2), _hw(), ops=OracleOps())
        if rank == 0:
            np.savez(out_path, coords=res.pattern.coords, costs=res.trace.costs())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,n_c", [(2, 6), (3, 7)])
def test_spatial_target_partition_matches_one(tmp_path, world, n_c):
    """The treecodes' multi-GPU layout (N-body targets split into Morton-order blocks,
    results all-gathered and returned to the shots' owners; engine.ShardedRun.spatial) on
    gloo ranks reproduces the single-rank run over a two-level schedule (uneven blocks
    and shot splits included)."""
    from cpu_ops import OracleOps

    single = spk.optimize(_cfg(n_c, 2), _hw(), ops=OracleOps())
    out = str(tmp_path / "s.npz")
    mp.spawn(_worker_spatial, args=(world, _free_port(), n_c, out), nprocs=world, join=True)
    got = np.load(out)
    assert np.allclose(got["costs"], single.trace.costs(), rtol=1e-12, atol=0)
    assert np.abs(got["coords"] - single.pattern.coords).max() <= 1e-9
