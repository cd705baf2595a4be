"""The multi-GPU code path (NCCL process group, sharded ShardedRun, all-gathers, max over
ranks) exercised on the one GPU this run has, as a world of size 1: every collective the
N-rank path issues runs through NCCL, and no rank waits on another.  N > 1 host logic is
covered by tests/test_distributed.py (gloo, world size 2)."""

import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

_WORKER = r'''
import os, sys, numpy as np, torch, torch.distributed as dist
sys.path.insert(0, sys.argv[1])
import paper_2108_02991_b200 as spk
cfg = spk.OptimizerConfig(n_c=16, n_s=64, dims=2, n_decim=1, n_git=6, n_pit=60, grad_mode="exact",
                          grid_n=16, seed=3, perturbation=0.25)
hw = spk.HardwareSpec(g_max=0.04, s_max=180.0, gamma=42.576e6, raster_dt=1e-5, dwell_dt=1e-5,
                      fov=0.192, matrix=32, dims=2)
if sys.argv[2] == "nccl":
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
res = spk.optimize(cfg, hw)
np.savez(sys.argv[3], coords=res.pattern.coords, costs=res.trace.costs())
if dist.is_initialized():
    dist.destroy_process_group()
'''


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_nccl_world1_optimize_is_bitwise(tmp_path):
    env = dict(os.environ, MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_port()))
    out = {}
    for mode in ("plain", "nccl"):
        path = str(tmp_path / f"{mode}.npz")
        subprocess.run([sys.executable, "-c", _WORKER, REPO, mode, path], check=True, env=env,
                       timeout=600)
        out[mode] = np.load(path)
    assert np.array_equal(out["plain"]["coords"], out["nccl"]["coords"])
    assert np.array_equal(out["plain"]["costs"], out["nccl"]["costs"])


def test_bench_under_torchrun_world1(tmp_path):
    """bench.py's N-rank arm (NCCL init, barriers, max-over-ranks, sharded e2e) at N = 1."""
    env = dict(os.environ, SPK_BENCH_DIST="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "1",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), "bench.py",
           "--config", "c1", "--gpus", "1", "--steps", "2", "--warmup", "3",
           "--no-cpu-baseline"]
    res = subprocess.run(cmd, cwd=REPO, env=env, capture_output=True, text=True, timeout=900)
    assert res.returncode == 0, res.stderr[-2000:]
    line = json.loads(res.stdout.strip().splitlines()[-1])
    assert line["n_gpus"] == 1 and line["value"] > 0 and line["gpu_launches"] > 0
    assert line["e2e"]["h2d_bytes_per_step"] > 0
