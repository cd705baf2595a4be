"""The C ABI from plain C (examples/abi_demo.c: cudaMalloc'd buffers, no PyTorch):
repulsion raw sums vs the fp64 oracle, and the batched projection bit-identical to the
oracle (outputs and sweep counts)."""

import os
import subprocess

import numpy as np
import pytest

from oracle import oracle as orc

pytestmark = pytest.mark.gpu
REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(REPO, "paper_2108_02991_b200", "_lib")


def _build(tmp_path):
    exe = str(tmp_path / "abi_demo")
    subprocess.run(["gcc", "-O2", "-I", os.path.join(REPO, "include"), "-I", "/usr/local/cuda/include",
                    os.path.join(REPO, "examples", "abi_demo.c"), "-L", LIB, "-lsparkling_b200",
                    "-L", "/usr/local/cuda/lib64", "-lcudart", "-o", exe], check=True)
    return exe


def test_c_consumer_matches_oracle(tmp_path):
    import paper_2108_02991_b200 as spk  # builds/locates the library

    exe = _build(tmp_path)
    rng = np.random.default_rng(21)
    p, dims, n_shots, n_s, pin = 3000, 3, 12, 256, 128
    pts = rng.uniform(-1, 1, (p, dims))
    shots = rng.uniform(-1.2, 1.2, (n_shots, n_s, dims))
    eps, a, b, tol = 1e-3, 0.05, 0.01, 1e-7
    tau = 1.0 / spk.projection.stacked_operator_norm(n_s, pin)
    pin_val = np.array([0.05, -0.02, 0.0])
    with open(tmp_path / "in.bin", "wb") as fh:
        fh.write(np.array([p, dims, n_shots, n_s, pin], dtype=np.int64).tobytes())
        fh.write(np.array([eps, a, b, tau, tol, *pin_val], dtype=np.float64).tobytes())
        fh.write(pts.tobytes())
        fh.write(shots.tobytes())
    env = dict(os.environ, LD_LIBRARY_PATH=LIB + ":" + os.environ.get("LD_LIBRARY_PATH", ""))
    res = subprocess.run([exe, str(tmp_path / "in.bin"), str(tmp_path / "out.bin")], env=env,
                         capture_output=True, text=True, timeout=300)
    assert res.returncode == 0, res.stderr
    raw = (tmp_path / "out.bin").read_bytes()
    f64 = np.frombuffer(raw[: (p + p * dims + shots.size) * 8], dtype=np.float64)
    val, grad = f64[:p], f64[p:p + p * dims].reshape(p, dims)
    proj = f64[p + p * dims:].reshape(shots.shape)
    sweeps = np.frombuffer(raw[(p + p * dims + shots.size) * 8:], dtype=np.int32)
    vref, gref = orc.direct_sums(pts, eps * eps)
    assert np.linalg.norm(val - vref) / np.linalg.norm(vref) <= 1e-5
    assert np.linalg.norm(grad - gref) / np.linalg.norm(gref) <= 1e-4
    ref, rsw = orc.project_all(shots, a, b, pin, pin_val, 100, tau, tol)
    assert np.array_equal(sweeps, rsw)
    assert np.array_equal(proj, ref)
