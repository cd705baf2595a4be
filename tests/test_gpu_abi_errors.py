"""C-ABI error paths: invalid arguments return SPK_ERR_ARG (-> ValueError), an
undersized workspace SPK_ERR_WORKSPACE (-> NativeError), each with spk_last_error()
naming the problem, and a failed call launches nothing and leaves the library usable."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def env():
    import paper_2108_02991_b200  # noqa: F401
    from paper_2108_02991_b200 import _device, _native

    return _device, _native


def test_argument_errors(env):
    _device, _native = env
    pts = _device.h2d(np.zeros((8, 2)))
    p4 = _device.pack_positions(pts)
    val = torch.empty(8, dtype=torch.float64, device=pts.device)
    grad = torch.empty((8, 2), dtype=torch.float64, device=pts.device)
    ws = _device.workspace(_native.query("spk_nbody_workspace_bytes", 8, 0, 8), "err")
    with pytest.raises(ValueError, match="dims"):
        _native.call("spk_direct_sums", p4.data_ptr(), 8, p4.data_ptr(), 8, 4, 1e-6,
                     val.data_ptr(), grad.data_ptr(), ws.data_ptr(), ws.numel(),
                     _device.stream())
    out = torch.empty((2, 1, 2), dtype=torch.float64, device=pts.device)
    pws = _device.workspace(_native.query("spk_project_workspace_bytes", 2, 1, 2, 0), "err2")
    with pytest.raises(ValueError, match="at least 2 samples"):
        _native.call("spk_project_all", out.data_ptr(), None, 0.0, None, out.data_ptr(), 2, 1,
                     2, 0.1, 0.1, -1, _native.f64_array([0, 0]), 10, 0.05, 0, 1e-7, 100, None,
                     None, None, None, pws.data_ptr(), pws.numel(), _device.stream())
    with pytest.raises(ValueError, match="unknown mode"):
        g = _native.i64_array([4, 4])
        w = torch.zeros((8, 2), dtype=torch.float64, device=pts.device)
        o = torch.empty((16, 2), dtype=torch.float64, device=pts.device)
        nws = _device.workspace(_native.query("spk_nudft_workspace_bytes", 8, 2, g), "err3")
        _native.call("spk_nudft_adjoint", pts.data_ptr(), w.data_ptr(), 8, 2, g, 7,
                     o.data_ptr(), nws.data_ptr(), nws.numel(), _device.stream())


def test_workspace_too_small(env):
    _device, _native = env
    shots = _device.h2d(np.zeros((4, 64, 3)))
    out = torch.empty_like(shots)
    tiny = torch.empty(16, dtype=torch.uint8, device=shots.device)
    with pytest.raises(_native.NativeError, match="workspace"):
        _native.call("spk_project_all", shots.data_ptr(), None, 0.0, None, out.data_ptr(), 4,
                     64, 3, 0.1, 0.1, -1, _native.f64_array([0, 0, 0]), 10, 0.05, 0, 1e-7, 100,
                     None, None, None, None, tiny.data_ptr(), tiny.numel(), _device.stream())


def test_library_usable_after_errors(env):
    import paper_2108_02991_b200 as spk

    cost, grad = spk.eval_repulsion_direct(np.array([[0.0, 0.0], [1.0, 0.0]]), eps=0.0)
    assert abs(cost - 0.25) < 1e-7 and np.abs(grad).max() == pytest.approx(0.25, rel=1e-7)


def test_round2_entry_point_errors(env):
    """spk_grid_sums_shots / spk_polish_shots / spk_project_fista reject bad arguments and
    undersized workspaces like the other entry points."""
    _device, _native = env
    dev = _device.device()
    p4 = _device.pack_positions(_device.h2d(np.zeros((32, 3))))
    val = torch.empty(32, dtype=torch.float64, device=dev)
    grad = torch.empty((32, 3), dtype=torch.float64, device=dev)
    w = torch.zeros(28, dtype=torch.float32, device=dev)
    side = _native.i64_array([3, 3, 3])
    ids = torch.tensor([1, 3], dtype=torch.int32, device=dev)
    tiny = torch.empty(16, dtype=torch.uint8, device=dev)
    with pytest.raises(ValueError, match="null shot list"):
        _native.call("spk_grid_sums_shots", p4.data_ptr(), None, 2, 8, w.data_ptr(), side, 3,
                     1e-4, val.data_ptr(), grad.data_ptr(), None, tiny.data_ptr(),
                     tiny.numel(), _device.stream())
    with pytest.raises(_native.NativeError, match="workspace"):
        _native.call("spk_grid_sums_shots", p4.data_ptr(), ids.data_ptr(), 2, 8, w.data_ptr(),
                     side, 3, 1e-4, val.data_ptr(), grad.data_ptr(), None, tiny.data_ptr(),
                     tiny.numel(), _device.stream())
    shots = _device.h2d(np.zeros((4, 8, 3)))
    with pytest.raises(_native.NativeError, match="workspace"):
        _native.call("spk_polish_shots", shots.data_ptr(), ids.data_ptr(), 2, 4, 8, 3, 0.1, 0.1,
                     -1, _native.f64_array([0, 0, 0]), 1e-7, 100, None, None, None, None, 0,
                     0, tiny.data_ptr(), tiny.numel(), _device.stream())
    with pytest.raises(ValueError, match="n_pit"):
        _native.call("spk_project_fista", shots.data_ptr(), None, 0.0, None, shots.data_ptr(),
                     4, 8, 3, 0.1, 0.1, -1, _native.f64_array([0, 0, 0]), 0, 0.05, 0, None,
                     None, tiny.data_ptr(), tiny.numel(), _device.stream())
