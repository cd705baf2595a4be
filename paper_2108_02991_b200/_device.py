"""Device-memory plumbing (PyTorch tensors as buffers, one current stream).

No arithmetic of the hot path happens here; it only owns buffers and hands raw
pointers to the C ABI.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _native

_WS: dict = {}


def device() -> torch.device:
    """The CUDA device the kernels run on.  Raises if there is none (no CPU fallback)."""
    if not torch.cuda.is_available():
        raise RuntimeError(
            "paper_2108_02991_b200 needs a CUDA device (built for sm_100a / B200); "
            "there is no CPU fallback")
    _native.load()
    return torch.device("cuda", torch.cuda.current_device())


def stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def ptr(t):
    return None if t is None else t.data_ptr()


def workspace(nbytes: int, slot: str = "main") -> torch.Tensor:
    """A cached uint8 device buffer of at least ``nbytes`` (grown on demand)."""
    dev = device()
    key = (dev.index, slot)
    buf = _WS.get(key)
    if buf is None or buf.numel() < nbytes:
        buf = torch.empty(max(int(nbytes), 256), dtype=torch.uint8, device=dev)
        _WS[key] = buf
    return buf


def h2d(arr: np.ndarray, dtype=torch.float64) -> torch.Tensor:
    """Copy a host array to the device (synchronous; pageable source)."""
    host = torch.from_numpy(np.ascontiguousarray(arr))
    if host.dtype != dtype:
        host = host.to(dtype)
    return host.to(device(), non_blocking=False)


# Below this size the pinned staging buys nothing over a plain copy.
_PINNED_MIN_BYTES = 1 << 16


def d2h(t: torch.Tensor) -> np.ndarray:
    """Device -> host numpy array through page-locked memory: a pageable D2H runs at
    ~2 GB/s on the B200 boxes, a pinned one at full PCIe rate, and the array returned is a
    view of the pinned buffer (torch's caching host allocator keeps it alive and reuses
    it), so a later h2d of that array is a page-locked copy too."""
    t = t.detach()
    if t.device.type != "cuda" or t.numel() * t.element_size() < _PINNED_MIN_BYTES:
        return t.to("cpu").numpy()
    host = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
    host.copy_(t)  # synchronous copy into the page-locked buffer
    return host.numpy()


def pack_positions(coords: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
    """fp64 (..., d) coordinates -> float4 positions (p, 4) f32 via our kernel."""
    d = coords.shape[-1]
    p = coords.numel() // d
    if out is None:
        out = torch.empty((p, 4), dtype=torch.float32, device=coords.device)
    _native.call("spk_pack_positions", ptr(coords), p, d, ptr(out), stream())
    return out


def release_workspaces() -> None:
    """Drop the cached workspaces (e.g. between problem sizes in one process)."""
    _WS.clear()
    if torch.cuda.is_available():
        torch.cuda.empty_cache()
