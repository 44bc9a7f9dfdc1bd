"""Device plumbing: tensors in and out of the native library (PyTorch for
device memory and streams only -- all arithmetic happens in libwino)."""

from __future__ import annotations

import numpy as np

try:
    import torch
except ImportError as exc:  # pragma: no cover - torch is part of the image
    raise RuntimeError("paper_1803_10986_b200 needs PyTorch for device memory") from exc

from . import _native

_DT = {np.float32: torch.float32, np.float64: torch.float64}


def require_cuda() -> None:
    if not torch.cuda.is_available():
        raise RuntimeError("paper_1803_10986_b200 runs on a CUDA device (B200, sm_100a); "
                           "no CUDA device is visible and there is no CPU fallback")
    _native.lib()


def stream_handle() -> int:
    return torch.cuda.current_stream().cuda_stream


def to_device(a, np_dtype) -> tuple:
    """(contiguous CUDA tensor of np_dtype, came_from_host).  Casting follows
    numpy's astype (round to nearest even)."""
    require_cuda()
    tdt = _DT[np_dtype]
    if isinstance(a, torch.Tensor):
        t = a if a.is_cuda else a.to("cuda", non_blocking=False)
        return t.to(tdt).contiguous(), not a.is_cuda
    arr = np.asarray(a)
    if arr.dtype == object:
        arr = arr.astype(np.float64)
    if arr.dtype.kind not in "fiub":
        raise ValueError(f"unsupported input dtype {arr.dtype}")
    t = torch.from_numpy(np.ascontiguousarray(arr))
    return t.to("cuda").to(tdt).contiguous(), True


def shape_of(a) -> tuple:
    if isinstance(a, torch.Tensor):
        return tuple(a.shape)
    return np.shape(a)


def empty(shape, np_dtype):
    return torch.empty(tuple(shape), dtype=_DT[np_dtype], device="cuda")


def finish(t, host: bool):
    """Return a numpy array for host callers, the device tensor otherwise."""
    if host:
        return t.cpu().numpy()
    return t


def ptr(t):
    return _native.as_ptr(t)
