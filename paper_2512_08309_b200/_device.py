"""Device plumbing: the CUDA device/stream the package computes on, and small
host<->device helpers.  PyTorch is used only for memory and streams."""

from __future__ import annotations

import numpy as np
import torch

_device = None

# host<->device traffic issued through upload()/download() (bench e2e accounting)
traffic = {"h2d": 0, "d2h": 0}


def device() -> torch.device:
    global _device
    if _device is None:
        if not torch.cuda.is_available():
            raise RuntimeError("paper_2512_08309_b200 computes on a CUDA device (sm_100a); "
                               "none is visible and there is no CPU fallback")
        _device = torch.device("cuda", torch.cuda.current_device())
    return _device


def set_device(index: int):
    global _device
    torch.cuda.set_device(index)
    _device = torch.device("cuda", index)


def stream_ptr() -> int:
    return torch.cuda.current_stream(device()).cuda_stream


def torch_dtype(dtype) -> torch.dtype:
    if isinstance(dtype, torch.dtype):
        if dtype in (torch.float32, torch.float64):
            return dtype
        raise ValueError(f"unsupported dtype {dtype} (float32 or float64)")
    dt = np.dtype(dtype)
    if dt == np.float32:
        return torch.float32
    if dt == np.float64:
        return torch.float64
    raise ValueError(f"unsupported dtype {dt} (float32 or float64)")


def ig_dtype(dtype) -> int:
    dt = np.dtype(dtype) if not isinstance(dtype, torch.dtype) else (
        np.float32 if dtype == torch.float32 else np.float64)
    return 0 if np.dtype(dt) == np.float32 else 1


def empty(shape, dtype) -> torch.Tensor:
    return torch.empty(shape, dtype=torch_dtype(dtype) if not isinstance(dtype, torch.dtype)
                       else dtype, device=device())


def upload(arr: np.ndarray) -> torch.Tensor:
    """Host array -> device tensor via pinned staging (async on the current stream)."""
    a = np.ascontiguousarray(arr)
    if not a.flags.writeable:
        a = a.copy()
    t = torch.from_numpy(a)
    traffic["h2d"] += t.numel() * t.element_size()
    if t.numel() * t.element_size() >= 1 << 16:
        t = t.pin_memory()
    return t.to(device(), non_blocking=True)


def upload_i64(values) -> torch.Tensor:
    return upload(np.asarray(values, dtype=np.int64))


def download(t: torch.Tensor) -> np.ndarray:
    traffic["d2h"] += t.numel() * t.element_size()
    return t.detach().to("cpu").numpy()


def ptr(t) -> int:
    return 0 if t is None else t.data_ptr()
