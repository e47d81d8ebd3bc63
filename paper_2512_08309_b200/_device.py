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


class _Staging:
    """A small ring of grow-only pinned host buffers for host->device copies.
    Pinning a fresh buffer per upload (tensor.pin_memory()) cost ~2.6 ms per
    call on the analytic-Phi step; a slot is reused once the copy that last
    read it has executed (its event)."""

    SLOTS = 8

    def __init__(self):
        self.bufs = [None] * self.SLOTS
        self.events = [None] * self.SLOTS
        self.i = 0

    def upload(self, a: np.ndarray) -> torch.Tensor:
        nbytes = a.nbytes
        k = self.i
        self.i = (self.i + 1) % self.SLOTS
        buf = self.bufs[k]
        if buf is None or buf.numel() < nbytes:
            buf = self.bufs[k] = torch.empty(max(nbytes, 1 << 16), dtype=torch.uint8,
                                             pin_memory=True)
            self.events[k] = None
        if self.events[k] is not None:
            self.events[k].synchronize()
        host = buf[:nbytes]
        host.numpy()[:] = a.reshape(-1).view(np.uint8)
        out = torch.empty(a.shape, dtype=torch.from_numpy(np.empty(0, a.dtype)).dtype,
                          device=device())
        out.view(-1).view(torch.uint8).copy_(host, non_blocking=True)
        ev = torch.cuda.Event()
        ev.record()
        self.events[k] = ev
        return out


_staging = None


def upload(arr: np.ndarray) -> torch.Tensor:
    """Host array -> device tensor via pinned staging (async on the current stream)."""
    global _staging
    a = np.ascontiguousarray(arr)
    traffic["h2d"] += a.nbytes
    if a.nbytes == 0:
        return torch.from_numpy(a.copy()).to(device())
    if _staging is None:
        _staging = _Staging()
    return _staging.upload(a)


_reserved = 0


def reserve(nbytes: int):
    """Grow the CUDA caching allocator to `nbytes` once (allocate + free): a
    bounded window cache then fills from cached segments instead of calling
    cudaMalloc in the middle of a query (a new segment stalled a cfg4 query by
    ~45 ms, tools/cfg4_tail.py).  The memory stays with torch's allocator."""
    global _reserved
    device()
    free, _ = torch.cuda.mem_get_info()
    nbytes = min(int(nbytes), int(0.8 * (free + torch.cuda.memory_reserved())))
    if nbytes <= _reserved:
        return
    t = torch.empty(nbytes, dtype=torch.uint8, device=device())
    del t
    _reserved = nbytes


def upload_i64(values) -> torch.Tensor:
    return upload(np.asarray(values, dtype=np.int64))


def download(t: torch.Tensor) -> np.ndarray:
    """Device tensor -> numpy.  Large results land in a pinned block of torch's
    caching host allocator (direct DMA instead of the driver's pageable staging
    path); the returned array is a view that keeps the block alive, and the block
    goes back to the cache when the caller drops it."""
    nbytes = t.numel() * t.element_size()
    traffic["d2h"] += nbytes
    t = t.detach()
    if t.is_cuda and nbytes >= (1 << 20):
        host = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
        host.copy_(t)
        return host.numpy()
    return t.to("cpu").numpy()


def ptr(t) -> int:
    return 0 if t is None else t.data_ptr()
