"""Elevation transforms on the GPU (kernels K6): signed sqrt/square, box mean,
Laplacian encode / decode / stabilize.

API-compatible with infigrid/transforms.py.  Each function accepts a numpy
array (reference contract: numpy in, numpy out, via one upload/download) or
a CUDA ``torch.Tensor`` (stays on the device).  The Laplacian split keeps the
reference's float64 arithmetic (transforms.py:89-114): the residual must be
float64 for decode(encode(x)) == x to hold bit-exactly.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _device as dev
from ._native import DTYPE_F32, DTYPE_F64, call
from .errors import ShapeError


def _to_dev(x):
    if isinstance(x, torch.Tensor):
        return x.contiguous(), True
    arr = np.asarray(x)
    if arr.dtype not in (np.float32, np.float64):
        arr = arr.astype(np.float64)
    return dev.upload(arr), False


def _ret(t, was_dev):
    return t if was_dev else dev.download(t)


def _dt(t: torch.Tensor) -> int:
    if t.dtype == torch.float32:
        return DTYPE_F32
    if t.dtype == torch.float64:
        return DTYPE_F64
    raise ShapeError(f"unsupported dtype {t.dtype}")


def signed_sqrt(x):
    """sign(x) * sqrt(|x|)  (transforms.py:17-20)."""
    t, d = _to_dev(x)
    out = torch.empty_like(t)
    call("ig_signed_pow", t.data_ptr(), t.numel(), 0, _dt(t), out.data_ptr(), dev.stream_ptr())
    return _ret(out, d)


def signed_square(x):
    """sign(x) * x * x  (transforms.py:23-26)."""
    t, d = _to_dev(x)
    out = torch.empty_like(t)
    call("ig_signed_pow", t.data_ptr(), t.numel(), 1, _dt(t), out.data_ptr(), dev.stream_ptr())
    return _ret(out, d)


def _planes(t: torch.Tensor):
    if t.dim() < 2:
        raise ShapeError("need at least two (spatial) axes")
    h, w = t.shape[-2], t.shape[-1]
    return max(1, t.numel() // max(h * w, 1)), h, w


def box_mean(x, radius: int):
    """Separable (2r+1)^2 mean with edge clamp, rows then columns (transforms.py:29-51)."""
    if radius < 0:
        raise ValueError("radius must be >= 0")
    t, d = _to_dev(x)
    out = torch.empty_like(t)
    p, h, w = _planes(t)
    call("ig_box_mean", t.data_ptr(), p, h, w, radius, _dt(t), out.data_ptr(), dev.stream_ptr())
    return _ret(out, d)


def blur3_iterated(x, radius: int):
    """`radius` passes of the 3x3 box mean (transforms.py:54-58)."""
    for _ in range(radius):
        x = box_mean(x, 1)
    return x


def _blur_block_mean(t: torch.Tensor, blur_iters: int, factor: int) -> torch.Tensor:
    p, h, w = _planes(t)
    if h % factor or w % factor:
        raise ShapeError(f"spatial dims {h}x{w} not divisible by factor {factor}")
    low = torch.empty(t.shape[:-2] + (h // factor, w // factor), dtype=torch.float64,
                      device=t.device)
    scratch = torch.empty(2 * t.numel(), dtype=torch.float64, device=t.device)
    call("ig_blur_block_mean_f64", t.data_ptr(), _dt(t), p, h, w, blur_iters, factor,
         scratch.data_ptr(), low.data_ptr(), dev.stream_ptr())
    return low


def block_mean(x, factor: int):
    """factor x factor block average in float64 (transforms.py:61-67)."""
    t, d = _to_dev(x)
    if t.dtype != torch.float64:
        raise ShapeError("block_mean on the device is defined for float64 input "
                         "(the Laplacian path); widen the input first")
    return _ret(_blur_block_mean(t, 0, factor), d)


def upsample_nn(x, factor: int):
    """Nearest-neighbour replication on the last two axes (transforms.py:70-72)."""
    if isinstance(x, torch.Tensor):
        return x.repeat_interleave(factor, dim=-2).repeat_interleave(factor, dim=-1)
    return np.repeat(np.repeat(x, factor, axis=-2), factor, axis=-1)


@dataclass
class LaplacianPair:
    """float64 low band at 1/factor resolution plus the exact float64 residual."""

    low: object
    high: object
    factor: int
    dtype: np.dtype


def laplacian_encode(x, factor: int = 8, blur_radius: int = 1) -> LaplacianPair:
    """low = block_mean(blur(x64)), high = x64 - up(low)  (transforms.py:89-95)."""
    t, d = _to_dev(x)
    src_dtype = np.dtype(np.float32) if t.dtype == torch.float32 else np.dtype(np.float64)
    low = _blur_block_mean(t, blur_radius, factor)
    high = torch.empty(t.shape, dtype=torch.float64, device=t.device)
    p, h, w = _planes(t)
    call("ig_laplacian_residual", t.data_ptr(), _dt(t), low.data_ptr(), p, h, w, factor,
         high.data_ptr(), dev.stream_ptr())
    if not d:
        return LaplacianPair(dev.download(low), dev.download(high), factor, src_dtype)
    return LaplacianPair(low, high, factor, src_dtype)


def _merge(pair: LaplacianPair, out_dtype, square: bool):
    low, d = _to_dev(pair.low)
    high, _ = _to_dev(pair.high)
    low = low.to(torch.float64)
    high = high.to(torch.float64)
    p, h, w = _planes(high)
    tdt = dev.torch_dtype(out_dtype)
    out = torch.empty(high.shape, dtype=tdt, device=high.device)
    call("ig_laplacian_merge", low.data_ptr(), high.data_ptr(), p, h, w, pair.factor,
         _dt(out), int(square), out.data_ptr(), dev.stream_ptr())
    return out, d


def laplacian_decode(pair: LaplacianPair):
    """up(low) + high in float64, cast to the original dtype (transforms.py:98-101)."""
    out, d = _merge(pair, pair.dtype, False)
    return _ret(out, d)


def laplacian_decode_signed_square(pair: LaplacianPair):
    """signed_square(laplacian_decode(pair)) fused in one pass (elevation output)."""
    out, d = _merge(pair, pair.dtype, True)
    return _ret(out, d)


def laplacian_stabilize(pair: LaplacianPair, blur_radius: int = 1) -> LaplacianPair:
    """Re-extract the low band from the provisional decode (transforms.py:104-114)."""
    prov, d = _merge(pair, np.float64, False)
    low_hat = _blur_block_mean(prov, blur_radius, pair.factor)
    if not d:
        return LaplacianPair(dev.download(low_hat), pair.high, pair.factor, pair.dtype)
    return LaplacianPair(low_hat, pair.high, pair.factor, pair.dtype)


def normalize_heightmap_u8(batch) -> np.ndarray:
    """Algorithm 2 render normalisation (transforms.py:117-135).

    Out of the throughput path; evaluated on the host.
    """
    b = np.asarray(batch.detach().cpu().numpy() if isinstance(batch, torch.Tensor) else batch,
                   dtype=np.float64)
    if b.ndim == 3:
        b = b[:, None]
    if b.ndim != 4 or b.shape[1] != 1:
        raise ShapeError(f"expected (B, 1, H, W) or (B, H, W), got {b.shape}")
    lo = b.min(axis=(-2, -1), keepdims=True)
    hi = b.max(axis=(-2, -1), keepdims=True)
    span = np.maximum(hi - lo, 255.0)
    centre = (lo + hi) / 2.0
    scaled = np.clip(((b - centre) / span + 0.5) * 255.0, 0.0, 255.0)
    return np.repeat(np.rint(scaled).astype(np.uint8), 3, axis=1)
