"""Elevation transforms on the GPU (kernels K6): signed sqrt/square, box mean,
Laplacian encode / decode / stabilize.

API-compatible with infigrid/transforms.py.  Each function accepts a numpy
array (reference contract: numpy in, numpy out, via one upload/download) or
a CUDA ``torch.Tensor`` (stays on the device).  The Laplacian split keeps the
reference's float64 arithmetic (transforms.py:89-114): the residual must be
float64 for decode(encode(x)) == x to hold bit-exactly.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _device as dev
from ._native import DTYPE_F16, DTYPE_F32, DTYPE_F64, DTYPE_I32, DTYPE_I64, call
from .errors import ShapeError


_TORCH_OF = {np.dtype(np.float32): torch.float32, np.dtype(np.float64): torch.float64,
             np.dtype(np.float16): torch.float16, np.dtype(np.int32): torch.int32,
             np.dtype(np.int64): torch.int64}
_NP_OF = {v: k for k, v in _TORCH_OF.items()}
_CODE_OF = {torch.float32: DTYPE_F32, torch.float64: DTYPE_F64, torch.float16: DTYPE_F16,
            torch.int32: DTYPE_I32, torch.int64: DTYPE_I64}


def _to_dev(x):
    """(device tensor, numpy dtype of the caller's array, input was a tensor).

    float16/32/64 and int32/int64 arrays travel as they are; other integer and
    bool arrays are widened to int64 for the upload (lossless) and results are
    cast back to the caller's dtype where numpy would keep it."""
    if isinstance(x, torch.Tensor):
        t = x.contiguous()
        if t.dtype not in _CODE_OF:
            raise ShapeError(f"unsupported tensor dtype {t.dtype}")
        return t, _NP_OF[t.dtype], True
    arr = np.asarray(x)
    kind = arr.dtype.kind
    if arr.dtype in _TORCH_OF:
        return dev.upload(arr), arr.dtype, False
    if kind in "iub":
        return dev.upload(arr.astype(np.int64)), arr.dtype, False
    raise ShapeError(f"unsupported dtype {arr.dtype}")


def _ret(t, was_dev, want=None):
    """Device result -> the caller's side; `want` = numpy dtype the reference's
    expression yields when it differs from the device tensor's (narrow ints)."""
    if was_dev:
        return t
    out = dev.download(t)
    return out if want is None or out.dtype == want else out.astype(want)


def _code(t: torch.Tensor) -> int:
    return _CODE_OF[t.dtype]


def _dt(t: torch.Tensor) -> int:
    if t.dtype == torch.float32:
        return DTYPE_F32
    if t.dtype == torch.float64:
        return DTYPE_F64
    raise ShapeError(f"unsupported dtype {t.dtype}")


def _convert(t: torch.Tensor, to: torch.dtype) -> torch.Tensor:
    """astype on the device (exact widenings, RN narrowings; ig_convert)."""
    if t.dtype == to:
        return t
    out = torch.empty(t.shape, dtype=to, device=t.device)
    call("ig_convert", t.data_ptr(), _code(t), t.numel(), out.data_ptr(), _CODE_OF[to],
         dev.stream_ptr())
    return out


def _float_work(t: torch.Tensor) -> torch.Tensor:
    """The float tensor an elementwise numpy expression computes in: float32/64
    as is, float16 exactly widened to float32 (rounded back at the end),
    integers exactly widened to float64 (numpy's int -> float64 promotion)."""
    if t.dtype in (torch.float32, torch.float64):
        return t
    return _convert(t, torch.float32 if t.dtype == torch.float16 else torch.float64)


def signed_sqrt(x):
    """sign(x) * sqrt(|x|)  (transforms.py:17-20); integers give float64."""
    t, src, d = _to_dev(x)
    w = _float_work(t)
    out = torch.empty_like(w)
    call("ig_signed_pow", w.data_ptr(), w.numel(), 0, _dt(w), out.data_ptr(), dev.stream_ptr())
    if t.dtype == torch.float16:
        out = _convert(out, torch.float16)
    return _ret(out, d)


def signed_square(x):
    """sign(x) * x * x  (transforms.py:23-26), in the input's dtype (integers
    wrap like numpy's integer multiply)."""
    t, src, d = _to_dev(x)
    if t.dtype in (torch.int32, torch.int64):
        out = torch.empty_like(t)
        call("ig_signed_pow", t.data_ptr(), t.numel(), 1, _code(t), out.data_ptr(),
             dev.stream_ptr())
        return _ret(out, d, src)
    w = _float_work(t)
    out = torch.empty_like(w)
    call("ig_signed_pow", w.data_ptr(), w.numel(), 1, _dt(w), out.data_ptr(), dev.stream_ptr())
    if t.dtype == torch.float16:
        out = _convert(out, torch.float16)
    return _ret(out, d)


def _planes(t: torch.Tensor):
    if t.dim() < 2:
        raise ShapeError("need at least two (spatial) axes")
    h, w = t.shape[-2], t.shape[-1]
    return max(1, t.numel() // max(h * w, 1)), h, w


def box_mean(x, radius: int):
    """Separable (2r+1)^2 mean with edge clamp, rows then columns (transforms.py:29-51).

    Integer input: the reference sums in the integer dtype (exact) and divides
    into float64, which is the float64 kernel on the exactly widened input."""
    if radius < 0:
        raise ValueError("radius must be >= 0")
    t, src, d = _to_dev(x)
    if radius == 0:
        return _ret(t.clone(), d, src)
    if t.dtype == torch.float16:
        raise ShapeError("box_mean of float16 input is not supported on the device "
                         "(numpy rounds every partial sum to float16)")
    t = _float_work(t)
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
    """float64 low band of blur3_iterated(widen(t)) (f32/f64 sources read directly)."""
    if t.dtype not in (torch.float32, torch.float64):
        t = _convert(t, torch.float64)
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
    """factor x factor block average (transforms.py:61-67) with numpy .mean's
    dtype rules: float32 accumulates in float32, float16 in float32 and rounds
    back, integers (and bool) in float64."""
    t, src, d = _to_dev(x)
    p, h, w = _planes(t)
    if h % factor or w % factor:
        raise ShapeError(f"spatial dims {h}x{w} not divisible by factor {factor}")
    acc = torch.float32 if t.dtype in (torch.float32, torch.float16) else torch.float64
    tw = _convert(t, acc)
    low = torch.empty(t.shape[:-2] + (h // factor, w // factor), dtype=acc, device=t.device)
    call("ig_block_mean", tw.data_ptr(), _dt(tw), p, h, w, factor, low.data_ptr(),
         dev.stream_ptr())
    if t.dtype == torch.float16:
        low = _convert(low, torch.float16)
    return _ret(low, d)


def upsample_nn(x, factor: int):
    """Nearest-neighbour replication on the last two axes (transforms.py:70-72)."""
    if factor < 1:
        raise ValueError("factor must be >= 1")
    t, src, d = _to_dev(x)
    if t.dim() < 2:
        raise ShapeError("need at least two (spatial) axes")
    p, h, w = _planes(t)
    out = torch.empty(t.shape[:-2] + (h * factor, w * factor), dtype=t.dtype, device=t.device)
    call("ig_upsample_nn", t.data_ptr(), t.element_size(), p, h, w, factor, out.data_ptr(),
         dev.stream_ptr())
    return _ret(out, d, src)


@dataclass
class LaplacianPair:
    """float64 low band at 1/factor resolution plus the exact float64 residual;
    `dtype` is the encoded input's dtype, restored by laplacian_decode."""

    low: object
    high: object
    factor: int
    dtype: np.dtype


def laplacian_encode(x, factor: int = 8, blur_radius: int = 1) -> LaplacianPair:
    """low = block_mean(blur(x64)), high = x64 - up(low)  (transforms.py:89-95)."""
    t, src, d = _to_dev(x)
    if t.dtype not in (torch.float32, torch.float64):
        t = _convert(t, torch.float64)        # x.astype(np.float64), exact
    low = _blur_block_mean(t, blur_radius, factor)
    high = torch.empty(t.shape, dtype=torch.float64, device=t.device)
    p, h, w = _planes(t)
    call("ig_laplacian_residual", t.data_ptr(), _dt(t), low.data_ptr(), p, h, w, factor,
         high.data_ptr(), dev.stream_ptr())
    if not d:
        return LaplacianPair(dev.download(low), dev.download(high), factor, src)
    return LaplacianPair(low, high, factor, src)


def _merge(pair: LaplacianPair, out_dtype, square: bool):
    low, _, d = _to_dev(pair.low)
    high, _, _ = _to_dev(pair.high)
    low = _convert(low, torch.float64)
    high = _convert(high, torch.float64)
    p, h, w = _planes(high)
    want = _NP_OF[out_dtype] if isinstance(out_dtype, torch.dtype) else np.dtype(out_dtype)
    tdt = _TORCH_OF.get(want, torch.int64 if want.kind in "iub" else None)
    if tdt is None:
        raise ShapeError(f"unsupported decode dtype {want}")
    out = torch.empty(high.shape, dtype=tdt, device=high.device)
    call("ig_laplacian_merge", low.data_ptr(), high.data_ptr(), p, h, w, pair.factor,
         _CODE_OF[tdt], int(square), out.data_ptr(), dev.stream_ptr())
    return out, d, want


def laplacian_decode(pair: LaplacianPair):
    """up(low) + high in float64, cast to the original dtype (transforms.py:98-101)."""
    out, d, want = _merge(pair, pair.dtype, False)
    return _ret(out, d, want)


def laplacian_decode_signed_square(pair: LaplacianPair):
    """signed_square(laplacian_decode(pair)) fused in one pass (elevation output)."""
    out, d, want = _merge(pair, pair.dtype, True)
    return _ret(out, d, want)


def laplacian_stabilize(pair: LaplacianPair, blur_radius: int = 1) -> LaplacianPair:
    """Re-extract the low band from the provisional decode (transforms.py:104-114)."""
    prov, d, _ = _merge(pair, np.float64, False)
    low_hat = _blur_block_mean(prov, blur_radius, pair.factor)
    if not d:
        return LaplacianPair(dev.download(low_hat), pair.high, pair.factor, pair.dtype)
    return LaplacianPair(low_hat, pair.high, pair.factor, pair.dtype)


def hillshade_u8(elev, azimuth_deg: float = 315.0, altitude_deg: float = 45.0):
    """Horn 3x3 slope shading to uint8 on the device (reference cli.py:230-249):
    float64 arithmetic in the reference's operation order; the light's
    cos / sin are evaluated on the host with numpy, as the reference does.
    numpy in -> numpy out; a CUDA tensor stays on the device."""
    was_dev = isinstance(elev, torch.Tensor)
    if was_dev:
        t = elev.contiguous()
        if t.dtype not in (torch.float32, torch.float64):
            t = _convert(t, torch.float64)
    else:
        arr = np.asarray(elev)
        if arr.dtype not in (np.float32, np.float64):
            arr = arr.astype(np.float64)
        t = dev.upload(np.ascontiguousarray(arr))
    if t.dim() != 2:
        raise ShapeError(f"hillshade expects a 2-D raster, got {tuple(t.shape)}")
    zen = math.radians(90.0 - altitude_deg)
    azi = math.radians(360.0 - azimuth_deg + 90.0)
    h, w = t.shape
    out = torch.empty((h, w), dtype=torch.uint8, device=t.device)
    call("ig_hillshade_u8", t.data_ptr(), _dt(t), h, w, float(np.cos(zen)), float(np.sin(zen)),
         azi, out.data_ptr(), dev.stream_ptr())
    return out if was_dev else dev.download(out)


def normalize_heightmap_u8(batch):
    """Algorithm 2 render normalisation (transforms.py:117-135) on the device:
    per image, centre on (min + max) / 2, scale by max(range, 255), shift to
    [0, 255], round half to even, clamp, replicate to 3 channels (uint8).
    Every step is an IEEE float64 operation, so the bytes equal numpy's.
    numpy in -> numpy out; a CUDA tensor stays on the device."""
    was_dev = isinstance(batch, torch.Tensor)
    if was_dev:
        t = batch.contiguous()
        if t.dtype not in (torch.float32, torch.float64):
            t = _convert(t, torch.float64)
    else:
        arr = np.asarray(batch)
        if arr.dtype not in (np.float32, np.float64):
            arr = arr.astype(np.float64)         # numpy's float64 view of the input
        t = dev.upload(np.ascontiguousarray(arr))
    if t.dim() == 3:
        t = t[:, None]
    if t.dim() != 4 or t.shape[1] != 1:
        raise ShapeError(f"expected (B, 1, H, W) or (B, H, W), got {tuple(t.shape)}")
    b, _, h, w = t.shape
    out = torch.empty((b, 3, h, w), dtype=torch.uint8, device=t.device)
    mm = torch.empty(2 * max(b, 1), dtype=torch.int64, device=t.device)
    call("ig_normalize_u8", t.data_ptr(), _dt(t), b, h * w, mm.data_ptr(), out.data_ptr(),
         dev.stream_ptr())
    return out if was_dev else dev.download(out)
