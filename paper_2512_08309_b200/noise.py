"""Coordinate-keyed Gaussian noise, evaluated on the GPU (kernel K1).

API-compatible with infigrid/noise.py.  The field value at (seed, stream, x,
y, channel) is the reference's SplitMix64-absorb + Box-Muller construction
(noise.py:39-64), rounded to float32; ``csrc/ig_noise.cuh`` documents how the
device reproduces the float64 libm results bit-exactly.
"""

from __future__ import annotations

from typing import NamedTuple

import numpy as np
import torch

from . import _device as dev
from ._native import DTYPE_F32, call
from .grid import Region

STREAM_BASE = 0            # initial noise of the sampler recursion (noise.py:27)
STREAM_CONDITIONING = 101  # conditioning hole fill (noise.py:28)
STREAM_CORRUPTION = 201    # user-map corruption, + channel (noise.py:29)
STREAM_PROCEDURAL = 7      # ProceduralMap lattice (pipeline.py:94)
STREAM_RENOISE = 301       # consistency-step renoise of the UNet Phi (+ outer step); new

_U64 = (1 << 64) - 1
_U32 = (1 << 32) - 1


class NoiseStream(NamedTuple):
    """(seed, stream id) naming one independent field (noise.py:32-36)."""

    seed: int
    stream: int = STREAM_BASE


def noise_region_device(stream: NoiseStream, r: Region, channels: int = 1,
                        dtype=np.float32, out: torch.Tensor | None = None,
                        ch0: int = 0) -> torch.Tensor:
    """Device (channels, h, w) block; entry (c, py, px) = G(x0+px, y0+py, ch0+c)."""
    tdt = dev.torch_dtype(dtype)
    if out is None:
        out = torch.empty((channels, r.height, r.width), dtype=tdt, device=dev.device())
    call("ig_noise_region", stream.seed & _U64, stream.stream & _U32, r.x0, r.y0, r.width,
         r.height, ch0, channels, dev.ig_dtype(tdt), out.data_ptr(), None, dev.stream_ptr())
    return out


def noise_region(stream: NoiseStream, r: Region, channels: int = 1) -> np.ndarray:
    """Dense float32 (channels, height, width) block (noise.py:74-86)."""
    return dev.download(noise_region_device(stream, r, channels))


def noise_at(stream: NoiseStream, x: int, y: int, channel: int = 0) -> float:
    """Single deviate (noise.py:67-71)."""
    out = torch.empty((1, 1, 1), dtype=torch.float32, device=dev.device())
    call("ig_noise_region", stream.seed & _U64, stream.stream & _U32, x, y, 1, 1, channel, 1,
         DTYPE_F32, out.data_ptr(), None, dev.stream_ptr())
    return float(out.item())
