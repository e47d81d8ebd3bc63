"""Dense finite-canvas evaluation of the fused trajectory, on the device.

The reference ships these as its verification oracle (`infigrid.oracle`,
oracle.py:23-116): every step's image over a finite canvas evaluated directly
from its defining weighted sum, with float64 accumulation.  The CLI's
``verify oracle`` mode (cli.py:379-394) compares the lazy store against it.

Here the same definition runs through the product kernels in float64 --
noise (K1) widened to f64, the batched analytic Phi (K3) on the f64 canvas,
and the weighted canonical-order blend (K5) with the f64 weight table and the
B > 0 division -- orchestrated densely (union covers, outermost first)
instead of through the window cache.  The per-pixel operation sequence is the
reference's: num += fl(w64 * phi) over windows in (j, i) order, den += w64,
out = num / den where den > 0, else 0.

This is an API mirror for the CLI, not the test oracle (that is oracle/,
which the package never imports).
"""

from __future__ import annotations

import numpy as np
import torch

from . import _device as dev
from ._native import call
from .denoise import DenoiserSpec, apply, apply_batch
from .grid import (Region, WindowIndex, WindowLayout, index_box, region_union_cover,
                   window_region, windows_overlapping)
from .noise import NoiseStream, noise_region_device


class CropError(AssertionError, ValueError):
    """A crop outside the canvas (the reference asserts, oracle.py:30)."""


class DenseCanvas:
    """A finite multi-channel tensor with explicit lattice bounds (oracle.py:23-32).

    ``data`` is the float64 (C, H, W) numpy array, as in the reference; the
    device copy the dense steps compute on is ``device()``.  Either side is
    materialised on first use, once."""

    def __init__(self, region: Region, data):
        self.region = region
        if isinstance(data, torch.Tensor):
            self._dev, self._host = data, None
        else:
            self._dev, self._host = None, np.asarray(data, dtype=np.float64)

    @property
    def data(self) -> np.ndarray:
        if self._host is None:
            self._host = dev.download(self._dev)
        return self._host

    def device(self) -> torch.Tensor:
        if self._dev is None:
            self._dev = dev.upload(np.ascontiguousarray(self._host))
        return self._dev

    def crop(self, r: Region) -> np.ndarray:
        if not self.region.contains(r):
            raise CropError(f"{r} outside canvas {self.region}")
        ys = slice(r.y0 - self.region.y0, r.y1 - self.region.y0)
        xs = slice(r.x0 - self.region.x0, r.x1 - self.region.x0)
        if self._host is not None:
            return self._host[:, ys, xs].copy()
        return dev.download(self._dev[:, ys, xs])


def dense_fusion_step(canvas: DenseCanvas, target: Region, layout: WindowLayout,
                      weights: np.ndarray, spec: DenoiserSpec, t: int,
                      conditioning=None) -> DenseCanvas:
    """One fusion step over ``target`` from its defining weighted sum
    (oracle.py:35-68): Phi of every window overlapping target on the canvas,
    weighted average in canonical window order, float64."""
    c = int(canvas.device().shape[0])
    win = layout.window
    idxs = windows_overlapping(layout, target)
    i_lo, i_hi, j_lo, j_hi = index_box(layout, target)
    ni, nj = i_hi - i_lo + 1, j_hi - j_lo + 1
    src = canvas.device().to(torch.float64).contiguous()
    if conditioning is None and spec.kind != "unet":
        ij = np.asarray(idxs, dtype=np.int64).reshape(-1, 2)
        wxy = dev.upload(ij * layout.stride + np.asarray(layout.offset, dtype=np.int64))
        for idx in idxs:
            if not canvas.region.contains(window_region(layout, idx)):
                raise ValueError(f"window {idx} outside canvas {canvas.region}")
        phi = apply_batch(spec, src, canvas.region, wxy, win, t).contiguous()
    else:
        wins = []
        for idx in idxs:
            r = window_region(layout, idx)
            x = src[:, r.y0 - canvas.region.y0:r.y1 - canvas.region.y0,
                    r.x0 - canvas.region.x0:r.x1 - canvas.region.x0].contiguous()
            if spec.kind == "unet":
                from .unet import unet_phi_batch
                wxy1 = dev.upload_i64([[r.x0, r.y0]])
                y = unet_phi_batch(spec.unet, x.to(torch.float32)[None], None, wxy1, win, t,
                                   None)[0].to(torch.float64)
            else:
                y = apply(spec, x, conditioning(idx) if conditioning is not None else None, t)
            wins.append(y.to(torch.float64))
        phi = torch.stack(wins).contiguous()
    table = np.zeros(ni * nj, dtype=np.int64)
    nbytes = c * win * win * 8
    for k, (i, j) in enumerate(idxs):
        table[(j - j_lo) * ni + (i - i_lo)] = phi.data_ptr() + k * nbytes
    ptrs = dev.upload(table)
    w64 = dev.upload(np.ascontiguousarray(np.asarray(weights, dtype=np.float64)))
    out = torch.empty((c, target.height, target.width), dtype=torch.float64,
                      device=dev.device())
    ox, oy = layout.offset
    call("ig_blend", ptrs.data_ptr(), i_lo, j_lo, ni, nj, win, layout.stride, ox, oy, c, 1,
         w64.data_ptr(), target.x0, target.y0, target.width, target.height, 1,
         dev.ig_dtype(torch.float64), out.data_ptr(), dev.stream_ptr())
    torch.cuda.current_stream().synchronize()   # phi / ptrs / w64 die here
    return DenseCanvas(region=target, data=out)


def dense_trajectory(seed: int, steps: int, layout: WindowLayout, weights: np.ndarray,
                     spec: DenoiserSpec, target: Region,
                     channels: int = 1) -> dict[int, DenseCanvas]:
    """Every step's image over ``target`` (oracle.py:71-92): canvases shrink
    outward-in from the noise level T to the requested region."""
    regions = {0: target}
    for t in range(1, steps + 1):
        regions[t] = region_union_cover(layout, regions[t - 1])
    noise = noise_region_device(NoiseStream(seed), regions[steps], channels).to(torch.float64)
    out = {steps: DenseCanvas(regions[steps], noise)}
    for t in range(steps - 1, -1, -1):
        out[t] = dense_fusion_step(out[t + 1], regions[t], layout, weights, spec, t + 1)
    return out


def brute_force_windows(layout: WindowLayout, r: Region,
                        search_radius: int) -> set[WindowIndex]:
    """Windows intersecting r by exhaustive scan of |i|, |j| <= search_radius
    (oracle.py:95-102) -- integer host logic."""
    found = set()
    for j in range(-search_radius, search_radius + 1):
        for i in range(-search_radius, search_radius + 1):
            if window_region(layout, (i, j)).intersection(r) is not None:
                found.add((i, j))
    return found


def count_denoiser_calls_naive(steps: int, layout: WindowLayout, r: Region) -> int:
    """Uncached recursion-tree count of Phi calls (oracle.py:105-116)."""

    def cost(t: int, region: Region) -> int:
        if t == steps:
            return 0
        total = 0
        for idx in windows_overlapping(layout, region):
            total += 1 + cost(t + 1, window_region(layout, idx))
        return total

    return cost(0, r)
