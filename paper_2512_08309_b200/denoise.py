"""The Phi plugin boundary and per-window conditioning, on the GPU.

API-compatible with infigrid/denoise.py (KINDS, Conditioning, DenoiserSpec,
apply, conditioning_for_window, coarse_patch_features) plus one new kind,
``"unet"``: the consistency-distilled UNet Phi the north star names (no
reference implementation exists; see unet.py and DESIGN.md).

`apply` keeps the reference's single-window calling contract
(denoise.py:89-113).  The sampler does not call it per window: it hands whole
batches of windows to :func:`apply_batch`, which launches one kernel (analytic
kinds) or one UNet forward per batch.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _device as dev
from ._native import PHI_COND_AFFINE, PHI_IDENTITY, PHI_SHRINK_SMOOTH, call
from .errors import CoverageError, ShapeError
from .grid import Region, WindowIndex, WindowLayout, window_region
from .noise import STREAM_CONDITIONING  # noqa: F401  (re-exported as in denoise.py:19)

KINDS = ("identity", "shrink_smooth", "cond_affine", "multistep", "unet")
_KIND_CODE = {"identity": PHI_IDENTITY, "shrink_smooth": PHI_SHRINK_SMOOTH,
              "cond_affine": PHI_COND_AFFINE}


@dataclass(frozen=True)
class Conditioning:
    """Window-resolution conditioning: channels, side scalars, 0/1 mask (denoise.py:25-36)."""

    channels: object
    scalars: tuple[float, ...] = ()
    mask: object = None


@dataclass(frozen=True)
class DenoiserSpec:
    """One Phi configuration (denoise.py:39-72); ``unet`` carries a UNetConfig."""

    kind: str = "shrink_smooth"
    radius: int = 1
    lambdas: tuple[float, ...] = (0.5,)
    inner_kind: str = "shrink_smooth"
    inner_steps: int = 1
    lambda_start: float = 0.9
    lambda_end: float = 0.1
    channels: int = 1
    unet: object = None

    def __post_init__(self):
        if self.kind not in KINDS:
            raise ValueError(f"unknown denoiser kind {self.kind!r}")
        if self.kind == "multistep" and self.inner_kind not in ("shrink_smooth", "cond_affine"):
            raise ValueError("multistep inner kind must be shrink_smooth or cond_affine")
        if self.kind == "unet" and self.unet is None:
            raise ValueError("kind 'unet' needs a UNetConfig in `unet`")

    def lambda_for(self, t: int) -> float:
        """Shrink factor of outer step t (1-based); the last entry repeats."""
        if not self.lambdas:
            return 0.5
        return self.lambdas[min(t, len(self.lambdas)) - 1]

    def inner_lambdas(self) -> list[float]:
        """Geometric multistep schedule (denoise.py:104-112), Python floats."""
        k = self.inner_steps
        out = []
        for step in range(k):
            frac = step / (k - 1) if k > 1 else 0.0
            out.append(self.lambda_start * (self.lambda_end / self.lambda_start) ** frac)
        return out


# ---------------------------------------------------------------------------
# batched device entry (used by the sampler)

@dataclass
class CondSource:
    """A coarse parent slab feeding conditioning_for_window for a batch."""

    parent: torch.Tensor          # (pc, ph, pw) on the device
    region: Region                # lattice footprint of `parent`
    scale: int
    mask_channel: int | None
    seed: int
    scalars: tuple[float, ...] = ()
    fill: bool = True             # False: holes were filled already (materialised y)

    def check_covers(self, layout: WindowLayout, idxs):
        for idx in idxs:
            need = window_region(layout, idx).scale_down(self.scale)
            if not self.region.contains(need):
                raise CoverageError(
                    f"parent data over {self.region} does not cover required region {need}",
                    missing=need)


def _phi_launch(kind_code, radius, lam, src, batched, sx0, sy0, wxy, n, win, cond, out):
    dt = out.dtype
    channels = out.shape[1]
    sh, sw = (src.shape[-2], src.shape[-1])
    if cond is not None:
        cp = cond.parent
        call("ig_phi_analytic", kind_code, radius, float(lam), dev.ig_dtype(dt), src.data_ptr(),
             int(batched), sx0, sy0, sw, sh, channels, wxy.data_ptr(), n, win,
             cp.data_ptr(), cond.region.x0, cond.region.y0, cp.shape[-1], cp.shape[-2],
             cp.shape[0], cond.scale, -1 if cond.mask_channel is None else cond.mask_channel,
             cond.seed & ((1 << 64) - 1), int(cond.fill), out.data_ptr(), dev.stream_ptr())
    else:
        call("ig_phi_analytic", kind_code, radius, float(lam), dev.ig_dtype(dt), src.data_ptr(),
             int(batched), sx0, sy0, sw, sh, channels, wxy.data_ptr(), n, win,
             None, 0, 0, 0, 0, 0, 1, -1, 0, 0, out.data_ptr(), dev.stream_ptr())


def apply_batch(spec: DenoiserSpec, src: torch.Tensor, src_region: Region | None,
                wxy: torch.Tensor, win: int, t: int, cond: CondSource | None = None,
                seed: int = 0, steps: int | None = None) -> torch.Tensor:
    """Phi over n windows at outer step t (1-based).

    src: canvas (C, h, w) covering every window (src_region = its footprint)
    or a window batch (n, C, win, win) (src_region None).  wxy: device int64
    (n, 2) window origins.  Returns (n, C, win, win) in src's dtype.
    """
    n = int(wxy.shape[0])
    channels = src.shape[-3]
    batched = src_region is None
    sx0, sy0 = (0, 0) if batched else (src_region.x0, src_region.y0)
    out = torch.empty((n, channels, win, win), dtype=src.dtype, device=src.device)
    if n == 0:
        return out
    if spec.kind == "unet":
        from .unet import unet_phi_batch
        return unet_phi_batch(spec.unet, src, src_region, wxy, win, t, cond, seed, steps)
    if spec.kind in _KIND_CODE:
        code = _KIND_CODE[spec.kind]
        _phi_launch(code, spec.radius, spec.lambda_for(t), src, batched, sx0, sy0, wxy, n, win,
                    cond if spec.kind == "cond_affine" else None, out)
        return out
    # multistep: inner one-step rule iterated over a ping-pong window batch
    if spec.inner_steps <= 0:
        _phi_launch(PHI_IDENTITY, 0, 0.0, src, batched, sx0, sy0, wxy, n, win, None, out)
        return out
    code = _KIND_CODE[spec.inner_kind]
    cur, cur_batched = src, batched
    for lam_j in spec.inner_lambdas():
        nxt = torch.empty_like(out)
        _phi_launch(code, spec.radius, lam_j, cur, cur_batched, sx0, sy0, wxy, n, win,
                    cond if spec.inner_kind == "cond_affine" else None, nxt)
        cur, cur_batched = nxt, True
    return cur


# ---------------------------------------------------------------------------
# reference-shaped single-window API

def apply(spec: DenoiserSpec, x, y: Conditioning | None, t: int, *,
          origin: tuple[int, int] = (0, 0), seed: int = 0):
    """Phi on one (C, H, W) window at outer step t (denoise.py:89-113).

    The analytic kinds are pure functions of (x, y, t), as in the reference.
    The ``"unet"`` kind (no reference counterpart) also depends on where the
    window sits: its consistency renoise at steps t < T draws coordinate noise
    (stream 301 + t) and conditioning holes are filled from stream 101, both
    keyed on the window's lattice ``origin`` and the sampler ``seed`` -- pass
    the window's origin and seed to reproduce the sampler's Phi exactly."""
    was_dev = isinstance(x, torch.Tensor)
    xa = x if was_dev else np.asarray(x)
    if xa.ndim != 3:
        raise ShapeError(f"window tensor must be (C, H, W), got shape {tuple(xa.shape)}")
    ych = None
    if y is not None:
        ych = y.channels
        if tuple(ych.shape[-2:]) != tuple(xa.shape[-2:]):
            raise ShapeError(f"conditioning spatial shape {tuple(ych.shape[-2:])} != window "
                             f"{tuple(xa.shape[-2:])}")
    if xa.shape[-1] != xa.shape[-2]:
        raise ShapeError("windows are square")
    xt = xa.contiguous() if was_dev else dev.upload(np.ascontiguousarray(xa))
    if xt.dtype not in (torch.float32, torch.float64):
        xt = xt.to(torch.float64)
    win = xt.shape[-1]
    wxy = dev.upload_i64([[0, 0]])
    cond = None
    if y is not None and y.mask is not None:
        # a materialised Conditioning: channel 0 is the target (holes already
        # filled), the mask rides along as an extra parent channel
        ch = y.channels if isinstance(y.channels, torch.Tensor) else dev.upload(
            np.ascontiguousarray(np.asarray(y.channels)))
        mk = y.mask if isinstance(y.mask, torch.Tensor) else dev.upload(
            np.ascontiguousarray(np.asarray(y.mask)))
        par = torch.cat([ch[:1].to(xt.dtype), mk.reshape(1, win, win).to(xt.dtype)], dim=0)
        cond = CondSource(par.contiguous(), Region(0, 0, win, win), 1, 1, 0, fill=False)
    if spec.kind == "unet":
        out = _apply_unet(spec, xt, y, t, origin, seed)
    else:
        out = apply_batch(spec, xt[None], None, wxy, win, t, cond)[0]
    return out if was_dev else dev.download(out)


def _apply_unet(spec: DenoiserSpec, xt: torch.Tensor, y, t: int, origin, seed: int):
    """One window through the batched UNet path (a batch of one; the kernels
    are batch invariant, so this is bit-identical to the sampler's Phi)."""
    from .unet import unet_phi_batch
    cfg = spec.unet
    steps = len(cfg.sigmas)
    if not 1 <= t <= steps:
        raise ValueError(f"outer step {t} outside [1, {steps}] for a {steps}-step UNet")
    C, H, W = xt.shape
    if C != cfg.data_channels:
        raise ShapeError(f"window has {C} channels, the UNet expects {cfg.data_channels}")
    x0, y0 = int(origin[0]), int(origin[1])
    cond = None
    if cfg.cond_channels:
        if y is None:
            raise ShapeError(f"the UNet takes {cfg.cond_channels} conditioning channels; "
                             "y is None")
        ch = y.channels if isinstance(y.channels, torch.Tensor) else dev.upload(
            np.ascontiguousarray(np.asarray(y.channels, dtype=np.float32)))
        mk = y.mask if isinstance(y.mask, torch.Tensor) else dev.upload(
            np.ascontiguousarray(np.asarray(y.mask, dtype=np.float32)))
        k = ch.shape[0]
        # the materialised conditioning as a scale-1 parent slab at the window's
        # own footprint, the mask as its last channel (holes are re-filled from
        # the same stream-101 noise at the same coordinates: a no-op)
        par = torch.cat([ch.float(), mk.reshape(1, H, W).float()], dim=0).contiguous()
        cond = CondSource(par, Region(x0, y0, W, H), 1, k, seed)
    wxy = dev.upload_i64([[x0, y0]])
    return unet_phi_batch(cfg, xt.float()[None].contiguous(), None, wxy, W, t, cond, seed,
                          steps)[0]


def conditioning_for_window(parent, parent_region: Region, scale: int, layout: WindowLayout,
                            idx: WindowIndex, scalars: tuple[float, ...] = (), seed: int = 0,
                            mask=None) -> Conditioning:
    """NN-upsampled parent crop + mask + stream-101 hole fill (denoise.py:116-163)."""
    was_dev = isinstance(parent, torch.Tensor)
    p = parent if was_dev else np.asarray(parent)
    if p.ndim == 2:
        p = p[None]
    win = window_region(layout, idx)
    need = win.scale_down(scale)
    if not parent_region.contains(need):
        raise CoverageError(
            f"parent data over {parent_region} does not cover required region {need}",
            missing=need)
    pt = p.contiguous() if was_dev else dev.upload(np.ascontiguousarray(p))
    if pt.dtype not in (torch.float32, torch.float64):
        pt = pt.to(torch.float64)
    mask_channel = -1
    if mask is not None:
        m = mask if isinstance(mask, torch.Tensor) else np.asarray(mask)
        if tuple(m.shape) != tuple(pt.shape[-2:]):
            raise ShapeError(f"mask shape {tuple(m.shape)} != parent spatial "
                             f"{tuple(pt.shape[-2:])}")
        mt = m if isinstance(m, torch.Tensor) else dev.upload(np.ascontiguousarray(m))
        pt = torch.cat([pt, mt.reshape(1, *mt.shape).to(pt.dtype)], dim=0).contiguous()
        mask_channel = pt.shape[0] - 1
    pc = pt.shape[0] - (1 if mask_channel >= 0 else 0)
    H = layout.window
    out = torch.empty((1, pt.shape[0], H, H), dtype=pt.dtype, device=pt.device)
    mout = torch.empty((1, H, H), dtype=pt.dtype, device=pt.device)
    wxy = dev.upload_i64([[win.x0, win.y0]])
    call("ig_condition_window", pt.data_ptr(), parent_region.x0, parent_region.y0,
         pt.shape[-1], pt.shape[-2], pt.shape[0], scale, mask_channel, seed & ((1 << 64) - 1),
         wxy.data_ptr(), 1, H, dev.ig_dtype(pt.dtype), out.data_ptr(), mout.data_ptr(),
         dev.stream_ptr())
    ch = out[0, :pc]
    mk = mout[0]
    if not was_dev:
        ch, mk = dev.download(ch), dev.download(mk)
    return Conditioning(channels=ch, scalars=tuple(scalars), mask=mk)


def percentile_rank(patch: int) -> int:
    """Lower nearest-rank index of the 5th percentile (denoise.py:181-182)."""
    return max(math.ceil(0.05 * patch * patch), 1)


def patch_features_device(elev: torch.Tensor, patch: int, n: int = 1,
                          tile_stride: int | None = None) -> torch.Tensor:
    """(n, 3, h/p, w/p) features of n elevation tiles (h, w) laid out every
    `tile_stride` elements (default: contiguous)."""
    h, w = elev.shape[-2], elev.shape[-1]
    if h % patch or w % patch:
        raise ShapeError(f"region {h}x{w} not divisible by patch size {patch}")
    stride = h * w if tile_stride is None else tile_stride
    out = torch.empty((n, 3, h // patch, w // patch), dtype=elev.dtype, device=elev.device)
    call("ig_patch_features", elev.data_ptr(), stride, n, h, w, patch, percentile_rank(patch),
         dev.ig_dtype(elev.dtype), out.data_ptr(), dev.stream_ptr())
    return out


def coarse_patch_features(elevation, patch: int):
    """(mean, 5th percentile, 1) per patch (denoise.py:166-185)."""
    was_dev = isinstance(elevation, torch.Tensor)
    e = elevation if was_dev else np.asarray(elevation)
    if e.ndim == 3:
        e = e[0]
    h, w = e.shape
    if h % patch or w % patch:
        raise ShapeError(f"region {h}x{w} not divisible by patch size {patch}")
    et = e.contiguous() if was_dev else dev.upload(np.ascontiguousarray(e))
    if et.dtype not in (torch.float32, torch.float64):
        et = et.to(torch.float64)
    out = patch_features_device(et, patch)[0]
    return out if was_dev else dev.download(out)
