"""Profiling driver: one cfg2-shaped UNet Phi batch (or a full bench step) for ncu.

python tools/prof_step.py [--windows N] [--full]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2512_08309_b200 as ig  # noqa: E402
from paper_2512_08309_b200 import unet  # noqa: E402
from paper_2512_08309_b200.grid import Region, WindowLayout  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--windows", type=int, default=64)
ap.add_argument("--full", action="store_true")
ap.add_argument("--variant", type=int, default=None, help="ig_conv_set_variant (A/B timing)")
ap.add_argument("--fused-pool", action="store_true", help="unet.FUSED_POOL = True (A/B timing)")
args = ap.parse_args()
from paper_2512_08309_b200._native import check, lib  # noqa: E402
if args.variant is not None:   # else IG_CONV_VARIANT (read at load) stands
    check(lib().ig_conv_set_variant(args.variant))
unet.FUSED_POOL = unet.FUSED_POOL or args.fused_pool
cfg = unet.UNetConfig()
if args.full:
    scfg = ig.SamplerConfig(steps=2, layout=WindowLayout(256, 128), seed=0,
                            denoiser=ig.DenoiserSpec(kind="unet", unet=cfg))
    for k in range(2):
        ig.SamplerState(scfg, ig.TileStore()).query_device(0, Region(2048 * k, 0, 2048, 2048))
else:
    n = args.windows
    wxy = torch.tensor([[256 * k, 0] for k in range(n)], dtype=torch.int64, device="cuda")
    src = torch.randn(n, 1, 256, 256, device="cuda")
    for _ in range(2):
        unet.unet_phi_batch(cfg, src, None, wxy, 256, 1, None, seed=0, steps=2)
torch.cuda.synchronize()
print("done")
