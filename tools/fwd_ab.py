"""A/B timing of one UNet Phi batch (default UNetConfig, 256^2 windows):
CUDA events around `--reps` forwards after warm-up.  Environment toggles
(IG_RES_V8, IG_ATT_POLY, ...) are read by the library at load time, so run
one process per variant and alternate them:

for v in 0 1 0 1; do IG_RES_V8=$v python tools/fwd_ab.py --tag res_v8=$v; done
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2512_08309_b200 import unet  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--windows", type=int, default=128)
ap.add_argument("--reps", type=int, default=6)
ap.add_argument("--tag", default="")
ap.add_argument("--variant", type=int, default=None, help="ig_conv_set_variant (A/B)")
args = ap.parse_args()
from paper_2512_08309_b200._native import check, lib  # noqa: E402
if args.variant is not None:   # else IG_CONV_VARIANT (read at load) stands
    check(lib().ig_conv_set_variant(args.variant))
cfg = unet.UNetConfig()
n = args.windows
wxy = torch.tensor([[256 * k, 0] for k in range(n)], dtype=torch.int64, device="cuda")
src = torch.randn(n, 1, 256, 256, device="cuda", generator=torch.Generator("cuda").manual_seed(0))
for _ in range(2):
    out = unet.unet_phi_batch(cfg, src, None, wxy, 256, 1, None, seed=0, steps=2)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize()
e0.record()
for _ in range(args.reps):
    out = unet.unet_phi_batch(cfg, src, None, wxy, 256, 1, None, seed=0, steps=2)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / args.reps
print(f"{args.tag}: {ms:.3f} ms per {n}-window forward ({ms / n * 64:.3f} ms per 64), "
      f"checksum {out.double().sum().item():.6f}")
