"""Timing of the attention block's 1x1 convs (qkv, proj) at cfg2 geometry
(64 windows, 32^2, 256 channels): CUDA events around --reps launches.
Environment toggles (IG_CONV_VARIANT, IG_DBG) are read at library load."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2512_08309_b200 import unet  # noqa: E402
from paper_2512_08309_b200._native import ConvParams, check, lib  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--windows", type=int, default=64)
ap.add_argument("--reps", type=int, default=20)
ap.add_argument("--tag", default="")
args = ap.parse_args()
n, h, w, c = args.windows, 32, 32, 256
x = torch.randn(n, h, w, c, device="cuda").bfloat16()
r = torch.randn(n, h, w, c, device="cuda").bfloat16()
wq = (torch.randn(3 * c, c, device="cuda") / 16).bfloat16()
wp = (torch.randn(c, c, device="cuda") / 16).bfloat16()
o = [torch.empty_like(x) for _ in range(3)]
st = torch.cuda.current_stream().cuda_stream


def qkv():
    p = ConvParams(n, h, w, c, 0, c, 1, x.data_ptr(), None, wq.data_ptr(), None, None, None,
                   0.0, 1.0, 1.0, o[0].data_ptr(), None)
    p.head_norm, p.head_scale = 1, unet.Q_SCALE
    check(lib().ig_conv_qkv(p, o[1].data_ptr(), o[2].data_ptr(), st))


def proj():
    p = ConvParams(n, h, w, c, 0, c, 1, x.data_ptr(), None, wp.data_ptr(), None, None,
                   r.data_ptr(), float(unet.ATTN_RA), float(unet.ATTN_RB), unet.MP_SILU_GAIN,
                   o[0].data_ptr(), o[1].data_ptr())
    check(lib().ig_conv_tc(p, None, st))


flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for name, fn in (("qkv", qkv), ("proj", proj)):
    for _ in range(3):
        fn()
    tot = 0.0
    for _ in range(args.reps):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        tot += e0.elapsed_time(e1)
    print(f"{args.tag} {name}: {1000 * tot / args.reps:.1f} us")
