"""Is a conv epilogue-bound?  Times one c2-shaped conv (3x3 + fused skip GEMM)
with both outputs (x, mp_silu(x)), x only, and mp_silu(x) only.

python tools/epi_probe.py
"""
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2512_08309_b200._native import ConvParams, check, lib  # noqa: E402

DEV = "cuda"


def run(n, h, w, ca, cout, csa, outs, reps=10):
    g = torch.Generator(device=DEV).manual_seed(0)
    a = torch.randn(n, h, w, ca, device=DEV, generator=g).bfloat16()
    sk = torch.randn(n, h, w, csa, device=DEV, generator=g).bfloat16()
    wgt = (torch.randn(cout, 9 * ca, device=DEV, generator=g) / math.sqrt(9 * ca)).bfloat16()
    wsk = (torch.randn(cout, csa, device=DEV, generator=g) / math.sqrt(csa)).bfloat16()
    scale = torch.rand(cout, device=DEV, generator=g) + 0.5
    o0 = torch.empty(n, h, w, cout, device=DEV, dtype=torch.bfloat16) if "x" in outs else None
    o1 = torch.empty(n, h, w, cout, device=DEV, dtype=torch.bfloat16) if "xa" in outs else None
    p = ConvParams(n, h, w, ca, 0, cout, 9, a.data_ptr(), 0, wgt.data_ptr(), scale.data_ptr(), 0, 0,
                   0.0, 1.0, 1.6778524, 0 if o0 is None else o0.data_ptr(),
                   0 if o1 is None else o1.data_ptr(), csa, 0, sk.data_ptr(), 0, wsk.data_ptr())
    st = torch.cuda.current_stream().cuda_stream
    for _ in range(3):
        check(lib().ig_conv_tc(p, None, st))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        check(lib().ig_conv_tc(p, None, st))
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


for (name, n, h, w, ca, cout, csa) in [("enc0.0.c2", 64, 256, 256, 64, 64, 64),
                                        ("dec0.1.c2", 64, 256, 256, 64, 64, 128),
                                        ("dec1.0.c2", 64, 128, 128, 128, 128, 256),
                                        ("enc0.0.c1-like", 64, 256, 256, 64, 64, 0)]:
    if csa == 0:
        csa = 64   # keep the skip path shape-valid; c1-like = one chunk + small skip
    res = {o: run(n, h, w, ca, cout, csa, o) for o in (("x", "xa"), ("x",), ("xa",))}
    print(name, "  ".join(f"{'+'.join(k)}: {v:7.1f} us" for k, v in res.items()))
