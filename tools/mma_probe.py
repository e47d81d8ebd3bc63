"""Probe: achievable tcgen05 throughput of ig_conv_tc as a plain GEMM
(1x1 conv, large K) per N, to separate MMA/SMEM limits from epilogue/memory."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2512_08309_b200._native import ConvParams, check, lib

dev = "cuda"
st = torch.cuda.current_stream().cuda_stream
res = {}
for taps, cin in ((1, 1024), (9, 128)):
    for N in (64, 128, 256):
        n, h, w = 8, 128, 256      # 262144 px
        a = torch.randn(n, h, w, cin, device=dev).bfloat16()
        wgt = torch.randn(N, taps * cin, device=dev).bfloat16()
        o1 = torch.empty(n, h, w, N, device=dev, dtype=torch.bfloat16)
        p = ConvParams(n, h, w, cin, 0, N, taps, a.data_ptr(), 0, wgt.data_ptr(), 0, 0, 0,
                       0.0, 1.0, 1.0, 0, o1.data_ptr())
        for variant in (0, 1):
            check(lib().ig_conv_set_variant(variant))
            for _ in range(3):
                check(lib().ig_conv_tc(p, None, st))
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(10):
                check(lib().ig_conv_tc(p, None, st))
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / 10
            fl = 2.0 * n * h * w * cin * N * taps
            res[f"taps{taps}_cin{cin}_N{N}_v{variant}"] = round(fl / ms / 1e9, 1)
check(lib().ig_conv_set_variant(0))
print(json.dumps(res, indent=1))
