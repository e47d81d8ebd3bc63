"""A/B timing of the attention kernel alone (64 windows of 32^2 tokens, 256
channels = 4 heads): CUDA events over 20 launches after warm-up, for the
current IG_ATT_POLY (set in the environment), plus its max error against an
fp32 softmax(QK^T)V reference.

for p in 0 4 6 8; do IG_ATT_POLY=$p python tools/attn_ab.py; done
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2512_08309_b200._native import call  # noqa: E402

n, hw, c = 64, 1024, 256
g = torch.Generator(device="cuda").manual_seed(0)


def unit_heads(x):
    x = x.view(n, hw, c // 64, 64)
    return (x / x.pow(2).mean(-1, keepdim=True).sqrt()).view(n, hw, c)


q = unit_heads(torch.randn(n, hw, c, device="cuda", generator=g))
k = unit_heads(torch.randn(n, hw, c, device="cuda", generator=g))
v = unit_heads(torch.randn(n, hw, c, device="cuda", generator=g))
qd = (q * (0.125 * 1.4426950408889634)).bfloat16().contiguous()
kd = k.bfloat16().contiguous()
vd = v.half().contiguous()
y = torch.empty(n, hw, c, dtype=torch.bfloat16, device="cuda")
s = torch.cuda.current_stream().cuda_stream


def run():
    call("ig_attention", qd.data_ptr(), kd.data_ptr(), vd.data_ptr(), n, hw, c, y.data_ptr(), s)


for _ in range(5):
    run()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize()
e0.record()
for _ in range(20):
    run()
e1.record()
torch.cuda.synchronize()
us = e0.elapsed_time(e1) / 20 * 1e3
# reference on 4 windows
qh = qd[:4].float().view(4, hw, 4, 64).transpose(1, 2)
kh = kd[:4].float().view(4, hw, 4, 64).transpose(1, 2)
vh = vd[:4].float().view(4, hw, 4, 64).transpose(1, 2)
p = torch.softmax((qh @ kh.transpose(-1, -2)) * 0.6931471805599453, dim=-1)
ref = (p @ vh).transpose(1, 2).reshape(4, hw, c)
err = (y[:4].float() - ref).abs()
print(f"IG_ATT_POLY={os.environ.get('IG_ATT_POLY', 'default')}: {us:.1f} us per 64 windows, "
      f"max err {err.max().item():.3e}, rms err {err.pow(2).mean().sqrt().item():.3e}")
