"""Where does the GPU sit idle inside a bench step?  (torch.profiler timeline)

python tools/host_gaps.py [--phi analytic]
Runs the cfg2 UNet step (bench.py's workload) twice to warm up, profiles one
more with CPU + CUDA activities, and prints the device span, summed kernel
time, the largest idle gaps between consecutive kernels, and the top host
functions by self CPU time.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import paper_2512_08309_b200 as ig  # noqa: E402
from paper_2512_08309_b200 import unet  # noqa: E402
from paper_2512_08309_b200.grid import Region, WindowLayout  # noqa: E402

cfg = unet.UNetConfig()
analytic = "--phi" in sys.argv and sys.argv[sys.argv.index("--phi") + 1] == "analytic"
spec = (ig.DenoiserSpec(kind="shrink_smooth", radius=1, lambdas=(0.6, 0.4)) if analytic
        else ig.DenoiserSpec(kind="unet", unet=cfg))
scfg = ig.SamplerConfig(steps=2, layout=WindowLayout(256, 128), seed=0, denoiser=spec,
                        name="bench")


def step(k):
    st = ig.SamplerState(scfg, ig.TileStore())
    return st.query_device(0, Region(2048 * k, 0, 2048, 2048))


for k in range(2):
    step(100 + k)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    step(7)
    torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA
      and e.time_range.elapsed_us() > 0]
ev.sort(key=lambda e: e.time_range.start)
busy = sum(e.time_range.elapsed_us() for e in ev)
span = ev[-1].time_range.end - ev[0].time_range.start
print(f"kernels {len(ev)}  busy {busy/1e3:.2f} ms  span {span/1e3:.2f} ms")
gaps = []
for a, b in zip(ev, ev[1:]):
    g = b.time_range.start - a.time_range.end
    if g > 20:
        gaps.append((g, a.name[:40], b.name[:40]))
gaps.sort(reverse=True)
print(f"gaps > 20us: {len(gaps)}  total {sum(g for g, _, _ in gaps)/1e3:.2f} ms")
for g, a, b in gaps[:15]:
    print(f"  {g/1e3:7.2f} ms  after {a}  before {b}")
print(prof.key_averages().table(sort_by="self_cpu_time_total", row_limit=25))
