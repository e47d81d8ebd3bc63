"""cfg4: how busy is the GPU inside a 512^2 query?  torch.profiler over a few
warm queries; prints wall time per query, summed kernel time and the largest
idle gaps between consecutive kernels.

python tools/cfg4_busy.py [--queries 5]
"""
import os
import random
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import paper_2512_08309_b200 as ig  # noqa: E402
from paper_2512_08309_b200 import unet  # noqa: E402
from paper_2512_08309_b200.grid import Region, WindowLayout  # noqa: E402

n = int(sys.argv[sys.argv.index("--queries") + 1]) if "--queries" in sys.argv else 5
scfg = ig.SamplerConfig(steps=2, layout=WindowLayout(256, 128), seed=0,
                        denoiser=ig.DenoiserSpec(kind="unet", unet=unet.UNetConfig()),
                        name="stream", cache_limit=8 << 30)
state = ig.SamplerState(scfg, ig.TileStore())
rng = random.Random(0 ^ 0xB1E55ED)
org = [(rng.randrange(-10 ** 6, 10 ** 6), rng.randrange(-10 ** 6, 10 ** 6)) for _ in range(n + 5)]
for x, y in org[:5]:
    state.query(0, Region(x, y, 512, 512))
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    t0 = time.perf_counter()
    for x, y in org[5:]:
        state.query(0, Region(x, y, 512, 512))
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
ev = sorted((e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA
             and e.time_range.elapsed_us() > 0), key=lambda e: e.time_range.start)
busy = sum(e.time_range.elapsed_us() for e in ev)
print(f"{n} queries: wall {wall * 1e3 / n:.2f} ms/query, kernels {busy / 1e3 / n:.2f} ms/query, "
      f"{len(ev) / n:.0f} launches/query")
gaps = sorted(((b.time_range.start - a.time_range.end, a.name[:40], b.name[:40])
               for a, b in zip(ev, ev[1:])), reverse=True)
print(f"idle between kernels: {sum(g for g, _, _ in gaps if g > 0) / 1e3 / n:.2f} ms/query")
for g, a, b in gaps[:8]:
    print(f"  {g / 1e3:6.2f} ms  after {a}  before {b}")
