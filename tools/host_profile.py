"""cProfile of warm cfg2 steps (host-side hot spots of the sampler/store path).

python tools/host_profile.py [--phi analytic|unet] [--steps 5]
"""
import cProfile
import os
import pstats
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2512_08309_b200 as ig  # noqa: E402
from paper_2512_08309_b200 import unet  # noqa: E402
from paper_2512_08309_b200.grid import Region, WindowLayout  # noqa: E402

phi = sys.argv[sys.argv.index("--phi") + 1] if "--phi" in sys.argv else "analytic"
steps = int(sys.argv[sys.argv.index("--steps") + 1]) if "--steps" in sys.argv else 5
spec = (ig.DenoiserSpec(kind="shrink_smooth", radius=1, lambdas=(0.6, 0.4)) if phi == "analytic"
        else ig.DenoiserSpec(kind="unet", unet=unet.UNetConfig()))
scfg = ig.SamplerConfig(steps=2, layout=WindowLayout(256, 128), seed=0, denoiser=spec,
                        name="bench")


def step(k):
    st = ig.SamplerState(scfg, ig.TileStore())
    return st.query_device(0, Region(2048 * k, 0, 2048, 2048))


for k in range(3):
    step(100 + k)
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
for k in range(steps):
    step(k)
torch.cuda.synchronize()
pr.disable()
st = pstats.Stats(pr)
st.sort_stats("tottime").print_stats(25)
st.print_callers("built-in method torch.empty")
