"""cfg4 tail diagnosis: per-query latency of the analytic-Phi serving loop
(numpy out) with the slowest queries' index and Phi count."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gc  # noqa: E402

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2512_08309_b200 as ig  # noqa: E402
from paper_2512_08309_b200.grid import WindowLayout  # noqa: E402

mode = sys.argv[1] if len(sys.argv) > 1 else "query"
st = ig.SamplerState(ig.SamplerConfig(steps=2, layout=WindowLayout(256, 128), seed=0, name="a",
                                      denoiser=ig.DenoiserSpec(kind="shrink_smooth", radius=1,
                                                               lambdas=(0.6, 0.4)),
                                      cache_limit=8 << 30), ig.TileStore())
lat = []
for k, (x, y) in enumerate(bench._cfg4_origins(1003, False)):
    if k == 3:
        gc.collect()
        gc.freeze()
    c0 = st.total_denoiser_calls()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    if mode == "query":
        st.query(0, ig.Region(x, y, 512, 512))
    else:
        st.query_device(0, ig.Region(x, y, 512, 512))
    torch.cuda.synchronize()
    lat.append(((time.perf_counter() - t0) * 1e3, k, st.total_denoiser_calls() - c0))
lat = lat[3:]
srt = sorted(lat)
print(mode, "p50", srt[len(srt) // 2][0], "p99", srt[int(0.99 * len(srt))][0])
print("slowest", [(round(a, 1), k, c) for a, k, c in srt[-15:]])
