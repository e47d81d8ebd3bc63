"""cfg4 latency tail: per-query wall time with allocator / cache counters, to
see what the slow queries have in common.

python tools/cfg4_tail.py [--queries 300] [--snap]
"""
import os
import random
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2512_08309_b200 as ig  # noqa: E402
from paper_2512_08309_b200 import unet  # noqa: E402
from paper_2512_08309_b200.grid import WindowLayout  # noqa: E402

n = int(sys.argv[sys.argv.index("--queries") + 1]) if "--queries" in sys.argv else 300
snap = "--snap" in sys.argv
scfg = ig.SamplerConfig(steps=2, layout=WindowLayout(256, 128), seed=0,
                        denoiser=ig.DenoiserSpec(kind="unet", unet=unet.UNetConfig()),
                        name="stream", cache_limit=8 << 30)
store = ig.TileStore()
state = ig.SamplerState(scfg, store)
rng = random.Random(0 ^ 0xB1E55ED)
origins = [(rng.randrange(-10 ** 6, 10 ** 6), rng.randrange(-10 ** 6, 10 ** 6))
           for _ in range(n + 3)]
if snap:
    origins = [(x - x % 128, y - y % 128) for x, y in origins]
import gc  # noqa: E402
_gc = {"t": 0.0, "t0": 0.0, "n2": 0}


def _gc_cb(phase, info):
    if phase == "start":
        _gc["t0"] = time.perf_counter()
    else:
        _gc["t"] += time.perf_counter() - _gc["t0"]
        _gc["n2"] += info.get("generation", 0) == 2


gc.callbacks.append(_gc_cb)
_ev = {"t": 0.0, "n": 0}
_orig_evict = type(store)._evict_one


def _timed_evict(self, t):
    a = time.perf_counter()
    r = _orig_evict(self, t)
    _ev["t"] += time.perf_counter() - a
    _ev["n"] += 1
    return r


type(store)._evict_one = _timed_evict
rows = []
freeze = "--freeze" in sys.argv
for k, (x, y) in enumerate(origins):
    if freeze and k == 3:          # as bench.py run_cfg4
        gc.collect()
        gc.freeze()
    g0, n20 = _gc["t"], _gc["n2"]
    s0 = torch.cuda.memory_stats()
    c0 = state.total_denoiser_calls()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    state.query_device(0, ig.Region(x, y, 512, 512))
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    s1 = torch.cuda.memory_stats()
    rows.append((k, (t2 - t0) * 1e3, (t1 - t0) * 1e3, state.total_denoiser_calls() - c0,
                 s1.get("num_alloc_retries", 0) - s0.get("num_alloc_retries", 0),
                 s1.get("segment.all.allocated", 0) - s0.get("segment.all.allocated", 0),
                 s1.get("segment.all.freed", 0) - s0.get("segment.all.freed", 0),
                 (_gc["t"] - g0) * 1e3, _gc["n2"] - n20, _ev["t"] * 1e3, _ev["n"]))
    _ev["t"], _ev["n"] = 0.0, 0
lat = sorted(r[1] for r in rows[3:])
print(f"p50 {lat[len(lat)//2]:.2f} ms  p99 {lat[int(0.99*len(lat))]:.2f} ms  max {lat[-1]:.2f}")
print("k  ms  host_ms  phi  alloc_retries  seg_alloc  seg_freed  gc_ms  gen2  evict_ms  evicts")
for r in sorted(rows[3:], key=lambda r: -r[1])[:15]:
    print(*[f"{v:.2f}" if isinstance(v, float) else v for v in r])
print("median-ish rows:")
for r in rows[3:8]:
    print(*[f"{v:.2f}" if isinstance(v, float) else v for v in r[:7]])
