"""Device memory lifetime: a dropped SamplerState / TileStore releases its
buffers immediately (reference counting), without waiting for the cyclic GC.
A reference cycle here made every bench step allocate fresh device memory."""

import gc

import pytest
import torch

pytestmark = pytest.mark.gpu

import paper_2512_08309_b200 as ig  # noqa: E402
from paper_2512_08309_b200.grid import Region, WindowLayout  # noqa: E402


def test_state_releases_device_memory_without_gc():
    spec = ig.DenoiserSpec(kind="shrink_smooth", radius=1, lambdas=(0.6, 0.4))
    cfg = ig.SamplerConfig(steps=2, layout=WindowLayout(64, 32), seed=3, denoiser=spec)

    def step(k):
        st = ig.SamplerState(cfg, ig.TileStore())
        return float(st.query_device(0, Region(512 * k, 0, 256, 256)).sum())

    step(0)
    torch.cuda.synchronize()
    gc.collect()
    base = torch.cuda.memory_allocated()
    gc.disable()
    try:
        for k in range(1, 4):
            step(k)
        torch.cuda.synchronize()
        assert torch.cuda.memory_allocated() == base
    finally:
        gc.enable()
