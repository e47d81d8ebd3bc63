"""Sharded region query on the device tile store: ranks emulated in one
process (one GPU; the halo exchange is an in-process mailbox), every rank
with its own TileStore.  The concatenated strips must be bitwise equal to a
single-store query and no Phi may be evaluated twice."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

import paper_2512_08309_b200 as ig  # noqa: E402
from paper_2512_08309_b200 import shard  # noqa: E402
from paper_2512_08309_b200.grid import Region, WindowLayout  # noqa: E402


def _cfg(kind, steps, H, s):
    if kind == "unet":
        from paper_2512_08309_b200.unet import UNetConfig
        spec = ig.DenoiserSpec(kind="unet", unet=UNetConfig(base=64, mults=(1, 2), blocks=1))
    else:
        spec = ig.DenoiserSpec(kind="shrink_smooth", radius=1, lambdas=(0.6, 0.4))
    return ig.SamplerConfig(steps=steps, layout=WindowLayout(H, s), denoiser=spec, seed=4,
                            name=f"sh_{kind}")


@pytest.mark.parametrize("kind,steps,H,s,world,region", [
    ("shrink", 2, 16, 8, 3, (-37, 11, 70, 90)),
    ("shrink", 3, 16, 8, 4, (0, 0, 64, 96)),
    ("shrink", 2, 256, 128, 2, (0, 0, 512, 768)),
    ("unet", 2, 64, 32, 2, (0, 0, 128, 192)),
])
def test_sharded_equals_single(kind, steps, H, s, world, region):
    cfg = _cfg(kind, steps, H, s)
    r = Region(*region)
    single = ig.SamplerState(cfg, ig.TileStore())
    want = single.query(0, r)
    p = shard.plan([WindowLayout(H, s)] * steps, r, world)
    states = [ig.SamplerState(cfg, ig.TileStore()) for _ in range(world)]
    strips = shard.run_emulated(p, [shard.StoreExecutor(st) for st in states])
    got = np.concatenate([s_.cpu().numpy() for s_ in strips], axis=1)
    np.testing.assert_array_equal(got.view(np.uint32), want.view(np.uint32))
    assert sum(st.total_denoiser_calls() for st in states) == single.total_denoiser_calls()
