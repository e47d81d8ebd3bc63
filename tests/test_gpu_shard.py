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
    if kind == "unet_prod":
        # the bench's network: default UNetConfig (attention at 32^2, CTA-pair
        # four-row kernels at 256^2, gutter layout at 64^2)
        from paper_2512_08309_b200.unet import UNetConfig
        spec = ig.DenoiserSpec(kind="unet", unet=UNetConfig())
    elif kind == "unet":
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
    ("unet_prod", 2, 256, 128, 3, (-256, 128, 512, 768)),
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


# ---------------------------------------------------------------------------
# Peer-memory halo exchange (shard.IpcExchange): real processes, each with its
# own CUDA context; on the round-end box they share one GPU (CUDA IPC memory
# and interprocess events work between processes on the same device exactly as
# across NVLink peers).  A consumer's stream waits on the producer's pack event
# (device-side ordering; the producers never wait on their consumers within a
# query, so time-sliced contexts always make progress).  Two queries run
# through the same exchange (buffer reuse behind the release events).  The
# gathered strips must be bitwise equal to one-process queries and the
# boundary windows must have been read in place (PeerWindow slots).

def _ipc_worker(rank, world, port_, kind, steps, H, s, region, q):
    import os

    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port_))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        cfg = _cfg(kind, steps, H, s)
        assert shard.ipc_supported(dist)
        xch = shard.ipc_exchange(dist, (1, H, H), torch.float32)
        out = []
        for shift in (0, 8 * s):
            st = ig.SamplerState(cfg, ig.TileStore())
            r = Region(region[0] + shift, region[1], region[2], region[3])
            p = shard.plan([WindowLayout(H, s)] * steps, r, world)
            strip = shard.run(p, rank, shard.StoreExecutor(st), xch).cpu().numpy()
            peers = sum(1 for t in range(steps)
                        for slot in st.store._tensor(st.handles[t]).lru.values()
                        if getattr(slot.data, "is_peer", False))
            out.append((strip, st.total_denoiser_calls(), peers))
        xch.close()
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("kind,steps,H,s,world,region", [
    ("shrink", 2, 16, 8, 2, (-37, 11, 70, 90)),
    ("shrink", 3, 16, 8, 3, (0, 0, 64, 96)),
    ("unet", 2, 64, 32, 2, (0, 0, 128, 192)),
    ("unet_prod", 2, 256, 128, 2, (0, 0, 512, 512)),
])
def test_ipc_exchange_bitwise(kind, steps, H, s, world, region):
    import multiprocessing as mp
    import socket

    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port_ = so.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_ipc_worker, args=(k, world, port_, kind, steps, H, s, region, q))
             for k in range(world)]
    for pr in procs:
        pr.start()
    res = sorted([q.get(timeout=300) for _ in range(world)], key=lambda x: x[0])
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    cfg = _cfg(kind, steps, H, s)
    for k, shift in enumerate((0, 8 * s)):
        single = ig.SamplerState(cfg, ig.TileStore())
        want = single.query(0, Region(region[0] + shift, region[1], region[2], region[3]))
        got = np.concatenate([r_[1][k][0] for r_ in res], axis=1)
        np.testing.assert_array_equal(got.view(np.uint32), want.view(np.uint32))
        assert sum(r_[1][k][1] for r_ in res) == single.total_denoiser_calls()  # no Phi twice
        assert sum(r_[1][k][2] for r_ in res) > 0    # boundary windows were read in place
