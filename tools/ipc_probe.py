"""Where does the time of a sharded step go with the IPC vs the send/recv halo
exchange?  Two ranks (gloo) on one GPU, a 4096^2 cfg5-shaped region with the
analytic Phi; rank 0 prints cProfile's top entries for one warm step.

python tools/ipc_probe.py [ipc|nccl]
"""
import cProfile
import multiprocessing as mp
import os
import pstats
import socket
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def worker(rank, world, port, mode):
    import torch
    import torch.distributed as dist

    import paper_2512_08309_b200 as ig
    from paper_2512_08309_b200 import shard
    from paper_2512_08309_b200.grid import Region, WindowLayout

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    spec = ig.DenoiserSpec(kind="shrink_smooth", radius=1, lambdas=(0.6, 0.4))
    cfg = ig.SamplerConfig(steps=2, layout=WindowLayout(256, 128), denoiser=spec, seed=0)

    def step(k):
        st = ig.SamplerState(cfg, ig.TileStore())
        r = Region(4096 * k - 10 ** 6, 10 ** 5, 4096, 4096)
        p = shard.plan([WindowLayout(256, 128)] * 2, r, world)
        xch = (shard.ipc_exchange(dist, (1, 256, 256), torch.float32) if mode == "ipc" else
               shard.p2p_exchange(dist, torch.device("cuda", 0), (1, 256, 256), torch.float32))
        out = shard.run(p, rank, shard.StoreExecutor(st), xch)
        if hasattr(xch, "close"):
            xch.close()
        torch.cuda.synchronize()
        dist.barrier()
        return out

    step(0)
    step(1)
    t0 = time.perf_counter()
    pr = cProfile.Profile()
    pr.enable()
    step(2)
    pr.disable()
    if rank == 0:
        print(f"{mode}: step {1e3 * (time.perf_counter() - t0):.1f} ms")
        pstats.Stats(pr).sort_stats("tottime").print_stats(14)
    dist.destroy_process_group()


if __name__ == "__main__":
    mode = sys.argv[1] if len(sys.argv) > 1 else "ipc"
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    ctx = mp.get_context("spawn")
    ps = [ctx.Process(target=worker, args=(k, 2, port, mode)) for k in range(2)]
    for p in ps:
        p.start()
    for p in ps:
        p.join()
